// ubench_idp.cu -- issue rate of the integer dot products (dp2a / dp4a) on
// sm_100a, alone and mixed with LOP3, against FHFMA: can a decode loop that
// multiplies int4 codes by 16-bit fixed-point x beat the FHFMA loop's ~2.4
// warp-instr/clk/SM co-issue limit?  8 independent chains per thread.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_idp tools/ubench_idp.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

template <int MODE>
__global__ void __launch_bounds__(512, 1) kern(long long* cyc, int* sink, uint32_t seed) {
    int acc[8];
    uint32_t a[8], b[8];
    for (int i = 0; i < 8; ++i) { acc[i] = 0; a[i] = seed * (i + 1) + threadIdx.x; b[i] = seed ^ (i * 77 + threadIdx.x); }
    float facc[8];
    for (int i = 0; i < 8; ++i) facc[i] = 0.f;
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (MODE == 0) {        // dp2a.lo
                asm volatile("dp2a.lo.s32.s32 %0, %1, %2, %0;" : "+r"(acc[i]) : "r"(a[i]), "r"(b[i]));
            } else if (MODE == 1) { // dp4a
                asm volatile("dp4a.s32.s32 %0, %1, %2, %0;" : "+r"(acc[i]) : "r"(a[i]), "r"(b[i]));
            } else if (MODE == 2) { // dp2a + LOP3 (the unpack)
                asm volatile("dp2a.lo.s32.s32 %0, %1, %2, %0;" : "+r"(acc[i]) : "r"(a[i]), "r"(b[i]));
                asm volatile("lop3.b32 %0, %0, %1, 0x0F0F0F0F, 0xc0;" : "+r"(b[i]) : "r"(a[i]));
            } else if (MODE == 3) { // FHFMA reference
                uint16_t h = static_cast<uint16_t>(a[i]), g = static_cast<uint16_t>(b[i]);
                asm volatile("fma.rn.f32.f16 %0, %1, %2, %0;" : "+f"(facc[i]) : "h"(h), "h"(g));
            } else if (MODE == 4) { // 2 dp2a + 1 LOP3 (the mix a dp2a decode loop needs: 4 dp2a + ~1.5 ALU per 8 codes)
                asm volatile("dp2a.lo.s32.s32 %0, %1, %2, %0;" : "+r"(acc[i]) : "r"(a[i]), "r"(b[i]));
                asm volatile("dp2a.hi.s32.s32 %0, %1, %2, %0;" : "+r"(acc[i]) : "r"(a[i]), "r"(b[i]));
                asm volatile("lop3.b32 %0, %0, %1, 0x0F0F0F0F, 0xc0;" : "+r"(b[i]) : "r"(a[i]));
            }
        }
    }
    const long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    int s = 0;
    for (int i = 0; i < 8; ++i) s += acc[i] + static_cast<int>(facc[i]) + b[i];
    if (s == 0x7fffffff) *sink = s;
}

template <int MODE>
static void run(const char* name, int instr_per_iter) {
    long long* d; int* sink;
    cudaMalloc(&d, 148 * sizeof(long long)); cudaMalloc(&sink, 4);
    kern<MODE><<<148, 512>>>(d, sink, 12345u);
    cudaDeviceSynchronize();
    kern<MODE><<<148, 512>>>(d, sink, 12345u);
    cudaError_t e = cudaDeviceSynchronize();
    long long c[148];
    cudaMemcpy(c, d, sizeof c, cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int i = 0; i < 148; ++i) mx = c[i] > mx ? c[i] : mx;
    const double warp_instr = 16.0 * ITERS * 8 * instr_per_iter;   // 16 warps per SM
    printf("%-34s %.2f warp-instr/clk/SM (%s)\n", name, warp_instr / mx, cudaGetErrorString(e));
    cudaFree(d); cudaFree(sink);
}

int main() {
    run<0>("dp2a.lo", 1);
    run<1>("dp4a", 1);
    run<2>("dp2a + LOP3", 2);
    run<3>("FHFMA (fma.rn.f32.f16)", 1);
    run<4>("2 dp2a + LOP3", 3);
    return 0;
}
