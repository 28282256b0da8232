// ubench.cu -- per-SM issue throughput of the instructions the GEMV inner
// loop is made of (FHFMA = fma.rn.f32.f16, FFMA, HFMA2, LOP3), measured with
// clock64 on one CTA per SM, 8 independent chains per thread.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench tools/ubench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

template <int OP>
__global__ void kern(float* out, uint32_t seed, long long* cycles) {
    float a[8];
    uint32_t u[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) { a[i] = (float)(threadIdx.x + i); u[i] = seed * (i + 1) + threadIdx.x; }
    const uint32_t h = 0x3c003c00u ^ (seed & 1);
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (OP == 0) {        // FHFMA
                asm volatile("fma.rn.f32.f16 %0, %1, %2, %0;" : "+f"(a[i]) : "h"((unsigned short)(h & 0xffff)), "h"((unsigned short)(u[i] & 0xffff)));
            } else if (OP == 1) { // FFMA 3-reg
                asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(__uint_as_float(u[i])), "f"(__uint_as_float(h)));
            } else if (OP == 2) { // HFMA2
                asm volatile("fma.rn.f16x2 %0, %0, %1, %2;" : "+r"(u[i]) : "r"(h), "r"(seed));
            } else if (OP == 3) { // LOP3
                asm volatile("lop3.b32 %0, %0, %1, %2, 0xea;" : "+r"(u[i]) : "r"(h), "r"(seed));
            } else if (OP == 5) { // LOP3 + 2 FFMA
                asm volatile("lop3.b32 %0, %0, %1, %2, 0xea;" : "+r"(u[i]) : "r"(h), "r"(seed));
                asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(__uint_as_float(u[i])), "f"(__uint_as_float(h)));
                asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(__uint_as_float(seed)), "f"(__uint_as_float(u[i])));
            } else if (OP == 6) { // LOP3 + HFMA2 (1:1)
                asm volatile("lop3.b32 %0, %0, %1, %2, 0xea;" : "+r"(u[i]) : "r"(h), "r"(seed));
                asm volatile("fma.rn.f16x2 %0, %0, %1, %2;" : "+r"(u[(i + 4) & 7]) : "r"(h), "r"(seed));
            } else if (OP == 7) { // FHFMA + HFMA2 (1:1)
                asm volatile("fma.rn.f32.f16 %0, %1, %2, %0;" : "+f"(a[i]) : "h"((unsigned short)(h & 0xffff)), "h"((unsigned short)(u[i] & 0xffff)));
                asm volatile("fma.rn.f16x2 %0, %0, %1, %2;" : "+r"(u[(i + 4) & 7]) : "r"(h), "r"(seed));
            } else if (OP == 8) { // FHFMA + FFMA (1:1)
                asm volatile("fma.rn.f32.f16 %0, %1, %2, %0;" : "+f"(a[i]) : "h"((unsigned short)(h & 0xffff)), "h"((unsigned short)(u[i] & 0xffff)));
                asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[(i + 4) & 7]) : "f"(__uint_as_float(u[i])), "f"(__uint_as_float(h)));
            } else if (OP == 9) { // FHFMA with immediate-ish reuse: same b operand for all chains
                asm volatile("fma.rn.f32.f16 %0, %1, %2, %0;" : "+f"(a[i]) : "h"((unsigned short)(u[i] & 0xffff)), "h"((unsigned short)(h & 0xffff)));
            } else {              // mixed: 1 LOP3 + 2 FHFMA (the ZPF GEMV ratio ~ 5:8)
                asm volatile("lop3.b32 %0, %0, %1, %2, 0xea;" : "+r"(u[i]) : "r"(h), "r"(seed));
                asm volatile("fma.rn.f32.f16 %0, %1, %2, %0;" : "+f"(a[i]) : "h"((unsigned short)(u[i] & 0xffff)), "h"((unsigned short)(h >> 16)));
                asm volatile("fma.rn.f32.f16 %0, %1, %2, %0;" : "+f"(a[i]) : "h"((unsigned short)(u[i] >> 16)), "h"((unsigned short)(h & 0xffff)));
            }
        }
    }
    long long t1 = clock64();
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += a[i] + (float)u[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

int main() {
    float* out;
    long long* cyc;
    cudaMalloc(&out, 148 * 1024 * 4);
    cudaMalloc(&cyc, 148 * 8);
    const char* names[] = {"FHFMA", "FFMA(3reg)", "HFMA2", "LOP3", "LOP3+2FHFMA", "LOP3+2FFMA", "LOP3+HFMA2", "FHFMA+HFMA2", "FHFMA+FFMA", "FHFMA(b-shared)"};
    for (int op = 0; op < 10; ++op) {
        for (int threads : {512}) {
            auto launch = [&] {
                switch (op) {
                    case 0: kern<0><<<148, threads>>>(out, 7, cyc); break;
                    case 1: kern<1><<<148, threads>>>(out, 7, cyc); break;
                    case 2: kern<2><<<148, threads>>>(out, 7, cyc); break;
                    case 3: kern<3><<<148, threads>>>(out, 7, cyc); break;
                    case 4: kern<4><<<148, threads>>>(out, 7, cyc); break;
                    case 5: kern<5><<<148, threads>>>(out, 7, cyc); break;
                    case 6: kern<6><<<148, threads>>>(out, 7, cyc); break;
                    case 7: kern<7><<<148, threads>>>(out, 7, cyc); break;
                    case 8: kern<8><<<148, threads>>>(out, 7, cyc); break;
                    default: kern<9><<<148, threads>>>(out, 7, cyc); break;
                }
            };
            launch();
            cudaDeviceSynchronize();
            launch();
            cudaDeviceSynchronize();
            long long c[148];
            cudaMemcpy(c, cyc, sizeof c, cudaMemcpyDeviceToHost);
            long long mx = 0;
            for (int i = 0; i < 148; ++i) mx = c[i] > mx ? c[i] : mx;
            const double ninst = (double)ITERS * 8 * (op == 4 || op == 5 ? 3 : (op >= 6 && op <= 8) ? 2 : 1) * threads / 32;   // warp instructions per SM
            printf("%-12s threads=%4d  warp-inst/clk/SM = %.2f  lanes/clk/SM = %.1f\n", names[op], threads,
                   ninst / mx, ninst * 32 / mx);
        }
    }
    return 0;
}
