// ubench_tc.cu -- tcgen05.mma kind::f16 issue throughput on one SM per CTA:
// A operand from TMEM ("ts", what gemm_tc.cu uses) vs from SMEM ("ss"), for
// M = 128 and N in {64, 128, 256}, cta_group::1.  One elected thread issues
// ITERS back-to-back MMAs (K = 16 each) into one accumulator, commits, waits.
// Operand contents are irrelevant (garbage in, throughput out).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2311_02103_b200/csrc -o tools/ubench_tc tools/ubench_tc.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "ptx.cuh"

using namespace rq4;

constexpr int ITERS = 4096;

__device__ __forceinline__ void mma_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                       uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
        :: "r"(d_tmem), "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(acc) : "memory");
}

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) kern(long long* cycles) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tbase;
    __shared__ __align__(8) uint64_t bar;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) { tmem_alloc<512>(&tbase); tmem_relinquish(); }
    if (threadIdx.x == 32) { mbar_init(&bar, 1); fence_mbar_init(); }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tm = tbase;
    const uint32_t sa = smem_u32(smem);                 // A: 128 x 16 fp16 K-major SW128 (16 KB region)
    const uint32_t sb = sa + 16384;                     // B: N x 16
    const uint32_t idesc = idesc_f16_f32(128, N);
    long long t0 = 0, t1 = 0;
    if (threadIdx.x == 0) {
        t0 = clock64();
        for (int i = 0; i < ITERS; ++i) {
            const uint64_t bd = smem_desc_k_sw128(sb + (i & 3) * 32);
            if (TS) tc_mma_ts(tm, tm + 256, bd, idesc, i > 0);                 // A in TMEM cols 256..
            else mma_ss(tm, smem_desc_k_sw128(sa + (i & 3) * 32), bd, idesc, i > 0);
        }
        tc_commit(&bar);
        mbar_wait(&bar, 0);
        t1 = clock64();
        cycles[blockIdx.x] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) tmem_dealloc<512>(tm);
}

template <int N, bool TS>
static void run(long long* d) {
    const int smem = 16384 + 32768 + 1024;
    cudaFuncSetAttribute(kern<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    kern<N, TS><<<148, 128, smem>>>(d);
    cudaDeviceSynchronize();
    kern<N, TS><<<148, 128, smem>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    long long c[148];
    cudaMemcpy(c, d, sizeof c, cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int i = 0; i < 148; ++i) mx = c[i] > mx ? c[i] : mx;
    const double macs = 128.0 * N * 16 * ITERS;
    printf("%s M=128 N=%3d K=16: %.1f clk/MMA, %.0f MAC/clk/SM (%s)\n", TS ? "TS (A in TMEM)" : "SS (A in SMEM)", N,
           (double)mx / ITERS, macs / mx, cudaGetErrorString(e));
}

int main() {
    long long* d;
    cudaMalloc(&d, 148 * sizeof(long long));
    run<64, true>(d);  run<64, false>(d);
    run<128, true>(d); run<128, false>(d);
    run<256, true>(d); run<256, false>(d);
    return 0;
}
