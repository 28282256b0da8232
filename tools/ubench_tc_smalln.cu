// ubench_tc_smalln.cu -- tcgen05.mma kind::f16 issue throughput at small N
// (16, 32, 64) for M = 128, cta_group::1: one accumulator vs D rotating over
// NACC independent accumulators, A from TMEM (ts) or SMEM (ss).  Decides
// whether a decode (n = 1..16) kernel can feed the tensor pipe with narrow
// tiles: weights per clock per SM = 128 * 16 / (clk per MMA).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2311_02103_b200/csrc -o tools/ubench_tc_smalln tools/ubench_tc_smalln.cu
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

template <int N, bool TS, int NACC>
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
    const uint32_t sa = smem_u32(smem);
    const uint32_t sb = sa + 16384;
    const uint32_t idesc = idesc_f16_f32(128, N);
    if (threadIdx.x == 0) {
        const long long t0 = clock64();
        for (int i = 0; i < ITERS; ++i) {
            const uint64_t bd = smem_desc_k_sw128(sb + (i & 3) * 32);
            const uint32_t d = tm + (i % NACC) * N;                 // accumulators in cols [0, NACC*N)
            if (TS) tc_mma_ts(d, tm + 256 + (i & 3) * 8, bd, idesc, i >= NACC);
            else mma_ss(d, smem_desc_k_sw128(sa + (i & 3) * 32), bd, idesc, i >= NACC);
        }
        tc_commit(&bar);
        mbar_wait(&bar, 0);
        cycles[blockIdx.x] = clock64() - t0;
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) tmem_dealloc<512>(tm);
}

template <int N, bool TS, int NACC>
static void run(long long* d) {
    const int smem = 16384 + 32768 + 1024;
    cudaFuncSetAttribute(kern<N, TS, NACC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    kern<N, TS, NACC><<<148, 128, smem>>>(d);
    cudaDeviceSynchronize();
    kern<N, TS, NACC><<<148, 128, smem>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    long long c[148];
    cudaMemcpy(c, d, sizeof c, cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int i = 0; i < 148; ++i) mx = c[i] > mx ? c[i] : mx;
    const double clk = (double)mx / ITERS;
    printf("%s M=128 N=%3d NACC=%d: %.1f clk/MMA, %.0f weights(A elems)/clk/SM, %.0f MAC/clk/SM (%s)\n",
           TS ? "TS" : "SS", N, NACC, clk, 128.0 * 16 / clk, 128.0 * N * 16 / clk, cudaGetErrorString(e));
}

int main() {
    long long* d;
    cudaMalloc(&d, 148 * sizeof(long long));
    run<16, true, 1>(d); run<16, true, 4>(d); run<16, true, 8>(d);
    run<16, false, 1>(d); run<16, false, 4>(d); run<16, false, 8>(d);
    run<32, true, 1>(d); run<32, true, 4>(d);
    run<32, false, 1>(d); run<32, false, 4>(d);
    run<64, true, 1>(d); run<64, true, 2>(d);
    run<64, false, 1>(d); run<64, false, 2>(d);
    return 0;
}
