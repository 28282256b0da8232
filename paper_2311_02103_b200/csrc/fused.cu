// fused.cu -- the RMSNorm prologue as its own kernel, for the tensor-core
// path of relax_q4_matmul_fused (the decode GEMV normalises x in registers).
//
// Llama RMSNorm (include/relax_q4.h RELAX_OP_RMSNORM_X):
//   r_t = 1 / sqrt(mean_k x[t][k]^2 + eps)     (fp32)
//   xn[t][k] = fp16_RNE(fp16_RNE(x[t][k] * r_t) * gamma[k])
// One CTA per token row; 16-B vector loads; fixed-order block reduction, so
// the result is deterministic.  HBM-bound (4 bytes per element moved).
#include <cstdint>
#include <cuda_fp16.h>
#include "internal.h"
#include "ptx.cuh"

namespace rq4 {

constexpr int kRmsThreads = 256;

__global__ void __launch_bounds__(kRmsThreads) rmsnorm_kernel(const uint16_t* __restrict__ x, int64_t K,
                                                              const uint16_t* __restrict__ gamma, float eps,
                                                              uint16_t* __restrict__ out) {
    __shared__ float red[kRmsThreads / 32];
    pdl_wait();                                  // x may come from the previous kernel
    pdl_launch_dependents();
    const int64_t t = blockIdx.x;
    const uint4* xv = reinterpret_cast<const uint4*>(x + t * K);
    const uint4* gv = reinterpret_cast<const uint4*>(gamma);
    uint4* ov = reinterpret_cast<uint4*>(out + t * K);
    const int64_t nv = K / 8;
    float acc = 0.f;
    for (int64_t i = threadIdx.x; i < nv; i += kRmsThreads) {
        const uint4 v = xv[i];
        const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const float2 f = __half22float2(u32_as_h2(w4[u]));
            acc = fmaf(f.x, f.x, acc);
            acc = fmaf(f.y, f.y, acc);
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    float tot = 0.f;
#pragma unroll
    for (int w = 0; w < kRmsThreads / 32; ++w) tot += red[w];
    const float r = 1.0f / sqrtf(tot / static_cast<float>(K) + eps);
    for (int64_t i = threadIdx.x; i < nv; i += kRmsThreads) {
        const uint4 v = xv[i];
        const uint4 g = gv[i];
        uint32_t w4[4] = {v.x, v.y, v.z, v.w};
        const uint32_t g4[4] = {g.x, g.y, g.z, g.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const float2 f = __half22float2(u32_as_h2(w4[u]));
            const __half2 hn = __floats2half2_rn(f.x * r, f.y * r);
            w4[u] = h2_as_u32(__hmul2(hn, u32_as_h2(g4[u])));
        }
        ov[i] = make_uint4(w4[0], w4[1], w4[2], w4[3]);
    }
}

int launch_rmsnorm(const uint16_t* x, int64_t n, int64_t K, const uint16_t* gamma, float eps,
                   uint16_t* out, bool pdl, cudaStream_t stream) {
    if (n <= 0) return 0;
    if (K % 8 != 0) return static_cast<int>(cudaErrorInvalidValue);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(n));
    cfg.blockDim = dim3(kRmsThreads);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return static_cast<int>(cudaLaunchKernelEx(&cfg, rmsnorm_kernel, x, K, gamma, eps, out));
}

}  // namespace rq4
