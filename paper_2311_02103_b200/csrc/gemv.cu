// gemv.cu -- small-n path: bandwidth-bound q4f16 GEMV on CUDA cores, and the
// bit-exact dequant export kernel.
//
// y[t][j] = sum_k x[t][k] * W(k, j),  W(k, j) = (q(k,j) - 7) * s(k/32, j)
// (dequant fused into the matmul as one kernel; the token
// count n stays a runtime argument while K, N shape the launch).
//
// Work decomposition:
//   * an "item" = 4 consecutive output rows x one 1024-k chunk; lane l of the
//     warp owns group g = 32*chunk + l, i.e. one 16-byte LDG.128 of codes per
//     row (= exactly one 32-code group with one scale) -- 128-bit coalesced
//     loads, 512 contiguous bytes per warp instruction;
//   * each CTA owns a contiguous block of rows (balanced to +-1 row block);
//     its 8 warps stride over the (row-block, chunk) items;
//   * per lane: sum_{32 k} (q-7) * x in fp32 with FHFMA (fp16 x fp16 -> fp32
//     accumulate, exact products), times the group scale (one FFMA);
//   * warp-shuffle butterfly reduction across the 32 groups of a chunk, then a
//     fixed-order sum over chunks from shared memory: deterministic;
//   * x (n x K fp16) is staged once per CTA in shared memory, swizzled so the
//     4 LDS.128 a lane issues per group are bank-conflict free;
//   * PDL: the first batch of weight loads is issued before
//     griddepcontrol.wait (weights never depend on the previous kernel), so
//     back-to-back GEMVs overlap their latency ramps.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include "internal.h"
#include "ptx.cuh"
#include "q4_unpack.cuh"
#include "knobs.h"

namespace rq4 {

constexpr int kGemvThreads = 256;
constexpr int kGemvWarps = kGemvThreads / 32;
constexpr int kGemvRows = 4;    // rows per item: x reuse factor
constexpr int kGemvBatch = 2;   // items in flight per warp
constexpr int kGemvCtasPerSM = 2;
constexpr size_t kGemvSmemCap = 100 * 1024;

struct GemvArgs {
    const uint16_t* x;     // [NT][K] fp16 (already offset to the first token)
    const uint32_t* w;     // [N][K/8]
    const uint16_t* s;     // [N][K/32]
    uint16_t* y;           // [NT][N] fp16
    int64_t K;
    int64_t N;
};

__device__ __forceinline__ int xs_slot(int g, int q) { return g * 4 + (q ^ ((g >> 1) & 3)); }

template <int NT>
__global__ void __launch_bounds__(kGemvThreads, kGemvCtasPerSM)
q4_decode_generic_kernel(const __grid_constant__ GemvArgs a) {
    extern __shared__ __align__(16) uint8_t smem[];
    uint4* xs = reinterpret_cast<uint4*>(smem);
    const int64_t K = a.K, N = a.N;
    const int K8 = static_cast<int>(K / 8);
    const int G = static_cast<int>(K / kGroup);
    const int C = (G + 31) / 32;
    const int64_t RB = (N + kGemvRows - 1) / kGemvRows;
    const int64_t rb0 = static_cast<int64_t>(blockIdx.x) * RB / gridDim.x;
    const int64_t rb1 = static_cast<int64_t>(blockIdx.x + 1) * RB / gridDim.x;
    const int nrb = static_cast<int>(rb1 - rb0);
    const int items = nrb * C;
    float* part = reinterpret_cast<float*>(smem + static_cast<size_t>(NT) * K * 2);
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint64_t pol = policy_evict_first();

    pdl_launch_dependents();

    uint4 cw[kGemvBatch][kGemvRows];
    uint16_t sc[kGemvBatch][kGemvRows];
    auto load_item = [&](int it, int b) {
        const int rbl = it / C;
        const int g = (it - rbl * C) * 32 + lane;
#pragma unroll
        for (int r = 0; r < kGemvRows; ++r) {
            const int64_t row = (rb0 + rbl) * kGemvRows + r;
            if (g < G && row < N) {
                cw[b][r] = ldg_stream_v4(a.w + row * K8 + g * 4, pol);
                sc[b][r] = ldg_stream_u16(a.s + row * G + g, pol);
            } else {
                cw[b][r] = make_uint4(0u, 0u, 0u, 0u);
                sc[b][r] = 0;
            }
        }
    };

    // Prologue: weights for the first batch, before waiting on the producer of x.
#pragma unroll
    for (int b = 0; b < kGemvBatch; ++b)
        if (warp + b * kGemvWarps < items) load_item(warp + b * kGemvWarps, b);

    pdl_wait();
    {
        const uint4* xg = reinterpret_cast<const uint4*>(a.x);
        for (int i = threadIdx.x; i < NT * K8; i += kGemvThreads) {
            const int t = i / K8;
            const int m = i - t * K8;
            xs[t * K8 + xs_slot(m >> 2, m & 3)] = xg[static_cast<int64_t>(t) * K8 + m];
        }
    }
    __syncthreads();

    for (int it = warp; it < items; it += kGemvBatch * kGemvWarps) {
        if (it != warp) {
#pragma unroll
            for (int b = 0; b < kGemvBatch; ++b)
                if (it + b * kGemvWarps < items) load_item(it + b * kGemvWarps, b);
        }
#pragma unroll
        for (int b = 0; b < kGemvBatch; ++b) {
            const int itb = it + b * kGemvWarps;
            if (itb >= items) break;                       // warp-uniform
            const int rbl = itb / C;
            const int c = itb - rbl * C;
            const int g = c * 32 + lane;
            float acc[kGemvRows][NT];
#pragma unroll
            for (int r = 0; r < kGemvRows; ++r)
#pragma unroll
                for (int t = 0; t < NT; ++t) acc[r][t] = 0.f;
            if (g < G) {
                uint4 xv[NT][4];
#pragma unroll
                for (int t = 0; t < NT; ++t)
#pragma unroll
                    for (int q = 0; q < 4; ++q) xv[t][q] = xs[t * K8 + xs_slot(g, q)];
#pragma unroll
                for (int r = 0; r < kGemvRows; ++r) {
                    const uint32_t words[4] = {cw[b][r].x, cw[b][r].y, cw[b][r].z, cw[b][r].w};
                    float gacc[NT];
#pragma unroll
                    for (int t = 0; t < NT; ++t) gacc[t] = 0.f;
#pragma unroll
                    for (int wi = 0; wi < 4; ++wi) {
                        __half2 cc[4];
                        unpack_centered_interleaved(words[wi], cc);
                        const uint32_t c0 = h2_as_u32(cc[0]), c1 = h2_as_u32(cc[1]);
                        const uint32_t c2 = h2_as_u32(cc[2]), c3 = h2_as_u32(cc[3]);
#pragma unroll
                        for (int t = 0; t < NT; ++t) {
                            // x pairs: X.x = (k0,k1) X.y = (k2,k3) X.z = (k4,k5) X.w = (k6,k7)
                            const uint4 X = xv[t][wi];
                            const uint32_t X0 = X.x, X1 = X.y, X2 = X.z, X3 = X.w;
                            float s0 = gacc[t];
                            s0 = fhfma(lo16(c0), lo16(X0), s0);   // k0
                            s0 = fhfma(lo16(c1), hi16(X0), s0);   // k1
                            s0 = fhfma(lo16(c2), lo16(X1), s0);   // k2
                            s0 = fhfma(lo16(c3), hi16(X1), s0);   // k3
                            s0 = fhfma(hi16(c0), lo16(X2), s0);   // k4
                            s0 = fhfma(hi16(c1), hi16(X2), s0);   // k5
                            s0 = fhfma(hi16(c2), lo16(X3), s0);   // k6
                            s0 = fhfma(hi16(c3), hi16(X3), s0);   // k7
                            gacc[t] = s0;
                        }
                    }
                    const float s = __half2float(__ushort_as_half(sc[b][r]));
#pragma unroll
                    for (int t = 0; t < NT; ++t) acc[r][t] = s * gacc[t];
                }
            }
#pragma unroll
            for (int r = 0; r < kGemvRows; ++r)
#pragma unroll
                for (int t = 0; t < NT; ++t) {
                    float v = acc[r][t];
#pragma unroll
                    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
                    acc[r][t] = v;
                }
            if (lane == 0) {
#pragma unroll
                for (int r = 0; r < kGemvRows; ++r)
#pragma unroll
                    for (int t = 0; t < NT; ++t)
                        part[((rbl * C + c) * kGemvRows + r) * NT + t] = acc[r][t];
            }
        }
    }
    __syncthreads();

    // Fixed-order sum over the chunks of each (row, token); fp32 -> fp16 RNE.
    for (int o = threadIdx.x; o < nrb * kGemvRows * NT; o += kGemvThreads) {
        const int t = o % NT;
        const int rr = o / NT;                 // rbl * R + r
        const int rbl = rr / kGemvRows;
        const int r = rr - rbl * kGemvRows;
        const int64_t row = (rb0 + rbl) * kGemvRows + r;
        if (row >= N) continue;
        float sum = 0.f;
        for (int c = 0; c < C; ++c) sum += part[((rbl * C + c) * kGemvRows + r) * NT + t];
        a.y[static_cast<int64_t>(t) * N + row] = __half_as_ushort(__float2half_rn(sum));
    }
}

static size_t gemv_smem_bytes(int nt, int64_t K, int64_t N, int grid) {
    const int64_t RB = (N + kGemvRows - 1) / kGemvRows;
    const int64_t nrb_max = (RB + grid - 1) / grid;
    const int64_t C = (K / kGroup + 31) / 32;
    return static_cast<size_t>(nt) * K * 2 + static_cast<size_t>(nrb_max * C * kGemvRows * nt) * 4;
}

static int gemv_grid(int64_t N) {
    const int64_t RB = (N + kGemvRows - 1) / kGemvRows;
    const int64_t gmax = static_cast<int64_t>(kGemvCtasPerSM) * num_sms();
    return static_cast<int>(RB < gmax ? RB : gmax);
}

bool gemv_fits(int nt, int64_t K) {
    // x for nt tokens must fit the per-CTA budget next to the partial sums
    // (two CTAs per SM); checked against the largest N the partials allow.
    return static_cast<size_t>(nt) * K * 2 + 16 * 1024 <= kGemvSmemCap;
}

template <int NT>
static int launch_gemv_nt(const GemvArgs& a, bool pdl, cudaStream_t stream) {
    const int grid = gemv_grid(a.N);
    const size_t smem = gemv_smem_bytes(NT, a.K, a.N, grid);
    if (smem > 227 * 1024) return static_cast<int>(cudaErrorInvalidConfiguration);
    const cudaError_t e = ensure_kernel_attrs(reinterpret_cast<const void*>(q4_decode_generic_kernel<NT>), 227 * 1024);
    if (e != cudaSuccess) return static_cast<int>(e);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kGemvThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return static_cast<int>(cudaLaunchKernelEx(&cfg, q4_decode_generic_kernel<NT>, a));
}

int launch_gemv(const uint16_t* x, int64_t n, int64_t K, int64_t N, const uint32_t* w,
                const uint16_t* s, uint16_t* y, int nt, bool pdl, cudaStream_t stream) {
    // Decode kernels: the streamed CUDA-core kernel (gemv_stream.cu) for
    // n <= 2 when the shape fits it, else the generic one below (any K % 32 == 0,
    // up to 8 tokens per launch).  The experiments build can pin one of the
    // measured-slower variants kept in experiments/csrc (RELAX_Q4_GEMV_IMPL =
    // mma | bdmma | row | v1).
    int impl = 0;
#ifdef RQ4_EXPERIMENTS
    static const int impl_env = knob_is("RELAX_Q4_GEMV_IMPL", "mma") ? 1 : knob_is("RELAX_Q4_GEMV_IMPL", "row") ? 2
                              : knob_is("RELAX_Q4_GEMV_IMPL", "v1") ? 3 : knob_is("RELAX_Q4_GEMV_IMPL", "bdmma") ? 4 : 0;
    impl = impl_env;
    if (impl == 4 && n == 1 && gemv_bdmma_ok(K, N))
        return launch_gemv_mma(x, n, K, N, w, s, y, pdl, stream, true);
    if (n == 1 && impl == 2 && gemv_row_ok(K))
        return launch_gemv_row(x, n, K, N, w, s, y, pdl, stream);
    if (impl == 1 && nt <= 2 && gemv_mma_ok(n >= 2 ? 2 : 1, K, N))
        return launch_gemv_mma(x, n, K, N, w, s, y, pdl, stream);
#endif
    if (impl <= 1 && nt <= 2 && gemv_stream_ok(nt, K, N))
        return launch_gemv_stream(x, n, K, N, w, s, y, pdl, stream);
    if (nt < 1 || nt > kGemvMaxNT) nt = kGemvMaxNT;
    for (int64_t t0 = 0; t0 < n; t0 += nt) {
        const int cnt = static_cast<int>((n - t0) < nt ? (n - t0) : nt);
        GemvArgs a{x + t0 * K, w, s, y + t0 * N, K, N};
        int rc = 0;
        switch (cnt) {
            case 1: rc = launch_gemv_nt<1>(a, pdl, stream); break;
            case 2: rc = launch_gemv_nt<2>(a, pdl, stream); break;
            case 3: rc = launch_gemv_nt<3>(a, pdl, stream); break;
            case 4: rc = launch_gemv_nt<4>(a, pdl, stream); break;
            case 5: rc = launch_gemv_nt<5>(a, pdl, stream); break;
            case 6: rc = launch_gemv_nt<6>(a, pdl, stream); break;
            case 7: rc = launch_gemv_nt<7>(a, pdl, stream); break;
            default: rc = launch_gemv_nt<8>(a, pdl, stream); break;
        }
        if (rc != 0) return rc;
    }
    return 0;
}

// ---------------------------------------------------------------------------
// Dequant export: w_out[j][k] = fp16_RNE((q - 7) * s), bit-exact (reading 5).
// One thread per 32-code group: one LDG.128 of codes, one scale, 64 B out.
__global__ void __launch_bounds__(256)
dequant_q4_kernel(const uint32_t* __restrict__ w, const uint16_t* __restrict__ s,
                  int64_t K, int64_t N, uint16_t* __restrict__ out) {
    const int64_t G = K / kGroup;
    const int64_t total = N * G;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t row = i / G;
        const int64_t g = i - row * G;
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(w + row * (K / 8) + g * 4));
        const __half sh = __ushort_as_half(__ldg(s + row * G + g));
        const __half2 s2 = __halves2half2(sh, sh);
        const uint32_t words[4] = {v.x, v.y, v.z, v.w};
        uint4* dst = reinterpret_cast<uint4*>(out + row * K + g * kGroup);
#pragma unroll
        for (int wi = 0; wi < 4; ++wi) {
            uint32_t o[4];
            dequant_word_natural(words[wi], s2, o);
            dst[wi] = make_uint4(o[0], o[1], o[2], o[3]);
        }
    }
}

int launch_dequant(const uint32_t* w, const uint16_t* s, int64_t K, int64_t N,
                   uint16_t* out, cudaStream_t stream) {
    const int64_t total = N * (K / kGroup);
    if (total == 0) return 0;
    int64_t blocks = (total + 255) / 256;
    const int64_t bmax = 8 * static_cast<int64_t>(num_sms());
    if (blocks > bmax) blocks = bmax;
    dequant_q4_kernel<<<static_cast<unsigned>(blocks), 256, 0, stream>>>(w, s, K, N, out);
    return static_cast<int>(cudaGetLastError());
}

}  // namespace rq4
