// attention.cu -- decode attention over a symbolic KV length (SURVEY §8(f)
// F4; "the KV-cache context length" as a dynamic dimension
// single-batch Llama-2 decode), and the KV-cache append.
//
// One query token per sequence (reading 21; include/relax_q4.h):
//   s_j = (q . k_j) / sqrt(D),  p = softmax_j<len[b](s),  out = sum_j p_j v_j
// with grouped-query attention (query head h reads kv head h / G, G = Hq/Hkv)
// and fp16 q, caches and output, fp32 arithmetic.
//
// HBM-bound: every cached key and value of every sequence is read once
// (2 * len * Hkv * D * 2 bytes per sequence).  Split-KV ("flash decoding"):
//   attn_partial_kernel  grid (chunks of 256 keys, Hkv, batch), 256 threads:
//       the G query heads of one kv head against one chunk -- an 8-lane group
//       scores one key per step (coalesced 32-B slices of the key row, q
//       broadcast from shared memory, 3-shuffle reduction),
//       per-head max / exp / sum by warp reductions, then p . V with 64
//       threads per key row (coalesced half2 loads) in 4 key quarters summed
//       in fixed order; writes the chunk's (m, l, o) to the workspace;
//   attn_combine_kernel  grid (Hq, batch), 128 threads: rescales and sums the
//       chunks in fixed order -> fp16.  Deterministic.
// Both wait for the previous kernel (griddepcontrol.wait) before reading.
#include <cuda_fp16.h>
#include "internal.h"
#include "ptx.cuh"

namespace rq4 {

constexpr int kAttD = 128;          // head_dim (every Llama-2 size)
constexpr int kAttChunk = 256;      // keys per partial CTA
constexpr int kAttThreads = 256;
constexpr int kAttMaxG = 8;         // query heads per kv head

struct AttArgs {
    const uint16_t* q;              // [batch][Hq][D]
    const uint16_t* k;              // [batch][Hkv][Lmax][D]
    const uint16_t* v;
    const int32_t* lens;            // [batch]
    uint16_t* out;                  // [batch][Hq][D]
    float* part_o;                  // [batch][Hq][nch][D]
    float* part_ml;                 // [batch][Hq][nch][2]  (max, sum)
    int64_t Lmax;
    int Hq, Hkv, nch;
    int chunk;                      // keys per partial CTA (multiple of 32, <= kAttChunk)
    float scale;                    // 1 / sqrt(D)
};

template <int G>
__global__ void __launch_bounds__(kAttThreads) attn_partial_kernel(const __grid_constant__ AttArgs a) {
    __shared__ __align__(16) float qs[G][kAttD];
    __shared__ float sc[G][kAttChunk];
    __shared__ float red[(G <= 2) ? 1 : 4][G][kAttD];
    __shared__ float red16[(G <= 2) ? 16 : 1][G][kAttD];
    __shared__ float ml[G][2];
    pdl_launch_dependents();
    pdl_wait();                                          // q and the caches come from earlier kernels
    const int b = blockIdx.z, g = blockIdx.y, c = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int L = a.lens[b];
    const int CH = a.chunk;
    const int k0 = c * CH;
    if (k0 >= L) return;                                 // the combine only reads chunks below len
    const int nk = L - k0 < CH ? L - k0 : CH;
    // q of the G heads of this kv head, fp32
    for (int i = tid; i < G * kAttD / 8; i += kAttThreads) {
        const int gg = i / (kAttD / 8), d8 = i - gg * (kAttD / 8);
        const uint4 v4 = *reinterpret_cast<const uint4*>(a.q + (static_cast<int64_t>(b) * a.Hq + g * G + gg) * kAttD + d8 * 8);
        const uint32_t w4[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const float2 f = __half22float2(u32_as_h2(w4[u]));
            qs[gg][d8 * 8 + 2 * u] = f.x;
            qs[gg][d8 * 8 + 2 * u + 1] = f.y;
        }
    }
    __syncthreads();
    const int64_t kvbase = (static_cast<int64_t>(b) * a.Hkv + g) * a.Lmax;
    if constexpr (G >= 4) {
        // scores, G >= 4 (GQA): thread t scores key k0 + t for all G heads (16-B
        // loads of its key row, q broadcast from shared memory) -- G dots per
        // key row read, no shuffles (measured faster than the 8-lane groups at
        // G = 8: 28 vs 51 us for the 70B heads at L = 4096)
        float acc[G];
#pragma unroll
        for (int gg = 0; gg < G; ++gg) acc[gg] = 0.f;
        if (tid < nk) {
            const uint4* kp = reinterpret_cast<const uint4*>(a.k + (kvbase + k0 + tid) * kAttD);
#pragma unroll 4
            for (int d8 = 0; d8 < kAttD / 8; ++d8) {
                const uint4 v4 = __ldg(kp + d8);
                const uint32_t w4[4] = {v4.x, v4.y, v4.z, v4.w};
                float kf[8];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const float2 f = __half22float2(u32_as_h2(w4[u]));
                    kf[2 * u] = f.x;
                    kf[2 * u + 1] = f.y;
                }
#pragma unroll
                for (int gg = 0; gg < G; ++gg) {
                    const float4 qa = *reinterpret_cast<const float4*>(&qs[gg][d8 * 8]);
                    const float4 qb = *reinterpret_cast<const float4*>(&qs[gg][d8 * 8 + 4]);
                    float s2 = acc[gg];
                    s2 = fmaf(qa.x, kf[0], s2); s2 = fmaf(qa.y, kf[1], s2); s2 = fmaf(qa.z, kf[2], s2);
                    s2 = fmaf(qa.w, kf[3], s2); s2 = fmaf(qb.x, kf[4], s2); s2 = fmaf(qb.y, kf[5], s2);
                    s2 = fmaf(qb.z, kf[6], s2); s2 = fmaf(qb.w, kf[7], s2);
                    acc[gg] = s2;
                }
            }
        }
#pragma unroll
        for (int gg = 0; gg < G; ++gg) sc[gg][tid] = tid < nk ? acc[gg] * a.scale : -INFINITY;
    } else {
        // scores, G <= 2: 8-lane groups, one key per group per step (a group reads
        // the key's 256-B row as 8 x 32 B, so a warp reads 4 consecutive rows =
        // 1 KB contiguous); lane `sub` holds d in [16 sub, 16 sub + 16); the
        // partial dots are reduced over the group with 3 shuffles
        const int grp = lane >> 3, sub = lane & 7;
        // all 8 steps' key slices loaded first (16 x 16 B per lane in flight),
        // then the dots: the phase is one memory round trip, not eight
        uint4 kv[8][2];
#pragma unroll
        for (int it = 0; it < 8; ++it) {
            const int t = warp * 4 + grp + 32 * it;
            if (t < nk) {
                const uint4* kp = reinterpret_cast<const uint4*>(a.k + (kvbase + k0 + t) * kAttD + sub * 16);
                kv[it][0] = __ldg(kp);
                kv[it][1] = __ldg(kp + 1);
            } else {
                kv[it][0] = make_uint4(0u, 0u, 0u, 0u);
                kv[it][1] = make_uint4(0u, 0u, 0u, 0u);
            }
        }
#pragma unroll
        for (int it = 0; it < 8; ++it) {
            const int t = warp * 4 + grp + 32 * it;
            const uint32_t w8[8] = {kv[it][0].x, kv[it][0].y, kv[it][0].z, kv[it][0].w,
                                    kv[it][1].x, kv[it][1].y, kv[it][1].z, kv[it][1].w};
            float kf[16];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const float2 f = __half22float2(u32_as_h2(w8[u]));
                kf[2 * u] = f.x;
                kf[2 * u + 1] = f.y;
            }
#pragma unroll
            for (int gg = 0; gg < G; ++gg) {
                const float4* qp = reinterpret_cast<const float4*>(&qs[gg][sub * 16]);
                float s2 = 0.f;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const float4 qv = qp[i];
                    s2 = fmaf(qv.x, kf[4 * i], s2);
                    s2 = fmaf(qv.y, kf[4 * i + 1], s2);
                    s2 = fmaf(qv.z, kf[4 * i + 2], s2);
                    s2 = fmaf(qv.w, kf[4 * i + 3], s2);
                }
                s2 += __shfl_xor_sync(0xffffffffu, s2, 1);
                s2 += __shfl_xor_sync(0xffffffffu, s2, 2);
                s2 += __shfl_xor_sync(0xffffffffu, s2, 4);
                if (sub == 0) sc[gg][t] = t < nk ? s2 * a.scale : -INFINITY;
            }
        }
    }
    __syncthreads();
    // per-head max, exp, sum: warp gg owns head gg (G <= 8 warps)
    if (warp < G) {
        float m = -INFINITY;
        for (int t = lane; t < kAttChunk; t += 32) m = fmaxf(m, sc[warp][t]);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
        float l = 0.f;
        for (int t = lane; t < kAttChunk; t += 32) {
            const float p = t < nk ? __expf(sc[warp][t] - m) : 0.f;
            sc[warp][t] = p;
            l += p;
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) l += __shfl_xor_sync(0xffffffffu, l, off);
        if (lane == 0) { ml[warp][0] = m; ml[warp][1] = l; }
    }
    __syncthreads();
    if constexpr (G <= 2) {
        // p . V, G <= 2: thread (key group kg, d8) accumulates columns 8 d8 .. 8 d8 + 7
        // over keys kg, kg + 16, ... -- 16-B loads, 16 threads per value row
        const int d8 = tid & 15, kg = tid >> 4;
        float o[G][8];
#pragma unroll
        for (int gg = 0; gg < G; ++gg)
#pragma unroll
            for (int i = 0; i < 8; ++i) o[gg][i] = 0.f;
        const uint4* vp = reinterpret_cast<const uint4*>(a.v + (kvbase + k0) * kAttD) + d8;
#pragma unroll 8
        for (int t = kg; t < nk; t += 16) {
            const uint4 v4 = __ldg(vp + static_cast<int64_t>(t) * (kAttD / 8));
            const uint32_t w4[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
            for (int gg = 0; gg < G; ++gg) {
                const float p = sc[gg][t];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const float2 f = __half22float2(u32_as_h2(w4[u]));
                    o[gg][2 * u] = fmaf(p, f.x, o[gg][2 * u]);
                    o[gg][2 * u + 1] = fmaf(p, f.y, o[gg][2 * u + 1]);
                }
            }
        }
        // the 16 key groups' partial rows go through shared memory and are
        // summed in fixed order below
#pragma unroll
        for (int gg = 0; gg < G; ++gg)
#pragma unroll
            for (int i = 0; i < 8; ++i) red16[kg][gg][d8 * 8 + i] = o[gg][i];
    } else {
    // p . V: thread (quarter, d2) accumulates columns 2*d2, 2*d2+1 over keys
    // quarter, quarter + 4, ... (a key row is 64 threads x 4 B, coalesced)
    {
        const int d2 = tid & 63, qt = tid >> 6;
        float o[G][2];
#pragma unroll
        for (int gg = 0; gg < G; ++gg) { o[gg][0] = 0.f; o[gg][1] = 0.f; }
        const uint32_t* vp = reinterpret_cast<const uint32_t*>(a.v + (kvbase + k0) * kAttD) + d2;
#pragma unroll 4
        for (int t = qt; t < nk; t += 4) {
            const float2 vf = __half22float2(u32_as_h2(__ldg(vp + static_cast<int64_t>(t) * (kAttD / 2))));
#pragma unroll
            for (int gg = 0; gg < G; ++gg) {
                const float p = sc[gg][t];
                o[gg][0] = fmaf(p, vf.x, o[gg][0]);
                o[gg][1] = fmaf(p, vf.y, o[gg][1]);
            }
        }
#pragma unroll
        for (int gg = 0; gg < G; ++gg) { red[qt][gg][2 * d2] = o[gg][0]; red[qt][gg][2 * d2 + 1] = o[gg][1]; }
    }
    }
    __syncthreads();
    for (int i = tid; i < G * kAttD; i += kAttThreads) {
        const int gg = i / kAttD, d = i - gg * kAttD;
        float s;
        if constexpr (G <= 2) {
            s = 0.f;
#pragma unroll
            for (int kg = 0; kg < 16; ++kg) s += red16[kg][gg][d];
        } else {
            s = ((red[0][gg][d] + red[1][gg][d]) + red[2][gg][d]) + red[3][gg][d];
        }
        const int64_t row = (static_cast<int64_t>(b) * a.Hq + g * G + gg) * a.nch + c;
        a.part_o[row * kAttD + d] = s;
        if (d == 0) { a.part_ml[row * 2] = ml[gg][0]; a.part_ml[row * 2 + 1] = ml[gg][1]; }
    }
}

__global__ void __launch_bounds__(kAttD) attn_combine_kernel(const __grid_constant__ AttArgs a) {
    __shared__ float wts[kAttD * 2];                    // per-chunk weights exp(m_c - M) (<= 256 chunks)
    __shared__ float red[kAttD / 32];
    pdl_launch_dependents();
    pdl_wait();
    const int b = blockIdx.y, h = blockIdx.x, d = threadIdx.x;
    const int L = a.lens[b];
    uint16_t* dst = a.out + (static_cast<int64_t>(b) * a.Hq + h) * kAttD + d;
    if (L <= 0) { *dst = 0; return; }
    const int nc = (L + a.chunk - 1) / a.chunk;          // <= 2 * kAttD (chunk >= 64, L <= 16384)
    const int64_t base = (static_cast<int64_t>(b) * a.Hq + h) * a.nch;
    // all chunk maxima in parallel (thread c), the max by a block reduction
    float mloc = -INFINITY, m2 = -INFINITY;
    if (d < nc) mloc = a.part_ml[(base + d) * 2];
    if (d + kAttD < nc) m2 = a.part_ml[(base + d + kAttD) * 2];
    float M = fmaxf(mloc, m2);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
    if ((d & 31) == 0) red[d >> 5] = M;
    __syncthreads();
    M = fmaxf(fmaxf(red[0], red[1]), fmaxf(red[2], red[3]));
    if (d < nc) wts[d] = __expf(mloc - M);
    if (d + kAttD < nc) wts[d + kAttD] = __expf(m2 - M);
    __syncthreads();
    float num = 0.f, den = 0.f;
#pragma unroll 8
    for (int c = 0; c < nc; ++c) {                       // fixed order: deterministic
        const float w = wts[c];
        den = fmaf(w, a.part_ml[(base + c) * 2 + 1], den);
        num = fmaf(w, a.part_o[(base + c) * kAttD + d], num);
    }
    *dst = __half_as_ushort(__float2half_rn(num / den));
}

__global__ void __launch_bounds__(64) kv_append_kernel(const uint16_t* __restrict__ kn, const uint16_t* __restrict__ vn,
                                                       const int32_t* __restrict__ pos, int64_t Lmax, int Hkv,
                                                       uint16_t* __restrict__ kc, uint16_t* __restrict__ vc) {
    pdl_launch_dependents();
    pdl_wait();
    const int b = blockIdx.y, h = blockIdx.x, i = threadIdx.x;      // i: one 4-B pair of the row
    const int p = pos[b];
    if (p < 0 || p >= Lmax) return;                                  // out of range: nothing written
    const int64_t src = (static_cast<int64_t>(b) * Hkv + h) * kAttD;
    const int64_t dst = ((static_cast<int64_t>(b) * Hkv + h) * Lmax + p) * kAttD;
    reinterpret_cast<uint32_t*>(kc + dst)[i] = reinterpret_cast<const uint32_t*>(kn + src)[i];
    reinterpret_cast<uint32_t*>(vc + dst)[i] = reinterpret_cast<const uint32_t*>(vn + src)[i];
}

static cudaLaunchConfig_t att_cfg(dim3 grid, dim3 block, bool pdl, cudaStream_t st, cudaLaunchAttribute* attr) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cfg;
}

// Keys per partial CTA: enough CTAs for two per SM when the grid is short
// (64..256, a multiple of 64; 7B decode with a 512-key cache 656 -> 728
// tok/s), else 256.
static int attn_chunk(int64_t batch, int64_t Hkv, int64_t G, int64_t Lmax) {
    // (the combine holds <= 256 chunk weights: chunk 256 for Lmax <= 65536, and
    // smaller chunks only while the grid is short, i.e. for short caches)
    if (G >= 4 || Lmax > 16384) return kAttChunk;        // thread-per-key scoring wants full chunks
    const int64_t target = 2 * static_cast<int64_t>(num_sms());
    int ch = kAttChunk;
    while (ch > 64 && batch * Hkv * ((Lmax + ch - 1) / ch) < target) ch -= 64;
    return ch;
}

size_t attn_workspace_bytes(int64_t batch, int64_t Hq, int64_t Lmax) {
    // sized for the smallest chunk any launch with these (batch, Lmax) may pick
    const int64_t nch = (Lmax + 63) / 64;
    return static_cast<size_t>(batch * Hq * nch) * (kAttD + 2) * 4;
}

template <int G>
static int launch_partial(const AttArgs& a, int64_t batch, bool pdl, cudaStream_t st) {
    cudaLaunchAttribute attr[1];
    cudaLaunchConfig_t cfg = att_cfg(dim3(static_cast<unsigned>(a.nch), static_cast<unsigned>(a.Hkv),
                                          static_cast<unsigned>(batch)), dim3(kAttThreads), pdl, st, attr);
    return static_cast<int>(cudaLaunchKernelEx(&cfg, attn_partial_kernel<G>, a));
}

int launch_attention_decode(const uint16_t* q, const uint16_t* k, const uint16_t* v, const int32_t* lens,
                            int64_t batch, int64_t Hq, int64_t Hkv, int64_t Lmax, uint16_t* out, void* ws,
                            bool pdl, cudaStream_t st) {
    AttArgs a;
    a.q = q; a.k = k; a.v = v; a.lens = lens; a.out = out;
    a.Lmax = Lmax;
    a.Hq = static_cast<int>(Hq);
    a.Hkv = static_cast<int>(Hkv);
    a.chunk = attn_chunk(batch, Hkv, Hq / Hkv, Lmax);
    a.nch = static_cast<int>((Lmax + a.chunk - 1) / a.chunk);
    a.scale = 0.08838834764831845f;                      // 1 / sqrt(128)
    a.part_o = static_cast<float*>(ws);
    a.part_ml = a.part_o + static_cast<size_t>(batch * Hq * a.nch) * kAttD;
    int rc = 0;
    if (a.nch > 0) {
        switch (Hq / Hkv) {
            case 1: rc = launch_partial<1>(a, batch, pdl, st); break;
            case 2: rc = launch_partial<2>(a, batch, pdl, st); break;
            case 4: rc = launch_partial<4>(a, batch, pdl, st); break;
            case 8: rc = launch_partial<8>(a, batch, pdl, st); break;
            default: return static_cast<int>(cudaErrorInvalidValue);
        }
        if (rc) return rc;
    }
    cudaLaunchAttribute attr[1];
    cudaLaunchConfig_t cfg = att_cfg(dim3(static_cast<unsigned>(Hq), static_cast<unsigned>(batch)), dim3(kAttD),
                                     pdl, st, attr);
    return static_cast<int>(cudaLaunchKernelEx(&cfg, attn_combine_kernel, a));
}

int launch_kv_append(const uint16_t* kn, const uint16_t* vn, const int32_t* pos, int64_t batch, int64_t Hkv,
                     int64_t Lmax, uint16_t* kc, uint16_t* vc, bool pdl, cudaStream_t st) {
    cudaLaunchAttribute attr[1];
    cudaLaunchConfig_t cfg = att_cfg(dim3(static_cast<unsigned>(Hkv), static_cast<unsigned>(batch)), dim3(kAttD / 2),
                                     pdl, st, attr);
    return static_cast<int>(cudaLaunchKernelEx(&cfg, kv_append_kernel, kn, vn, pos, Lmax, static_cast<int>(Hkv),
                                               kc, vc));
}

}  // namespace rq4
