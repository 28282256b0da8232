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
//   attn_partial_kernel  grid (chunks of 64 keys, Hkv, batch), 128 threads:
//       the chunk's keys and values arrive by four 2-D TMA loads (64 keys x 64
//       dims each, 128-B swizzle) issued at once -- 32 KB in flight per CTA,
//       six CTAs per SM; the G query heads of one kv head are the N dimension
//       of warp-level tensor-core MMAs (mma.sync m16n8k16, fp16 in, fp32 out):
//           S^T[key][head]  = K[key][dim] . Q^T[dim][head]     (warp w: keys 16w..16w+15)
//           O^T[dim][head]  = V^T[dim][key] . P^T[key][head]   (warp w: dims 32w..32w+31)
//       with the softmax of the chunk (max, exp, sum per head) in between
//       (P rounded to fp16 once; its sum uses the same rounded values); writes
//       the chunk's (m, l, o) to the workspace;
//   attn_combine_kernel  grid (Hq, batch), 128 threads: rescales and sums the
//       chunks in fixed order -> fp16.  Deterministic.
// Both wait for the previous kernel (griddepcontrol.wait) before reading.
#include <cuda_fp16.h>
#include "internal.h"
#include "ptx.cuh"

namespace rq4 {

constexpr int kAttD = 128;          // head_dim (every Llama-2 size)
constexpr int kAttChunk = 64;       // keys per partial CTA
constexpr int kAttThreads = 128;    // 4 warps
constexpr int kAttMaxG = 8;         // query heads per kv head (the MMA's N)
constexpr int kAttMaxChunks = 1024; // combine capacity: Lmax <= 65536
constexpr uint32_t kAttTile = kAttChunk * kAttD * 2;        // one TMA box: 64 keys x 128 dims fp16 = 16 KB
constexpr size_t kAttSmem = 1024 + 2 * 2 * kAttTile;        // align pad + 2 stages of (K, V)

struct AttArgs {
    const uint16_t* q;              // [batch][Hq][D]
    const int32_t* lens;            // [batch]
    uint16_t* out;                  // [batch][Hq][D]
    float* part_o;                  // [batch][Hq][nch][D]
    float* part_ml;                 // [batch][Hq][nch][2]  (max, sum)
    int64_t Lmax;
    int Hq, Hkv, nch, batch;
    int chunk;                      // keys per work item
    float scale;                    // 1 / sqrt(D)
};

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], uint32_t addr) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], uint32_t addr) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(addr));
}
__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                 "{%0,%1,%2,%3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// byte offset of (row, 16-B chunk c of the 64-dim half) in a 128-B swizzled box
__device__ __forceinline__ uint32_t sw128(int row, int c) { return row * 128 + ((c ^ (row & 7)) << 4); }
// (key, 16-B dim chunk 0..15) of a [64 keys][2 halves][64 dims] tile: 128-B row 2 key + half
__device__ __forceinline__ uint32_t kv_off(int key, int dch) { return sw128(2 * key + (dch >> 3), dch & 7); }

template <int G>
__global__ void __launch_bounds__(kAttThreads) attn_partial_kernel(const __grid_constant__ CUtensorMap mk,
                                                                   const __grid_constant__ CUtensorMap mv,
                                                                   const __grid_constant__ AttArgs a) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    __shared__ __align__(16) uint16_t ps[kAttMaxG][kAttChunk + 8];   // P as fp16 [head][key] (+8: bank spread)
    __shared__ float wmax[4][kAttMaxG], wsum[4][kAttMaxG];
    __shared__ uint64_t bar[2];
    uint8_t* kv0 = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    pdl_launch_dependents();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int gq = lane >> 2, tq = lane & 3;             // MMA fragment coordinates
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
    }
    pdl_wait();                                          // q, lens and the caches come from earlier kernels
    // the lengths, staged once (a global load per work item would put an L2
    // round trip on every item's critical path)
    __shared__ int lens_s[256];
    for (int i = tid; i < a.batch && i < 256; i += kAttThreads) lens_s[i] = a.lens[i];
    __syncthreads();
    auto len_of = [&](int b) { return b < 256 ? lens_s[b] : a.lens[b]; };
    // work items (chunk c, kv head g, sequence b), c fastest, strided over the
    // grid; items at or past the sequence's length have nothing to do
    const int total = a.nch * a.Hkv * a.batch;
    auto valid_from = [&](int it) {
        for (; it < total; it += gridDim.x) {
            const int c = it % a.nch, b = it / (a.nch * a.Hkv);
            if (c * kAttChunk < len_of(b)) return it;
        }
        return total;
    };
    auto issue = [&](int it, int st) {
        const int c = it % a.nch, rest = it / a.nch, g = rest % a.Hkv, b = rest / a.Hkv;
        const int32_t row = static_cast<int32_t>((static_cast<int64_t>(b) * a.Hkv + g) * a.Lmax + c * kAttChunk);
        uint8_t* ks = kv0 + st * 2 * kAttTile;
        const uint64_t pol = policy_evict_first();
        fence_proxy_async_smem();                        // after generic writes (zeroed rows) to this buffer
        mbar_arrive_expect_tx(&bar[st], 2 * kAttTile);
        tma_load_3d(ks, &mk, &bar[st], 0, 0, row, pol);
        tma_load_3d(ks + kAttTile, &mv, &bar[st], 0, 0, row, pol);
    };
    int cur = valid_from(blockIdx.x);
    if (tid == 0 && cur < total) issue(cur, 0);
    int st = 0;
    uint32_t ph[2] = {0u, 0u};
    while (cur < total) {
        const int nxt = valid_from(cur + gridDim.x);
        if (tid == 0 && nxt < total) issue(nxt, st ^ 1);   // the other buffer was released at the loop end
        const int c = cur % a.nch, rest = cur / a.nch, g = rest % a.Hkv, b = rest / a.Hkv;
        const int L = len_of(b);
        const int k0 = c * kAttChunk;
        const int nk = L - k0 < kAttChunk ? L - k0 : kAttChunk;
        uint8_t* ks = kv0 + st * 2 * kAttTile;           // K tile [key][half][64 dims], 128-B swizzle
        uint8_t* vs = ks + kAttTile;                     // V tile, likewise
        // B fragments of Q^T (k = dims, n = head gq): q[head gq][16 s + 2 tq (+8)], heads >= G zero
        uint32_t qb[8][2];
        {
            const bool hv = gq < G;
            const uint32_t* qp = reinterpret_cast<const uint32_t*>(
                a.q + (static_cast<int64_t>(b) * a.Hq + g * G + (hv ? gq : 0)) * kAttD);
#pragma unroll
            for (int s8 = 0; s8 < 8; ++s8) {
                qb[s8][0] = hv ? qp[(16 * s8 + 2 * tq) / 2] : 0u;
                qb[s8][1] = hv ? qp[(16 * s8 + 8 + 2 * tq) / 2] : 0u;
            }
        }
        mbar_wait(&bar[st], ph[st]);
        ph[st] ^= 1u;
        if (nk < kAttChunk) {
            // value rows past len may hold anything (NaN): zero them, p = 0 there
            for (int i = tid; i < (kAttChunk - nk) * 16; i += kAttThreads) {
                const int r = nk + (i >> 4), u = i & 15;   // 16-B unit u of the row's 2 x 128 B
                *reinterpret_cast<uint4*>(vs + r * 256 + u * 16) = make_uint4(0u, 0u, 0u, 0u);
            }
        }
        // ---- scores S^T = K . Q^T: warp w, keys 16 w .. 16 w + 15
        float sacc[4] = {0.f, 0.f, 0.f, 0.f};
        {
            const int r = 16 * warp + (lane & 7) + 8 * ((lane >> 3) & 1);
#pragma unroll
            for (int s8 = 0; s8 < 8; ++s8) {
                uint32_t af[4];
                const int cch = 2 * (s8 & 3) + (lane >> 4);
                ldsm_x4(af, smem_u32(ks + kv_off(r, 8 * (s8 >> 2) + cch)));
                mma16816(sacc, af, qb[s8][0], qb[s8][1]);
            }
        }
        // sacc: keys (16w + gq, 16w + gq + 8) x heads (2 tq, 2 tq + 1)
        const int kA = 16 * warp + gq, kB = kA + 8;
        float sv[4];
        sv[0] = kA < nk ? sacc[0] * a.scale : -INFINITY;
        sv[1] = kA < nk ? sacc[1] * a.scale : -INFINITY;
        sv[2] = kB < nk ? sacc[2] * a.scale : -INFINITY;
        sv[3] = kB < nk ? sacc[3] * a.scale : -INFINITY;
        // per-head max over the chunk: lanes of equal tq (xor 4, 8, 16), then the 4 warps
        float m0 = fmaxf(sv[0], sv[2]), m1 = fmaxf(sv[1], sv[3]);
#pragma unroll
        for (int off = 4; off < 32; off <<= 1) {
            m0 = fmaxf(m0, __shfl_xor_sync(0xffffffffu, m0, off));
            m1 = fmaxf(m1, __shfl_xor_sync(0xffffffffu, m1, off));
        }
        if (gq == 0) { wmax[warp][2 * tq] = m0; wmax[warp][2 * tq + 1] = m1; }
        __syncthreads();
        const float M0 = fmaxf(fmaxf(wmax[0][2 * tq], wmax[1][2 * tq]), fmaxf(wmax[2][2 * tq], wmax[3][2 * tq]));
        const float M1 = fmaxf(fmaxf(wmax[0][2 * tq + 1], wmax[1][2 * tq + 1]),
                               fmaxf(wmax[2][2 * tq + 1], wmax[3][2 * tq + 1]));
        // p in fp16 (the MMA operand); the sum over the same rounded values
        const __half p0 = __float2half_rn(kA < nk ? __expf(sv[0] - M0) : 0.f);
        const __half p1 = __float2half_rn(kA < nk ? __expf(sv[1] - M1) : 0.f);
        const __half p2 = __float2half_rn(kB < nk ? __expf(sv[2] - M0) : 0.f);
        const __half p3 = __float2half_rn(kB < nk ? __expf(sv[3] - M1) : 0.f);
        ps[2 * tq][kA] = __half_as_ushort(p0);
        ps[2 * tq + 1][kA] = __half_as_ushort(p1);
        ps[2 * tq][kB] = __half_as_ushort(p2);
        ps[2 * tq + 1][kB] = __half_as_ushort(p3);
        float l0 = __half2float(p0) + __half2float(p2), l1 = __half2float(p1) + __half2float(p3);
#pragma unroll
        for (int off = 4; off < 32; off <<= 1) {
            l0 += __shfl_xor_sync(0xffffffffu, l0, off);
            l1 += __shfl_xor_sync(0xffffffffu, l1, off);
        }
        if (gq == 0) { wsum[warp][2 * tq] = l0; wsum[warp][2 * tq + 1] = l1; }
        __syncthreads();                                 // ps, wsum and the zeroed V rows visible
        // ---- O^T = V^T . P^T: warp w, dims 32 w .. 32 w + 31 (two 16-dim tiles), keys in 4 k-steps
        float o[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
        for (int ks4 = 0; ks4 < 4; ++ks4) {
            // B = P^T[key][head]: P[head gq][16 ks4 + 2 tq (+8)]
            const uint32_t pb0 = *reinterpret_cast<const uint32_t*>(&ps[gq][16 * ks4 + 2 * tq]);
            const uint32_t pb1 = *reinterpret_cast<const uint32_t*>(&ps[gq][16 * ks4 + 8 + 2 * tq]);
#pragma unroll
            for (int mt = 0; mt < 2; ++mt) {
                // A = V^T tile (dims d0 .. d0+15, keys 16 ks4 .. +15) via ldmatrix.trans of V rows
                const int d0 = 32 * warp + 16 * mt;
                const int j = lane >> 3, i = lane & 7;
                const int key = 16 * ks4 + i + 8 * (j >> 1);
                const int dch = (d0 >> 3) + (j & 1);       // 16-B dim chunk 0..15
                uint32_t af[4];
                ldsm_x4_t(af, smem_u32(vs + kv_off(key, dch)));
                mma16816(o[mt], af, pb0, pb1);
            }
        }
        // o[mt]: dims (d0 + gq, d0 + gq + 8) x heads (2 tq, 2 tq + 1)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
            const int head = 2 * tq + hh;
            if (head >= G) continue;
            const int64_t row = (static_cast<int64_t>(b) * a.Hq + g * G + head) * a.nch + c;
            float* po = a.part_o + row * kAttD;
#pragma unroll
            for (int mt = 0; mt < 2; ++mt) {
                const int d0 = 32 * warp + 16 * mt;
                po[d0 + gq] = o[mt][hh];
                po[d0 + gq + 8] = o[mt][2 + hh];
            }
            if (warp == 0 && gq == 0) {
                a.part_ml[row * 2] = hh ? M1 : M0;
                a.part_ml[row * 2 + 1] = ((wsum[0][head] + wsum[1][head]) + wsum[2][head]) + wsum[3][head];
            }
        }
        __syncthreads();                                 // buffer st, ps, wmax, wsum free again
        cur = nxt;
        st ^= 1;
    }
}

__global__ void __launch_bounds__(kAttD) attn_combine_kernel(const __grid_constant__ AttArgs a) {
    __shared__ float wts[kAttMaxChunks];                // per-chunk weights exp(m_c - M)
    __shared__ float red[kAttD / 32];
    pdl_launch_dependents();
    pdl_wait();
    const int b = blockIdx.y, h = blockIdx.x, d = threadIdx.x;
    const int L = a.lens[b];
    uint16_t* dst = a.out + (static_cast<int64_t>(b) * a.Hq + h) * kAttD + d;
    if (L <= 0) { *dst = 0; return; }
    const int nc = (L + a.chunk - 1) / a.chunk;          // <= kAttMaxChunks (L <= 65536)
    const int64_t base = (static_cast<int64_t>(b) * a.Hq + h) * a.nch;
    // the first 32 chunks' partials are requested together with the chunk
    // maxima (one memory round trip for caches up to 2048 keys)
    float pv[32], lv[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        const int cc = j < nc ? j : nc - 1;
        pv[j] = a.part_o[(base + cc) * kAttD + d];
        lv[j] = a.part_ml[(base + cc) * 2 + 1];
    }
    // all chunk maxima in parallel (thread d: chunks d, d + 128, ...), the max by a block reduction
    float M = -INFINITY;
    for (int cc = d; cc < nc; cc += kAttD) M = fmaxf(M, a.part_ml[(base + cc) * 2]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
    if ((d & 31) == 0) red[d >> 5] = M;
    __syncthreads();
    M = fmaxf(fmaxf(red[0], red[1]), fmaxf(red[2], red[3]));
    for (int cc = d; cc < nc; cc += kAttD) wts[cc] = __expf(a.part_ml[(base + cc) * 2] - M);
    __syncthreads();
    // summed in chunk order (fixed order: deterministic), 32 chunks per round trip
    float num = 0.f, den = 0.f;
    for (int c0 = 0; c0 < nc; c0 += 32) {
        if (c0 > 0) {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const int cc = c0 + j < nc ? c0 + j : nc - 1;
                pv[j] = a.part_o[(base + cc) * kAttD + d];
                lv[j] = a.part_ml[(base + cc) * 2 + 1];
            }
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            if (c0 + j < nc) {
                const float w = wts[c0 + j];
                den = fmaf(w, lv[j], den);
                num = fmaf(w, pv[j], num);
            }
        }
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

size_t attn_workspace_bytes(int64_t batch, int64_t Hq, int64_t Lmax) {
    const int64_t nch = (Lmax + kAttChunk - 1) / kAttChunk;
    return static_cast<size_t>(batch * Hq * nch) * (kAttD + 2) * 4;
}

template <int G>
static int launch_partial(const CUtensorMap& mk, const CUtensorMap& mv, const AttArgs& a, int64_t batch, bool pdl,
                          cudaStream_t st) {
    const cudaError_t e = ensure_kernel_attrs(reinterpret_cast<const void*>(attn_partial_kernel<G>),
                                              static_cast<int>(kAttSmem));
    if (e != cudaSuccess) return static_cast<int>(e);
    cudaLaunchAttribute attr[1];
    // a persistent grid: 3 CTAs per SM (66 KB of shared memory each), each
    // streaming its strided share of the (chunk, kv head, sequence) items
    // through a two-stage TMA ring
    const int64_t items = static_cast<int64_t>(a.nch) * a.Hkv * batch;
    const int64_t cap = 3 * static_cast<int64_t>(num_sms());
    (void)batch;
    cudaLaunchConfig_t cfg = att_cfg(dim3(static_cast<unsigned>(items < cap ? items : cap)), dim3(kAttThreads), pdl,
                                     st, attr);
    cfg.dynamicSmemBytes = kAttSmem;
    return static_cast<int>(cudaLaunchKernelEx(&cfg, attn_partial_kernel<G>, mk, mv, a));
}

int launch_attention_decode(const uint16_t* q, const uint16_t* k, const uint16_t* v, const int32_t* lens,
                            int64_t batch, int64_t Hq, int64_t Hkv, int64_t Lmax, uint16_t* out, void* ws,
                            bool pdl, cudaStream_t st) {
    AttArgs a;
    a.q = q; a.lens = lens; a.out = out;
    a.Lmax = Lmax;
    a.Hq = static_cast<int>(Hq);
    a.Hkv = static_cast<int>(Hkv);
    a.chunk = kAttChunk;
    a.nch = static_cast<int>((Lmax + a.chunk - 1) / a.chunk);
    a.batch = static_cast<int>(batch);
    a.scale = 0.08838834764831845f;                      // 1 / sqrt(128)
    a.part_o = static_cast<float*>(ws);
    a.part_ml = a.part_o + static_cast<size_t>(batch * Hq * a.nch) * kAttD;
    if (a.nch > kAttMaxChunks) return static_cast<int>(cudaErrorInvalidValue);
    int rc = 0;
    if (a.nch > 0) {
        // caches as 3-D {64 dims, 2 halves, batch * Hkv * Lmax rows} fp16: one box
        // of {64, 2, 64} is a whole 64-key tile (16 KB), 128-B swizzled
        CUtensorMap mk, mv;
        const uint64_t rows = static_cast<uint64_t>(batch * Hkv * Lmax);
        const uint64_t dims[3] = {64, 2, rows};
        const uint64_t strides[2] = {128, kAttD * 2};
        const uint32_t box[3] = {64, 2, kAttChunk};
        rc = make_tensor_map(&mk, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, k, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
        if (rc) return rc;
        rc = make_tensor_map(&mv, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, v, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
        if (rc) return rc;
        switch (Hq / Hkv) {
            case 1: rc = launch_partial<1>(mk, mv, a, batch, pdl, st); break;
            case 2: rc = launch_partial<2>(mk, mv, a, batch, pdl, st); break;
            case 4: rc = launch_partial<4>(mk, mv, a, batch, pdl, st); break;
            case 8: rc = launch_partial<8>(mk, mv, a, batch, pdl, st); break;
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
