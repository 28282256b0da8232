// gemv_mma.cu -- the decode path (n = 1, 2) on the warp-level tensor cores.
//
// y[t][j] = sum_k x[t][k] * W(k, j),  W = (q - 7) * s   (dequant fused
// into the matmul; K, N static per call, n runtime).
//
// Why a tensor-core GEMV: in a chain of decode GEMVs under
// programmatic dependent launch every kernel's weights are already streaming
// into shared memory while the previous kernel runs, so what is left on the
// critical path after griddepcontrol.wait is the MATH on resident data.  On
// the CUDA cores that math is one FHFMA per weight plus the unpack, and FHFMA
// shares the ALU pipe (2.4 warp-instr/clk/SM measured, profiles/ubench_r01.txt)
// -> <= ~47 weights/clk/SM.  mma.sync m16n8k16 (fp16 x fp16 -> fp32) does 256
// weight-MACs per instruction (0.5 MMA/clk/SM measured, tools/ubench_mma.cu),
// so the unpack alone bounds the rate: ~85 weights/clk/SM.
//
// Arithmetic -- factored zero point, exact products:
//   codes enter the MMA as fp16 SUBNORMALS, no conversion at all: the masks
//   w & 0x000F000F and (w >> 8) & 0x000F000F give the half2 pairs
//   (q0, q4), (q2, q6) * 2^-24; w & 0x00F000F0 and (w >> 8) & 0x00F000F0 give
//   (q1, q5), (q3, q7) * 2^-20.  Two chained MMAs per (16 rows x 32-code group):
//     u = A(q even) . x + A(q odd) . (x / 16) + C,  C = -7 * 2^-24 * sum_group x
//       = 2^-24 sum (q - 7) x
//   (the tensor core keeps fp16 subnormals -- tools/ubench_mma.cu; x / 16 is
//   exact in fp16 unless |x| < 2^-10, where it rounds in the subnormal range),
//   acc += s * u per group in fp32, y = 2^24 * acc -> fp16 RNE.
//
// Data movement:
//   * each CTA owns a contiguous, row-balanced block of output rows; its
//     weights are cut into stages of (16 rows x 2048 k) = 16 KB of codes +
//     2 KB of scales, each ONE tensor-map TMA load issued by one thread:
//     codes through a 3-D map {32 words, rows, 128-B chunks} with the 128-B
//     swizzle, so a stage lands as [chunk][row][128 B] with the 16-B units of
//     row r XOR-ed by r mod 8 -- the MMA fragment loads (8 rows x 4 words per
//     instruction) are bank-conflict free; scales through a 2-D map, same
//     swizzle.  Out-of-range k (last chunk) and rows (past N) are zero-filled
//     by the TMA and never used;
//   * stages go chunk-major (all row blocks of k-chunk 0, then chunk 1, ...)
//     so each consumer warp keeps the B fragments (x, permuted to the code
//     order) of its groups in registers for a whole chunk; x is staged once
//     per CTA in shared memory already in fragment order;
//   * warp kw of W consumer warps owns groups [kw*64/W, (kw+1)*64/W) of every
//     chunk; its per-row partials accumulate in shared memory (only this warp
//     touches its slots) and are summed over the W warps in fixed order at the
//     end: deterministic;
//   * PDL: the producer streams weights before griddepcontrol.wait; only the
//     x staging and the y stores wait for the previous kernel.
#include <cstdlib>
#include <cstdio>
#include "internal.h"
#include "relax_q4.h"
#include "ptx.cuh"

namespace rq4 {

constexpr int kGmRows = 16;                          // MMA M
constexpr int kGmChunkG = 64;                        // groups per k-chunk
constexpr int kGmChunkK = kGmChunkG * kGroup;        // 2048 k
constexpr uint32_t kGmCodeBytes = kGmRows * kGmChunkK / 2;      // 16 KB
constexpr uint32_t kGmScaleBytes = kGmRows * kGmChunkG * 2;     // 2 KB
constexpr uint32_t kGmStageBytes = kGmCodeBytes + kGmScaleBytes;  // 18 KB (multiple of 1 KB)

struct GmArgs {
    const uint16_t* x;     // [NT][K] fp16
    uint16_t* y;           // [NT][N]
    int64_t N;
    int K, G, NS, nkc;
    uint32_t xtab_bytes, mtab_bytes;
};

struct GmConfig {
    int W, NS, grid, rows_cta_max, threads;
    uint32_t xtab_bytes, mtab_bytes;
    size_t smem;
    bool ok;
};

__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1,
                                         float c0, float c1, float c2, float c3) {
    asm(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%10,%11,%12,%13};"
        : "=f"(d[0]), "=f"(d[1]), "=f"(d[2]), "=f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1),
          "f"(c0), "f"(c1), "f"(c2), "f"(c3));
}

__device__ __forceinline__ void bar_consumers(int nthreads) {
    asm volatile("bar.sync 1, %0;" :: "r"(nthreads) : "memory");
}

// One warp, one stage: groups jj0 .. jj0+GPW-1 (of the 64 in the chunk) of a
// 16-row block.  acc[0/1] = row g (token 0/1), acc[2/3] = row g + 8, in units
// of 2^-24 (file comment).  GUARD: skip groups jj >= gc (last, partial chunk).
// xt: this lane's B fragments of the chunk's groups (stride NT*4 uint4 per group);
// mt: the zero-point terms {m_tok0, m_tok1, m_tok0, m_tok1} of the chunk's groups.
// Stage layout (128-B swizzle): code word t of group jj, row r at
//   (jj/8)*2048 + r*128 + ((jj%8) ^ (r%8))*16 + 4t;  scale of (r, jj) at
//   16384 + r*128 + ((jj/8) ^ (r%8))*16 + (jj%8)*2.
template <int NT, int GPW, bool GUARD>
__device__ __forceinline__ void gm_groups(float (&acc)[4], const uint8_t* stage, int g, int t, int jj0, int gc,
                                          const uint4* xt, const float4* mt) {
    uint32_t wa[GPW], wb[GPW];
    uint16_t sa[GPW], sb[GPW];
    const uint8_t* srow = stage + kGmCodeBytes + g * 128 + ((((jj0 >> 3) ^ g)) << 4) + (jj0 & 7) * 2;
    if (GPW == 8) {
        const uint4 va = *reinterpret_cast<const uint4*>(srow);
        const uint4 vb = *reinterpret_cast<const uint4*>(srow + 1024);
        const uint32_t A[4] = {va.x, va.y, va.z, va.w}, B[4] = {vb.x, vb.y, vb.z, vb.w};
#pragma unroll
        for (int i = 0; i < GPW; ++i) {
            sa[i] = static_cast<uint16_t>(A[i >> 1] >> ((i & 1) * 16));
            sb[i] = static_cast<uint16_t>(B[i >> 1] >> ((i & 1) * 16));
        }
    } else {
#pragma unroll
        for (int i = 0; i < GPW; ++i) {
            sa[i] = *reinterpret_cast<const uint16_t*>(srow + i * 2);
            sb[i] = *reinterpret_cast<const uint16_t*>(srow + 1024 + i * 2);
        }
    }
    const uint8_t* crow = stage + g * 128 + 4 * t;
#pragma unroll
    for (int i = 0; i < GPW; ++i) {
        const int jj = jj0 + i;
        if (!GUARD || jj < gc) {
            const uint8_t* p = crow + (jj >> 3) * 2048 + (((jj & 7) ^ g) << 4);
            wa[i] = *reinterpret_cast<const uint32_t*>(p);
            wb[i] = *reinterpret_cast<const uint32_t*>(p + 1024);
        }
    }
    // four groups per phase: all unpacks, then all MMAs (independent), then
    // the scale FMAs -- keeps several MMA chains in flight per warp
    constexpr int PH = GPW < 4 ? GPW : 4;
#pragma unroll
    for (int i0 = 0; i0 < GPW; i0 += PH) {
        uint32_t a1[PH][4], a2[PH][4];
        float d1[PH][4], d2[PH][4];
#pragma unroll
        for (int q = 0; q < PH; ++q) {
            const int i = i0 + q;
            const uint32_t wa8 = wa[i] >> 8, wb8 = wb[i] >> 8;
            a1[q][0] = wa[i] & 0x000F000Fu; a1[q][1] = wb[i] & 0x000F000Fu;
            a1[q][2] = wa8 & 0x000F000Fu;   a1[q][3] = wb8 & 0x000F000Fu;
            a2[q][0] = wa[i] & 0x00F000F0u; a2[q][1] = wb[i] & 0x00F000F0u;
            a2[q][2] = wa8 & 0x00F000F0u;   a2[q][3] = wb8 & 0x00F000F0u;
        }
#pragma unroll
        for (int q = 0; q < PH; ++q) {
            const int i = i0 + q, jj = jj0 + i;
            if (!GUARD || jj < gc) {
                const float4 c = mt[jj];
                const uint4 xv = xt[jj * NT * 4];
                mma16816(d1[q], a1[q], xv.x, xv.y, c.x, c.y, c.z, c.w);
                mma16816(d2[q], a2[q], xv.z, xv.w, 0.f, 0.f, 0.f, 0.f);
            }
        }
#pragma unroll
        for (int q = 0; q < PH; ++q) {
            const int i = i0 + q, jj = jj0 + i;
            if (!GUARD || jj < gc) {
                const float fa = __half2float(__ushort_as_half(sa[i]));
                const float fb = __half2float(__ushort_as_half(sb[i]));
                acc[0] = fmaf(fa, d1[q][0] + d2[q][0], acc[0]);
                acc[2] = fmaf(fb, d1[q][2] + d2[q][2], acc[2]);
                if (NT == 2) {
                    acc[1] = fmaf(fa, d1[q][1] + d2[q][1], acc[1]);
                    acc[3] = fmaf(fb, d1[q][3] + d2[q][3], acc[3]);
                }
            }
        }
    }
}

// Block-diagonal variant (BD = 1, n = 1): the MMA's 8
// columns are this warp's GPW groups of the chunk instead of tokens.  Lane
// (g, t) supplies B only for the MMAs of its own group column g (zero
// otherwise), so the 2 * GPW MMAs of a stage leave in column c the per-group
// dot product of group c for rows g and g + 8; 4 independent accumulator
// chains; the zero point enters once as the C operand of chain 0; the scales
// are applied once per stage (4 FFMA) instead of once per group.
template <int GPW>
__device__ __forceinline__ void gm_groups_bd(float (&acc)[2], const uint8_t* stage, int g, int t, int jj0,
                                             const uint32_t (&xb)[4], float m0, float m1) {
    float dd[4][4];
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int q = 0; q < 4; ++q) dd[c][q] = 0.f;
    dd[0][0] = m0; dd[0][1] = m1; dd[0][2] = m0; dd[0][3] = m1;
    const uint8_t* crow = stage + g * 128 + 4 * t;
#pragma unroll
    for (int i = 0; i < GPW; ++i) {
        const int jj = jj0 + i;
        const uint8_t* p = crow + (jj >> 3) * 2048 + (((jj & 7) ^ g) << 4);
        const uint32_t wa = *reinterpret_cast<const uint32_t*>(p);
        const uint32_t wb = *reinterpret_cast<const uint32_t*>(p + 1024);
        const uint32_t wa8 = wa >> 8, wb8 = wb >> 8;
        const uint32_t a1[4] = {wa & 0x000F000Fu, wb & 0x000F000Fu, wa8 & 0x000F000Fu, wb8 & 0x000F000Fu};
        const uint32_t a2[4] = {wa & 0x00F000F0u, wb & 0x00F000F0u, wa8 & 0x00F000F0u, wb8 & 0x00F000F0u};
        const bool mine = g == i;
        float d1[4], d2[4];
        mma16816(d1, a1, mine ? xb[0] : 0u, mine ? xb[1] : 0u, dd[(2 * i) & 3][0], dd[(2 * i) & 3][1],
                 dd[(2 * i) & 3][2], dd[(2 * i) & 3][3]);
#pragma unroll
        for (int q = 0; q < 4; ++q) dd[(2 * i) & 3][q] = d1[q];
        mma16816(d2, a2, mine ? xb[2] : 0u, mine ? xb[3] : 0u, dd[(2 * i + 1) & 3][0], dd[(2 * i + 1) & 3][1],
                 dd[(2 * i + 1) & 3][2], dd[(2 * i + 1) & 3][3]);
#pragma unroll
        for (int q = 0; q < 4; ++q) dd[(2 * i + 1) & 3][q] = d2[q];
    }
    float d[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) d[q] = (dd[0][q] + dd[1][q]) + (dd[2][q] + dd[3][q]);
    // scales of groups jj0 + 2t, jj0 + 2t + 1 for rows g, g + 8 (one 4-B load each)
    const int c0 = 2 * t;
    const uint8_t* sp = stage + kGmCodeBytes + g * 128 + ((((jj0 + c0) >> 3) ^ g) << 4) + ((jj0 + c0) & 7) * 2;
    const uint32_t sa = c0 < GPW ? *reinterpret_cast<const uint32_t*>(sp) : 0u;
    const uint32_t sb = c0 < GPW ? *reinterpret_cast<const uint32_t*>(sp + 1024) : 0u;
    const float2 fa = __half22float2(u32_as_h2(sa));
    const float2 fb = __half22float2(u32_as_h2(sb));
    acc[0] = fmaf(fa.x, d[0], fmaf(fa.y, d[1], acc[0]));
    acc[1] = fmaf(fb.x, d[2], fmaf(fb.y, d[3], acc[1]));
}

// W consumer warps + 1 producer warp; GPW = 64 / W groups per warp per chunk.
template <int NT, int GPW, int BD>
__global__ void __launch_bounds__((64 / GPW + 1) * 32, 2)
gemv_mma_kernel(const __grid_constant__ CUtensorMap mw, const __grid_constant__ CUtensorMap ms,
                const __grid_constant__ GmArgs a) {
    constexpr int W = kGmChunkG / GPW;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);   // provably warp-uniform
    const int lane = threadIdx.x & 31;
    // [pad to 1 KB][ring NS x 18 KB][barriers 256 B][xtab][mtab][part]
    uint8_t* ring = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + static_cast<size_t>(a.NS) * kGmStageBytes);
    uint64_t* empty = full + a.NS;
    uint4* xtab = reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(full) + 256);
    float4* mtab = reinterpret_cast<float4*>(reinterpret_cast<uint8_t*>(xtab) + a.xtab_bytes);
    float* part = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(mtab) + a.mtab_bytes);

    const int64_t row0 = static_cast<int64_t>(blockIdx.x) * a.N / gridDim.x;
    const int64_t row1 = static_cast<int64_t>(blockIdx.x + 1) * a.N / gridDim.x;
    const int rows = static_cast<int>(row1 - row0);
    const int nrb = (rows + kGmRows - 1) / kGmRows;
    const int nst = nrb * a.nkc;

    if (threadIdx.x == 0) {
        for (int i = 0; i < a.NS; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], W); }
        fence_mbar_init();
    }
    __syncthreads();
    pdl_launch_dependents();

    if (warp == W) {
        // ------------------------------------------------ producer (one thread)
        if (lane == 0) {
            tma_prefetch_desc(&mw);
            tma_prefetch_desc(&ms);
            const uint64_t pol = policy_evict_first();
            int slot = 0, rb = 0, kc = 0;
            uint32_t phase = 0;
            for (int st = 0; st < nst; ++st) {
                mbar_wait(&empty[slot], phase ^ 1);
                uint8_t* stage = ring + static_cast<size_t>(slot) * kGmStageBytes;
                const int r = static_cast<int>(row0) + rb * kGmRows;
                mbar_arrive_expect_tx(&full[slot], kGmStageBytes);
                tma_load_3d(stage, &mw, &full[slot], 0, r, kc * (kGmChunkK / 256), pol);
                tma_load_2d(stage + kGmCodeBytes, &ms, &full[slot], kc * kGmChunkG, r, pol);
                if (++slot == a.NS) { slot = 0; phase ^= 1; }
                if (++rb == nrb) { rb = 0; ++kc; }
            }
        }
    } else {
        // ------------------------------------------------ consumers
        pdl_wait();
        if constexpr (BD) {
            // x straight from global: lane (g, t) needs, per chunk, the 8 x of
            // its own group column (kw * GPW + g) at slots 8t..8t+7, and the
            // zero-point terms of columns 2t, 2t + 1 (quad sums, shuffled).
            const int g = lane >> 2, t = lane & 3;
            const int kw = warp;
            auto xload = [&](int kc) -> uint4 {
                const int j = kc * kGmChunkG + kw * GPW + g;
                return (g < GPW && kc < a.nkc && j < a.G)
                       ? *reinterpret_cast<const uint4*>(a.x + static_cast<int64_t>(j) * 32 + t * 8)
                       : make_uint4(0u, 0u, 0u, 0u);
            };
            uint4 vn = xload(0), vn2 = xload(1);
            uint32_t xb[4];
            float m0 = 0.f, m1 = 0.f;
            const __half2 sixteenth = __float2half2_rn(0.0625f);
            int slot = 0, rb = 0, kc = 0;
            uint32_t phase = 0;
            for (int st = 0; st < nst; ++st) {
                if (rb == 0) {
                    const uint4 v = vn;
                    vn = vn2;
                    vn2 = xload(kc + 2);
                    xb[0] = prmt(v.x, v.z, 0x5410u);
                    xb[1] = prmt(v.y, v.w, 0x5410u);
                    xb[2] = h2_as_u32(__hmul2(u32_as_h2(prmt(v.x, v.z, 0x7632u)), sixteenth));
                    xb[3] = h2_as_u32(__hmul2(u32_as_h2(prmt(v.y, v.w, 0x7632u)), sixteenth));
                    const uint32_t ws[4] = {v.x, v.y, v.z, v.w};
                    float p2[2] = {0.f, 0.f};
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const float2 f = __half22float2(u32_as_h2(ws[u]));
                        p2[u & 1] += f.x + f.y;
                    }
                    float sum = p2[0] + p2[1];
                    sum += __shfl_xor_sync(0xffffffffu, sum, 1);
                    sum += __shfl_xor_sync(0xffffffffu, sum, 2);      // group of column g, at lanes 4g..4g+3
                    const float mc0 = __shfl_sync(0xffffffffu, sum, (2 * t) * 4);
                    const float mc1 = __shfl_sync(0xffffffffu, sum, (2 * t + 1) * 4);
                    m0 = -7.0f * 5.9604644775390625e-08f * mc0;
                    m1 = -7.0f * 5.9604644775390625e-08f * mc1;
                }
                mbar_wait(&full[slot], phase);
                const uint8_t* stage = ring + static_cast<size_t>(slot) * kGmStageBytes;
                float acc[2] = {0.f, 0.f};
                gm_groups_bd<GPW>(acc, stage, g, t, kw * GPW, xb, m0, m1);
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[slot]);
                // row sums over the quad (columns 2t, 2t + 1 -> all of the warp's groups)
#pragma unroll
                for (int r = 0; r < 2; ++r) {
                    acc[r] += __shfl_xor_sync(0xffffffffu, acc[r], 1);
                    acc[r] += __shfl_xor_sync(0xffffffffu, acc[r], 2);
                }
                if (t == 0) {
                    const int ra = rb * kGmRows + g, rbb = ra + 8;
                    if (ra < rows) {
                        float* p = &part[static_cast<size_t>(ra) * W + kw];
                        *p = kc == 0 ? acc[0] : *p + acc[0];
                    }
                    if (rbb < rows) {
                        float* p = &part[static_cast<size_t>(rbb) * W + kw];
                        *p = kc == 0 ? acc[1] : *p + acc[1];
                    }
                }
                if (++slot == a.NS) { slot = 0; phase ^= 1; }
                if (++rb == nrb) { rb = 0; ++kc; }
            }
        } else {
        // x in fragment order: xtab[(j*NT + tok)*4 + t] = {(x0,x4), (x2,x6), (x1,x5)/16, (x3,x7)/16}
        // with xi = x[tok][32 j + 8 t + i]; mtab[j] = -7 * 2^-24 * (sum of group j)
        // as {tok0, tok1, tok0, tok1} (the MMA C operand).  G*NT*4 is a multiple of
        // 32, so every warp runs whole iterations and the quad shuffles are safe.
        const int nthr = W * 32;
        const __half2 sixteenth = __float2half2_rn(0.0625f);
        for (int idx = threadIdx.x; idx < a.G * NT * 4; idx += nthr) {
            const int j = idx / (NT * 4);
            const int rem = idx - j * (NT * 4);
            const int tok = rem >> 2, t = rem & 3;
            const uint4 v = *reinterpret_cast<const uint4*>(a.x + static_cast<int64_t>(tok) * a.K + j * 32 + t * 8);
            xtab[idx] = make_uint4(prmt(v.x, v.z, 0x5410u), prmt(v.y, v.w, 0x5410u),
                                   h2_as_u32(__hmul2(u32_as_h2(prmt(v.x, v.z, 0x7632u)), sixteenth)),
                                   h2_as_u32(__hmul2(u32_as_h2(prmt(v.y, v.w, 0x7632u)), sixteenth)));
            const uint32_t ws[4] = {v.x, v.y, v.z, v.w};
            float sum = 0.f;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const float2 f = __half22float2(u32_as_h2(ws[u]));
                sum += f.x + f.y;
            }
            sum += __shfl_xor_sync(0xffffffffu, sum, 1);
            sum += __shfl_xor_sync(0xffffffffu, sum, 2);
            const float m = -7.0f * 5.9604644775390625e-08f * sum;     // -7 * 2^-24 * sum
            if (t == 0) {
                float* mp = reinterpret_cast<float*>(&mtab[j]);
                if (NT == 1) { mp[0] = m; mp[1] = m; mp[2] = m; mp[3] = m; }
                else { mp[tok] = m; mp[tok + 2] = m; }
            }
        }
        bar_consumers(nthr);

        const int g = lane >> 2, t = lane & 3;
        const int tok_b = (NT == 2 && g == 1) ? 1 : 0;      // B column g <- token (cols >= NT unused)
        const int kw = warp;
        int slot = 0, rb = 0, kc = 0;
        uint32_t phase = 0;
        for (int st = 0; st < nst; ++st) {
            const int gc = a.G - kc * kGmChunkG < kGmChunkG ? a.G - kc * kGmChunkG : kGmChunkG;
            mbar_wait(&full[slot], phase);
            const uint8_t* stage = ring + static_cast<size_t>(slot) * kGmStageBytes;
            float acc[4] = {0.f, 0.f, 0.f, 0.f};
            const float4* mt = mtab + kc * kGmChunkG;
            const uint4* xt = xtab + static_cast<size_t>(kc) * kGmChunkG * NT * 4 + tok_b * 4 + t;
            if (gc == kGmChunkG) gm_groups<NT, GPW, false>(acc, stage, g, t, kw * GPW, gc, xt, mt);
            else gm_groups<NT, GPW, true>(acc, stage, g, t, kw * GPW, gc, xt, mt);
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[slot]);
            if (t == 0) {
                const int ra = rb * kGmRows + g, rbb = ra + 8;
#pragma unroll
                for (int tok = 0; tok < NT; ++tok) {
                    if (ra < rows) {
                        float* p = &part[(static_cast<size_t>(ra) * W + kw) * NT + tok];
                        *p = kc == 0 ? acc[tok] : *p + acc[tok];
                    }
                    if (rbb < rows) {
                        float* p = &part[(static_cast<size_t>(rbb) * W + kw) * NT + tok];
                        *p = kc == 0 ? acc[2 + tok] : *p + acc[2 + tok];
                    }
                }
            }
            if (++slot == a.NS) { slot = 0; phase ^= 1; }
            if (++rb == nrb) { rb = 0; ++kc; }
        }
        }
    }
    __syncthreads();
    // fixed-order sum over the W warps; y = 2^24 * acc -> fp16 RNE
    for (int o = threadIdx.x; o < rows * NT; o += blockDim.x) {
        const int rl = o / NT;
        const int tok = o - rl * NT;
        float sum = 0.f;
        for (int c = 0; c < W; ++c) sum += part[(static_cast<size_t>(rl) * W + c) * NT + tok];
        a.y[static_cast<int64_t>(tok) * a.N + row0 + rl] = __half_as_ushort(__float2half_rn(sum * 16777216.0f));
    }
}

// Shared memory per CTA is capped so that two GEMV CTAs (this kernel and the
// next one under PDL) fit on an SM: 2 x (smem + 1 KB reserved) <= 228 KB.
constexpr size_t kGmSmemCap = 113 * 1024;

static int gm_warps() {
    static int v = [] {
        const char* e = std::getenv("RELAX_Q4_GM_WARPS");
        const int w = e ? std::atoi(e) : 8;
        return (w == 8 || w == 16) ? w : 8;
    }();
    return v;
}

// CTAs per SM of one launch (RELAX_Q4_GM_CTAS = 1 | 2).
static int gm_ctas() {
    static int v = [] {
        const char* e = std::getenv("RELAX_Q4_GM_CTAS");
        return (e && std::atoi(e) == 2) ? 2 : 1;
    }();
    return v;
}

static GmConfig gm_config(int nt, int64_t K, int64_t N, bool bd = false) {
    GmConfig c{};
    c.ok = false;
    if (K % 256 != 0 || K <= 0 || N <= 0 || nt < 1 || nt > 2) return c;
    c.W = gm_warps();
    c.threads = (c.W + 1) * 32;
    const int64_t G = K / kGroup;
    c.xtab_bytes = bd ? 0u : static_cast<uint32_t>(G * nt * 64);
    c.mtab_bytes = bd ? 0u : static_cast<uint32_t>(((G * 16) + 127) / 128 * 128);
    const int64_t gmax = static_cast<int64_t>(num_sms()) * gm_ctas();
    c.grid = static_cast<int>(N < gmax ? N : gmax);
    c.rows_cta_max = static_cast<int>((N + c.grid - 1) / c.grid);
    const size_t fixed = 1024 + 256 + c.xtab_bytes + c.mtab_bytes + static_cast<size_t>(c.rows_cta_max) * c.W * nt * 4;
    if (fixed + 2 * static_cast<size_t>(kGmStageBytes) > kGmSmemCap) return c;
    const int ns = static_cast<int>((kGmSmemCap - fixed) / kGmStageBytes);
    c.NS = ns > 15 ? 15 : ns;
    c.smem = fixed + static_cast<size_t>(c.NS) * kGmStageBytes;
    c.ok = true;
    return c;
}

bool gemv_mma_ok(int nt, int64_t K, int64_t N) { return gm_config(nt, K, N).ok; }
bool gemv_bdmma_ok(int64_t K, int64_t N) { return gm_config(1, K, N, true).ok; }

template <int NT, int GPW, int BD>
static int launch_gm_t(const CUtensorMap& mw, const CUtensorMap& ms, const GmArgs& a, const GmConfig& c,
                       bool pdl, cudaStream_t stream) {
    auto k = gemv_mma_kernel<NT, GPW, BD>;
    static bool set = false;
    if (!set) {
        cudaError_t e = set_kernel_smem(reinterpret_cast<const void*>(k), static_cast<int>(kGmSmemCap));
        if (e != cudaSuccess) return static_cast<int>(e);
        set = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(c.grid);
    cfg.blockDim = dim3(c.threads);
    cfg.dynamicSmemBytes = c.smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return static_cast<int>(cudaLaunchKernelEx(&cfg, k, mw, ms, a));
}

int launch_gemv_mma(const uint16_t* x, int64_t n, int64_t K, int64_t N, const uint32_t* w,
                    const uint16_t* s, uint16_t* y, bool pdl, cudaStream_t stream, bool bd) {
    // codes: {32 words, N rows, K/256 chunks of 128 B}; scales: {K/32, N}
    CUtensorMap mw, ms;
    {
        const uint64_t dims[3] = {32, static_cast<uint64_t>(N), static_cast<uint64_t>(K / 256)};
        const uint64_t strides[2] = {static_cast<uint64_t>(K / 2), 128};
        const uint32_t box[3] = {32, kGmRows, kGmChunkK / 256};
        int rc = make_tensor_map(&mw, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, w, dims, strides, box,
                                 CU_TENSOR_MAP_SWIZZLE_128B);
        if (rc) return rc;
        const uint64_t sdims[2] = {static_cast<uint64_t>(K / kGroup), static_cast<uint64_t>(N)};
        const uint64_t sstrides[1] = {static_cast<uint64_t>(K / kGroup) * 2};
        const uint32_t sbox[2] = {kGmChunkG, kGmRows};
        rc = make_tensor_map(&ms, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, s, sdims, sstrides, sbox,
                             CU_TENSOR_MAP_SWIZZLE_128B);
        if (rc) return rc;
    }
    for (int64_t t0 = 0; t0 < n; t0 += 2) {
        const int cnt = (n - t0) >= 2 ? 2 : 1;
        const GmConfig c = gm_config(cnt, K, N, bd && cnt == 1);
        if (!c.ok) return static_cast<int>(cudaErrorInvalidConfiguration);
        if (std::getenv("RELAX_Q4_GS_PRINT"))
            fprintf(stderr, "gemv_mma K=%lld N=%lld NT=%d W=%d NS=%d grid=%d smem=%zu\n", (long long)K,
                    (long long)N, cnt, c.W, c.NS, c.grid, c.smem);
        GmArgs a;
        a.x = x + t0 * K;
        a.y = y + t0 * N;
        a.N = N;
        a.K = static_cast<int>(K);
        a.G = static_cast<int>(K / kGroup);
        a.NS = c.NS;
        a.nkc = static_cast<int>((K + kGmChunkK - 1) / kGmChunkK);
        a.xtab_bytes = c.xtab_bytes;
        a.mtab_bytes = c.mtab_bytes;
        int rc;
        if (bd && cnt == 1) rc = c.W == 16 ? launch_gm_t<1, 4, 1>(mw, ms, a, c, pdl, stream)
                                           : launch_gm_t<1, 8, 1>(mw, ms, a, c, pdl, stream);
        else if (c.W == 16) rc = cnt == 1 ? launch_gm_t<1, 4, 0>(mw, ms, a, c, pdl, stream) : launch_gm_t<2, 4, 0>(mw, ms, a, c, pdl, stream);
        else rc = cnt == 1 ? launch_gm_t<1, 8, 0>(mw, ms, a, c, pdl, stream) : launch_gm_t<2, 8, 0>(mw, ms, a, c, pdl, stream);
        if (rc != 0) return rc;
    }
    return 0;
}

}  // namespace rq4
