// gemm_tc_persist.cu -- the prefill path for large n: a persistent tcgen05
// kernel whose accumulator is double-buffered in TMEM, so the epilogue of one
// tile runs while the next tile's k-loop streams (SURVEY §8(f) / verdict r1
// "persistent tcgen05 with a double-buffered accumulator").
//
// y[t][j] = sum_k x[t][k] * W(k, j) with W = fp16_RNE((q-7) s), the
// dequant producer fused into the matmul, n a runtime argument
// (P:409-413); the tile schedule is the dynamic-shape-aware loop schedule of
// P:588-592 made persistent.
//
// Same "swap AB" mapping as gemm_tc.cu (MMA M = 128 weight rows, N = 256
// tokens, K = 16), one CTA per SM, CTA pairs (thread-block clusters of 2)
// walking pair tiles p = cluster + i * clusters (two m-tiles of one token
// tile; each CTA loads half of every x stage and multicasts it to both):
//   warp 0      W producer : TMA codes (128 rows x 128 B, SW128) + scales per
//                            256-k stage, across tile boundaries
//   warp 3      x producer : TMA x (its 128 of the 256 tokens x 64 k, SW128,
//                            multicast to the pair) per 64-k sub-block (OOB
//                            tokens zero-filled); TMEM owner
//   warp 1      MMA issuer : tcgen05.mma.kind::f16, A (dequantised W) AND B
//                            from shared memory, D into accumulator i % 2
//   warps 4-11  transform  : thread m = row m dequantises its codes bit-exactly
//                            and writes the fp16 row into an SMEM A slot in
//                            the canonical K-major SW128 layout (rows 128 B
//                            apart, 16-B chunk c of row m at c ^ (m % 8))
//   warps 12-15 epilogue   : tcgen05.ld of accumulator i % 2 while the MMA
//                            fills the other one, fp32 -> fp16 RNE, y stores
// TMEM: 2 x 256 fp32 columns (all 512); A lives in SMEM (4 x 16 KB slots),
// which is what frees the second accumulator.  PDL: weights stream before
// griddepcontrol.wait; x loads and y stores wait.
//
// Experiments build only (measured slower): the stream-K
// schedule (TpArgs::sk; full waves whole, the rest cut into k units reduced
// through the workspace with deferred column-slice fixups) and the pair-MMA
// form (C2: one tcgen05.mma.cta_group::2, M = 256, per k-step for the CTA
// pair).  The product dispatch offers this kernel up to 24 k-stages (abi.cpp).
#include <cstdio>
#include "internal.h"
#include "knobs.h"
#include "relax_q4.h"
#include "ptx.cuh"
#include "q4_unpack.cuh"

#ifndef RQ4_C2_ASLOTS
#define RQ4_C2_ASLOTS 4
#endif

namespace rq4 {

constexpr int kPWStages = 3;
constexpr uint32_t kPCodes = kTcBM * (kTcWStageK / 2);                    // 16 KB
constexpr uint32_t kPScales = kTcBM * (kTcWStageK / kGroup) * 2;          // 2 KB
constexpr uint32_t kPASlotBytes = kTcBM * kTcXStageK * 2;                 // 16 KB
constexpr int kPThreads = 16 * 32;

// BN = token tile (MMA N): 256 (long prefill) or 128 (more tiles for n ~ 512).
// C2: the CTA pair runs ONE M = 256 MMA (tcgen05 cta_group::2): each CTA holds
// its 128 weight rows of A and its BN/2 tokens of B, so an x stage is half as
// large and the MMA reads half as much B per CTA (shared-memory bandwidth
// bounds the cta_group::1 form).
template <int BN, bool C2>
struct PCfg {
    static constexpr int kXStages = C2 ? 4 : 3;                            // 64-k x stages
    // 64-k A slots (C2: deeper, the leader's MMA waits for both CTAs' transforms)
    static constexpr int kASlots = C2 ? RQ4_C2_ASLOTS : 4;
    static constexpr uint32_t kXStageBytes = (C2 ? BN / 2 : BN) * kTcXStageK * 2;   // per CTA
    static constexpr uint32_t kNumBars = 2 * kPWStages + 2 * kASlots + 2 * kXStages + 4;
    static constexpr uint32_t kOffCodes = 0;
    static constexpr uint32_t kOffScales = kOffCodes + kPWStages * kPCodes;       // 48 KB
    static constexpr uint32_t kOffA = kOffScales + kPWStages * kPScales + 2048;   // 56 KB (1 KB aligned)
    static constexpr uint32_t kOffX = kOffA + kASlots * kPASlotBytes;             // 120 KB (C1)
    static constexpr uint32_t kOffBar = kOffX + kXStages * kXStageBytes;
    static constexpr uint32_t kSmemBytes = kOffBar + kNumBars * 8 + 16 + 1024;  // + align slack
    static constexpr uint32_t kTmemCols = 2 * BN;                          // two accumulators
    static_assert(kOffA % 1024 == 0 && kOffX % 1024 == 0, "SW128 operands need 1 KB alignment");
    static_assert(kSmemBytes <= 227 * 1024, "shared memory budget");
};

struct TpArgs {
    int64_t n, K, N;
    uint16_t* y;
    int kt;                   // 256-k W stages per tile (= K / 256)
    int64_t m_tiles, tiles;   // m-tile pairs, and pair tiles = m_tiles * ceil(n / 256), pairs fastest
    // stream-K (sk = 1): the pair tiles [sk_tile0, tiles) are cut into units
    // (pair tile, 256-k stage), units = (tiles - sk_tile0) * kt of them, split
    // into one contiguous range per cluster; a tile whose range is cut between
    // clusters is reduced through the workspace by the last cluster to finish
    // it (fp32 partials, fixed cluster order).  The whole tiles [0, sk_tile0)
    // (a multiple of the cluster count: the full waves) go round-robin, AFTER
    // each cluster's units, so the fixups of the cut tiles run in the
    // epilogue while the MMA streams a whole tile (sk_tile0 = 0: pure stream-K).
    int sk;
    int64_t units, sk_tile0;
    float* part;              // [cluster][rank][slot 0/1][BN/4][128 rows][4] fp32
    uint32_t* tick;           // [pair tile][rank], zero before and after every call
    int trace;                // experiments build: per-CTA segment timeline
    int64_t ldy;              // row stride of y (N, or the full width for a row range)
};

// Experiments build (RELAX_Q4_TRACE=1): per CTA {smid, segments, t_setup,
// per segment (<= kPtSegs) {p, t_acc_full, t_partial_written, t_all_partials,
// t_done}, t_end} in globaltimer ns (relax_debug_ptrace_read)
constexpr int kPtSegs = 8;
constexpr int kPtWords = 3 + kPtSegs * 5 + 1;
#if RQ4_TRACE
__device__ uint64_t g_ptrace[512 * kPtWords];
#define PT_STAMP(w, v) do { if (a.trace && lane == 0 && warp == 12) g_ptrace[blockIdx.x * kPtWords + (w)] = (v); } while (0)
#else
#define PT_STAMP(w, v) do { } while (0)
#endif

// The work of one cluster: whole pair tiles p = cluster + i * clusters
// (sk = 0), or the stages [kb0, kb1) of the pair tiles its unit range covers
// followed by its whole tiles (sk = 1).  Every warp role walks the same sequence.
struct Seg {
    int64_t p;
    int kb0, kb1;
};
struct SegIter {
    int64_t cur, end, step, dp, dpend;
    int kt, sk;
    __device__ SegIter(const TpArgs& a, int64_t cid, int64_t nclu) : kt(a.kt), sk(a.sk) {
        if (a.sk) {
            const int64_t base = a.sk_tile0 * a.kt;
            cur = base + cid * a.units / nclu;
            end = base + (cid + 1) * a.units / nclu;
            dp = cid; dpend = a.sk_tile0; step = nclu;
        } else { cur = cid; end = a.tiles; step = nclu; dp = dpend = 0; }
    }
    __device__ bool next(Seg& g) {
        if (!sk) {
            if (cur >= end) return false;
            g.p = cur; g.kb0 = 0; g.kb1 = kt; cur += step; return true;
        }
        if (cur < end) {
            g.p = cur / kt;
            g.kb0 = static_cast<int>(cur - g.p * kt);
            const int64_t left = end - cur;
            g.kb1 = static_cast<int>(left < kt - g.kb0 ? g.kb0 + left : kt);
            cur += g.kb1 - g.kb0;
            return true;
        }
        if (dp >= dpend) return false;
        g.p = dp; g.kb0 = 0; g.kb1 = kt; dp += step;
        return true;
    }
};
// stream-K bookkeeping (global unit u = pair tile * kt + stage): first unit of
// cluster c, the cluster owning unit u, and the partial slot cluster c uses
// for tile p (0: its range starts in the tile, 1: the tile is the last of its range)
__device__ __forceinline__ int64_t sk_start(const TpArgs& a, int64_t c, int64_t nclu) {
    return a.sk_tile0 * a.kt + c * a.units / nclu;
}
__device__ __forceinline__ int64_t sk_owner(const TpArgs& a, int64_t u, int64_t nclu) {
    return ((u - a.sk_tile0 * a.kt + 1) * nclu + a.units - 1) / a.units - 1;
}
// the fixup loads the partials of up to this many clusters at once
constexpr int kSkMaxP = 8;
// fp32 partial of (cluster, rank, slot): float4 j of row m at [j][m], so a
// warp's 32 rows of one float4 column are 512 contiguous bytes
__device__ __forceinline__ float4* sk_part(const TpArgs& a, int64_t c, uint32_t rank, int64_t slot, int bn) {
    return reinterpret_cast<float4*>(a.part + ((c * 2 + rank) * 2 + slot) * kTcBM * bn);
}

__device__ __forceinline__ void tc_mma_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                          uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
        :: "r"(d_tmem), "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate) : "memory");
}

// x tile load multicast to both CTAs of the pair (same SMEM offset and
// mbarrier in each; every destination's barrier receives the bytes).
__device__ __forceinline__ void tma_load_2d_mc(void* smem_dst, const void* desc, uint64_t* bar, int32_t c0,
                                               int32_t c1, uint16_t mask, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
        ".L2::cache_hint [%0], [%1, {%3, %4}], [%2], %5, %6;"
        :: "r"(smem_u32(smem_dst)), "l"(desc), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "h"(mask), "l"(policy)
        : "memory");
}
// Arrive on the same mbarrier of every CTA in `mask` once this thread's prior MMAs complete.
__device__ __forceinline__ void tc_commit_mc(uint64_t* bar, uint16_t mask) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 :: "r"(smem_u32(bar)), "h"(mask) : "memory");
}

// cta_group::2 forms (C2): the leader CTA issues the pair's MMA; its commits
// arrive on the same barrier of both CTAs; a TMA load into this CTA's shared
// memory completes on the LEADER's barrier; arrivals from either CTA go to the
// leader's barrier.
__device__ __forceinline__ void tc_mma_ss2(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                           uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}"
        :: "r"(d_tmem), "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate) : "memory");
}
__device__ __forceinline__ void tc_commit2_mc(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 :: "r"(smem_u32(bar)), "h"(static_cast<uint16_t>(3)) : "memory");
}
__device__ __forceinline__ void tma_load_2d_2sm(void* smem_dst, const void* desc, uint32_t leader_bar, int32_t c0,
                                                int32_t c1, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%3, %4}], [%2], %5;"
        :: "r"(smem_u32(smem_dst)), "l"(desc), "r"(leader_bar), "r"(c0), "r"(c1), "l"(policy) : "memory");
}
__device__ __forceinline__ void mbar_arrive_leader(uint64_t* bar) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];"
                 :: "r"(mapa_shared(smem_u32(bar), 0)) : "memory");
}

template <int BN, bool C2>
__global__ void __launch_bounds__(kPThreads, 1)
tc_q4_persist_kernel(const __grid_constant__ CUtensorMap tm_w, const __grid_constant__ CUtensorMap tm_s,
                     const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ TpArgs a) {
    using C = PCfg<BN, C2>;
    constexpr int kPBN = BN;
    constexpr uint32_t kPXStageBytes = C::kXStageBytes;
    constexpr int kPXStages = C::kXStages;
    constexpr int kPASlots = C::kASlots;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* codes_sm = smem + C::kOffCodes;
    uint8_t* scales_sm = smem + C::kOffScales;
    uint8_t* a_sm = smem + C::kOffA;
    uint8_t* x_sm = smem + C::kOffX;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
    uint64_t* w_full = bars;
    uint64_t* w_empty = w_full + kPWStages;
    uint64_t* a_full = w_empty + kPWStages;
    uint64_t* a_empty = a_full + kPASlots;
    uint64_t* x_full = a_empty + kPASlots;
    uint64_t* x_empty = x_full + kPXStages;
    uint64_t* acc_full = x_empty + kPXStages;     // [2]
    uint64_t* acc_empty = acc_full + 2;           // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + C::kNumBars);

    const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
    const int lane = threadIdx.x & 31;
    // CTA pairs (clusters of 2) share each token tile: pair p covers m-tiles
    // 2 (p % m_pairs) + {0, 1} of token tile p / m_pairs; each CTA loads half
    // of every x stage and multicasts it to both, halving the L2 -> SM traffic
    // of x, which bounds this kernel (x is re-read once per m-tile).
    const uint32_t rank = cluster_ctarank();
    const int64_t cid = blockIdx.x >> 1, nclu = gridDim.x >> 1;

    pdl_launch_dependents();
    if (threadIdx.x == 0) {
        for (int i = 0; i < kPWStages; ++i) { mbar_init(&w_full[i], 1); mbar_init(&w_empty[i], 8); }
        // C2: the leader's a_full / acc_empty count the warps of both CTAs;
        // x_empty gets the pair MMA's one multicast commit (else one commit
        // from each CTA's MMA)
        for (int i = 0; i < kPASlots; ++i) { mbar_init(&a_full[i], C2 ? 8 : 4); mbar_init(&a_empty[i], 1); }
        for (int i = 0; i < kPXStages; ++i) { mbar_init(&x_full[i], 1); mbar_init(&x_empty[i], C2 ? 1 : 2); }
        for (int i = 0; i < 2; ++i) { mbar_init(&acc_full[i], 1); mbar_init(&acc_empty[i], C2 ? 8 : 4); }
        fence_mbar_init();
    }
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tm_w);
        tma_prefetch_desc(&tm_s);
        tma_prefetch_desc(&tm_x);
    }
    if (warp == 3) {
        if constexpr (C2) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;"
                         :: "r"(smem_u32(tmem_slot)), "n"(C::kTmemCols) : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
        } else {
            tmem_alloc<C::kTmemCols>(tmem_slot);
            tmem_relinquish();
        }
    }
    tc_fence_before();
    __syncthreads();
    cluster_arrive_release();
    cluster_wait_acquire();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ---------------- W producer (weights never depend on the previous kernel)
        if (elect_one()) {
            const uint64_t pol = policy_evict_last();           // W tiles are re-read by later token tiles
            int slot = 0;
            uint32_t ph = 0;
            SegIter it(a, cid, nclu);
            Seg g;
            while (it.next(g)) {
                const int32_t m0 = static_cast<int32_t>((2 * (g.p % a.m_tiles) + rank) * kTcBM);
                for (int i = g.kb0; i < g.kb1; ++i) {
                    mbar_wait(&w_empty[slot], ph ^ 1);
                    mbar_arrive_expect_tx(&w_full[slot], kPCodes + kPScales);
                    tma_load_2d(codes_sm + slot * kPCodes, &tm_w, &w_full[slot], i * (kTcWStageK / 2), m0, pol);
                    tma_load_2d(scales_sm + slot * kPScales, &tm_s, &w_full[slot], i * (kTcWStageK / kGroup), m0, pol);
                    if (++slot == kPWStages) { slot = 0; ph ^= 1; }
                }
            }
        }
    } else if (warp == 3) {
        // ---------------- x producer: the only input that depends on the previous kernel
        if (elect_one()) {
            pdl_wait();
            const uint64_t pol = policy_evict_last();
            int slot = 0;
            uint32_t ph = 0;
            SegIter it(a, cid, nclu);
            Seg g;
            while (it.next(g)) {
                const int32_t n0 = static_cast<int32_t>((g.p / a.m_tiles) * kPBN + rank * (kPBN / 2));
                for (int j = g.kb0 * 4; j < g.kb1 * 4; ++j) {
                    mbar_wait(&x_empty[slot], ph ^ 1);                // both CTAs released the slot
                    if constexpr (C2) {
                        // this CTA's BN/2 tokens into its own slot, completing on the leader's barrier
                        if (rank == 0) mbar_arrive_expect_tx(&x_full[slot], 2 * kPXStageBytes);
                        tma_load_2d_2sm(x_sm + slot * kPXStageBytes, &tm_x, mapa_shared(smem_u32(&x_full[slot]), 0),
                                        j * kTcXStageK, n0, pol);
                    } else {
                        mbar_arrive_expect_tx(&x_full[slot], kPXStageBytes);     // own half + the peer's half
                        tma_load_2d_mc(x_sm + slot * kPXStageBytes + rank * (kPXStageBytes / 2), &tm_x,
                                       &x_full[slot], j * kTcXStageK, n0, 0x3, pol);
                    }
                    if (++slot == kPXStages) { slot = 0; ph ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer (C2: the leader CTA only, for the pair)
        if ((!C2 || rank == 0) && elect_one()) {
            constexpr uint32_t idesc = idesc_f16_f32(C2 ? 2 * kTcBM : kTcBM, kPBN);
            int as = 0, xs = 0;
            uint32_t aph = 0, xph = 0;
            int it = 0;
            SegIter si(a, cid, nclu);
            Seg g;
            for (; si.next(g); ++it) {
                const int b = it & 1;
                mbar_wait(&acc_empty[b], ((it >> 1) & 1) ^ 1);        // the epilogue drained it
                tc_fence_after();
                const uint32_t d = tmem_base + static_cast<uint32_t>(b * kPBN);
                const int j0 = g.kb0 * 4;
                for (int j = j0; j < g.kb1 * 4; ++j) {
                    mbar_wait(&a_full[as], aph);
                    mbar_wait(&x_full[xs], xph);
                    tc_fence_after();
                    const uint64_t adesc = smem_desc_k_sw128(smem_u32(a_sm + as * kPASlotBytes));
                    const uint64_t bdesc = smem_desc_k_sw128(smem_u32(x_sm + xs * kPXStageBytes));
                    if constexpr (C2) {
#pragma unroll
                        for (int kk = 0; kk < kTcXStageK / 16; ++kk)
                            tc_mma_ss2(d, adesc + static_cast<uint64_t>(kk * 2), bdesc + static_cast<uint64_t>(kk * 2),
                                       idesc, (j != j0 || kk != 0) ? 1u : 0u);
                        tc_commit2_mc(&a_empty[as]);                  // both CTAs' A slot
                        tc_commit2_mc(&x_empty[xs]);                  // both CTAs' x slot
                    } else {
#pragma unroll
                        for (int kk = 0; kk < kTcXStageK / 16; ++kk)
                            tc_mma_ss(d, adesc + static_cast<uint64_t>(kk * 2), bdesc + static_cast<uint64_t>(kk * 2),
                                      idesc, (j != j0 || kk != 0) ? 1u : 0u);
                        tc_commit(&a_empty[as]);
                        tc_commit_mc(&x_empty[xs], 0x3);              // release the slot in both CTAs
                    }
                    if (++as == kPASlots) { as = 0; aph ^= 1; }
                    if (++xs == kPXStages) { xs = 0; xph ^= 1; }
                }
                if constexpr (C2) tc_commit2_mc(&acc_full[b]); else tc_commit(&acc_full[b]);
            }
        }
    } else if (warp >= 4 && warp < 12) {
        // ---------------- transform: warp (q, h) dequantises rows 32q..32q+31 of the
        // sub-blocks with parity h into SMEM A slots (slot j % 4 for sub-block j)
        const int tw = warp - 4;
        const int q = tw & 3;
        const int h = tw >> 2;
        const int m = q * 32 + lane;
        const uint32_t rbase = static_cast<uint32_t>((m >> 3) * 1024 + (m & 7) * 128);
        int ws = 0, as = h;
        uint32_t wph = 0, aph = 0;
        SegIter si(a, cid, nclu);
        Seg g;
        while (si.next(g)) {
            for (int i = g.kb0; i < g.kb1; ++i) {
                mbar_wait(&w_full[ws], wph);
                const uint8_t* crow = codes_sm + ws * kPCodes + m * 128;
                const uint32_t* srow = reinterpret_cast<const uint32_t*>(scales_sm + ws * kPScales + m * 16);
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const int sub = h + 2 * u;                    // 64-k sub-block of this stage
                    uint32_t v[2][4][4];
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int chunk = 2 * sub + e;            // 16-B code chunk = one 32-group
                        const uint4 c = *reinterpret_cast<const uint4*>(crow + ((chunk ^ (m & 7)) << 4));
                        const uint32_t sp = srow[sub];
                        const __half sh = __ushort_as_half(e ? hi16(sp) : lo16(sp));
                        const __half2 s2 = __halves2half2(sh, sh);
                        const uint32_t words[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
                        for (int w = 0; w < 4; ++w) dequant_word_natural(words[w], s2, v[e][w]);
                    }
                    mbar_wait(&a_empty[as], aph ^ 1);
                    uint8_t* slot = a_sm + as * kPASlotBytes + rbase;
#pragma unroll
                    for (int e = 0; e < 2; ++e)
#pragma unroll
                        for (int w = 0; w < 4; ++w) {
                            const int c8 = e * 4 + w;             // 8-k chunk of the row's 64 k
                            *reinterpret_cast<uint4*>(slot + ((c8 ^ (m & 7)) << 4)) =
                                make_uint4(v[e][w][0], v[e][w][1], v[e][w][2], v[e][w][3]);
                        }
                    fence_proxy_async_smem();                     // generic stores -> MMA (async proxy)
                    __syncwarp();
                    if (lane == 0) {
                        if constexpr (C2) mbar_arrive_leader(&a_full[as]); else mbar_arrive(&a_full[as]);
                    }
                    as += 2;
                    if (as >= kPASlots) { as -= kPASlots; aph ^= 1; }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&w_empty[ws]);
                if (++ws == kPWStages) { ws = 0; wph ^= 1; }
            }
        }
    } else if (warp >= 12) {
        // ---------------- epilogue: accumulator it % 2 -> fp16 y while the MMA
        // fills the other one
        const int q = warp & 3;                                   // TMEM lanes 32q..32q+31
        const int m = q * 32 + lane;
        const uint32_t lane_base = static_cast<uint32_t>(q * 32) << 16;
        int it = 0;
        bool waited = false;
        SegIter si(a, cid, nclu);
        Seg g;
#ifdef RQ4_EXPERIMENTS
        // stream-K: the cut tiles whose partial this cluster has written and
        // whose slice it still has to sum (a cluster's cut tiles come first in
        // its sequence, at most kSkPending of them, and are summed only once
        // all their partials are written, so no partial waits behind a sum)
        constexpr int kSkPending = 4;
        int64_t pend[kSkPending];
        int npend = 0;
        int pend_it[kSkPending];
        // Sum column slice k of cut tile p over the P partials of clusters
        // ca..cb in cluster order and store it (fp16 RNE).
        auto sk_fixup = [&](const int64_t p, const int tr) {
            const int64_t row = (2 * (p % a.m_tiles) + rank) * kTcBM + m;
            const int64_t n0 = (p / a.m_tiles) * kPBN;
            const bool row_ok = row < a.N;
            const int64_t ca = sk_owner(a, p * a.kt, nclu), cb = sk_owner(a, (p + 1) * a.kt - 1, nclu);
            const int P = static_cast<int>(cb - ca + 1);
            const int k = static_cast<int>(cid - ca);
            uint32_t* tick = &a.tick[p * 2 + rank];
            if (warp == 12 && lane == 0) {
                const uint64_t t0 = globaltimer();
                while (ld_acquire_gpu_u32(tick) < static_cast<uint32_t>(P)) {
                    __nanosleep(64);
                    if (globaltimer() - t0 > 10000000000ull) __trap();   // a partial never came: fail loudly
                }
            }
            asm volatile("bar.sync 5, 128;" ::: "memory");
            if (tr < kPtSegs) PT_STAMP(6 + tr * 5, globaltimer());
            // column slice k: float4 columns [j0, j1) of the tile
            const int nj = kPBN / 4;
            const int j0 = k * nj / P, j1 = (k + 1) * nj / P;
            // source c = 0 is cluster ca (slot 1 if the tile is the second of
            // its range); every later contributor's range starts in the tile (slot 0)
            const float4* src0 = sk_part(a, ca, rank, sk_start(a, ca, nclu) >= p * a.kt ? 0 : 1, kPBN) + m;
            const float4* src1 = sk_part(a, ca + 1, rank, 0, kPBN) + m;
            constexpr int64_t kSrcStride = 4 * kTcBM * kPBN / 4;     // float4s between clusters' slot-0 partials
            // (column j, source c) pairs in order, kSkMaxP loads in flight
            // per batch; each column summed over c = 0..P-1 in order
            const int L = (j1 - j0) * P;
            int jl = j0, cl = 0;
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 1
            for (int q0 = 0; q0 < L; q0 += kSkMaxP) {
                float4 f[kSkMaxP];
                int jq = jl, cq = cl;
#pragma unroll
                for (int t = 0; t < kSkMaxP; ++t) {
                    if (q0 + t < L) {
                        const float4* src = cq == 0 ? src0 : src1 + (cq - 1) * kSrcStride;
                        f[t] = __ldcg(src + jq * kTcBM);
                        if (++cq == P) { cq = 0; ++jq; }
                    }
                }
#pragma unroll
                for (int t = 0; t < kSkMaxP; ++t) {
                    if (q0 + t < L) {
                        if (cl == 0) acc = f[t];
                        else { acc.x += f[t].x; acc.y += f[t].y; acc.z += f[t].z; acc.w += f[t].w; }
                        if (cl == P - 1) {
                            const float o[4] = {acc.x, acc.y, acc.z, acc.w};
#pragma unroll
                            for (int i = 0; i < 4; ++i) {
                                const int64_t tok = n0 + 4 * jl + i;
                                if (row_ok && tok < a.n)
                                    a.y[tok * a.ldy + row] = __half_as_ushort(__float2half_rn(o[i]));
                            }
                        }
                        if (++cl == P) { cl = 0; ++jl; }
                    }
                }
            }
            asm volatile("bar.sync 5, 128;" ::: "memory");           // every row of the slice read
            if (tr < kPtSegs) PT_STAMP(7 + tr * 5, globaltimer());
            if (warp == 12 && lane == 0) {
                // the last of the P clusters to finish its slice zeroes the counter for the next call
                if (atomicAdd(tick, 1u) == static_cast<uint32_t>(2 * P - 1)) *tick = 0u;
            }
        };
#endif
        PT_STAMP(2, globaltimer());
        for (; si.next(g); ++it) {
            const int64_t p = g.p;
            const int b = it & 1;
#ifdef RQ4_EXPERIMENTS
            const bool whole = !a.sk || (g.kb0 == 0 && g.kb1 == a.kt);
            if (whole) {
                for (int i = 0; i < npend; ++i) sk_fixup(pend[i], pend_it[i]);
                npend = 0;
            }
#else
            constexpr bool whole = true;              // the product never schedules stream-K (abi.cpp)
#endif
            const int64_t row = (2 * (p % a.m_tiles) + rank) * kTcBM + m;
            const int64_t n0 = (p / a.m_tiles) * kPBN;
            mbar_wait(&acc_full[b], (it >> 1) & 1);
            tc_fence_after();
            if (it < kPtSegs) { PT_STAMP(3 + it * 5, static_cast<uint64_t>(p) | (static_cast<uint64_t>(g.kb0) << 32) | (static_cast<uint64_t>(g.kb1) << 48)); PT_STAMP(4 + it * 5, globaltimer()); }
            if (!waited) { pdl_wait(); waited = true; }           // y / workspace may still be used by the previous kernel
            const uint32_t col0 = tmem_base + lane_base + static_cast<uint32_t>(b * kPBN);
            const bool row_ok = row < a.N;
            if (whole) {
                // the whole k range of the tile: fp16 stores straight from TMEM
                uint32_t v0[16], v1[16];
                tmem_ld_32x32b_x16(col0, v0);
                tc_wait_ld();
#pragma unroll 1
                for (int c0 = 0; c0 < kPBN; c0 += 32) {
                    tmem_ld_32x32b_x16(col0 + c0 + 16, v1);
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const int64_t tok = n0 + c0 + i;
                        if (row_ok && tok < a.n) a.y[tok * a.ldy + row] = __half_as_ushort(__float2half_rn(__uint_as_float(v0[i])));
                    }
                    tc_wait_ld();
                    if (c0 + 32 < kPBN) tmem_ld_32x32b_x16(col0 + c0 + 32, v0);
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const int64_t tok = n0 + c0 + 16 + i;
                        if (row_ok && tok < a.n) a.y[tok * a.ldy + row] = __half_as_ushort(__float2half_rn(__uint_as_float(v1[i])));
                    }
                    tc_wait_ld();
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    if constexpr (C2) mbar_arrive_leader(&acc_empty[b]); else mbar_arrive(&acc_empty[b]);
                }
                if (it < kPtSegs) PT_STAMP(7 + it * 5, globaltimer());
            }
#ifdef RQ4_EXPERIMENTS
            else {
                // stream-K: a part of the tile's k range, shared by the P clusters
                // ca..cb.  Each writes its fp32 partial, releases the accumulator
                // at once and counts itself in; when all P partials are in,
                // cluster ca + k sums column slice k (sk_fixup, deferred until
                // this cluster's cut tiles are all written).  The P clusters are
                // co-resident (one persistent CTA pair per SM pair) and no
                // partial write waits for a sum, so every wait ends.
                const int64_t slot = sk_start(a, cid, nclu) >= p * a.kt ? 0 : 1;
                float4* mine = sk_part(a, cid, rank, slot, kPBN);
#pragma unroll 1
                for (int c0 = 0; c0 < kPBN; c0 += 16) {
                    uint32_t v[16];
                    tmem_ld_32x32b_x16(col0 + c0, v);
                    tc_wait_ld();
#pragma unroll
                    for (int i = 0; i < 16; i += 4)
                        mine[((c0 + i) / 4) * kTcBM + m] =
                            make_float4(__uint_as_float(v[i]), __uint_as_float(v[i + 1]), __uint_as_float(v[i + 2]),
                                        __uint_as_float(v[i + 3]));
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&acc_empty[b]);               // the MMA may refill it now
                __threadfence();                                         // this thread's partial is visible GPU-wide
                asm volatile("bar.sync 5, 128;" ::: "memory");           // the 4 epilogue warps wrote their rows
                if (warp == 12 && lane == 0) atomicAdd(&a.tick[p * 2 + rank], 1u);
                if (it < kPtSegs) PT_STAMP(5 + it * 5, globaltimer());
                if (npend == kSkPending) {                               // (not reached: <= 2 cut tiles per range)
                    sk_fixup(pend[0], pend_it[0]);
                    for (int i = 1; i < npend; ++i) { pend[i - 1] = pend[i]; pend_it[i - 1] = pend_it[i]; }
                    --npend;
                }
                pend[npend] = p;
                pend_it[npend] = it;
                ++npend;
            }
#endif
        }
#ifdef RQ4_EXPERIMENTS
        for (int i = 0; i < npend; ++i) sk_fixup(pend[i], pend_it[i]);
#endif
#if RQ4_TRACE
        uint32_t sm_id;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(sm_id));
        PT_STAMP(0, static_cast<uint64_t>(sm_id) | (static_cast<uint64_t>(it) << 32));
#endif
        PT_STAMP(1, static_cast<uint64_t>(cid));
        PT_STAMP(kPtWords - 1, globaltimer());
    }

    tc_fence_before();
    __syncthreads();
    cluster_arrive_release();          // the peer may still multicast into / commit onto this CTA
    cluster_wait_acquire();
    tc_fence_after();
    if (warp == 3) {
        if constexpr (C2)
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" :: "r"(tmem_base), "n"(C::kTmemCols)
                         : "memory");
        else
            tmem_dealloc<C::kTmemCols>(tmem_base);
    }
}

// Workspace of the stream-K schedule: the ticket region (zero before and after
// every call) and one fp32 partial tile per (cluster, rank, slot).
size_t persist_sk_ws_bytes(int bn) {
    return kTicketBytes + static_cast<size_t>(num_sms() / 2) * 2 * 2 * kTcBM * bn * 4;
}

template <int BN, bool C2>
static int launch_tc_persist_bn(const uint16_t* x, int64_t n, int64_t K, int64_t N, const uint32_t* w,
                                const uint16_t* s, uint16_t* y, int mode, void* ws, bool pdl, cudaStream_t stream,
                                int64_t ldy) {
    using C = PCfg<BN, C2>;
    CUtensorMap mw, ms, mx;
    int rc = make_map_2d(&mw, CU_TENSOR_MAP_DATA_TYPE_UINT8, w, K / 2, N, K / 2, kTcWStageK / 2, kTcBM,
                         CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) return rc;
    rc = make_map_2d(&ms, CU_TENSOR_MAP_DATA_TYPE_UINT16, s, K / kGroup, N, (K / kGroup) * 2, kTcWStageK / kGroup,
                     kTcBM, CU_TENSOR_MAP_SWIZZLE_NONE);
    if (rc) return rc;
    rc = make_map_2d(&mx, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, x, K, n, K * 2, kTcXStageK, BN / 2,
                     CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) return rc;
    const cudaError_t e = ensure_kernel_attrs(reinterpret_cast<const void*>(tc_q4_persist_kernel<BN, C2>),
                                              static_cast<int>(C::kSmemBytes), true);
    if (e != cudaSuccess) return static_cast<int>(e);
    TpArgs a;
    a.n = n; a.K = K; a.N = N; a.y = y;
    a.ldy = ldy > 0 ? ldy : N;
    a.kt = static_cast<int>(K / kTcWStageK);
    a.m_tiles = ((N + kTcBM - 1) / kTcBM + 1) / 2;             // m-tile PAIRS (an odd last one is zero-filled)
    a.tiles = a.m_tiles * ((n + BN - 1) / BN);                  // pair tiles
    const int64_t clusters = num_sms() / 2;
    const bool sk = mode == 2 && !C2;
    a.sk = sk ? 1 : 0;
    // stream-K: the full waves of whole tiles, the rest cut into units
    a.sk_tile0 = sk ? (a.tiles / clusters) * clusters : 0;
    if (sk && a.sk_tile0 == a.tiles) a.sk = 0;                 // no partial wave: whole tiles only
    // every cluster needs a non-empty unit range (the fixup sums the partials
    // of every cluster between a tile's first and last owner): fold one full
    // wave into the units when the rest alone has fewer units than clusters
    if (a.sk && (a.tiles - a.sk_tile0) * a.kt < clusters && a.sk_tile0 >= clusters) a.sk_tile0 -= clusters;
    a.units = (a.tiles - a.sk_tile0) * a.kt;
    a.tick = static_cast<uint32_t*>(ws);
    a.trace = RQ4_TRACE ? knob_int("RELAX_Q4_TRACE", 0) : 0;
    a.part = a.sk ? reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + kTicketBytes) : nullptr;
    if (a.sk && (!ws || a.tiles * 2 > static_cast<int64_t>(kTicketBytes / 4))) return static_cast<int>(cudaErrorInvalidValue);
    // stream-K keeps every cluster busy (units >= clusters); whole tiles use at most one cluster per tile
    const int64_t grid_clusters = a.sk ? (a.units < clusters && a.sk_tile0 == 0 ? a.units : clusters)
                                       : (a.tiles < clusters ? a.tiles : clusters);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(2 * grid_clusters));
    cfg.blockDim = dim3(kPThreads);
    cfg.dynamicSmemBytes = C::kSmemBytes;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = 2;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    return static_cast<int>(cudaLaunchKernelEx(&cfg, tc_q4_persist_kernel<BN, C2>, mw, ms, mx, a));
}

int launch_tc_persist(const uint16_t* x, int64_t n, int64_t K, int64_t N, const uint32_t* w, const uint16_t* s,
                      uint16_t* y, int bn, int mode, void* ws, bool pdl, cudaStream_t stream, int64_t ldy) {
    if (K % kTcWStageK != 0 || n <= 0) return static_cast<int>(cudaErrorInvalidValue);
#ifdef RQ4_EXPERIMENTS
    // BN = 128 tiles: measured slower than both BN = 256 and one tile per CTA at
    // every n (the A transform is re-done per 128 tokens; profiles/r02/sweep_persist_bn_r02.txt)
    if (bn == 128) return launch_tc_persist_bn<128, false>(x, n, K, N, w, s, y, mode, ws, pdl, stream, ldy);
#endif
    // the pair MMA (cta_group::2) for whole tiles; stream-K keeps the per-CTA form
#ifdef RQ4_EXPERIMENTS
    static const bool c2 = knob_int("RELAX_Q4_PERSIST_C2", 0) != 0;
    if (bn == 256 && c2 && mode != 2) return launch_tc_persist_bn<256, true>(x, n, K, N, w, s, y, mode, ws, pdl, stream, ldy);
#endif
    if (bn == 256) return launch_tc_persist_bn<256, false>(x, n, K, N, w, s, y, mode, ws, pdl, stream, ldy);
    return static_cast<int>(cudaErrorInvalidValue);
}

}  // namespace rq4

#if RQ4_TRACE
extern "C" RELAX_API int relax_debug_ptrace_read(void* host, size_t bytes) {
    const size_t n = sizeof(rq4::g_ptrace) < bytes ? sizeof(rq4::g_ptrace) : bytes;
    return cudaMemcpyFromSymbol(host, rq4::g_ptrace, n) == cudaSuccess ? RELAX_OK : RELAX_ERR_CUDA;
}
#endif
