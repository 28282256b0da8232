// gemm_tc.cu -- the tensor-core path: fused q4f16 dequant + tcgen05 GEMM.
//
// y[t][j] = sum_k x[t][k] * W(k, j) with W = fp16_RNE((q-7) s), the
// dequant producer fused into the matmul, specialised on the
// static (K, N) with n a runtime argument, and split-K partials in
// a caller-planned workspace (workspace lifting; upper-bound
// planning).
//
// "Swap AB" mapping: MMA M = 128 weight rows (output
// features), MMA N = BN tokens, K = 16 per instruction.
//   warp 0   W producer : TMA of packed codes (128 rows x 128 B, SW128) and
//                         scales (128 rows x 16 B) per 256-k stage
//   warp 3   x producer : TMA of x (BN rows x 64 k, SW128) per 64-k sub-block;
//                         out-of-range tokens / k are zero-filled by TMA
//                         (warp 3 also allocates/frees TMEM)
//   warp 2   x permuter : BN <= 64 only -- reorders k inside every 16-B chunk
//                         to match the PRMT-free interleaved dequant
//   warps 4-11 transform: warp (q, h), thread m = 32q + lane owns weight row m
//                         (= TMEM lane m) and dequantises the 64-k sub-blocks of
//                         parity h: reads its row's codes from SMEM, bit-exact
//                         fp16 in registers, tcgen05.st 32x32b straight into a
//                         TMEM A ring -- A never touches HBM or SMEM in fp16;
//                         the first ring-full is done before x even arrives
//   warp 1   MMA issuer : one thread issues tcgen05.mma.kind::f16 with A from
//                         TMEM, B (x) from SMEM, fp32 D in TMEM
//   warps 4-7 epilogue  : tcgen05.ld of D, fp32 -> fp16 RNE, store y.
//   split-K             : cluster mode -- the S CTAs of a tile form a thread-
//                         block cluster and reduce through DSMEM in fixed rank
//                         order; workspace mode (S > 8 or forced) -- fp32
//                         partials in the caller's workspace, the last CTA of a
//                         tile (atomic ticket) sums them in fixed split order.
//                         Both deterministic.
#include <cuda.h>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include "internal.h"
#include "relax_q4.h"
#include "ptx.cuh"
#include "q4_unpack.cuh"
#include "fusion.cuh"
#include "knobs.h"

namespace rq4 {

// Transform warps: 4 TMEM lane quarters x 2 sub-block parities (x 2 k-halves
// with 16).  8 for every tile: 16 for BN >= 128 (one CTA per SM) was measured
// 20-40% slower at n = 512..4096, so the knob stays at 8.
template <int BN> constexpr int tc_transform_warps() { return 8; }
constexpr int kWStages = 4;            // 256-k codes+scales stages in flight
constexpr uint32_t kCodesStageBytes = kTcBM * (kTcWStageK / 2);     // 16 KB
constexpr uint32_t kScalesStageBytes = kTcBM * (kTcWStageK / kGroup) * 2;  // 2 KB
constexpr int kSubPerStage = kTcWStageK / kTcXStageK;                // 4

// ---- optional per-CTA role timing (RELAX_Q4_TRACE=1): wait cycles per role
struct TcTrace { uint32_t cta, smid, nsub, pad; uint64_t t0, t_end;
                 uint64_t w_prod, x_prod, perm, tr_w, tr_a, mma_a, mma_x, epi;
                 uint64_t t_mma0, t_acc, t_epi;       // globaltimer: first MMA issued, accumulator ready, stores done
                 uint64_t t_cb1, t_cred, t_cb2; };    // cluster split: after 1st barrier, after reduce, after 2nd barrier
#if RQ4_TRACE
constexpr int kTcTraceMax = 1 << 14;
__device__ TcTrace g_tctrace[kTcTraceMax];
__device__ uint32_t g_tctrace_n;
#endif

template <bool T>
__device__ __forceinline__ void mbar_wait_t(uint64_t* bar, uint32_t parity, uint64_t& acc) {
    if (T) {
        const uint64_t c0 = clock64();
        mbar_wait(bar, parity);
        acc += clock64() - c0;
    } else {
        mbar_wait(bar, parity);
    }
}

struct TcArgs {
    int64_t n, K, N;
    const uint16_t* xptr;  // x fp16 [n][K] (the permuted-x producer reads it directly)
    uint16_t* y;
    float* part;          // workspace split-K: [split][n][N] fp32 partials
    uint32_t* cnt;        // workspace split-K: per-tile tickets, zero between calls
    int split;
    int kt;               // number of 256-k W stages covering K
    int cluster;          // 1: split-K partials reduced through DSMEM of the cluster
    int trace;            // record role wait cycles (debug)
    uint32_t ops;         // fused epilogue (RELAX_OP_SILU_MUL / RESIDUAL; RMSNORM_X runs before)
    const uint16_t* res;  // RESIDUAL: fp16 [n][Nout]
    int64_t Nout;         // N/2 with SILU_MUL, else N (row stride of y)
    int ytma;             // 1: tm_y is valid (N % 8 == 0) and the FU = 0 epilogue stores by TMA
    int64_t ldy;          // FU = 0: row stride of y (N, or the full width when this launch is a row range)
};

// Final store of output element (tok, row) with value f (fp32 sum) under the
// fused epilogue.  SILU_MUL pairs rows (2j, 2j+1), which sit in adjacent
// lanes of the calling warp: every lane of `mask` must call this (the pair
// exchange is a shuffle), and only the even row of a valid pair stores.
template <int FU>
__device__ __forceinline__ void tc_store(const TcArgs& a, unsigned mask, int64_t tok, int64_t row, float f,
                                         bool valid) {
    if (!FU) {                          // plain matmul: the unfused store, nothing else compiled
        if (valid) a.y[tok * a.ldy + row] = __half_as_ushort(__float2half_rn(f));
        return;
    }
    if (a.ops & RELAX_OP_SILU_MUL) {
        const float fp = __shfl_xor_sync(mask, f, 1);
        if (valid && (row & 1) == 0) {
            const int64_t idx = tok * a.Nout + row / 2;
            a.y[idx] = epilogue_value(silu_mul_value(f, fp), a.ops, a.res, idx);
        }
    } else if (valid) {
        const int64_t idx = tok * a.Nout + row;
        a.y[idx] = epilogue_value(__half_as_ushort(__float2half_rn(f)), a.ops, a.res, idx);
    }
}

// Four consecutive rows rr..rr+3 of token tok (rr % 4 == 0): the cluster
// reduction's vector path.  SiLU-mul pairs (rr, rr+1), (rr+2, rr+3) are
// inside the thread; rows past N are skipped (N is even with SILU_MUL).
template <int FU>
__device__ __forceinline__ void tc_store4(const TcArgs& a, int64_t tok, int64_t rr, const float (&f)[4]) {
    if (tok >= a.n) return;
    if (FU && (a.ops & RELAX_OP_SILU_MUL)) {
#pragma unroll
        for (int j = 0; j < 4; j += 2) {
            if (rr + j < a.N) {
                const int64_t idx = tok * a.Nout + (rr + j) / 2;
                a.y[idx] = epilogue_value(silu_mul_value(f[j], f[j + 1]), a.ops, a.res, idx);
            }
        }
        return;
    }
    if (!FU && rr + 3 < a.N && ((tok * a.ldy + rr) & 3) == 0) {    // one 8-B store
        const uint32_t lo = static_cast<uint32_t>(__half_as_ushort(__float2half_rn(f[0]))) |
                            (static_cast<uint32_t>(__half_as_ushort(__float2half_rn(f[1]))) << 16);
        const uint32_t hi = static_cast<uint32_t>(__half_as_ushort(__float2half_rn(f[2]))) |
                            (static_cast<uint32_t>(__half_as_ushort(__float2half_rn(f[3]))) << 16);
        *reinterpret_cast<uint2*>(a.y + tok * a.ldy + rr) = make_uint2(lo, hi);
        return;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        if (rr + j < a.N) {
            if (FU) {
                const int64_t idx = tok * a.Nout + rr + j;
                a.y[idx] = epilogue_value(__half_as_ushort(__float2half_rn(f[j])), a.ops, a.res, idx);
            } else {
                a.y[tok * a.ldy + rr + j] = __half_as_ushort(__float2half_rn(f[j]));
            }
        }
    }
}

template <int BN>
struct TcCfg {
    // BN <= 64: x is staged by a whole warp with LDG + PRMT + STS into the
    // SW128 B layout, k permuted to match dequant_word_interleaved (no byte
    // permutes in the transform).  BN >= 128: x by TMA, natural k order.
    static constexpr bool kPermX = BN <= 64;
    static constexpr int kTW = tc_transform_warps<BN>();            // transform warps
    static constexpr int kKH = 16 / kTW;                             // 32-k halves per warp and sub-block
    static constexpr int kThreads = (4 + kTW) * 32;
    static constexpr int kCtasPerSm = BN <= 64 ? 2 : 1;
    static constexpr uint32_t kTmemCols = BN <= 64 ? 256 : 512;
    static constexpr uint32_t kA0 = (BN < 32 ? 32 : BN);                 // TMEM col of A ring
    static constexpr int kAStages = static_cast<int>((kTmemCols - kA0) / 32);   // 64-k A slots
    static constexpr uint32_t kXStageBytes = BN * 128;
    static constexpr uint32_t kXBudget = BN <= 64 ? 32 * 1024 : 128 * 1024;
    static constexpr int kXRaw = static_cast<int>(kXBudget / kXStageBytes);
    static constexpr int kXStages = kXRaw < kAStages ? kXRaw : kAStages;
    static constexpr uint32_t kOffCodes = 0;
    static constexpr uint32_t kOffScales = kOffCodes + kWStages * kCodesStageBytes;
    static constexpr uint32_t kOffX = kOffScales + kWStages * kScalesStageBytes;
    static constexpr uint32_t kOffBar = kOffX + kXStages * kXStageBytes;
    static constexpr uint32_t kNumBars = 2 * kWStages + 2 * kAStages + 3 * kXStages + 1;
    static constexpr uint32_t kSmemBytes = kOffBar + kNumBars * 8 + 16 + 1024;  // + align slack
    static_assert(128u * BN * 4u <= kOffBar, "cluster reduction buffer must fit in the rings");
};

// FU = 0: plain matmul (fused-epilogue code compiled out, so the kernel is the
// unfused one register for register); FU = 1: a.ops (SILU_MUL / RESIDUAL).
template <int BN, int FU>
__global__ void __launch_bounds__(TcCfg<BN>::kThreads, TcCfg<BN>::kCtasPerSm)
tc_q4_kernel(const __grid_constant__ CUtensorMap tm_w, const __grid_constant__ CUtensorMap tm_s,
             const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_y,
             const __grid_constant__ TcArgs a) {
    using Cfg = TcCfg<BN>;
    constexpr int AS = Cfg::kAStages;
    constexpr int XS = Cfg::kXStages;
    extern __shared__ uint8_t smem_raw[];
    // 1024-B alignment for the 128B-swizzle atoms.
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* codes_sm = smem + Cfg::kOffCodes;
    uint8_t* scales_sm = smem + Cfg::kOffScales;
    uint8_t* x_sm = smem + Cfg::kOffX;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::kOffBar);
    uint64_t* w_full = bars;
    uint64_t* w_empty = w_full + kWStages;
    uint64_t* a_full = w_empty + kWStages;
    uint64_t* a_empty = a_full + AS;
    uint64_t* x_full = a_empty + AS;
    uint64_t* x_empty = x_full + XS;
    uint64_t* x_perm = x_empty + XS;
    uint64_t* acc_full = x_perm + XS;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + Cfg::kNumBars);
    uint32_t* flag_slot = tmem_slot + 1;

    // warp index through a shuffle: provably warp-uniform, so the per-warp
    // TMEM addresses of the transform stay in uniform registers
    const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
    const int lane = threadIdx.x & 31;
    const int64_t m0 = static_cast<int64_t>(blockIdx.x) * kTcBM;
    const int64_t n0 = static_cast<int64_t>(blockIdx.y) * BN;
    const int z = blockIdx.z;
    const int ks0 = static_cast<int>(static_cast<int64_t>(z) * a.kt / a.split);
    const int ks1 = static_cast<int>(static_cast<int64_t>(z + 1) * a.kt / a.split);
    const int nst = ks1 - ks0;              // >= 1 (split <= kt)
    const int nsub = nst * kSubPerStage;
    __shared__ uint64_t tr_slots[14];
    if (threadIdx.x < 14) tr_slots[threadIdx.x] = 0;
    const uint64_t t_start = (RQ4_TRACE && a.trace) ? globaltimer() : 0;
    uint64_t wacc = 0, wacc2 = 0, wacc3 = 0, wacc4 = 0;

    pdl_launch_dependents();

    if (threadIdx.x == 0) {
        for (int i = 0; i < kWStages; ++i) { mbar_init(&w_full[i], 1); mbar_init(&w_empty[i], Cfg::kTW); }
        for (int i = 0; i < AS; ++i) { mbar_init(&a_full[i], Cfg::kTW / 2); mbar_init(&a_empty[i], 1); }
        for (int i = 0; i < XS; ++i) { mbar_init(&x_full[i], 1); mbar_init(&x_empty[i], 1); mbar_init(&x_perm[i], 1); }
        mbar_init(acc_full, 1);
        fence_mbar_init();
    }
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tm_w);
        tma_prefetch_desc(&tm_s);
        tma_prefetch_desc(&tm_x);
    }
    if (warp == 3) {
        tmem_alloc<Cfg::kTmemCols>(tmem_slot);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ---------------- W producer (weights never depend on the previous kernel)
        if (elect_one()) {
            const uint64_t pol = policy_evict_first();
            int slot = 0;
            uint32_t ph = 0;
            for (int i = 0; i < nst; ++i, slot = (slot + 1 == kWStages) ? 0 : slot + 1, ph ^= (slot == 0)) {
                if ((RQ4_TRACE && a.trace)) mbar_wait_t<true>(&w_empty[slot], ph ^ 1, wacc); else mbar_wait(&w_empty[slot], ph ^ 1);
                mbar_arrive_expect_tx(&w_full[slot], kCodesStageBytes + kScalesStageBytes);
                const int kb = ks0 + i;
                tma_load_2d(codes_sm + slot * kCodesStageBytes, &tm_w, &w_full[slot],
                            kb * (kTcWStageK / 2), static_cast<int32_t>(m0), pol);
                tma_load_2d(scales_sm + slot * kScalesStageBytes, &tm_s, &w_full[slot],
                            kb * (kTcWStageK / kGroup), static_cast<int32_t>(m0), pol);
            }
        }
    } else if (warp == 3) {
        // ---------------- x producer (TMA): the only input that depends on the previous kernel
        if (elect_one()) {
            pdl_wait();
            const uint64_t pol = policy_evict_last();
            int slot = 0;
            uint32_t ph = 0;
            for (int j = 0; j < nsub; ++j, slot = (slot + 1 == XS) ? 0 : slot + 1, ph ^= (slot == 0)) {
                if ((RQ4_TRACE && a.trace)) mbar_wait_t<true>(&x_empty[slot], ph ^ 1, wacc); else mbar_wait(&x_empty[slot], ph ^ 1);
                mbar_arrive_expect_tx(&x_full[slot], Cfg::kXStageBytes);
                const int32_t k = (ks0 * kSubPerStage + j) * kTcXStageK;
                tma_load_2d(x_sm + slot * Cfg::kXStageBytes, &tm_x, &x_full[slot], k,
                            static_cast<int32_t>(n0), pol);
            }
        }
    } else if (warp == 2) {
        // ---------------- x permuter (BN <= 64): reorder the 8 k of every 16-B
        // chunk in place to (0,4,1,5,2,6,3,7) so B matches the A columns of
        // dequant_word_interleaved.  The 128B swizzle moves whole 16-B chunks,
        // so the in-chunk permutation is layout-independent.
        if constexpr (Cfg::kPermX) {
            int slot = 0;
            uint32_t ph = 0;
            for (int j = 0; j < nsub; ++j, slot = (slot + 1 == XS) ? 0 : slot + 1, ph ^= (slot == 0)) {
                if ((RQ4_TRACE && a.trace)) mbar_wait_t<true>(&x_full[slot], ph, wacc); else mbar_wait(&x_full[slot], ph);
                uint4* xt = reinterpret_cast<uint4*>(x_sm + slot * Cfg::kXStageBytes);
#pragma unroll
                for (int it = 0; it < (BN * 8) / 32; ++it) {
                    uint4* p = xt + it * 32 + lane;
                    *p = permute_x8(*p);
                }
                fence_proxy_async_smem();             // generic-proxy writes -> UMMA (async proxy)
                __syncwarp();
                if (lane == 0) mbar_arrive(&x_perm[slot]);
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer
        if (elect_one()) {
            constexpr uint32_t idesc = idesc_f16_f32(kTcBM, BN);
            int as = 0, xs = 0;
            uint32_t aph = 0, xph = 0;
            for (int j = 0; j < nsub; ++j, as = (as + 1 == AS) ? 0 : as + 1, aph ^= (as == 0),
                                           xs = (xs + 1 == XS) ? 0 : xs + 1, xph ^= (xs == 0)) {
                if ((RQ4_TRACE && a.trace)) {
                    mbar_wait_t<true>(&a_full[as], aph, wacc);
                    mbar_wait_t<true>(Cfg::kPermX ? &x_perm[xs] : &x_full[xs], xph, wacc2);
                } else {
                    mbar_wait(&a_full[as], aph);
                    mbar_wait(Cfg::kPermX ? &x_perm[xs] : &x_full[xs], xph);
                }
                tc_fence_after();
                if ((RQ4_TRACE && a.trace) && j == 0) tr_slots[8] = globaltimer();
                const uint64_t bdesc = smem_desc_k_sw128(smem_u32(x_sm + xs * Cfg::kXStageBytes));
#pragma unroll
                for (int kk = 0; kk < kTcXStageK / 16; ++kk) {
                    tc_mma_ts(tmem_base, tmem_base + Cfg::kA0 + as * 32 + kk * 8,
                              bdesc + static_cast<uint64_t>(kk * 2),  // +32 B along K in the atom
                              idesc, (j | kk) != 0 ? 1u : 0u);
                }
                tc_commit(&a_empty[as]);
                tc_commit(&x_empty[xs]);
            }
            tc_commit(acc_full);
        }
    } else if (warp >= 4) {
        // ---------------- transform: 8 warps; warp (q, h) dequantises rows 32q..32q+31
        // of the sub-blocks with parity h into the TMEM A ring.  Slots are free
        // up front, so the first AS sub-blocks are dequantised before x arrives.
        const int tw = warp - 4;
        const int q = tw & 3;                 // TMEM lanes 32q..32q+31 = rows
        const int h = (tw >> 2) & 1;          // sub-block parity
        const int kh0 = (tw >> 3) * Cfg::kKH;   // first k-half (32 k = 4 words) of the sub-block
        const int m = q * 32 + lane;
        const uint32_t lane_base = static_cast<uint32_t>(q * 32) << 16;
        int ws = 0, as = h;                 // this warp's sub-blocks: j = h, h+2, h+4, ...
        uint32_t wph = 0, aph = 0;
        for (int i = 0; i < nst; ++i) {
            if ((RQ4_TRACE && a.trace)) mbar_wait_t<true>(&w_full[ws], wph, wacc); else mbar_wait(&w_full[ws], wph);
            const uint8_t* crow = codes_sm + ws * kCodesStageBytes + m * 128;
            const uint32_t* srow = reinterpret_cast<const uint32_t*>(scales_sm + ws * kScalesStageBytes + m * 16);
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int sub = h + 2 * u;
                uint32_t v[Cfg::kKH][4][4];
#pragma unroll
                for (int e = 0; e < Cfg::kKH; ++e) {
                    const int kh = kh0 + e;
                    const int chunk = 2 * sub + kh;     // 16-B chunk = 32 codes = one group
                    const uint4 c = *reinterpret_cast<const uint4*>(crow + ((chunk ^ (m & 7)) << 4));
                    const uint32_t sp = srow[sub];      // scales of groups 2*sub, 2*sub+1
                    const __half sh = __ushort_as_half(kh ? hi16(sp) : lo16(sp));
                    const __half2 s2 = __halves2half2(sh, sh);
                    const uint32_t words[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
                    for (int w = 0; w < 4; ++w) {
                        if constexpr (Cfg::kPermX) dequant_word_interleaved(words[w], s2, v[e][w]);
                        else dequant_word_natural(words[w], s2, v[e][w]);
                    }
                }
                if ((RQ4_TRACE && a.trace)) mbar_wait_t<true>(&a_empty[as], aph ^ 1, wacc2); else mbar_wait(&a_empty[as], aph ^ 1);
                tc_fence_after();
#pragma unroll
                for (int e = 0; e < Cfg::kKH; ++e) {
                    const uint32_t acol = tmem_base + lane_base + Cfg::kA0 + as * 32 + (kh0 + e) * 16;
#pragma unroll
                    for (int w = 0; w < 4; ++w)
                        tmem_st_32x32b_x4(acol + 4 * w, v[e][w][0], v[e][w][1], v[e][w][2], v[e][w][3]);
                }
                if ((RQ4_TRACE && a.trace)) {
                    const uint64_t c0 = clock64();
                    tc_wait_st();
                    wacc3 += clock64() - c0;
                } else {
                    tc_wait_st();
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&a_full[as]);
                as += 2;
                if (as >= AS) { as -= AS; aph ^= 1; }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&w_empty[ws]);
            if (++ws == kWStages) { ws = 0; wph ^= 1; }
        }
    }

    if ((RQ4_TRACE && a.trace) && lane == 0) {
        if (warp == 0) tr_slots[0] = wacc;                    // W producer: waits for free W slots
        if (warp == 3) tr_slots[1] = wacc;                    // x producer: waits for free x slots
        if (warp == 2) tr_slots[2] = wacc;                    // permuter: waits for x data
        if (warp == 4) { tr_slots[3] = wacc; tr_slots[4] = wacc2; tr_slots[7] = wacc3; }   // transform: W data / A slot / wait::st
        if (warp == 1) { tr_slots[5] = wacc; tr_slots[6] = wacc2; }   // MMA: A ready / x ready
    }
    // ------------------------------------------------------------ epilogue
    const bool epi = warp >= 4 && warp < 8;          // TMEM lanes 32q..32q+31 (transform warps 0-3)
    const int q = warp & 3;
    const int m = q * 32 + lane;
    const uint32_t lane_base = static_cast<uint32_t>(q * 32) << 16;
    const int64_t row = m0 + m;
    const bool row_ok = row < a.N;
    if (a.split == 1) {
        // Direct store: the 8 transform warps split the columns (warps w and
        // w + 4 share TMEM lanes 32 (w % 4) ..), and the TMEM load of the next
        // 16 columns is issued before the stores of the current ones.
        constexpr int kCols = BN >= 32 ? BN / 2 : BN;
        const bool mine = BN >= 32 ? (warp >= 4 && warp < 12) : epi;
        const int cbeg = BN >= 32 ? ((warp - 4) >> 2) * kCols : 0;
        if (mine) {
            mbar_wait(acc_full, 0);
            tc_fence_after();
            if ((RQ4_TRACE && a.trace) && warp == 4 && lane == 0) tr_slots[9] = globaltimer();
            pdl_wait();
            // FU = 0: the fp16 tile is staged in the drained rings as
            // [token][row] (rows contiguous, as in y) and written by one TMA
            // tensor store (out-of-range rows / tokens are clipped by the TMA).
            uint16_t* ytile = reinterpret_cast<uint16_t*>(smem);
            uint32_t v0[16], v1[16];
            tmem_ld_32x32b_x16(tmem_base + lane_base + cbeg, v0);
            tc_wait_ld();
#pragma unroll 1
            for (int c0 = cbeg; c0 < cbeg + kCols; c0 += 32) {
                if (c0 + 16 < cbeg + kCols) tmem_ld_32x32b_x16(tmem_base + lane_base + c0 + 16, v1);
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    if (FU || !a.ytma) tc_store<FU>(a, 0xffffffffu, n0 + c0 + i, row, __uint_as_float(v0[i]),
                                                    row_ok && n0 + c0 + i < a.n);
                    else ytile[(c0 + i) * kTcBM + m] = __half_as_ushort(__float2half_rn(__uint_as_float(v0[i])));
                }
                tc_wait_ld();
                if (c0 + 16 >= cbeg + kCols) break;
                if (c0 + 32 < cbeg + kCols) tmem_ld_32x32b_x16(tmem_base + lane_base + c0 + 32, v0);
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    if (FU || !a.ytma) tc_store<FU>(a, 0xffffffffu, n0 + c0 + 16 + i, row, __uint_as_float(v1[i]),
                                                    row_ok && n0 + c0 + 16 + i < a.n);
                    else ytile[(c0 + 16 + i) * kTcBM + m] = __half_as_ushort(__float2half_rn(__uint_as_float(v1[i])));
                }
                tc_wait_ld();
            }
            if (!FU && a.ytma) {
                fence_proxy_async_smem();                     // generic STS -> async-proxy TMA read
                constexpr int kEpiThreads = (BN >= 32 ? 8 : 4) * 32;
                asm volatile("bar.sync 2, %0;" :: "n"(kEpiThreads) : "memory");
                if (warp == 4 && lane == 0) {
                    tma_store_2d(&tm_y, ytile, static_cast<int32_t>(m0), static_cast<int32_t>(n0));
                    bulk_commit_group();
                    bulk_wait_group_read0();                  // SMEM may be released after this
                }
            }
        }
    } else if (!a.cluster) {
        if (epi) {
            mbar_wait(acc_full, 0);
            tc_fence_after();
            if ((RQ4_TRACE && a.trace) && warp == 4 && lane == 0) tr_slots[9] = globaltimer();
            pdl_wait();
            const bool split = true;
#pragma unroll 1
            for (int c0 = 0; c0 < BN; c0 += 16) {
                uint32_t v[16];
                tmem_ld_32x32b_x16(tmem_base + lane_base + c0, v);
                tc_wait_ld();
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const int64_t tok = n0 + c0 + i;
                    const float f = __uint_as_float(v[i]);
                    if (split) {
                        if (row_ok && tok < a.n) a.part[(static_cast<int64_t>(z) * a.n + tok) * a.N + row] = f;
                    } else {
                        tc_store<FU>(a, 0xffffffffu, tok, row, f, row_ok && tok < a.n);
                    }
                }
            }
            if (split) {
                // workspace split-K: the last CTA of the tile (atomic ticket) sums
                // the partials in fixed split order.
                __threadfence();
                asm volatile("bar.sync 1, 128;" ::: "memory");
                if (warp == 4 && lane == 0) {
                    const uint32_t tile = blockIdx.y * gridDim.x + blockIdx.x;
                    const uint32_t old = atomicInc(a.cnt + tile, static_cast<uint32_t>(a.split - 1));
                    *flag_slot = (old == static_cast<uint32_t>(a.split - 1)) ? 1u : 0u;
                }
                asm volatile("bar.sync 1, 128;" ::: "memory");
                if (*flag_slot) {
                    __threadfence();
#pragma unroll 1
                    for (int c0 = 0; c0 < BN; c0 += 8) {
                        float sum[8];
#pragma unroll
                        for (int u = 0; u < 8; ++u) sum[u] = 0.f;
                        if (row_ok) {
                            for (int s = 0; s < a.split; ++s) {
                                const float* ps = a.part + (static_cast<int64_t>(s) * a.n + n0 + c0) * a.N + row;
#pragma unroll
                                for (int u = 0; u < 8; ++u)
                                    if (n0 + c0 + u < a.n) sum[u] += __ldcg(ps + static_cast<int64_t>(u) * a.N);
                            }
                        }
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            const int64_t tok = n0 + c0 + u;
                            tc_store<FU>(a, 0xffffffffu, tok, row, sum[u], row_ok && tok < a.n);
                        }
                    }
                }
            }
        }
    } else {
        // Cluster split-K: each CTA parks its fp32 accumulator tile in its own
        // shared memory ([BN][128], reusing the drained rings), then CTA r of the
        // cluster sums element range r of the tile over all S CTAs through
        // distributed shared memory in fixed rank order (deterministic, no HBM
        // workspace).
        float* red = reinterpret_cast<float*>(smem);
        // park the tile: 8 warps split the columns (as in the direct store),
        // the next TMEM load issued before the current columns are written
        constexpr int kCols = BN >= 32 ? BN / 2 : BN;
        const bool mine = BN >= 32 ? (warp >= 4 && warp < 12) : epi;
        const int cbeg = BN >= 32 ? ((warp - 4) >> 2) * kCols : 0;
        if (mine) {
            mbar_wait(acc_full, 0);
            tc_fence_after();
            if ((RQ4_TRACE && a.trace) && warp == 4 && lane == 0) tr_slots[9] = globaltimer();
            uint32_t v0[16], v1[16];
            tmem_ld_32x32b_x16(tmem_base + lane_base + cbeg, v0);
            tc_wait_ld();
#pragma unroll 1
            for (int c0 = cbeg; c0 < cbeg + kCols; c0 += 32) {
                if (c0 + 16 < cbeg + kCols) tmem_ld_32x32b_x16(tmem_base + lane_base + c0 + 16, v1);
#pragma unroll
                for (int i = 0; i < 16; ++i) red[(c0 + i) * kTcBM + m] = __uint_as_float(v0[i]);
                tc_wait_ld();
                if (c0 + 16 >= cbeg + kCols) break;
                if (c0 + 32 < cbeg + kCols) tmem_ld_32x32b_x16(tmem_base + lane_base + c0 + 32, v0);
#pragma unroll
                for (int i = 0; i < 16; ++i) red[(c0 + 16 + i) * kTcBM + m] = __uint_as_float(v1[i]);
                tc_wait_ld();
            }
        }
        cluster_arrive_release();
        cluster_wait_acquire();
        if ((RQ4_TRACE && a.trace) && threadIdx.x == 128) tr_slots[11] = globaltimer();
        pdl_wait();
        const uint32_t S = static_cast<uint32_t>(a.split);
        const uint32_t r = cluster_ctarank();
        constexpr uint32_t E = kTcBM * BN;
        // element ranges in units of 4 (16-B DSMEM vector loads, one per rank;
        // 4 consecutive rows of one token, so a SiLU-mul pair stays in a thread)
        const uint32_t e0 = r * (E / 4) / S * 4, e1 = (r + 1) * (E / 4) / S * 4;
        const uint32_t red_addr = smem_u32(red);
        for (uint32_t e = e0 + 4 * threadIdx.x; e < e1; e += 4 * Cfg::kThreads) {
            float f[4] = {0.f, 0.f, 0.f, 0.f};
            for (uint32_t s = 0; s < S; ++s) {
                const float4 v = ld_dsmem_v4f32(mapa_shared(red_addr + e * 4u, s));
                f[0] += v.x; f[1] += v.y; f[2] += v.z; f[3] += v.w;
            }
            const int64_t tok = n0 + static_cast<int64_t>(e / kTcBM);
            const int64_t rr = m0 + static_cast<int64_t>(e % kTcBM);
            tc_store4<FU>(a, tok, rr, f);
        }
        if ((RQ4_TRACE && a.trace) && threadIdx.x == 128) tr_slots[12] = globaltimer();
        cluster_arrive_release();
        cluster_wait_acquire();
        if ((RQ4_TRACE && a.trace) && threadIdx.x == 128) tr_slots[13] = globaltimer();
    }

    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if ((RQ4_TRACE && a.trace) && threadIdx.x == 0) tr_slots[10] = globaltimer();
    if (warp == 3) tmem_dealloc<Cfg::kTmemCols>(tmem_base);
#if RQ4_TRACE
    if ((RQ4_TRACE && a.trace) && threadIdx.x == 0) {
        const uint32_t i = atomicAdd(&g_tctrace_n, 1u);
        if (i < kTcTraceMax) {
            TcTrace r;
            r.cta = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
            uint32_t sm; asm volatile("mov.u32 %0, %%smid;" : "=r"(sm)); r.smid = sm;
            r.nsub = nsub; r.pad = 0; r.t0 = t_start; r.t_end = globaltimer();
            r.w_prod = tr_slots[0]; r.x_prod = tr_slots[1]; r.perm = tr_slots[2];
            r.tr_w = tr_slots[3]; r.tr_a = tr_slots[4]; r.mma_a = tr_slots[5]; r.mma_x = tr_slots[6]; r.epi = tr_slots[7];
            r.t_mma0 = tr_slots[8]; r.t_acc = tr_slots[9]; r.t_epi = tr_slots[10];
            r.t_cb1 = tr_slots[11]; r.t_cred = tr_slots[12]; r.t_cb2 = tr_slots[13];
            g_tctrace[i] = r;
        }
    }
#endif
}

// ---------------------------------------------------------------------------
// Host side: tensor maps (driver entry point through the runtime, so the
// library needs no link-time libcuda) and the launch.
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode_fn() {
    static const EncodeTiledFn fn = []() -> EncodeTiledFn {     // thread-safe one-time lookup
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            return reinterpret_cast<EncodeTiledFn>(p);
        cudaGetLastError();
        return nullptr;
    }();
    return fn;
}

// Tiled tensor map of rank 2..3 (dims innermost first; strides in bytes for
// dims 1..rank-1).  Out-of-bounds box elements are zero-filled and still
// counted in the mbarrier transaction bytes.
int make_tensor_map(CUtensorMap* m, CUtensorMapDataType dt, int rank, const void* base,
                    const uint64_t* dims, const uint64_t* strides, const uint32_t* box,
                    CUtensorMapSwizzle sw) {
    EncodeTiledFn enc = get_encode_fn();
    if (!enc) return static_cast<int>(cudaErrorInitializationError);
    cuuint64_t d[3], st[2];
    cuuint32_t bx[3], estr[3] = {1, 1, 1};
    for (int i = 0; i < rank; ++i) { d[i] = dims[i]; bx[i] = box[i]; }
    for (int i = 0; i + 1 < rank; ++i) st[i] = strides[i];
    CUresult r = enc(m, dt, static_cast<cuuint32_t>(rank), const_cast<void*>(base), d, st, bx, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
#ifdef RQ4_EXPERIMENTS
    if (r != CUDA_SUCCESS && knob_int("RELAX_Q4_PRINT_ERR", 0))
        fprintf(stderr, "rq4: cuTensorMapEncodeTiled -> %d (rank %d base %p dims %llu %llu box %u %u align64 %d)\n",
                static_cast<int>(r), rank, base, (unsigned long long)d[0], (unsigned long long)d[1], bx[0], bx[1],
                static_cast<int>((reinterpret_cast<uintptr_t>(m) & 63u) == 0));
#endif
    return r == CUDA_SUCCESS ? 0 : static_cast<int>(cudaErrorInvalidValue);
}

// 2-D maps are cached per host thread (direct-mapped, keyed by everything the
// map encodes: a hit is exactly the map cuTensorMapEncodeTiled would return),
// so the steady-state dispatch of a call costs a hash probe per operand, not
// an encode (~0.5 us each).  No locking: thread_local.
struct MapKey {
    const void* base;
    uint64_t inner, outer, row_bytes;
    uint32_t box_inner, box_outer;
    int dt, sw;
    bool operator==(const MapKey& o) const {
        return base == o.base && inner == o.inner && outer == o.outer && row_bytes == o.row_bytes &&
               box_inner == o.box_inner && box_outer == o.box_outer && dt == o.dt && sw == o.sw;
    }
};
struct MapEntry { MapKey key; CUtensorMap map; bool valid; };
constexpr int kMapCacheSlots = 1024;

static size_t map_hash(const MapKey& k) {
    uint64_t h = reinterpret_cast<uintptr_t>(k.base) * 0x9E3779B97F4A7C15ull;
    h ^= (k.inner + 0x632BE59BD9B4E019ull + (h << 6) + (h >> 2));
    h ^= (k.outer * 0xD6E8FEB86659FD93ull + (h << 6) + (h >> 2));
    h ^= (k.row_bytes + (static_cast<uint64_t>(k.box_inner) << 20) + (static_cast<uint64_t>(k.box_outer) << 40) +
          (static_cast<uint64_t>(k.dt) << 8) + static_cast<uint64_t>(k.sw) + (h << 6) + (h >> 2));
    return static_cast<size_t>(h ^ (h >> 29));
}

int make_map_2d(CUtensorMap* m, CUtensorMapDataType dt, const void* base, uint64_t inner,
                uint64_t outer, uint64_t row_bytes, uint32_t box_inner, uint32_t box_outer,
                CUtensorMapSwizzle sw) {
    thread_local MapEntry* cache = nullptr;
    if (!cache) cache = new MapEntry[kMapCacheSlots]();       // per thread, lives as long as the thread
    const MapKey key{base, inner, outer, row_bytes, box_inner, box_outer, static_cast<int>(dt), static_cast<int>(sw)};
    MapEntry& e = cache[map_hash(key) % kMapCacheSlots];
    if (e.valid && e.key == key) {
        *m = e.map;
        return 0;
    }
    const uint64_t dims[2] = {inner, outer};
    const uint64_t strides[1] = {row_bytes};
    const uint32_t box[2] = {box_inner, box_outer};
    const int rc = make_tensor_map(m, dt, 2, base, dims, strides, box, sw);
    if (rc == 0) {
        e.key = key;
        e.map = *m;
        e.valid = true;
    }
    return rc;
}

template <int BN, int FU>
static int launch_tc_k(const CUtensorMap& mw, const CUtensorMap& ms, const uint16_t* x,
                        const TcArgs& a, bool pdl, cudaStream_t stream) {
    using Cfg = TcCfg<BN>;
    CUtensorMap mx;
    int rc = make_map_2d(&mx, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, x, a.K, a.n, a.K * 2, kTcXStageK, BN,
                         CU_TENSOR_MAP_SWIZZLE_128B);
#ifdef RQ4_EXPERIMENTS
    if (rc && knob_int("RELAX_Q4_PRINT_ERR", 0)) fprintf(stderr, "rq4: x map failed %d\n", rc);
#endif
    if (rc) return rc;
    const cudaError_t ae = ensure_kernel_attrs(reinterpret_cast<const void*>(tc_q4_kernel<BN, FU>),
                                               static_cast<int>(Cfg::kSmemBytes), true);
#ifdef RQ4_EXPERIMENTS
    if (ae && knob_int("RELAX_Q4_PRINT_ERR", 0)) fprintf(stderr, "rq4: attrs failed %d\n", static_cast<int>(ae));
#endif
    if (ae != cudaSuccess) return static_cast<int>(ae);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>((a.N + kTcBM - 1) / kTcBM),
                       static_cast<unsigned>((a.n + BN - 1) / BN), static_cast<unsigned>(a.split));
    cfg.blockDim = dim3(Cfg::kThreads);
    cfg.dynamicSmemBytes = Cfg::kSmemBytes;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (a.cluster && a.split > 1) {
        attr[1].id = cudaLaunchAttributeClusterDimension;
        attr[1].val.clusterDim.x = 1;
        attr[1].val.clusterDim.y = 1;
        attr[1].val.clusterDim.z = static_cast<unsigned>(a.split);
        cfg.numAttrs = 2;
    }
    // y [n][N] fp16 as a 2-D tensor map {N rows, n tokens}, box {128, BN}
    // (the FU = 0 direct epilogue stores whole tiles through it)
    CUtensorMap my = mx;                 // placeholder when unused (ytma = 0)
    if (a.ytma) {
        rc = make_map_2d(&my, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, a.y, a.N, a.n, a.ldy * 2, kTcBM, BN,
                         CU_TENSOR_MAP_SWIZZLE_NONE);
        if (rc) return rc;
    }
    const int lr = static_cast<int>(cudaLaunchKernelEx(&cfg, tc_q4_kernel<BN, FU>, mw, ms, mx, my, a));
#ifdef RQ4_EXPERIMENTS
    if (lr && knob_int("RELAX_Q4_PRINT_ERR", 0))
        fprintf(stderr, "rq4: tc launch BN=%d grid=(%u,%u,%u) cluster=%d smem=%u stream=%p: %d\n", BN, cfg.gridDim.x,
                cfg.gridDim.y, cfg.gridDim.z, a.cluster, static_cast<unsigned>(cfg.dynamicSmemBytes),
                static_cast<void*>(stream), lr);
#endif
    return lr;
}

template <int BN>
static int launch_tc_bn(const CUtensorMap& mw, const CUtensorMap& ms, const uint16_t* x,
                        const TcArgs& a, bool pdl, cudaStream_t stream) {
    return a.ops ? launch_tc_k<BN, 1>(mw, ms, x, a, pdl, stream) : launch_tc_k<BN, 0>(mw, ms, x, a, pdl, stream);
}

#ifdef RQ4_EXPERIMENTS
// How many thread-block clusters of `s` CTAs of the BN kernel can be resident
// at once (cudaOccupancyMaxActiveClusters: GPC placement, not just SM slots --
// with two CTAs per SM, 96 clusters of 3 do not fit in 296 slots).  Cached;
// -1 without a device.  DESIGN.md §6.
template <int BN>
static int max_clusters_bn(int s) {
    using Cfg = TcCfg<BN>;
    if (ensure_kernel_attrs(reinterpret_cast<const void*>(tc_q4_kernel<BN, 0>), static_cast<int>(Cfg::kSmemBytes),
                            true) != cudaSuccess) {
        cudaGetLastError();
        return -1;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(1, 1, static_cast<unsigned>(s));
    cfg.blockDim = dim3(Cfg::kThreads);
    cfg.dynamicSmemBytes = Cfg::kSmemBytes;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = static_cast<unsigned>(s);
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int m = 0;
    if (cudaOccupancyMaxActiveClusters(&m, tc_q4_kernel<BN, 0>, &cfg) != cudaSuccess) {
        cudaGetLastError();
        return -1;
    }
    return m;
}

int tc_max_active_clusters(int bn, int s) {
    if (s < 1 || s > 8) return -1;
    static std::mutex mu;
    static int cache[5][9];
    static bool init = false;
    const int bi = bn == 16 ? 0 : bn == 32 ? 1 : bn == 64 ? 2 : bn == 128 ? 3 : bn == 256 ? 4 : -1;
    if (bi < 0) return -1;
    std::lock_guard<std::mutex> lk(mu);
    if (!init) {
        for (auto& r : cache) for (int& v : r) v = -2;
        init = true;
    }
    int& v = cache[bi][s];
    if (v == -2) {
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess) { cudaGetLastError(); v = -1; return v; }
        switch (bn) {
            case 16: v = max_clusters_bn<16>(s); break;
            case 32: v = max_clusters_bn<32>(s); break;
            case 64: v = max_clusters_bn<64>(s); break;
            case 128: v = max_clusters_bn<128>(s); break;
            default: v = max_clusters_bn<256>(s); break;
        }
    }
    return v;
}

#endif

// Workspace layout (fixed ticket region first, so one buffer serves every n):
//   [0, kTicketBytes)            uint32 tickets, one per output tile (<= 1024)
//   [kTicketBytes, +split*n*N*4) fp32 split-K partials [split][n][N]
size_t tc_workspace_bytes(int64_t n, int64_t N, int bn, int split) {
    (void)bn;
    if (split <= 1) return 0;
    return kTicketBytes + static_cast<size_t>(split) * n * N * 4;
}

int launch_tc(const uint16_t* x, int64_t n, int64_t K, int64_t N, const uint32_t* w,
              const uint16_t* s, uint16_t* y, const Plan& plan, void* ws, bool pdl,
              cudaStream_t stream, const Fusion& fu, int64_t ldy) {
    CUtensorMap mw, ms;
    int rc = make_map_2d(&mw, CU_TENSOR_MAP_DATA_TYPE_UINT8, w, K / 2, N, K / 2, kTcWStageK / 2, kTcBM,
                         CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) return rc;
    rc = make_map_2d(&ms, CU_TENSOR_MAP_DATA_TYPE_UINT16, s, K / kGroup, N, (K / kGroup) * 2,
                     kTcWStageK / kGroup, kTcBM, CU_TENSOR_MAP_SWIZZLE_NONE);
    if (rc) return rc;
    TcArgs a;
    a.n = n; a.K = K; a.N = N; a.y = y; a.xptr = x;
    a.split = plan.split;
    a.kt = static_cast<int>((K + kTcWStageK - 1) / kTcWStageK);
    a.part = nullptr; a.cnt = nullptr;
    a.cluster = plan.cluster;
    a.ops = fu.ops & (RELAX_OP_SILU_MUL | RELAX_OP_RESIDUAL);
    a.res = fu.res;
    a.Nout = (fu.ops & RELAX_OP_SILU_MUL) ? N / 2 : N;
    a.ldy = ldy > 0 ? ldy : N;
    if (a.ldy != N && a.ops != 0) return static_cast<int>(cudaErrorInvalidValue);
    a.ytma = (a.ops == 0 && plan.split == 1 && N % 8 == 0 && a.ldy % 8 == 0) ? 1 : 0;
    static const int tr = RQ4_TRACE ? knob_int("RELAX_Q4_TRACE", 0) : 0;
    a.trace = tr;
    if (plan.split > 1 && !plan.cluster) {
        a.cnt = static_cast<uint32_t*>(ws);
        a.part = reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + kTicketBytes);
    }
    if (plan.persist && a.ops == 0)
        return launch_tc_persist(x, n, K, N, w, s, y, plan.bn, plan.persist, ws, pdl, stream, a.ldy);
    switch (plan.bn) {
        case 16: return launch_tc_bn<16>(mw, ms, x, a, pdl, stream);
        case 32: return launch_tc_bn<32>(mw, ms, x, a, pdl, stream);
        case 64: return launch_tc_bn<64>(mw, ms, x, a, pdl, stream);
        case 128: return launch_tc_bn<128>(mw, ms, x, a, pdl, stream);
        case 256: return launch_tc_bn<256>(mw, ms, x, a, pdl, stream);
        default: return static_cast<int>(cudaErrorInvalidValue);
    }
}

}  // namespace rq4

#ifdef RQ4_EXPERIMENTS
extern "C" RELAX_API int relax_debug_tc_max_clusters(int bn, int s) { return rq4::tc_max_active_clusters(bn, s); }
#endif

#if RQ4_TRACE
extern "C" RELAX_API int relax_debug_tctrace_read(void* host, size_t max_records, size_t* n_records, int reset) {
    uint32_t n = 0;
    if (cudaMemcpyFromSymbol(&n, rq4::g_tctrace_n, sizeof n) != cudaSuccess) return RELAX_ERR_CUDA;
    if (n > static_cast<uint32_t>(rq4::kTcTraceMax)) n = rq4::kTcTraceMax;
    const size_t m = n < max_records ? n : max_records;
    if (m && cudaMemcpyFromSymbol(host, rq4::g_tctrace, m * sizeof(rq4::TcTrace)) != cudaSuccess) return RELAX_ERR_CUDA;
    if (n_records) *n_records = m;
    if (reset) {
        const uint32_t z = 0;
        if (cudaMemcpyToSymbol(rq4::g_tctrace_n, &z, sizeof z) != cudaSuccess) return RELAX_ERR_CUDA;
    }
    return RELAX_OK;
}
#endif
