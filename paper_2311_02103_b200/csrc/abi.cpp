// abi.cpp -- the C-ABI boundary (include/relax_q4.h): O(1) validation,
// shape-specialised dispatch on the runtime token count n (P:409-413,
// P:432-433), the upper-bound workspace plan, and the
// launches.  No exceptions cross this boundary; nothing here allocates.
#include <cmath>
#include <vector>
#include "relax_q4.h"
#ifdef RQ4_EXPERIMENTS
#include "relax_q4_debug.h"
#endif

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <cuda_runtime.h>

#include "internal.h"
#include "knobs.h"

namespace rq4 {

int gemv_max_n() {
    // measured crossover (profiles/sweep_cross_r01.jsonl): DESIGN.md §6
    static const int v = [] { const int x = knob_int("RELAX_Q4_GEMV_MAX_N", 2); return x >= 0 ? x : 2; }();
    return v;
}

static int ctas_per_sm_tc(int bn) { return bn <= 64 ? 2 : 1; }

// Time model of the persistent BN = 256 kernel (us per 256-k stage per tile,
// one fill/drain per CTA); RELAX_Q4_PERSIST (experiments build) 0 disables it.
static const double kPersistStepUs = 1.3;
static const double kPersistFixedUs = 8.0;
static bool persist_enabled() { static const bool v = knob_int("RELAX_Q4_PERSIST", 1) != 0; return v; }

// Small batches (3 <= n <= 8): the warp-MMA streamed kernel or the split-K
// tcgen05 tiles.  Measured in the decode chain, not per kernel
// (profiles/r02/smalln_dispatch_ab_r02.txt): in isolated
// same-shape chains the tcgen05 kernel leads for long K (11008 x 4096 n = 8:
// 11.9 vs 13.4 us, profiles/r02/sweep_smalln_r02.jsonl), but its two 384-thread
// CTAs per SM leave no room for a neighbour under PDL, so a tcgen05 linear
// between streamed ones costs its neighbours their weight prefetch: 7B decode
// n = 8 4655 tok/s all-streamed vs 3637 with the down projection on tcgen05
// (13B: 2417 vs 1872).  Only the 70B down projection (K = 28672) still gains
// from the tensor-core tiles (560 vs 474 tok/s), and narrow outputs
// (N < 2048, the 70B k/v) keep them.
static bool smalln_preferred(int64_t n, int64_t K, int64_t N) {
    static const int64_t kmax = knob_int("RELAX_Q4_SMALLN_MAX_K", 16384);
    return n >= 3 && n <= smalln_max_n() && N >= 2048 && K <= kmax;
}

// Split-K clusters of s CTAs that all start in the first wave on a B200
// (148 SMs), measured per resident-CTA count by tools/tc_waves.py
// (profiles/tc_waves_r01.txt): the GPC placement of clusters holds fewer than
// slots / s of them (two CTAs per SM: 93 clusters of 3, not 98).  More tiles
// than this at split s run a second wave of clusters (4096 x 12288 at n = 8:
// 96 clusters of 3 took 22.6 us vs 17.1 us at s = 2).  Index s = 1..8.
// On a device with another SM count the B200 table is scaled by the SM ratio
// (rounded down), a conservative estimate: GPC placement is not measured there.
static int64_t cluster_capacity(int bn, int s) {
    static const int64_t two[9] = {0, 296, 148, 93, 71, 56, 45, 37, 33};
    static const int64_t one[9] = {0, 148, 74, 45, 33, 26, 22, 15, 15};
    if (s < 1 || s > 8) return 0;
    const int64_t v = ctas_per_sm_tc(bn) == 2 ? two[s] : one[s];
    const int sms = num_sms();
    return sms == kB200SMs ? v : v * sms / kB200SMs;
}

static int choose_bn(int64_t n, int64_t K, int64_t N) {
    if (n <= 16) return 16;
    if (n <= 32) return 32;
    if (n <= 64) {
        // 33..64 tokens, from the measured sweep (profiles/r02/bn_n33_64_r02.txt;
        // each BN with its automatic split): one 128-token tile for narrow
        // outputs at long K or 28..40 m-tiles at K >= 4096 (4096^2 10.1 -> 9.5 us,
        // 11008 x 4096 17.0 -> 15.5, 28672 x 2048 26.9 -> 21.6), two 32-token
        // tiles for narrow outputs at K >= 8192 (8192 x 1024 9.0 -> 7.4,
        // 14336 x 2048 15.4 -> 13.6), else 64-token tiles at two CTAs per SM
        // (28672 x 6144: 44.4 vs 51.4 us with 128)
        const int64_t tm = (N + kTcBM - 1) / kTcBM;
        if (K >= 16384 && tm <= 16) return 128;
        if (K >= 4096 && tm >= 28 && tm <= 40) return 128;
        if (K >= 8192 && tm <= 16) return 32;
        return 64;
    }
    return 128;                  // n > 64: refined jointly with the split (choose_tc_large)
}

// n > 64 (tensor-bound): pick the token tile BN in {128, 256} and the split-K
// factor s <= 8 together, minimising a wave-quantised time model fitted to
// the measured sweeps (profiles/sweep_c3_*.jsonl):
//   waves = ceil(tiles * s / 148)           (one CTA per SM at BN >= 128)
//   t(us) = waves * (ceil(kt / s) * step + fixed) + [s > 1] * 1  (DSMEM reduce)
//   step  = 0.92 / 1.3 us per 256-k stage, fixed = 5.7 / 8.0 us at BN = 128 / 256.
// Split-K only within one wave: a multi-wave grid of split-K clusters was
// measured far slower than the model (cluster placement), so s > 1 requires
// tiles * s <= 148.  The model only ranks schedules; results never depend on
// it (every BN/split meets the same tolerance).
static void choose_tc_large(int64_t n, int64_t N, int kt, int* bn_out, int* s_out, int* persist_out,
                            bool allow_persist, bool allow_sk, int64_t* rows_a_out, int* split_b_out,
                            int* persist_a_out) {
    *rows_a_out = 0;
    *split_b_out = 1;
    *persist_a_out = 0;
    const int64_t tm = (N + kTcBM - 1) / kTcBM;
    const int64_t sms = num_sms();
    double best = 1e300;
    int bb = 128, bs = 1;
    bool bp = false;
    static const int64_t min_per_sm = knob_int("RELAX_Q4_PERSIST_MIN_TILES", 4);
    static const int force_pbn = knob_int("RELAX_Q4_PERSIST_BN", 0);        // experiments: force the persistent BN
    if (allow_persist && (force_pbn == 128 || force_pbn == 256)) {
        *bn_out = force_pbn;
        *s_out = 1;
        *persist_out = 1;
        return;
    }
    // long K (experiments: RELAX_Q4_PERSIST_MAX_KT): the persistent kernel's SS-form
    // stage is slower than the one-tile kernel's TS form, which its fill/drain
    // saving no longer covers
    static const int persist_max_kt = knob_int("RELAX_Q4_PERSIST_MAX_KT", 24);
    if (allow_persist && kt <= persist_max_kt && tm * ((n + 255) / 256) >= min_per_sm * sms) {
        // persistent BN = 256 tiles (gemm_tc_persist.cu): the epilogue of a
        // tile overlaps the next tile's k-loop, so the fill/drain is paid once
        // per CTA, not per tile.  Measured (profiles/r02/sweep_persist_r02.jsonl):
        // +19-20% at >= 4 tiles per CTA (4096 x 11008 / 4096 x 32000 at
        // n = 4096: 1263 / 1278 vs 1054 / 1070 TFLOP/s), a loss below that
        // (11008 x 4096 n = 2048: 1167 vs 1315), so it is only offered there.
        const int64_t tiles = tm * ((n + 255) / 256);
        const int64_t per_cta = (tiles + sms - 1) / sms;
        const double t = static_cast<double>(per_cta) * kt * kPersistStepUs + kPersistFixedUs;
        best = t;
        bb = 256;
        bp = true;
    }
    // cost of the DSMEM split-K reduction in the model (experiments: RELAX_Q4_SPLIT_US)
    static const double split_us = knob_double("RELAX_Q4_SPLIT_US", 1.0);
    static const double split_short_us = knob_double("RELAX_Q4_SPLIT_SHORT_US", 3.0);
    static const int mw_min_ks = knob_int("RELAX_Q4_MW_SPLIT_MIN_KS", 16);
    for (int bn : {128, 256}) {
        const int64_t tiles = tm * ((n + bn - 1) / bn);
        const double step = bn == 256 ? 1.3 : 0.92;
        const double fixed = bn == 256 ? 8.0 : 5.7;
        for (int s = 1; s <= 8 && s <= kt; ++s) {
            const int ks = (kt + s - 1) / s;
            // several waves of split-K clusters: only 256-token tiles that keep
            // >= mw_min_ks stages per CTA (experiments: RELAX_Q4_MW_SPLIT_MIN_KS)
            const bool multi = bn == 256 && mw_min_ks > 0 && ks >= mw_min_ks && s <= 2;
            if (s > 1 && tiles > kMaxSplitTiles) break;
            if (s > 1 && !multi && tiles * s > sms) break;
            if (s > 1 && !multi && tiles > cluster_capacity(bn, s)) continue;   // clusters would not all be resident
            const int64_t cap = s > 1 ? cluster_capacity(bn, s) : sms;
            const int64_t waves = s > 1 ? (tiles + cap - 1) / cap : (tiles + sms - 1) / sms;
            // a split that leaves <= 2 stages per CTA pays its cluster reduction
            // unamortised once the unsplit grid already has >= 64 tiles (1024 x 8192
            // at n = 65..128: s = 2 8.2 us vs s = 1 6.8 us); with fewer tiles the
            // extra CTAs still win (1024 x 1024 n = 65: s = 4 5.2 vs s = 1 6.7 us;
            // profiles/r02/split_short_k_r02.txt)
            const double t = static_cast<double>(waves) * (ks * step + fixed) +
                             (s > 1 ? (ks <= 2 && tiles >= 64 ? split_short_us : split_us) : 0.0);
            // several waves of split clusters must win by 10% in the model: at a
            // smaller margin they measured up to 6% slower (profiles/r02/long_k_r02.txt)
            const double margin = s > 1 && tiles * s > sms ? 0.9 : 0.999;
            if (t < best * margin) { best = t; bb = bn; bs = s; bp = false; }
        }
    }
    int bpk = bp ? 1 : 0;
    // Stream-K on the persistent kernel (gemm_tc_persist.cu) for grids that
    // whole tiles quantise badly (4096 x 11008 at n = 512: 86 pair tiles on 74
    // CTA pairs): the full waves run as whole tiles, the W rest tiles are cut
    // into (tile, 256-k stage) units spread evenly over all pairs and run
    // FIRST, so the fixup of a cut tile (partials through the workspace) runs
    // in the epilogue while the MMA streams a whole tile.  Model: a pair's
    // stages x the persistent step + fill/drain (+ the exposed fixup of a
    // grid without whole tiles).
    // Measured slower than the whole-tile schedules on most 7B/70B shapes
    // (profiles/r02/streamk_ab_r02.txt: the fixup traffic of 128-KB fp32
    // partials per cut tile competes with the MMA operand stream in L2), so
    // the product never offers it; experiments build: RELAX_Q4_STREAMK=1.
#ifdef RQ4_EXPERIMENTS
    static const int sk_knob = knob_int("RELAX_Q4_STREAMK", 0);
#else
    const int sk_knob = 0;
#endif
    const int64_t clusters = sms / 2;
    const int64_t pair_tiles = ((tm + 1) / 2) * ((n + 255) / 256);
    if (allow_persist && allow_sk && sk_knob && n >= 256 && pair_tiles * 2 <= static_cast<int64_t>(kTicketBytes / 4)) {
        const int64_t full = pair_tiles / clusters, rest = pair_tiles - full * clusters;
        if (rest > 0 && (full > 0 || sk_knob == 2)) {
            // (a rest with fewer units than clusters takes one full wave with it, gemm_tc_persist.cu)
            const int64_t cut = rest * kt < clusters && full > 0 ? rest + clusters : rest;
            const int64_t stages = (pair_tiles - cut) / clusters * kt + (cut * kt + clusters - 1) / clusters;
            const double t = static_cast<double>(stages) * kPersistStepUs + kPersistFixedUs + (full ? 1.0 : 3.0);
            if (t < best * 0.9) { bb = 256; bs = 1; bpk = 2; }
        }
    }
    // Two-part schedule: when whole 256-token tiles leave a partial last wave,
    // run the full waves as whole tiles over the leading rows and the rest
    // rows as split-K clusters in a second launch (both existing kernels; the
    // rest costs ceil(kt / s) stages instead of kt).  Offered with a 3%
    // margin over the model's best (every point offered at that margin measured
    // 1-33% faster, profiles/r02/two_part_r02.txt).
#ifdef RQ4_EXPERIMENTS
    static const int two_part = knob_int("RELAX_Q4_TWO_PART", 1);
#else
    const int two_part = 1;
#endif
    static const double tp_margin = knob_double("RELAX_Q4_TWO_PART_MARGIN", 0.97);
    static const int two_part_bn128 = knob_int("RELAX_Q4_TWO_PART_BN128", 1);
    for (int bn : {256, 128}) {
        if (bn == 128 && two_part_bn128 == 0) continue;
        const double step = bn == 256 ? 1.3 : 0.92;
        const double fixed = bn == 256 ? 8.0 : 5.7;
        const int64_t tt = (n + bn - 1) / bn;
        const int64_t full = tm * tt / sms;
        // 128-token tiles: measured ahead for n <= 128 (4096 x 22016 38.2 -> 31.7 us,
        // 8192 x 57344 140.8 -> 120.2) and at K >= 11008, behind at n = 160..384 on
        // K <= 8192 (profiles/r02/two_part_r02.txt)
        if (bn == 128 && !(tt == 1 || kt >= 43)) continue;
        if (two_part && full >= 1 && tm * tt % sms != 0) {
            const int64_t ma = full * sms / tt;                   // m-tiles of the whole-tile part
            const int64_t tiles_b = (tm - ma) * tt;
            int sb = 0;
            for (int s = 8; s >= 2; --s)
                if ((kt + s - 1) / s >= 2 && tiles_b * s <= sms && tiles_b <= cluster_capacity(bn, s)) { sb = s; break; }
            if (ma > 0 && tiles_b > 0 && sb > 1) {
                const double ta = static_cast<double>((ma * tt + sms - 1) / sms) * (kt * step + fixed);
                const double tb = static_cast<double>((kt + sb - 1) / sb) * step + fixed + split_us;
                if (ta + tb < best * tp_margin) {
                    best = ta + tb; bb = bn; bs = 1; bpk = 0;
                    *rows_a_out = ma * kTcBM;
                    *split_b_out = sb;
                    *persist_a_out = 0;
                }
            }
        }
    }
    {
        const int64_t tt = (n + 255) / 256;
        // the same with the leading rows on the persistent kernel (whole rounds
        // of pair tiles over 256-row m-pairs), where that kernel is offered
        const int64_t pm = (tm + 1) / 2, nclu = sms / 2;
        const int64_t full_r = pm * tt / nclu;
        if (two_part == 1 && allow_persist && kt <= persist_max_kt && full_r >= 1 && pm * tt % nclu != 0) {
            const int64_t map = full_r * nclu / tt;               // m-pairs of the persistent part
            const int64_t tiles_b = (tm - 2 * map) * tt;
            int sb = 0;
            for (int s = 8; s >= 2; --s)
                if ((kt + s - 1) / s >= 2 && tiles_b * s <= sms && tiles_b <= cluster_capacity(256, s)) { sb = s; break; }
            if (map > 0 && tiles_b > 0 && sb > 1 && map * tt * 2 >= min_per_sm * sms) {
                const double ta = static_cast<double>((map * tt + nclu - 1) / nclu) * kt * kPersistStepUs + kPersistFixedUs;
                const double tb = static_cast<double>((kt + sb - 1) / sb) * 1.3 + 8.0 + split_us;
                if (ta + tb < best * tp_margin) {
                    best = ta + tb; bb = 256; bs = 1; bpk = 0;
                    *rows_a_out = map * 2 * kTcBM;
                    *split_b_out = sb;
                    *persist_a_out = 1;
                }
            }
        }
    }
    *bn_out = bb;
    *s_out = bs;
    *persist_out = bpk;
}

// Split-K factor for small n (<= 64, HBM-bound): aim for about two CTAs per
// SM -- the occupancy of the BN <= 64 tiles -- so every SM streams with two
// pipelines (RELAX_Q4_TC_CTAS_PER_SM scales the target; measured 1.0 vs 2.0
// in DESIGN.md §6: 2.0 is 3-20% faster on every 7B shape at n = 3..64).
static int choose_split(int64_t n, int64_t tiles, int kt, int bn) {
    (void)n;
    static const double f = [] {
        const double v = knob_double("RELAX_Q4_TC_CTAS_PER_SM", 2.0);
        return v > 0.1 && v <= 4.0 ? v : 2.0;
    }();
    const double target = f * num_sms();
    int s = static_cast<int>(target / static_cast<double>(tiles) + 0.5);
    if (s < 1) s = 1;
    if (s > 8) s = 8;            // portable cluster: DSMEM reduction, no workspace
    if (s > kt) s = kt;
    // one wave of clusters (cluster_capacity)
    while (s > 1 && tiles > cluster_capacity(bn, s)) --s;
    return s;
}

int make_plan(int64_t n, int64_t K, int64_t N, int force_variant, int force_split, int force_bn,
              Plan* out, bool force_ws, bool no_persist, bool allow_sk) {
    if (n < 0 || K <= 0 || N <= 0) return RELAX_ERR_INVALID_ARG;
    if (K % kGroup != 0) return RELAX_ERR_UNSUPPORTED_SHAPE;
    Plan p;
    const bool tc_ok = (K % kTcWStageK == 0);
    int v = force_variant;
    if (v == kVariantAuto) {
        const int nt = static_cast<int>(n < kGemvMaxNT ? n : kGemvMaxNT);
        const int nt1 = nt < 1 ? 1 : nt;
        if (n <= gemv_max_n() && (gemv_stream_ok(nt1, K, N) || gemv_fits(nt1, K))) v = kVariantGemv;
        else if (smalln_preferred(n, K, N) && smalln_mma_ok(n, K, N)) v = kVariantSmallN;
        else if (tc_ok) v = kVariantTc;
        else v = kVariantGemv;
    }
    if (v == kVariantGemv) {
        int nt = static_cast<int>(n < kGemvMaxNT ? n : kGemvMaxNT);
        if (nt < 1) nt = 1;
        while (nt > 1 && !gemv_fits(nt, K) && !(nt <= 2 && gemv_stream_ok(nt, K, N))) --nt;
        if (!gemv_fits(nt, K) && !gemv_stream_ok(nt, K, N)) return RELAX_ERR_UNSUPPORTED_SHAPE;
        p.variant = kVariantGemv;
        p.nt = nt;
        p.ws_bytes = 0;
    } else if (v == kVariantSmallN) {
        if (!smalln_mma_ok(n < 1 ? 1 : n, K, N)) return RELAX_ERR_UNSUPPORTED_SHAPE;
        p.variant = kVariantSmallN;
        p.nt = 8;
        p.ws_bytes = 0;
    } else if (v == kVariantTc) {
        if (!tc_ok) return RELAX_ERR_UNSUPPORTED_SHAPE;
        p.variant = kVariantTc;
        const int kt = static_cast<int>(K / kTcWStageK);
        int auto_split = 0;
        if (force_bn) {
            if (force_bn != 16 && force_bn != 32 && force_bn != 64 && force_bn != 128 && force_bn != 256)
                return RELAX_ERR_INVALID_ARG;
            p.bn = force_bn;
        } else if (n > 64 && force_split <= 0) {
            int persist = 0;
            choose_tc_large(n, N, kt, &p.bn, &auto_split, &persist, !no_persist && persist_enabled(), allow_sk,
                            &p.rows_a, &p.split_b, &p.persist_a);
            p.persist = persist;
        } else {
            p.bn = choose_bn(n, K, N);
        }
        const int64_t tiles = ((N + kTcBM - 1) / kTcBM) * ((n + p.bn - 1) / p.bn);
        int s = force_split > 0 ? force_split
              : auto_split > 0 ? auto_split
              : n > 64 ? 1 : choose_split(n, tiles, kt, p.bn);
        if (s > kt) s = kt;
        if (s < 1) s = 1;
        if (s > 1 && tiles > kMaxSplitTiles) {
            if (force_split > 1) return RELAX_ERR_UNSUPPORTED_SHAPE;
            s = 1;
        }
        p.split = s;
        // a forced BN = 256 without split also runs persistent unless told otherwise
        if (force_bn == 256 && s == 1 && !no_persist && persist_enabled()) p.persist = 1;
        if (s > 1) p.persist = 0;
        // split-K partials: reduced in a thread-block cluster through DSMEM when
        // the split fits a portable cluster (<= 8), else in the workspace.
        p.cluster = (s > 1 && s <= 8 && !force_ws) ? 1 : 0;
        p.ws_bytes = p.cluster ? 0 : tc_workspace_bytes(n, N, p.bn, s);
        if (p.persist == 2) p.ws_bytes = persist_sk_ws_bytes(p.bn);
    } else {
        return RELAX_ERR_INVALID_ARG;
    }
    *out = p;
    return RELAX_OK;
}

// ---------------------------------------------------------------------------
static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

static bool overlap(const void* a, size_t na, const void* b, size_t nb) {
    if (!a || !b || na == 0 || nb == 0) return false;
    const uintptr_t a0 = reinterpret_cast<uintptr_t>(a), b0 = reinterpret_cast<uintptr_t>(b);
    return a0 < b0 + nb && b0 < a0 + na;
}

static int check_device() {
    int dev = -1;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0) {
        cudaGetLastError();
        return RELAX_ERR_DEVICE;
    }
    static std::mutex mu;
    static int cc[64];           // 0 = unknown, else major*10+minor
    if (dev >= 64) return RELAX_ERR_DEVICE;
    int c;
    {
        std::lock_guard<std::mutex> lk(mu);
        c = cc[dev];
    }
    if (c == 0) {
        int major = 0, minor = 0;
        if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess) {
            cudaGetLastError();
            return RELAX_ERR_DEVICE;
        }
        c = major * 10 + minor;
        std::lock_guard<std::mutex> lk(mu);
        cc[dev] = c;
    }
    if (c != 100) return RELAX_ERR_DEVICE;
    // The tensor maps are encoded with the driver API (cuTensorMapEncodeTiled),
    // which needs the device's context current in the CALLING thread; a host
    // thread whose runtime calls so far did not bind it (seen after other
    // threads had driven the device) got CUDA_ERROR_INVALID_CONTEXT.  Bind the
    // primary context once per (thread, device).
    thread_local int bound_dev = -1;
    if (bound_dev != dev) {
        if (cudaSetDevice(dev) != cudaSuccess) {
            cudaGetLastError();
            return RELAX_ERR_DEVICE;
        }
        bound_dev = dev;
    }
    return RELAX_OK;
}

static int matmul_impl(const void* x, int64_t n, int64_t K, int64_t N, const uint32_t* packed_w,
                       const void* scales, void* y, void* ws, size_t ws_bytes, int variant,
                       int split_k, int bn, unsigned flags, void* stream) {
    if (n < 0 || K <= 0 || N <= 0) return RELAX_ERR_INVALID_ARG;
    if (K % kGroup != 0) return RELAX_ERR_UNSUPPORTED_SHAPE;
    if (variant < 0 || variant > 3 || split_k < 0) return RELAX_ERR_INVALID_ARG;
    if (n == 0) return RELAX_OK;
    if (!x || !packed_w || !scales || !y) return RELAX_ERR_INVALID_ARG;
    if (ws_bytes > 0 && !ws) return RELAX_ERR_INVALID_ARG;
    if (!aligned16(x) || !aligned16(packed_w) || !aligned16(scales) || !aligned16(y) ||
        (ws && !aligned16(ws)))
        return RELAX_ERR_MISALIGNED;
    const size_t xb = static_cast<size_t>(n) * K * 2, yb = static_cast<size_t>(n) * N * 2;
    const size_t wb = static_cast<size_t>(N) * K / 2, sb = static_cast<size_t>(N) * (K / kGroup) * 2;
    if (overlap(y, yb, x, xb) || overlap(y, yb, packed_w, wb) || overlap(y, yb, scales, sb) ||
        overlap(y, yb, ws, ws_bytes) || overlap(ws, ws_bytes, x, xb) ||
        overlap(ws, ws_bytes, packed_w, wb) || overlap(ws, ws_bytes, scales, sb))
        return RELAX_ERR_ALIAS;
    Plan plan;
    // Without a workspace the schedule is workspace-free (split-K = 1).
    const bool force_ws = (flags & RELAX_FLAG_SPLIT_WORKSPACE) != 0;
    const bool no_persist = (flags & RELAX_FLAG_TILE_PER_CTA) != 0;
    int rc = make_plan(n, K, N, variant, split_k, bn, &plan, force_ws, no_persist);
    if (rc == RELAX_OK && plan.persist == 2 && ws_bytes < plan.ws_bytes)         // stream-K needs its workspace
        rc = make_plan(n, K, N, variant, split_k, bn, &plan, force_ws, no_persist, false);
    if (rc == RELAX_OK && plan.ws_bytes > 0 && ws_bytes == 0 && !force_ws && split_k == 0) {
        // no workspace given: fall back to the largest cluster-reduced split
        int s = plan.split < 8 ? plan.split : 8;
        rc = make_plan(n, K, N, variant, s, bn, &plan, false, no_persist, false);
    }
    if (rc != RELAX_OK) return rc;
    if (plan.ws_bytes > ws_bytes) return RELAX_ERR_WORKSPACE;
    rc = check_device();
    if (rc != RELAX_OK) return rc;
    const bool pdl = (flags & RELAX_FLAG_NO_PDL) == 0;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    int e;
    if (plan.variant == kVariantGemv)
        e = launch_gemv(static_cast<const uint16_t*>(x), n, K, N, packed_w,
                        static_cast<const uint16_t*>(scales), static_cast<uint16_t*>(y), plan.nt, pdl, st);
    else if (plan.variant == kVariantSmallN)
        e = launch_smalln_mma(static_cast<const uint16_t*>(x), n, K, N, packed_w,
                              static_cast<const uint16_t*>(scales), static_cast<uint16_t*>(y), pdl, st);
    else if (plan.rows_a > 0) {
        // two-part schedule: the full waves of whole 256-token tiles over rows
        // [0, rows_a), then the remaining rows as split-K clusters (a second
        // launch: its CTAs take the SMs the first one frees, under PDL)
        Plan pa = plan, pb = plan;
        pa.rows_a = pb.rows_a = 0;
        pa.split = 1; pa.cluster = 0;
        pa.persist = plan.persist_a; pb.persist = 0;
        pb.split = plan.split_b; pb.cluster = 1;
        const uint16_t* sc = static_cast<const uint16_t*>(scales);
        uint16_t* yo = static_cast<uint16_t*>(y);
        e = launch_tc(static_cast<const uint16_t*>(x), n, K, plan.rows_a, packed_w, sc, yo, pa, nullptr, pdl, st,
                      Fusion(), N);
        if (e == 0)
            e = launch_tc(static_cast<const uint16_t*>(x), n, K, N - plan.rows_a, packed_w + plan.rows_a * (K / 8),
                          sc + plan.rows_a * (K / kGroup), yo + plan.rows_a, pb, nullptr, true, st, Fusion(), N);
    } else
        e = launch_tc(static_cast<const uint16_t*>(x), n, K, N, packed_w,
                      static_cast<const uint16_t*>(scales), static_cast<uint16_t*>(y), plan, ws, pdl, st);
    if (e != 0) {
#ifdef RQ4_EXPERIMENTS
        if (knob_int("RELAX_Q4_PRINT_ERR", 0))
            fprintf(stderr, "rq4: matmul n=%lld K=%lld N=%lld variant=%d bn=%d split=%d persist=%d: error %d (%s)\n",
                    (long long)n, (long long)K, (long long)N, plan.variant, plan.bn, plan.split, plan.persist, e,
                    cudaGetErrorString(static_cast<cudaError_t>(e)));
#endif
        cudaGetLastError();
        return RELAX_ERR_CUDA;
    }
    return RELAX_OK;
}

// ---------------------------------------------------------------------------
// Fused neighbours (relax_q4_matmul_fused; include/relax_q4.h).  The plain
// plan picks the variant; RMSNORM_X on the tensor-core path writes the
// normalised x into the workspace after the plan's own bytes.
static constexpr uint32_t kOpsAll = RELAX_OP_RMSNORM_X | RELAX_OP_SILU_MUL | RELAX_OP_RESIDUAL | RELAX_OP_KV_APPEND;

static size_t align16(size_t v) { return (v + 15) & ~static_cast<size_t>(15); }

// Where the tensor path's RMSNORM_X prologue puts the normalised x in a fused
// call's workspace: after the plan's own bytes and never inside the split-K
// ticket region [0, kTicketBytes), so a workspace shared with
// RELAX_FLAG_SPLIT_WORKSPACE calls still finds its tickets zero.
static size_t fused_xn_offset(size_t plan_bytes) { return align16(plan_bytes > kTicketBytes ? plan_bytes : kTicketBytes); }

static int fused_shape_check(int64_t K, int64_t N, uint32_t ops) {
    if (ops & ~kOpsAll) return RELAX_ERR_INVALID_ARG;
    if (ops != 0 && K % kTcWStageK != 0) return RELAX_ERR_UNSUPPORTED_SHAPE;
    if ((ops & RELAX_OP_SILU_MUL) && (N % 2) != 0) return RELAX_ERR_UNSUPPORTED_SHAPE;
    if ((ops & RELAX_OP_KV_APPEND) && (ops & RELAX_OP_SILU_MUL)) return RELAX_ERR_INVALID_ARG;
    return RELAX_OK;
}

static int fused_impl(const void* x, int64_t n, int64_t K, int64_t N, const uint32_t* packed_w,
                      const void* scales, void* y, const relax_q4_fusion* fz, void* ws, size_t ws_bytes,
                      void* stream) {
    const uint32_t ops = fz ? fz->ops : 0u;
    if (ops == 0) return matmul_impl(x, n, K, N, packed_w, scales, y, ws, ws_bytes, 0, 0, 0, 0u, stream);
    if (n < 0 || K <= 0 || N <= 0) return RELAX_ERR_INVALID_ARG;
    if (K % kGroup != 0) return RELAX_ERR_UNSUPPORTED_SHAPE;
    int rc = fused_shape_check(K, N, ops);
    if (rc != RELAX_OK) return rc;
    if ((ops & RELAX_OP_RMSNORM_X) && (!fz->rms_weight || !(fz->rms_eps >= 0.f) || !std::isfinite(fz->rms_eps)))
        return RELAX_ERR_INVALID_ARG;
    if ((ops & RELAX_OP_RESIDUAL) && !fz->residual) return RELAX_ERR_INVALID_ARG;
    const bool kva = (ops & RELAX_OP_KV_APPEND) != 0;
    if (kva && (!fz->k_cache || !fz->v_cache || !fz->kv_pos || fz->kv_len_max <= 0 || fz->kv_heads <= 0 ||
                fz->kv_row0 < 0 || static_cast<int64_t>(fz->kv_row0) + 2 * 128 * static_cast<int64_t>(fz->kv_heads) > N))
        return RELAX_ERR_INVALID_ARG;
    if (kva && n > 2) return RELAX_ERR_UNSUPPORTED_SHAPE;         // decode only
    if (n == 0) return RELAX_OK;
    if (!x || !packed_w || !scales || !y) return RELAX_ERR_INVALID_ARG;
    if (kva && (!aligned16(fz->k_cache) || !aligned16(fz->v_cache) || (reinterpret_cast<uintptr_t>(fz->kv_pos) & 3u)))
        return RELAX_ERR_MISALIGNED;
    if (ws_bytes > 0 && !ws) return RELAX_ERR_INVALID_ARG;
    const void* gamma = (ops & RELAX_OP_RMSNORM_X) ? fz->rms_weight : nullptr;
    const void* res = (ops & RELAX_OP_RESIDUAL) ? fz->residual : nullptr;
    if (!aligned16(x) || !aligned16(packed_w) || !aligned16(scales) || !aligned16(y) ||
        (ws && !aligned16(ws)) || (gamma && !aligned16(gamma)) || (res && !aligned16(res)))
        return RELAX_ERR_MISALIGNED;
    const int64_t Nout = (ops & RELAX_OP_SILU_MUL) ? N / 2 : N;
    const size_t xb = static_cast<size_t>(n) * K * 2, yb = static_cast<size_t>(n) * Nout * 2;
    const size_t wb = static_cast<size_t>(N) * K / 2, sb = static_cast<size_t>(N) * (K / kGroup) * 2;
    const size_t gb = gamma ? static_cast<size_t>(K) * 2 : 0;
    if (overlap(y, yb, x, xb) || overlap(y, yb, packed_w, wb) || overlap(y, yb, scales, sb) ||
        overlap(y, yb, gamma, gb) || overlap(y, yb, ws, ws_bytes) || overlap(ws, ws_bytes, x, xb) ||
        overlap(ws, ws_bytes, packed_w, wb) || overlap(ws, ws_bytes, scales, sb) ||
        overlap(ws, ws_bytes, gamma, gb) || overlap(ws, ws_bytes, res, res ? yb : 0) ||
        (res && res != y && overlap(y, yb, res, yb)))
        return RELAX_ERR_ALIAS;
    if (kva) {
        const size_t cb = static_cast<size_t>(n) * fz->kv_heads * fz->kv_len_max * 128 * 2;
        if (overlap(fz->k_cache, cb, y, yb) || overlap(fz->v_cache, cb, y, yb) || overlap(fz->k_cache, cb, x, xb) ||
            overlap(fz->v_cache, cb, x, xb) || overlap(fz->k_cache, cb, fz->v_cache, cb) ||
            overlap(fz->k_cache, cb, packed_w, wb) || overlap(fz->v_cache, cb, packed_w, wb))
            return RELAX_ERR_ALIAS;
    }
    Plan plan;
    rc = make_plan(n, K, N, kVariantAuto, 0, 0, &plan, false, false, false);
    if (rc == RELAX_OK && plan.ws_bytes > 0 && ws_bytes < plan.ws_bytes) {
        const int sp = plan.split < 8 ? plan.split : 8;
        rc = make_plan(n, K, N, kVariantAuto, sp, 0, &plan, false, false, false);
    }
    if (rc != RELAX_OK) return rc;
    if (plan.variant == kVariantSmallN ||
        (plan.variant == kVariantGemv && !gemv_stream_ok(n >= 2 ? 2 : 1, K, N, (ops & RELAX_OP_SILU_MUL) ? 2 : 1))) {
        // the fused neighbours live in the streamed decode kernel and the
        // tensor-core kernel only: a shape the former cannot hold takes the latter
        rc = make_plan(n, K, N, kVariantTc, 0, 0, &plan, false, false, false);
        if (rc != RELAX_OK) return rc;
    }
    if (kva && plan.variant != kVariantGemv) return RELAX_ERR_UNSUPPORTED_SHAPE;   // the decode kernel's epilogue only
    const bool tc_norm = plan.variant == kVariantTc && (ops & RELAX_OP_RMSNORM_X);
    const size_t xn_off = fused_xn_offset(plan.ws_bytes);
    const size_t need = tc_norm ? xn_off + xb : plan.ws_bytes;
    if (need > ws_bytes) return RELAX_ERR_WORKSPACE;
    rc = check_device();
    if (rc != RELAX_OK) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Fusion fu;
    fu.ops = ops;
    fu.eps = (ops & RELAX_OP_RMSNORM_X) ? fz->rms_eps : 0.f;
    fu.gamma = static_cast<const uint16_t*>(gamma);
    fu.res = static_cast<const uint16_t*>(res);
    if (kva) {
        fu.kc = static_cast<uint16_t*>(fz->k_cache);
        fu.vc = static_cast<uint16_t*>(fz->v_cache);
        fu.kv_pos = fz->kv_pos;
        fu.kv_lmax = fz->kv_len_max;
        fu.kv_heads = fz->kv_heads;
        fu.kv_row0 = fz->kv_row0;
    }
    int e;
    if (plan.variant == kVariantGemv) {
        e = launch_gemv_stream(static_cast<const uint16_t*>(x), n, K, N, packed_w,
                               static_cast<const uint16_t*>(scales), static_cast<uint16_t*>(y), true, st, fu);
    } else {
        const uint16_t* xin = static_cast<const uint16_t*>(x);
        e = 0;
        if (tc_norm) {
            uint16_t* xn = reinterpret_cast<uint16_t*>(static_cast<uint8_t*>(ws) + xn_off);
            e = launch_rmsnorm(xin, n, K, fu.gamma, fu.eps, xn, true, st);
            xin = xn;
        }
        if (e == 0)
            e = launch_tc(xin, n, K, N, packed_w, static_cast<const uint16_t*>(scales), static_cast<uint16_t*>(y),
                          plan, ws, true, st, fu);
    }
    if (e != 0) {
        cudaGetLastError();
        return RELAX_ERR_CUDA;
    }
    return RELAX_OK;
}

}  // namespace rq4

extern "C" {

int relax_plan_workspace_fused(int64_t n_max, int64_t K, int64_t N, uint32_t ops, size_t* ws_bytes) {
    if (!ws_bytes || n_max < 0 || K <= 0 || N <= 0) return RELAX_ERR_INVALID_ARG;
    if (K % rq4::kGroup != 0) return RELAX_ERR_UNSUPPORTED_SHAPE;
    int rc = rq4::fused_shape_check(K, N, ops);
    if (rc != RELAX_OK) return rc;
    const int64_t n_cap = static_cast<int64_t>(rq4::num_sms()) * 256;
    const int64_t hi = n_max < n_cap ? n_max : n_cap;
    const bool norm = (ops & RELAX_OP_RMSNORM_X) != 0;
    size_t best = 0;
    for (int64_t n = 1; n <= hi; ++n) {
        rq4::Plan p;
        rc = rq4::make_plan(n, K, N, rq4::kVariantAuto, 0, 0, &p, false, false, false);
        if (rc != RELAX_OK) return rc;
        // a GEMV plan the streamed decode kernel cannot hold runs on the TC path (fused_impl)
        if (p.variant == rq4::kVariantSmallN ||
            (p.variant == rq4::kVariantGemv &&
             !rq4::gemv_stream_ok(n >= 2 ? 2 : 1, K, N, (ops & RELAX_OP_SILU_MUL) ? 2 : 1))) {
            rc = rq4::make_plan(n, K, N, rq4::kVariantTc, 0, 0, &p, false, false, false);
            if (rc != RELAX_OK) return rc;
        }
        size_t need = p.ws_bytes;
        if (norm && p.variant == rq4::kVariantTc) need = rq4::fused_xn_offset(p.ws_bytes) + static_cast<size_t>(n) * K * 2;
        if (need > best) best = need;
    }
    if (norm && n_max > hi) {
        // beyond n_cap every schedule is split-free (no plan bytes) and takes the TC path
        const size_t need = rq4::fused_xn_offset(0) + static_cast<size_t>(n_max) * K * 2;
        if (need > best) best = need;
    }
    *ws_bytes = best;
    return RELAX_OK;
}

int relax_q4_matmul_fused(const void* x, int64_t n, int64_t K, int64_t N, const uint32_t* packed_w,
                          const void* scales, void* y, const relax_q4_fusion* fusion, void* workspace,
                          size_t ws_bytes, void* stream) {
    return rq4::fused_impl(x, n, K, N, packed_w, scales, y, fusion, workspace, ws_bytes, stream);
}

int relax_plan_workspace(int64_t n_max, int64_t K, int64_t N, size_t* ws_bytes) {
    if (!ws_bytes || n_max < 0 || K <= 0 || N <= 0) return RELAX_ERR_INVALID_ARG;
    if (K % rq4::kGroup != 0) return RELAX_ERR_UNSUPPORTED_SHAPE;
    // Beyond this n every schedule has >= one full wave of tiles, so split-K
    // (the only workspace user) is 1: the maximum is reached below it.
    const int64_t n_cap = static_cast<int64_t>(rq4::num_sms()) * 256;
    const int64_t hi = n_max < n_cap ? n_max : n_cap;
    size_t best = 0;
    for (int64_t n = 1; n <= hi; ++n) {
        rq4::Plan p;
        const int rc = rq4::make_plan(n, K, N, rq4::kVariantAuto, 0, 0, &p, false);
        if (rc != RELAX_OK) return rc;
        if (p.ws_bytes > best) best = p.ws_bytes;
    }
    *ws_bytes = best;
    return RELAX_OK;
}

int relax_query_schedule(int64_t n, int64_t K, int64_t N, int* variant, int* tile, int* split_k,
                         size_t* ws_bytes, int* persistent) {
    rq4::Plan p;
    const int rc = rq4::make_plan(n, K, N, rq4::kVariantAuto, 0, 0, &p, false);
    if (rc != RELAX_OK) return rc;
    if (variant) *variant = p.variant;
    if (tile) *tile = (p.variant == rq4::kVariantGemv || p.variant == rq4::kVariantSmallN) ? p.nt : p.bn;
    if (split_k) *split_k = p.split;
    if (ws_bytes) *ws_bytes = p.ws_bytes;
    if (persistent) *persistent = p.rows_a > 0 ? (p.persist_a ? 4 : 3) : p.persist;
    return RELAX_OK;
}

int relax_q4_matmul(const void* x, int64_t n, int64_t K, int64_t N, const uint32_t* packed_w,
                    const void* scales, void* y, void* stream) {
    return rq4::matmul_impl(x, n, K, N, packed_w, scales, y, nullptr, 0, 0, 0, 0, 0u, stream);
}

int relax_q4_matmul_grouped(const void* x, int64_t n, int64_t K, int count, const int64_t* N,
                            const uint32_t* const* packed_w, const void* const* scales, void* const* y,
                            void* stream) {
    if (count < 1 || count > 4 || !N || !packed_w || !scales || !y) return RELAX_ERR_INVALID_ARG;
    if (n < 0 || K <= 0) return RELAX_ERR_INVALID_ARG;
    for (int i = 0; i < count; ++i)
        if (N[i] <= 0) return RELAX_ERR_INVALID_ARG;
    if (K % rq4::kGroup != 0) return RELAX_ERR_UNSUPPORTED_SHAPE;
    if (n == 0) return RELAX_OK;
    if (!x) return RELAX_ERR_INVALID_ARG;
    const size_t xb = static_cast<size_t>(n) * K * 2;
    for (int i = 0; i < count; ++i) {
        if (!packed_w[i] || !scales[i] || !y[i]) return RELAX_ERR_INVALID_ARG;
        if (!rq4::aligned16(packed_w[i]) || !rq4::aligned16(scales[i]) || !rq4::aligned16(y[i]))
            return RELAX_ERR_MISALIGNED;
    }
    if (!rq4::aligned16(x)) return RELAX_ERR_MISALIGNED;
    for (int i = 0; i < count; ++i) {
        const size_t yb = static_cast<size_t>(n) * N[i] * 2;
        if (rq4::overlap(y[i], yb, x, xb)) return RELAX_ERR_ALIAS;
        for (int j = 0; j < count; ++j) {
            const size_t wb = static_cast<size_t>(N[j]) * K / 2, sb = static_cast<size_t>(N[j]) * (K / rq4::kGroup) * 2;
            if (rq4::overlap(y[i], yb, packed_w[j], wb) || rq4::overlap(y[i], yb, scales[j], sb)) return RELAX_ERR_ALIAS;
            if (j != i && rq4::overlap(y[i], yb, y[j], static_cast<size_t>(n) * N[j] * 2)) return RELAX_ERR_ALIAS;
        }
    }
    // one launch where the streamed decode kernel serves every member (n <= 2)
    if (n <= rq4::gemv_max_n() && rq4::gemv_stream_grouped_ok(n, K, count, N)) {
        const int rc = rq4::check_device();
        if (rc != RELAX_OK) return rc;
        const uint16_t* sp[4];
        uint16_t* yp[4];
        for (int i = 0; i < count; ++i) {
            sp[i] = static_cast<const uint16_t*>(scales[i]);
            yp[i] = static_cast<uint16_t*>(y[i]);
        }
        const int e = rq4::launch_gemv_stream_grouped(static_cast<const uint16_t*>(x), n, K, count, N, packed_w, sp,
                                                      yp, true, static_cast<cudaStream_t>(stream));
        if (e != 0) {
            cudaGetLastError();
            return RELAX_ERR_CUDA;
        }
        return RELAX_OK;
    }
    // small batches: one small-n launch for the whole group when the members
    // together are wide enough for it (the rule of smalln_preferred applied to
    // the group's total rows)
    {
        int64_t tot = 0;
        for (int i = 0; i < count; ++i) tot += N[i];
        if (rq4::smalln_preferred(n, K, tot) && rq4::smalln_mma_grouped_ok(n, K, count, N)) {
            const int rc = rq4::check_device();
            if (rc != RELAX_OK) return rc;
            const uint16_t* sp[4];
            uint16_t* yp[4];
            for (int i = 0; i < count; ++i) {
                sp[i] = static_cast<const uint16_t*>(scales[i]);
                yp[i] = static_cast<uint16_t*>(y[i]);
            }
            const int e = rq4::launch_smalln_mma_grouped(static_cast<const uint16_t*>(x), n, K, count, N, packed_w, sp,
                                                         yp, true, static_cast<cudaStream_t>(stream));
            if (e != 0) {
                cudaGetLastError();
                return RELAX_ERR_CUDA;
            }
            return RELAX_OK;
        }
    }
    // otherwise each member through the ordinary dispatch (same results)
    for (int i = 0; i < count; ++i) {
        const int rc = rq4::matmul_impl(x, n, K, N[i], packed_w[i], scales[i], y[i], nullptr, 0, 0, 0, 0, 0u, stream);
        if (rc != RELAX_OK) return rc;
    }
    return RELAX_OK;
}

#ifdef RQ4_EXPERIMENTS
// the persistent decode chain (experiments build; include/relax_q4_debug.h)
int relax_q4_chain_workspace(int count, size_t* ws_bytes) {
    if (!ws_bytes || count < 1 || count > rq4::chain_max_ops()) return RELAX_ERR_INVALID_ARG;
    *ws_bytes = rq4::chain_workspace_bytes(count);
    return RELAX_OK;
}

int relax_q4_chain_init(const relax_q4_chain_op* ops, int count, void* ws, size_t ws_bytes) {
    if (!ops || count < 1 || count > rq4::chain_max_ops() || !ws) return RELAX_ERR_INVALID_ARG;
    std::vector<rq4::ChainOpHost> h(static_cast<size_t>(count));
    for (int i = 0; i < count; ++i) {
        const relax_q4_chain_op& o = ops[i];
        if (!o.x || !o.packed_w || !o.scales || !o.y || o.K <= 0 || o.N <= 0 || o.reserved != 0)
            return RELAX_ERR_INVALID_ARG;
        if (!rq4::chain_op_ok(o.K, o.N)) return RELAX_ERR_UNSUPPORTED_SHAPE;
        if (!rq4::aligned16(o.x) || !rq4::aligned16(o.packed_w) || !rq4::aligned16(o.scales) || !rq4::aligned16(o.y))
            return RELAX_ERR_MISALIGNED;
        const size_t xb = static_cast<size_t>(o.K) * 2, yb = static_cast<size_t>(o.N) * 2;
        const size_t wb = static_cast<size_t>(o.N) * o.K / 2, sb = static_cast<size_t>(o.N) * (o.K / rq4::kGroup) * 2;
        if (rq4::overlap(o.y, yb, o.x, xb) || rq4::overlap(o.y, yb, o.packed_w, wb) ||
            rq4::overlap(o.y, yb, o.scales, sb) || rq4::overlap(o.y, yb, ws, ws_bytes))
            return RELAX_ERR_ALIAS;
        h[i].x = static_cast<const uint16_t*>(o.x);
        h[i].w = o.packed_w;
        h[i].s = static_cast<const uint16_t*>(o.scales);
        h[i].y = static_cast<uint16_t*>(o.y);
        h[i].K = o.K;
        h[i].N = o.N;
        h[i].after = o.after;
    }
    if (!rq4::aligned16(ws)) return RELAX_ERR_MISALIGNED;
    if (ws_bytes < rq4::chain_workspace_bytes(count)) return RELAX_ERR_WORKSPACE;
    const int rc = rq4::check_device();
    if (rc != RELAX_OK) return rc;
    if (rq4::chain_init(h.data(), count, ws) != 0) {
        cudaGetLastError();
        return RELAX_ERR_CUDA;
    }
    return RELAX_OK;
}

int relax_q4_chain_run(void* ws, void* stream) {
    if (!ws) return RELAX_ERR_INVALID_ARG;
    const int rc = rq4::check_device();
    if (rc != RELAX_OK) return rc;
    if (rq4::launch_chain(ws, true, static_cast<cudaStream_t>(stream)) != 0) {
        cudaGetLastError();
        return RELAX_ERR_CUDA;
    }
    return RELAX_OK;
}

#endif

int relax_tp_comm_bytes(int32_t world, int64_t N_max, size_t* bytes) {
    if (!bytes || world < 1 || world > RELAX_TP_MAX_WORLD || N_max <= 0) return RELAX_ERR_INVALID_ARG;
    *bytes = rq4::tp_comm_bytes(world, N_max);
    return RELAX_OK;
}

int relax_q4_matmul_allreduce(const relax_tp_comm* comm, const void* x, int64_t n, int64_t K, int64_t N,
                              const uint32_t* packed_w, const void* scales, const void* residual, void* y,
                              void* stream) {
    if (!comm || comm->world < 1 || comm->world > RELAX_TP_MAX_WORLD || comm->rank < 0 ||
        comm->rank >= comm->world || n < 0 || K <= 0 || N <= 0)
        return RELAX_ERR_INVALID_ARG;
    for (int p = 0; p < comm->world; ++p) {
        if (!comm->bufs[p]) return RELAX_ERR_INVALID_ARG;
        if (!rq4::aligned16(comm->bufs[p])) return RELAX_ERR_MISALIGNED;
    }
    if (comm->buf_bytes < rq4::tp_comm_bytes(comm->world, N)) return RELAX_ERR_WORKSPACE;
    if (K % rq4::kGroup != 0) return RELAX_ERR_UNSUPPORTED_SHAPE;
    // the fused exchange lives in the streamed decode kernel: n <= 2, K % 256 == 0
    if (n > 2 || !rq4::gemv_stream_ok(n >= 2 ? 2 : 1, K, N) || rq4::gemv_stream_grid(K, N) > rq4::kTpMaxCta)
        return RELAX_ERR_UNSUPPORTED_SHAPE;
    if (n == 0) return RELAX_OK;
    if (!x || !packed_w || !scales || !y) return RELAX_ERR_INVALID_ARG;
    if (!rq4::aligned16(x) || !rq4::aligned16(packed_w) || !rq4::aligned16(scales) || !rq4::aligned16(y) ||
        (residual && !rq4::aligned16(residual)))
        return RELAX_ERR_MISALIGNED;
    const size_t xb = static_cast<size_t>(n) * K * 2, yb = static_cast<size_t>(n) * N * 2;
    const size_t wb = static_cast<size_t>(N) * K / 2, sb = static_cast<size_t>(N) * (K / rq4::kGroup) * 2;
    const size_t cb = rq4::tp_comm_bytes(comm->world, N);
    if (rq4::overlap(y, yb, x, xb) || rq4::overlap(y, yb, packed_w, wb) || rq4::overlap(y, yb, scales, sb) ||
        rq4::overlap(y, yb, comm->bufs[comm->rank], cb) || (residual && residual != y && rq4::overlap(y, yb, residual, yb)))
        return RELAX_ERR_ALIAS;
    const int rc = rq4::check_device();
    if (rc != RELAX_OK) return rc;
    rq4::TpComm tc;
    tc.world = comm->world;
    tc.rank = comm->rank;
    for (int p = 0; p < comm->world; ++p) tc.bufs[p] = static_cast<uint8_t*>(comm->bufs[p]);
    rq4::Fusion fu;
    fu.ops = rq4::kOpTpAllReduce | (residual ? RELAX_OP_RESIDUAL : 0u);
    fu.res = static_cast<const uint16_t*>(residual);
    fu.tp = &tc;
    const int e = rq4::launch_gemv_stream(static_cast<const uint16_t*>(x), n, K, N, packed_w,
                                          static_cast<const uint16_t*>(scales), static_cast<uint16_t*>(y), true,
                                          static_cast<cudaStream_t>(stream), fu);
    if (e != 0) {
        cudaGetLastError();
        return RELAX_ERR_CUDA;
    }
    return RELAX_OK;
}

int relax_q4_matmul_ws(const void* x, int64_t n, int64_t K, int64_t N, const uint32_t* packed_w,
                       const void* scales, void* y, void* workspace, size_t ws_bytes, void* stream) {
    return rq4::matmul_impl(x, n, K, N, packed_w, scales, y, workspace, ws_bytes, 0, 0, 0, 0u, stream);
}

int relax_q4_matmul_ex(const void* x, int64_t n, int64_t K, int64_t N, const uint32_t* packed_w,
                       const void* scales, void* y, void* workspace, size_t ws_bytes, int variant,
                       int split_k, int bn, unsigned flags, void* stream) {
    return rq4::matmul_impl(x, n, K, N, packed_w, scales, y, workspace, ws_bytes, variant, split_k,
                            bn, flags, stream);
}

int relax_q4_dequant(const uint32_t* packed_w, const void* scales, int64_t K, int64_t N,
                     void* w_out, void* stream) {
    if (K <= 0 || N < 0) return RELAX_ERR_INVALID_ARG;
    if (K % rq4::kGroup != 0) return RELAX_ERR_UNSUPPORTED_SHAPE;
    if (N == 0) return RELAX_OK;
    if (!packed_w || !scales || !w_out) return RELAX_ERR_INVALID_ARG;
    if (!rq4::aligned16(packed_w) || !rq4::aligned16(scales) || !rq4::aligned16(w_out))
        return RELAX_ERR_MISALIGNED;
    const size_t ob = static_cast<size_t>(N) * K * 2;
    if (rq4::overlap(w_out, ob, packed_w, static_cast<size_t>(N) * K / 2) ||
        rq4::overlap(w_out, ob, scales, static_cast<size_t>(N) * (K / rq4::kGroup) * 2))
        return RELAX_ERR_ALIAS;
    const int rc = rq4::check_device();
    if (rc != RELAX_OK) return rc;
    const int e = rq4::launch_dequant(packed_w, static_cast<const uint16_t*>(scales), K, N,
                                      static_cast<uint16_t*>(w_out), static_cast<cudaStream_t>(stream));
    if (e != 0) {
        cudaGetLastError();
        return RELAX_ERR_CUDA;
    }
    return RELAX_OK;
}

int relax_q4_repack(const uint32_t* src_packed, const void* src_scales, int64_t K, int64_t N, int layout,
                    int group, uint32_t* packed_w, void* scales, void* stream) {
    if (K <= 0 || N < 0) return RELAX_ERR_INVALID_ARG;
    if (layout != RELAX_LAYOUT_NK && layout != RELAX_LAYOUT_KN && layout != RELAX_LAYOUT_NK3)
        return RELAX_ERR_INVALID_ARG;
    if (group != 32 && group != 64 && group != 128) return RELAX_ERR_UNSUPPORTED_SHAPE;
    if (K % group != 0) return RELAX_ERR_UNSUPPORTED_SHAPE;
    if (N == 0) return RELAX_OK;
    if (!src_packed || !src_scales || !packed_w || !scales) return RELAX_ERR_INVALID_ARG;
    if (!rq4::aligned16(src_packed) || !rq4::aligned16(src_scales) || !rq4::aligned16(packed_w) ||
        !rq4::aligned16(scales))
        return RELAX_ERR_MISALIGNED;
    const size_t wb = static_cast<size_t>(N) * K / 2;
    const size_t wb_in = layout == RELAX_LAYOUT_NK3 ? static_cast<size_t>(N) * (K / rq4::kGroup) * 12 : wb;
    const size_t sb_out = static_cast<size_t>(N) * (K / rq4::kGroup) * 2;
    const size_t sb_in = static_cast<size_t>(N) * (K / group) * 2;
    if (rq4::overlap(packed_w, wb, src_packed, wb_in) || rq4::overlap(packed_w, wb, src_scales, sb_in) ||
        rq4::overlap(scales, sb_out, src_packed, wb_in) || rq4::overlap(scales, sb_out, src_scales, sb_in) ||
        rq4::overlap(packed_w, wb, scales, sb_out))
        return RELAX_ERR_ALIAS;
    const int rc = rq4::check_device();
    if (rc != RELAX_OK) return rc;
    const int e = rq4::launch_repack(src_packed, static_cast<const uint16_t*>(src_scales), K, N, layout, group,
                                     packed_w, static_cast<uint16_t*>(scales), static_cast<cudaStream_t>(stream));
    if (e != 0) {
        cudaGetLastError();
        return RELAX_ERR_CUDA;
    }
    return RELAX_OK;
}

// ---------------------------------------------------------------------------
// Decode attention (F4; include/relax_q4.h).
static int attn_shape_check(int64_t batch, int64_t Hq, int64_t Hkv, int64_t D, int64_t Lmax) {
    if (batch < 0 || Hq <= 0 || Hkv <= 0 || D <= 0 || Lmax < 0) return RELAX_ERR_INVALID_ARG;
    if (D != 128 || Hq % Hkv != 0 || Lmax > 65536) return RELAX_ERR_UNSUPPORTED_SHAPE;
    const int64_t G = Hq / Hkv;
    if (G != 1 && G != 2 && G != 4 && G != 8) return RELAX_ERR_UNSUPPORTED_SHAPE;
    return RELAX_OK;
}

int relax_attn_decode_workspace(int64_t batch, int64_t n_heads, int64_t kv_len_max, size_t* ws_bytes) {
    if (!ws_bytes || batch < 0 || n_heads <= 0 || kv_len_max < 0) return RELAX_ERR_INVALID_ARG;
    *ws_bytes = rq4::attn_workspace_bytes(batch, n_heads, kv_len_max);
    return RELAX_OK;
}

int relax_attn_decode(const void* q, const void* k_cache, const void* v_cache, const int32_t* kv_lens,
                      int64_t batch, int64_t n_heads, int64_t n_kv_heads, int64_t head_dim, int64_t kv_len_max,
                      void* out, void* workspace, size_t ws_bytes, void* stream) {
    int rc = attn_shape_check(batch, n_heads, n_kv_heads, head_dim, kv_len_max);
    if (rc != RELAX_OK) return rc;
    if (batch == 0) return RELAX_OK;
    if (!q || !k_cache || !v_cache || !kv_lens || !out || (kv_len_max > 0 && !workspace)) return RELAX_ERR_INVALID_ARG;
    if (!rq4::aligned16(q) || !rq4::aligned16(k_cache) || !rq4::aligned16(v_cache) || !rq4::aligned16(out) ||
        (workspace && !rq4::aligned16(workspace)) || (reinterpret_cast<uintptr_t>(kv_lens) & 3u))
        return RELAX_ERR_MISALIGNED;
    const size_t need = rq4::attn_workspace_bytes(batch, n_heads, kv_len_max);
    if (ws_bytes < need) return RELAX_ERR_WORKSPACE;
    const size_t qb = static_cast<size_t>(batch * n_heads * head_dim) * 2;
    const size_t cb = static_cast<size_t>(batch * n_kv_heads * kv_len_max * head_dim) * 2;
    const size_t lb = static_cast<size_t>(batch) * 4;
    if (rq4::overlap(out, qb, q, qb) || rq4::overlap(out, qb, k_cache, cb) || rq4::overlap(out, qb, v_cache, cb) ||
        rq4::overlap(out, qb, kv_lens, lb) || rq4::overlap(out, qb, workspace, need) ||
        rq4::overlap(workspace, need, q, qb) || rq4::overlap(workspace, need, k_cache, cb) ||
        rq4::overlap(workspace, need, v_cache, cb) || rq4::overlap(workspace, need, kv_lens, lb))
        return RELAX_ERR_ALIAS;
    rc = rq4::check_device();
    if (rc != RELAX_OK) return rc;
    const int e = rq4::launch_attention_decode(static_cast<const uint16_t*>(q), static_cast<const uint16_t*>(k_cache),
                                               static_cast<const uint16_t*>(v_cache), kv_lens, batch, n_heads,
                                               n_kv_heads, kv_len_max, static_cast<uint16_t*>(out), workspace, true,
                                               static_cast<cudaStream_t>(stream));
    if (e != 0) {
        cudaGetLastError();
        return RELAX_ERR_CUDA;
    }
    return RELAX_OK;
}

int relax_kv_append(const void* k_new, const void* v_new, const int32_t* pos, int64_t batch, int64_t n_kv_heads,
                    int64_t head_dim, int64_t kv_len_max, void* k_cache, void* v_cache, void* stream) {
    int rc = attn_shape_check(batch, n_kv_heads, n_kv_heads, head_dim, kv_len_max);
    if (rc != RELAX_OK) return rc;
    if (batch == 0) return RELAX_OK;
    if (!k_new || !v_new || !pos || !k_cache || !v_cache) return RELAX_ERR_INVALID_ARG;
    if (!rq4::aligned16(k_new) || !rq4::aligned16(v_new) || !rq4::aligned16(k_cache) || !rq4::aligned16(v_cache) ||
        (reinterpret_cast<uintptr_t>(pos) & 3u))
        return RELAX_ERR_MISALIGNED;
    const size_t nb = static_cast<size_t>(batch * n_kv_heads * head_dim) * 2;
    const size_t cb = static_cast<size_t>(batch * n_kv_heads * kv_len_max * head_dim) * 2;
    if (rq4::overlap(k_cache, cb, v_cache, cb) || rq4::overlap(k_cache, cb, k_new, nb) ||
        rq4::overlap(k_cache, cb, v_new, nb) || rq4::overlap(v_cache, cb, k_new, nb) ||
        rq4::overlap(v_cache, cb, v_new, nb) || rq4::overlap(k_cache, cb, pos, batch * 4) ||
        rq4::overlap(v_cache, cb, pos, batch * 4))
        return RELAX_ERR_ALIAS;
    rc = rq4::check_device();
    if (rc != RELAX_OK) return rc;
    const int e = rq4::launch_kv_append(static_cast<const uint16_t*>(k_new), static_cast<const uint16_t*>(v_new), pos,
                                        batch, n_kv_heads, kv_len_max, static_cast<uint16_t*>(k_cache),
                                        static_cast<uint16_t*>(v_cache), true, static_cast<cudaStream_t>(stream));
    if (e != 0) {
        cudaGetLastError();
        return RELAX_ERR_CUDA;
    }
    return RELAX_OK;
}

const char* relax_status_str(int status) {
    switch (status) {
        case RELAX_OK: return "RELAX_OK";
        case RELAX_ERR_INVALID_ARG: return "RELAX_ERR_INVALID_ARG: null pointer, negative n, or non-positive K/N";
        case RELAX_ERR_UNSUPPORTED_SHAPE: return "RELAX_ERR_UNSUPPORTED_SHAPE: K % 32 != 0 or variant cannot run shape";
        case RELAX_ERR_MISALIGNED: return "RELAX_ERR_MISALIGNED: pointer not 16-byte aligned";
        case RELAX_ERR_ALIAS: return "RELAX_ERR_ALIAS: output overlaps an input or the workspace";
        case RELAX_ERR_WORKSPACE: return "RELAX_ERR_WORKSPACE: workspace smaller than the schedule needs";
        case RELAX_ERR_DEVICE: return "RELAX_ERR_DEVICE: no CUDA device or device is not sm_100";
        case RELAX_ERR_CUDA: return "RELAX_ERR_CUDA: CUDA launch or runtime call failed";
        default: return "RELAX_ERR_UNKNOWN";
    }
}

const char* relax_version(void) { return "relax_q4 0.1 sm_100a"; }

}  // extern "C"
