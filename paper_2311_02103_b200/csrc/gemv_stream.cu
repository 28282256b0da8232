// gemv_stream.cu -- the decode path (n = 1, 2): a streamed q4f16 GEMV.
//
// y[t][j] = sum_k x[t][k] * W(k, j),  W = (q - 7) * s   (dequant fused
// into the matmul; K, N static per call, n runtime).
//
// Design -- HBM-bound, so the whole kernel is organised
// around keeping >= 64 KB of weights in flight per SM with as few
// instructions per weight as possible:
//   * each CTA owns a contiguous, row-balanced block of output rows; since the
//     NK layout stores rows contiguously, its codes and scales are two
//     contiguous byte ranges, streamed through a shared-memory ring by ONE
//     producer thread with 1-D bulk async copies (cp.async.bulk, the TMA
//     engine, L2 evict-first): a stage is RS whole rows, 16-32 KB;
//   * consumer warp (h, kw): lane l owns the 32-code group g = 32*kw + l of
//     every row, so x[t][32g .. 32g+31] lives in 16 registers per token for
//     the whole kernel (x is read from HBM/L2 once per CTA, never from SMEM
//     in the loop); per row the lane issues one LDS.128 (its 16 B of codes:
//     one 32-code group) and one LDS.U16 (its scale), unpacks in registers
//     (LOP3/SHF magic-number trick + one HFMA2 per code pair, exact q - 7),
//     and accumulates sum (q-7)*x with FHFMA (fp16 x fp16 -> fp32, exact
//     products), then one FFMA by the scale;
//   * warp h of the kw column handles RPW consecutive rows of each stage and
//     reduces them across the 32 lanes with a transposed butterfly (RPW rows
//     in log2(RPW) exchange steps + plain steps), then the partials of the
//     WK K-columns are summed in shared memory in fixed order: deterministic;
//   * PDL: the producer starts streaming weights before griddepcontrol.wait;
//     only the x loads and the y stores wait for the previous kernel.
#include <cstdlib>
#include <cstdio>
#include "internal.h"
#include "relax_q4.h"
#include "ptx.cuh"
#include "q4_unpack.cuh"
#include "fusion.cuh"
#include "decode_math.cuh"
#include "knobs.h"

namespace rq4 {

constexpr int kGsMaxGroup = 4;   // matrices per grouped launch

struct GsArgs {
    const uint16_t* x;     // [NT][K] fp16
    const uint8_t* w;      // [N][K/2] bytes
    const uint8_t* s;      // [N][K/16] bytes (fp16 scales)
    uint16_t* y;           // [NT][N]
    int64_t N;
    int K, G, WK, H, RS, NS;
    uint32_t stage_bytes;  // RS * (K/2 + K/16)
    int rows_cta_max;
    uint32_t trace_seq;    // 0 = no trace, else launch sequence number
    int trace_xload;       // trace: stamp t_first after the x loads (1) or after the conversion (0)
    int prefetch;          // stages the producer issues before griddepcontrol.wait
    int l2_prefetch;       // bytes of codes beyond the ring pulled into L2 at the start (0: none)
    int trigger;           // where the CTA signals launch_dependents (0 start, 1 after x, 2 after stage 0)
    // fused neighbours (include/relax_q4.h RELAX_OP_*)
    uint32_t ops;
    float eps;             // RMSNORM_X
    const uint16_t* gamma; // RMSNORM_X: fp16 [K]
    const uint16_t* res;   // RESIDUAL: fp16 [NT][Nout]
    int64_t Nout;          // N/2 with SILU_MUL, else N (row stride of y and res)
    // grouped launch (relax_q4_matmul_grouped): matrices i = 1 .. nmat-1 take
    // CTAs [cta0[i], cta0[i+1]); matrix 0 is (w, s, y, N, Nout) above
    int nmat;
    int cta0[kGsMaxGroup + 1];
    const uint8_t* wgp[kGsMaxGroup];
    const uint8_t* sgp[kGsMaxGroup];
    uint16_t* ygp[kGsMaxGroup];
    int64_t Ngp[kGsMaxGroup];
    // RELAX_OP_KV_APPEND: rows kv_row0 .. are also stored into the caches
    uint16_t* kc;
    uint16_t* vc;
    const int32_t* kv_pos;
    int64_t kv_lmax;
    int kv_heads, kv_row0;
    // kOpTpAllReduce (relax_q4_matmul_allreduce): rank tp_rank of tp_world,
    // tp_bufs[p] = rank p's exchange buffer mapped on this device
    int tp_world, tp_rank;
    uint8_t* tp_bufs[kTpMaxWorld];
};

// Fused row-split all-reduce epilogue.  The
// CTA's fp32 partial of its rows (this rank's K slice) goes to every other
// rank as 8-byte words (epoch << 32 | value) stored straight into the peers'
// buffers over NVLink; the CTA then reads the same rows' words of every other
// rank from its own buffer, spinning until each carries this call's epoch,
// and sums the world partials in rank order 0..world-1 (its own from
// registers) -- the same order on every rank, so all ranks hold the same y
// bit for bit.  The epoch of a call is a per-CTA counter in the rank's own
// buffer (every rank makes the same sequence of calls, so the epochs agree);
// the word slots alternate with its parity, which is enough: a rank reaches
// call e + 2 only after it read every rank's words of call e + 1, which every
// rank wrote after it had finished reading the slots of call e.  No fences:
// the flag is part of the word (NCCL's LL idea).
template <int NT>
__device__ __forceinline__ void tp_allreduce_epilogue(const GsArgs& a, const float* part, int rows, int64_t row0,
                                                      float rescale, uint16_t* y, uint32_t ops, uint32_t e) {
    const int64_t N = a.N;
    const size_t slot0 = static_cast<size_t>(e & 1u) * a.tp_world;      // [parity][source rank]
    auto woff = [&](int src, int t, int64_t row) {
        return kTpHdrBytes + ((((slot0 + src) * 2 + t) * N) + row) * 8;
    };
    auto partial = [&](int rl, int t) {
        float sum = 0.f;
        for (int c = 0; c < a.WK; ++c) sum += part[(static_cast<size_t>(rl) * a.WK + c) * NT + t];
        return sum * rescale;
    };
    if (a.tp_world > 1) {
        for (int o = threadIdx.x; o < rows * NT; o += blockDim.x) {
            const int rl = o / NT;
            const int t = o - rl * NT;
            const uint64_t word = (static_cast<uint64_t>(e) << 32) | __float_as_uint(partial(rl, t));
            const size_t off = woff(a.tp_rank, t, row0 + rl);
            for (int p = 0; p < a.tp_world; ++p)
                if (p != a.tp_rank) st_relaxed_sys_u64(a.tp_bufs[p] + off, word);
        }
    }
    const uint8_t* own = a.tp_bufs[a.tp_rank];
    for (int o = threadIdx.x; o < rows * NT; o += blockDim.x) {
        const int rl = o / NT;
        const int t = o - rl * NT;
        const float mine = partial(rl, t);
        float acc = 0.f;
        for (int p = 0; p < a.tp_world; ++p) {
            float c = mine;
            if (p != a.tp_rank) {
                const uint8_t* src = own + woff(p, t, row0 + rl);
                uint64_t w = ld_relaxed_sys_u64(src);
                if (static_cast<uint32_t>(w >> 32) != e) {
                    const uint64_t t0 = globaltimer();
                    do {
                        // a rank that never arrives (call sequences that differ
                        // between ranks) fails the launch instead of hanging
                        if (globaltimer() - t0 > 10000000000ull) __trap();
                        w = ld_relaxed_sys_u64(src);
                    } while (static_cast<uint32_t>(w >> 32) != e);
                }
                c = __uint_as_float(static_cast<uint32_t>(w));
            }
            acc = p == 0 ? c : acc + c;
        }
        const int64_t idx = static_cast<int64_t>(t) * N + row0 + rl;
        y[idx] = residual_add(__half_as_ushort(__float2half_rn(acc)), ops,
                              (ops & RELAX_OP_RESIDUAL) ? a.res[idx] : uint16_t(0));
    }
}

// ---- optional per-CTA timeline (experiments build only, RELAX_Q4_TRACE=1;
// include/relax_q4_debug.h)
#if RQ4_TRACE
constexpr int kTraceMax = 1 << 16;                // records
struct TraceRec { uint32_t seq, cta, smid, pad; uint64_t t0, t_wait, t_first, t_end; };
__device__ TraceRec g_trace[kTraceMax];
__device__ uint32_t g_trace_n;
#endif

__device__ __forceinline__ uint64_t gtime() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ uint32_t smid() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
    return r;
}

struct GsConfig {
    int WK, H, RPW, RS, NS, threads, rows_cta_max, grid;
    size_t smem;
};

constexpr int kGsMaxConsumerWarps = 16;   // consumer warps per CTA (one CTA per SM)
// Ring budget per CTA: <= ~100 KB so that the next GEMV's CTA (programmatic
// dependent launch) fits on the SM beside this one and prefetches its whole
// share of weights while this kernel finishes.
static size_t gs_ring_budget() {
    static size_t v = [] {
        const int kb = knob_int("RELAX_Q4_GS_RING_KB", 112);
        return static_cast<size_t>(kb >= 72 && kb <= 190 ? kb : 112) * 1024;
    }();
    return v;
}

__device__ __forceinline__ uint4 lds128(const uint8_t* p) { return *reinterpret_cast<const uint4*>(p); }

// Per-lane contribution of one row: lane owns one 32-code group (16 B of
// codes `cw`, fp16 scale `sbits`), x for that group in xr[t][0..3].
//   ZPF = 0: exact centering -- (q - 7) as fp16 via the magic-number unpack
//            (1 SHF + 4 LOP3 + 4 HFMA2 per 8 codes), then 8 FHFMA;
//   ZPF = 1: factored zero point -- codes as fp16 subnormals q * 2^-24 (pure
//            masks, 1 SHF + 4 LOP3 per 8 codes), 8 FHFMA into an even-code and an
//            odd-code chain, and per group 2^-24 sum (q - 7) x =
//            (acc_e - z_e) + (acc_o - z_o) / 16, where (z_e, z_o) are the SAME two
//            FHFMA chains run once per kernel with every code = 7.  For an all-7
//            group the chains repeat z's operations bit for bit, so the group
//            contributes exactly 0 (r == 0 => y == +-0, reading 10);
//            the 2^24 is applied once per output.
template <int ZPF>
__device__ __forceinline__ void unpack_word(uint32_t word, uint32_t& c0, uint32_t& c1, uint32_t& c2, uint32_t& c3) {
    if (ZPF) {
        const uint32_t v8 = word >> 8;
        c0 = word & 0x000F000Fu;      // (q0, q4)   * 2^-24
        c1 = word & 0x00F000F0u;      // (q1, q5)   * 2^-20
        c2 = v8 & 0x000F000Fu;        // (q2, q6)   * 2^-24
        c3 = v8 & 0x00F000F0u;        // (q3, q7)   * 2^-20
    } else {
        __half2 cc[4];
        unpack_centered_interleaved(word, cc);
        c0 = h2_as_u32(cc[0]); c1 = h2_as_u32(cc[1]); c2 = h2_as_u32(cc[2]); c3 = h2_as_u32(cc[3]);
    }
}

// The even/odd FHFMA chains of one 32-code group (4 words), NT tokens; the
// codes are unpacked once and shared by the tokens.
template <int NT, int ZPF>
__device__ __forceinline__ void group_chains(const uint32_t (&words)[4], const uint4 (&xr)[NT][4],
                                             float (&e)[NT], float (&o)[NT]) {
#pragma unroll
    for (int wi = 0; wi < 4; ++wi) {
        uint32_t c0, c1, c2, c3;
        unpack_word<ZPF>(words[wi], c0, c1, c2, c3);
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            const uint4 x = xr[t][wi];            // (k0,k1) (k2,k3) (k4,k5) (k6,k7)
            e[t] = fhfma(lo16(c0), lo16(x.x), e[t]);   // k0
            o[t] = fhfma(lo16(c1), hi16(x.x), o[t]);   // k1
            e[t] = fhfma(lo16(c2), lo16(x.y), e[t]);   // k2
            o[t] = fhfma(lo16(c3), hi16(x.y), o[t]);   // k3
            e[t] = fhfma(hi16(c0), lo16(x.z), e[t]);   // k4
            o[t] = fhfma(hi16(c1), hi16(x.z), o[t]);   // k5
            e[t] = fhfma(hi16(c2), lo16(x.w), e[t]);   // k6
            o[t] = fhfma(hi16(c3), hi16(x.w), o[t]);   // k7
        }
    }
}

template <int NT, int ZPF>
__device__ __forceinline__ void row_dot(const uint4& cw, uint16_t sbits, const uint4 (&xr)[NT][4],
                                        const float (&ze)[NT], const float (&zo)[NT], float (&out)[NT]) {
    const uint32_t words[4] = {cw.x, cw.y, cw.z, cw.w};
    float e[NT], o[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) { e[t] = 0.f; o[t] = 0.f; }
    group_chains<NT, ZPF>(words, xr, e, o);
    const float sc = __half2float(__ushort_as_half(sbits));
#pragma unroll
    for (int t = 0; t < NT; ++t) {
        if (ZPF) out[t] = sc * fmaf(o[t] - zo[t], 0.0625f, e[t] - ze[t]);   // units of 2^-24
        else out[t] = sc * (e[t] + o[t]);
    }
}

// ---- fused neighbours (RELAX_OP_*, include/relax_q4.h) -------------------
// RMSNorm prologue on the x registers: r_t = 1/sqrt(mean x^2 + eps) over the
// whole row (per-lane sums -> warp shuffle -> one partial per K-column warp in
// shared memory -> every consumer sums the WK partials in fixed order), then
// x <- fp16(fp16(x * r_t) * gamma) in place.  `scratch`: WK * NT floats of
// static shared memory (not reused, so one barrier suffices).  gamma is a
// model parameter like the weights and is loaded before griddepcontrol.wait.
template <int NT>
__device__ __forceinline__ void rmsnorm_prologue(uint4 (&xr)[NT][4], const uint4 (&gm)[4], const GsArgs& a,
                                                 int lane, int kw, int h, int nwc, float* scratch) {
    float ss[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) {
        float pq[4];                                      // four independent chains (latency)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint32_t w4[4] = {xr[t][q].x, xr[t][q].y, xr[t][q].z, xr[t][q].w};
            float acc = 0.f;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const float2 f = __half22float2(u32_as_h2(w4[u]));
                acc = fmaf(f.x, f.x, acc);
                acc = fmaf(f.y, f.y, acc);
            }
            pq[q] = acc;
        }
        float acc = (pq[0] + pq[1]) + (pq[2] + pq[3]);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
        ss[t] = acc;
    }
    if (h == 0 && lane == 0)
#pragma unroll
        for (int t = 0; t < NT; ++t) scratch[kw * NT + t] = ss[t];
    asm volatile("bar.sync 1, %0;" :: "r"(nwc * 32) : "memory");
#pragma unroll
    for (int t = 0; t < NT; ++t) {
        float tot = 0.f;
        for (int c = 0; c < a.WK; ++c) tot += scratch[c * NT + t];
        const float r = 1.0f / sqrtf(tot / static_cast<float>(a.K) + a.eps);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            uint32_t w4[4] = {xr[t][q].x, xr[t][q].y, xr[t][q].z, xr[t][q].w};
            const uint32_t g4[4] = {gm[q].x, gm[q].y, gm[q].z, gm[q].w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const float2 f = __half22float2(u32_as_h2(w4[u]));
                const __half2 hn = __floats2half2_rn(f.x * r, f.y * r);        // cast back to fp16
                w4[u] = h2_as_u32(__hmul2(hn, u32_as_h2(g4[u])));              // fp16 * gamma, one rounding
            }
            xr[t][q] = make_uint4(w4[0], w4[1], w4[2], w4[3]);
        }
    }
}

// FU = 0: the plain matmul (the fused-neighbour code is compiled out, so the
// decode kernel of relax_q4_matmul is exactly the unfused one); FU = 1: a.ops.
template <int NT, int RPW, int ZPF, int FULLG, int MAXT, int FU>
__global__ void __launch_bounds__(MAXT, (MAXT <= 544 ? 2 : 1)) q4_decode_stream_kernel(const __grid_constant__ GsArgs a) {
    extern __shared__ __align__(128) uint8_t smem[];
    // NT = 2: the warp index through a shuffle (provably warp-uniform, so the
    // per-warp ring addressing moves to uniform registers): n = 2 decode
    // 1167 -> 1222 tok/s; at NT = 1 it measured 0.6% slower, so plain there.
    const int warp = NT > 1 ? __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0)
                            : static_cast<int>(threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    const int nwc = a.WK * a.H;                        // consumer warps
    // [barriers: 2*NS x 8 B, padded to 256][ring: NS stages + 1 KB pad][partials]
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + a.NS;
    uint8_t* ring = smem + 256;
    float* part = reinterpret_cast<float*>(ring + static_cast<size_t>(a.NS) * a.stage_bytes + 1024);

    // rows of this CTA; with SILU_MUL whole (gate, up) pairs
    const uint32_t ops = FU ? a.ops : 0u;
    const int psh = (ops & RELAX_OP_SILU_MUL) ? 1 : 0;       // log2 of the row unit
    // grouped launch: this CTA's matrix and its block of that matrix's rows
    const uint8_t* w_base = a.w;
    const uint8_t* s_base = a.s;
    uint16_t* y_base = a.y;
    int64_t Nm = a.N, Nout = a.Nout;
    int cb = static_cast<int>(blockIdx.x), nb = static_cast<int>(gridDim.x);
    if (a.nmat > 1) {
        int m = 0;
#pragma unroll 1
        for (int i = 1; i < a.nmat; ++i) if (static_cast<int>(blockIdx.x) >= a.cta0[i]) m = i;
        w_base = a.wgp[m]; s_base = a.sgp[m]; y_base = a.ygp[m];
        Nm = a.Ngp[m]; Nout = Nm;
        cb = static_cast<int>(blockIdx.x) - a.cta0[m];
        nb = a.cta0[m + 1] - a.cta0[m];
    }
    const int64_t units = Nm >> psh;
    const int64_t row0 = (static_cast<int64_t>(cb) * units / nb) << psh;
    const int64_t row1 = (static_cast<int64_t>(cb + 1) * units / nb) << psh;
    const int rows = static_cast<int>(row1 - row0);
    const int nst = (rows + a.RS - 1) / a.RS;
    const uint32_t cb_row = static_cast<uint32_t>(a.K / 2);
    const uint32_t sb_row = static_cast<uint32_t>(a.K / 16);
    const uint32_t codes_stage = static_cast<uint32_t>(a.RS) * cb_row;

    const uint64_t t_start = (RQ4_TRACE && a.trace_seq) ? gtime() : 0;
    __shared__ uint64_t tr_wait, tr_first;
    __shared__ float rms_red[(FU ? 32 : 1) * NT];        // RMSNorm partials (WK <= 32)
    __shared__ uint32_t tp_epoch;                         // kOpTpAllReduce: this call's epoch
    uint16_t res_pre = 0;                                 // RESIDUAL: prefetched first value
    if (threadIdx.x == 0) {
        for (int i = 0; i < a.NS; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], a.WK); }
        fence_mbar_init();
    }
    __syncthreads();
    if (a.trigger == 0) pdl_launch_dependents();

    if (warp == nwc) {
        // ------------------------------------------------ producer (one thread)
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            const uint8_t* wsrc = w_base + row0 * cb_row;
            const uint8_t* ssrc = s_base + row0 * sb_row;
#ifdef RQ4_EXPERIMENTS
            if (a.l2_prefetch > 0) {
                // experiments build: the rows beyond what the ring holds, pulled
                // into L2 at the start so HBM keeps streaming across the kernel
                // boundary -- measured slower (7B 1167 -> 967 tok/s at 192 KB
                // per CTA, profiles/r02/l2pf/)
                const int ring_rows = a.NS * a.RS;
                if (rows > ring_rows) {
                    uint64_t cbytes = static_cast<uint64_t>(rows - ring_rows) * cb_row;
                    uint64_t sbytes = static_cast<uint64_t>(rows - ring_rows) * sb_row;
                    const uint64_t cap = static_cast<uint64_t>(a.l2_prefetch);
                    if (cbytes > cap) { sbytes = sbytes * cap / cbytes & ~15ull; cbytes = cap; }
                    const uint8_t* cp = wsrc + static_cast<size_t>(ring_rows) * cb_row;
                    for (uint64_t o = 0; o < cbytes; o += 32768)
                        bulk_prefetch_l2(cp + o, static_cast<uint32_t>(cbytes - o < 32768 ? cbytes - o : 32768));
                    if (sbytes > 0) bulk_prefetch_l2(ssrc + static_cast<size_t>(ring_rows) * sb_row, static_cast<uint32_t>(sbytes));
                }
            }
#endif
            int slot = 0;
            uint32_t phase = 0;
            int issued = 0;
            for (int r = 0; r < rows; r += a.RS) {
                if (issued++ == a.prefetch) pdl_wait();     // stages streamed before the previous kernel ends
                mbar_wait(&empty[slot], phase ^ 1);
                const int nr = rows - r < a.RS ? rows - r : a.RS;
                const uint32_t bc = static_cast<uint32_t>(nr) * cb_row;
                const uint32_t bs = static_cast<uint32_t>(nr) * sb_row;
                uint8_t* dst = ring + static_cast<size_t>(slot) * a.stage_bytes;
                mbar_arrive_expect_tx(&full[slot], bc + bs);
                bulk_load(dst, wsrc + static_cast<size_t>(r) * cb_row, bc, &full[slot], pol);
                bulk_load(dst + codes_stage, ssrc + static_cast<size_t>(r) * sb_row, bs, &full[slot], pol);
                if (++slot == a.NS) { slot = 0; phase ^= 1; }
            }
        }
    } else {
        // ------------------------------------------------ consumers
        const int h = warp / a.WK;
        const int kw = warp - h * a.WK;
        const int g = kw * 32 + lane;
        const bool gv = g < a.G;
        uint4 gm[4];                                      // RMSNorm gamma of this lane's group
        if (ops & RELAX_OP_RMSNORM_X) {
#pragma unroll
            for (int q = 0; q < 4; ++q)
                gm[q] = gv ? reinterpret_cast<const uint4*>(a.gamma + g * 32)[q] : make_uint4(0u, 0u, 0u, 0u);
        }
        pdl_wait();
        if (RQ4_TRACE && a.trace_seq && warp == 0 && lane == 0) tr_wait = gtime();
        if (FU && (ops & kOpTpAllReduce) && threadIdx.x == 0) {
            // this call's epoch (the counter is touched by this CTA index only,
            // and the previous call has completed: griddepcontrol.wait)
            uint32_t* ctr = reinterpret_cast<uint32_t*>(a.tp_bufs[a.tp_rank]) + blockIdx.x;
            tp_epoch = *ctr + 1u;
            *ctr = tp_epoch;
        }
        uint4 xr[NT][4];
        float ze[NT], zo[NT];
#pragma unroll
        for (int t = 0; t < NT; ++t)
#pragma unroll
            for (int q = 0; q < 4; ++q)
                xr[t][q] = gv ? reinterpret_cast<const uint4*>(a.x + static_cast<int64_t>(t) * a.K + g * 32)[q]
                              : make_uint4(0u, 0u, 0u, 0u);
#if RQ4_TRACE
        // experiments: RELAX_Q4_TRACE_XLOAD=1 stamps t_first when the x loads have
        // landed (before the fixed-point conversion) instead of after it
        if (a.trace_seq && a.trace_xload && warp == 0 && lane == 0) {
            asm volatile("" ::"r"(xr[0][0].x), "r"(xr[0][3].w));
            tr_first = gtime() + ((xr[0][0].x ^ xr[0][3].w) == 0x9E3779B9u ? 1u : 0u);
        }
#endif
        if (ops & RELAX_OP_RMSNORM_X) rmsnorm_prologue<NT>(xr, gm, a, lane, kw, h, nwc, rms_red);
        // zero-point chains: the per-group FHFMA chains with every code = 7
        // (exactly what row_dot computes for an all-7 group)
#pragma unroll
        for (int t = 0; t < NT; ++t) { ze[t] = 0.f; zo[t] = 0.f; }
        if (ZPF == 1) {
            const uint32_t sevens[4] = {0x77777777u, 0x77777777u, 0x77777777u, 0x77777777u};
            group_chains<NT, 1>(sevens, xr, ze, zo);
        }
        // ZPF = 2: x of the group in 16-bit fixed point for the dp2a loop
        uint32_t xi[NT][4][4];
        int sx7[NT];
        float xinv[NT];
        if (ZPF == 2) {
#pragma unroll
            for (int t = 0; t < NT; ++t) x_to_fixed(xr[t], xi[t], sx7[t], xinv[t]);
        }
        if (ops & RELAX_OP_RESIDUAL) {
            // prefetch this thread's first residual value of the final loop (its
            // latency would otherwise sit on the kernel's tail)
            const int units_cta = (ops & RELAX_OP_SILU_MUL) ? rows / 2 : rows;
            if (static_cast<int>(threadIdx.x) < units_cta * NT) {
                const int o = threadIdx.x;
                const int ul = o / NT, t = o - ul * NT;
                const int64_t col = (ops & RELAX_OP_SILU_MUL) ? row0 / 2 + ul : row0 + ul;
                res_pre = a.res[static_cast<int64_t>(t) * Nout + col];
            }
        }
        if (RQ4_TRACE && a.trace_seq && !a.trace_xload && warp == 0 && lane == 0) tr_first = gtime();   // x in registers
        if (a.trigger == 1) pdl_launch_dependents();
        const int rsel = reduce_row_of_lane<RPW>(lane);
        const bool writer = (lane & (32 / RPW - 1)) == 0;
        // Stages (RPW rows each) go round-robin to the H row groups: warp (h, kw)
        // consumes stages h, h+H, ... and each stage is released by its WK
        // warps alone, so the producer refills slots at a fine grain.
        const uint32_t coff = static_cast<uint32_t>(g) * 16u;
        const uint32_t soff = codes_stage + static_cast<uint32_t>(g) * 2u;
        int slot = h;                                    // requires H <= NS
        uint32_t phase = 0;
        for (int st = h; st < nst; st += a.H) {
            const int r_base = st * a.RS;
            const int nr = rows - r_base < a.RS ? rows - r_base : a.RS;
            mbar_wait(&full[slot], phase);
            const uint8_t* stage = ring + static_cast<size_t>(slot) * a.stage_bytes;
            float acc[NT][RPW];
#pragma unroll
            for (int i = 0; i < RPW; ++i) {
                const uint4 cw = lds128(stage + coff + i * cb_row);
                uint16_t sbits = *reinterpret_cast<const uint16_t*>(stage + soff + i * sb_row);
                if (!FULLG && !gv) sbits = 0;                 // lanes past K: x = 0 and s = 0
                float o[NT];
                if (ZPF == 2) row_dot_idp<NT>(cw, sbits, xi, sx7, xinv, o);
                else row_dot<NT, ZPF>(cw, sbits, xr, ze, zo, o);
#pragma unroll
                for (int t = 0; t < NT; ++t) acc[t][i] = o[t];
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[slot]);      // stage bytes fully consumed
            if (a.trigger == 2) pdl_launch_dependents();
            slot += a.H;
            if (slot >= a.NS) { slot -= a.NS; phase ^= 1; }
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                const float v = reduce_rows<RPW>(acc[t], lane);
                if (writer && rsel < nr)
                    part[(static_cast<size_t>(r_base + rsel) * a.WK + kw) * NT + t] = v;
            }
        }
    }
    __syncthreads();
#if RQ4_TRACE
    __shared__ uint64_t tr_epi;                           // every stage consumed: the epilogue starts
    if (a.trace_seq && threadIdx.x == 0) tr_epi = gtime();
#endif
    // fixed-order sum over the WK K-columns; fp32 -> fp16 RNE
    const float rescale = ZPF == 1 ? 16777216.0f : 1.0f;     // exact power-of-two rescale
    if (FU && (ops & kOpTpAllReduce)) {
        tp_allreduce_epilogue<NT>(a, part, rows, row0, rescale, y_base, ops, tp_epoch);
    } else if (ops & RELAX_OP_SILU_MUL) {
        const int np = rows / 2;
        for (int o = threadIdx.x; o < np * NT; o += blockDim.x) {
            const int pl = o / NT;
            const int t = o - pl * NT;
            float sg = 0.f, su = 0.f;
            for (int c = 0; c < a.WK; ++c) {
                sg += part[(static_cast<size_t>(2 * pl) * a.WK + c) * NT + t];
                su += part[(static_cast<size_t>(2 * pl + 1) * a.WK + c) * NT + t];
            }
            const int64_t idx = static_cast<int64_t>(t) * Nout + row0 / 2 + pl;
            const bool pre = o == static_cast<int>(threadIdx.x) && warp < nwc;
            y_base[idx] = residual_add(silu_mul_value(sg * rescale, su * rescale), ops,
                                    (ops & RELAX_OP_RESIDUAL) ? (pre ? res_pre : a.res[idx]) : uint16_t(0));
        }
    } else {
        for (int o = threadIdx.x; o < rows * NT; o += blockDim.x) {
            const int rl = o / NT;
            const int t = o - rl * NT;
            float sum = 0.f;
            for (int c = 0; c < a.WK; ++c) sum += part[(static_cast<size_t>(rl) * a.WK + c) * NT + t];
            const int64_t idx = static_cast<int64_t>(t) * Nout + row0 + rl;
            const bool pre = o == static_cast<int>(threadIdx.x) && warp < nwc;
            const uint16_t v = residual_add(__half_as_ushort(__float2half_rn(sum * rescale)), ops,
                                            (ops & RELAX_OP_RESIDUAL) ? (pre ? res_pre : a.res[idx]) : uint16_t(0));
            y_base[idx] = v;
            if (FU && (ops & RELAX_OP_KV_APPEND)) {
                // the new token's key / value rows, also stored at its cache position
                const int64_t kr = row0 + rl - a.kv_row0;
                const int64_t span = static_cast<int64_t>(a.kv_heads) * 128;
                if (kr >= 0 && kr < 2 * span) {
                    const int p = a.kv_pos[t];
                    if (p >= 0 && p < a.kv_lmax) {
                        const bool isv = kr >= span;
                        const int64_t hr = isv ? kr - span : kr;
                        const int64_t hd = hr >> 7, d = hr & 127;
                        uint16_t* cache = isv ? a.vc : a.kc;
                        cache[((static_cast<int64_t>(t) * a.kv_heads + hd) * a.kv_lmax + p) * 128 + d] = v;
                    }
                }
            }
        }
    }
#if RQ4_TRACE
    if (a.trace_seq) {
        __syncthreads();
        if (threadIdx.x == 0) {
            const uint64_t t_end = gtime();               // before the record's own global atomic
            const uint32_t i = atomicAdd(&g_trace_n, 1u);
            if (i < kTraceMax) {
                TraceRec r;
                r.seq = a.trace_seq; r.cta = blockIdx.x; r.smid = smid();
                r.pad = static_cast<uint32_t>(tr_epi - t_start);   // ns from start to the epilogue
                r.t0 = t_start; r.t_wait = tr_wait; r.t_first = tr_first; r.t_end = t_end;
                g_trace[i] = r;
            }
        }
    }
#else
    (void)t_start;
#endif
}

static uint32_t g_launch_seq = 0;
static bool gs_trace() { return RQ4_TRACE && knob_int("RELAX_Q4_TRACE", 0) == 1; }
// stages the producer issues before griddepcontrol.wait (default: the whole ring)
static int gs_prefetch() { static const int v = knob_int("RELAX_Q4_GS_PREFETCH", -1); return v < 0 ? (1 << 30) : v; }
// where each CTA signals griddepcontrol.launch_dependents (0: at its start)
static int gs_trigger() { static const int v = knob_int("RELAX_Q4_GS_TRIGGER", 0); return v; }
// bytes of codes per CTA beyond the ring prefetched into L2 at kernel start
// (experiments build only; measured slower)
static int gs_l2_prefetch() { static const int v = knob_int("RELAX_Q4_GS_L2PF_KB", 0); return v > 0 ? v * 1024 : 0; }
// 2 = integer dot products (default); 1 = FHFMA with the factored
// zero point, 0 = exact centering (experiments build)
static int gs_zpf() { static const int v = knob_int("RELAX_Q4_GEMV_ZPF", 2); return v; }

static GsConfig gs_config(int64_t K, int64_t N, int pair = 1) {
    GsConfig c{};
    const int G = static_cast<int>(K / kGroup);
    c.WK = (G + 31) / 32;
    c.H = kGsMaxConsumerWarps / c.WK;
    if (c.H < 1) c.H = 1;
    const size_t row_bytes = static_cast<size_t>(K / 2 + K / 16);
    c.RPW = 4;
    { const int v = knob_int("RELAX_Q4_GS_H", 0); if (v >= 1 && v * c.WK <= 31) c.H = v; }
    { const int v = knob_int("RELAX_Q4_GS_RPW", 0); if (v == 1 || v == 2 || v == 4 || v == 8) c.RPW = v; }
    int mult = 1;
    { const int v = knob_int("RELAX_Q4_GS_GRID_MULT", 1); if (v >= 1 && v <= 4) mult = v; }
    const int64_t gmax = static_cast<int64_t>(num_sms()) * mult;
    c.grid = static_cast<int>(N < gmax ? N : gmax);
    const int64_t units = N / pair;                       // rows, or (gate, up) pairs
    c.rows_cta_max = static_cast<int>((units + c.grid - 1) / c.grid) * pair;
    const size_t part_bytes = static_cast<size_t>(c.rows_cta_max) * c.WK * 2 * 4;
    // Ring budget.  (Trimming it so that every CTA stays <= 113 KB -- for the
    // wide lm_head -- cost a ring slot per row group on the 70B shapes:
    // 114 -> 87 tok/s; the untrimmed budget is kept.)
    const size_t budget = gs_ring_budget();
    // at least max(H, 3) stages of RPW rows must fit the ring
    const int nsmin = c.H < 3 ? 3 : c.H;
    while (c.RPW > 1 && static_cast<size_t>(nsmin) * c.RPW * row_bytes > budget) c.RPW /= 2;
    c.RS = c.RPW;
    const size_t stage = static_cast<size_t>(c.RS) * row_bytes;
    int ns = static_cast<int>(budget / stage);
    if (ns < nsmin) c.H = ns < 1 ? 1 : ns;          // (only for huge K with RPW = 1)
    c.NS = ns < 2 ? 2 : ns > 16 ? 16 : ns;
    if (c.NS < c.H) c.H = c.NS;
    // NS a multiple of H: stage s -> slot s % NS then always belongs to row
    // group s % H, i.e. every group owns a private sub-ring of NS/H slots
    // (the classic one-consumer ring protocol per group).
    c.NS -= c.NS % c.H;
    c.threads = (c.WK * c.H + 1) * 32;
    c.smem = 256 + static_cast<size_t>(c.NS) * stage + 1024 + part_bytes;
    // At most two GEMV CTAs per SM (the running kernel and the next one under
    // PDL): a third co-resident kernel was observed to stall the chain.
    if (c.smem < 80 * 1024) c.smem = 80 * 1024;
    return c;
}

// Largest dynamic shared memory any decode-stream launch may request (the
// attribute set once per device and kernel).
constexpr int kGsSmemMax = 210 * 1024;

int gemv_stream_grid(int64_t K, int64_t N) { return gs_config(K, N).grid; }

bool gemv_stream_ok(int nt, int64_t K, int64_t N, int pair) {
    if (nt < 1 || nt > 2 || K % 256 != 0 || N < 1 || N >= (int64_t{1} << 24)) return false;
    if (pair != 1 && (pair != 2 || N % 2 != 0)) return false;
    const GsConfig c = gs_config(K, N, pair);
    return c.threads <= 1024 && c.smem <= static_cast<size_t>(kGsSmemMax);
}

template <int NT, int RPW, int ZPF, int FULLG, int MAXT, int FU>
static int launch_gs_k(const GsArgs& a, const GsConfig& c, bool pdl, cudaStream_t stream) {
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
    auto k = q4_decode_stream_kernel<NT, RPW, ZPF, FULLG, MAXT, FU>;
    const cudaError_t e = ensure_kernel_attrs(reinterpret_cast<const void*>(k), kGsSmemMax);
    if (e != cudaSuccess) return static_cast<int>(e);
    return static_cast<int>(cudaLaunchKernelEx(&cfg, k, a));
}

template <int NT, int RPW, int ZPF, int FULLG>
static int launch_gs_t(const GsArgs& a, const GsConfig& c, bool pdl, cudaStream_t stream) {
    const bool fu = a.ops != 0;
    if (c.threads <= 544)
        return fu ? launch_gs_k<NT, RPW, ZPF, FULLG, 544, 1>(a, c, pdl, stream)
                  : launch_gs_k<NT, RPW, ZPF, FULLG, 544, 0>(a, c, pdl, stream);
    // K > 16K: one CTA per SM
    return fu ? launch_gs_k<NT, RPW, ZPF, FULLG, 1024, 1>(a, c, pdl, stream)
              : launch_gs_k<NT, RPW, ZPF, FULLG, 1024, 0>(a, c, pdl, stream);
}

template <int NT, int ZPF, int FULLG>
static int launch_gs_nt(const GsArgs& a, const GsConfig& c, bool pdl, cudaStream_t stream) {
    switch (c.RPW) {
        case 8: return launch_gs_t<NT, 8, ZPF, FULLG>(a, c, pdl, stream);
        case 4: return launch_gs_t<NT, 4, ZPF, FULLG>(a, c, pdl, stream);
        case 2: return launch_gs_t<NT, 2, ZPF, FULLG>(a, c, pdl, stream);
        default: return launch_gs_t<NT, 1, ZPF, FULLG>(a, c, pdl, stream);
    }
}

template <int NT, int ZPF>
static int launch_gs_z(const GsArgs& a, const GsConfig& c, bool pdl, cudaStream_t stream) {
    return (a.G % 32 == 0) ? launch_gs_nt<NT, ZPF, 1>(a, c, pdl, stream)
                           : launch_gs_nt<NT, ZPF, 0>(a, c, pdl, stream);
}

int launch_gemv_stream(const uint16_t* x, int64_t n, int64_t K, int64_t N, const uint32_t* w,
                       const uint16_t* s, uint16_t* y, bool pdl, cudaStream_t stream, const Fusion& fu) {
    const int64_t Nout = (fu.ops & RELAX_OP_SILU_MUL) ? N / 2 : N;
    const int pair = (fu.ops & RELAX_OP_SILU_MUL) ? 2 : 1;
    if (!gemv_stream_ok(n >= 2 ? 2 : 1, K, N, pair)) return static_cast<int>(cudaErrorInvalidValue);
    const GsConfig c = gs_config(K, N, pair);
    if (knob_int("RELAX_Q4_GS_PRINT", 0))
        fprintf(stderr, "gemv_stream K=%lld N=%lld WK=%d H=%d RPW=%d RS=%d NS=%d threads=%d grid=%d smem=%zu\n",
                (long long)K, (long long)N, c.WK, c.H, c.RPW, c.RS, c.NS, c.threads, c.grid, c.smem);
    const int zpf = gs_zpf();
    for (int64_t t0 = 0; t0 < n; t0 += 2) {
        const int cnt = (n - t0) >= 2 ? 2 : 1;
        GsArgs a;
        a.x = x + t0 * K;
        a.w = reinterpret_cast<const uint8_t*>(w);
        a.s = reinterpret_cast<const uint8_t*>(s);
        a.y = y + t0 * Nout;
        a.N = N;
        a.K = static_cast<int>(K);
        a.G = static_cast<int>(K / kGroup);
        a.WK = c.WK; a.H = c.H; a.RS = c.RS; a.NS = c.NS;
        a.ops = fu.ops;
        a.eps = fu.eps;
        a.gamma = fu.gamma;
        a.kc = fu.kc;
        a.vc = fu.vc;
        a.kv_pos = fu.kv_pos ? fu.kv_pos + t0 : nullptr;
        a.kv_lmax = fu.kv_lmax;
        a.kv_heads = fu.kv_heads;
        a.kv_row0 = fu.kv_row0;
        if (fu.kc) {
            const int64_t per_tok = static_cast<int64_t>(fu.kv_heads) * fu.kv_lmax * 128;
            a.kc = fu.kc + t0 * per_tok;
            a.vc = fu.vc + t0 * per_tok;
        }
        a.res = fu.res ? fu.res + t0 * Nout : nullptr;
        a.Nout = Nout;
        a.nmat = 1;
        a.stage_bytes = static_cast<uint32_t>(c.RS * (K / 2 + K / 16));
        a.rows_cta_max = c.rows_cta_max;
        a.prefetch = gs_prefetch();
        a.trigger = gs_trigger();
        a.l2_prefetch = gs_l2_prefetch();
        a.trace_seq = gs_trace() ? ++g_launch_seq : 0u;
        a.trace_xload = knob_int("RELAX_Q4_TRACE_XLOAD", 0);
        a.tp_world = 0;
        a.tp_rank = 0;
        for (int p = 0; p < kTpMaxWorld; ++p) a.tp_bufs[p] = nullptr;
        if (fu.tp) {
            if (c.grid > kTpMaxCta) return static_cast<int>(cudaErrorInvalidConfiguration);
            a.tp_world = fu.tp->world;
            a.tp_rank = fu.tp->rank;
            for (int p = 0; p < fu.tp->world; ++p) a.tp_bufs[p] = fu.tp->bufs[p];
        }
        int rc;
#ifdef RQ4_EXPERIMENTS
        if (zpf == 0) rc = cnt == 1 ? launch_gs_z<1, 0>(a, c, pdl, stream) : launch_gs_z<2, 0>(a, c, pdl, stream);
        else if (zpf == 1) rc = cnt == 1 ? launch_gs_z<1, 1>(a, c, pdl, stream) : launch_gs_z<2, 1>(a, c, pdl, stream);
        else
#else
        (void)zpf;
#endif
        rc = cnt == 1 ? launch_gs_z<1, 2>(a, c, pdl, stream) : launch_gs_z<2, 2>(a, c, pdl, stream);
        if (rc != 0) return rc;
    }
    return 0;
}

// Grouped launch (relax_q4_matmul_grouped): `count` matrices sharing x and K
// in ONE launch -- the CTAs are split among the matrices in proportion to
// their rows, each CTA streaming a row block of one matrix, so independent
// linears that read the same x (q/k/v, gate/up) are one dependent step of the
// PDL chain instead of `count`.
bool gemv_stream_grouped_ok(int64_t n, int64_t K, int count, const int64_t* N) {
    if (n < 1 || n > 2 || count < 1 || count > kGsMaxGroup) return false;
    int64_t tot = 0;
    for (int i = 0; i < count; ++i) {
        if (!gemv_stream_ok(static_cast<int>(n), K, N[i])) return false;
        tot += N[i];
    }
    if (tot < 2 * count) return false;
    const GsConfig c = gs_config(K, tot);
    return c.smem <= static_cast<size_t>(kGsSmemMax);
}

int launch_gemv_stream_grouped(const uint16_t* x, int64_t n, int64_t K, int count, const int64_t* N,
                               const uint32_t* const* w, const uint16_t* const* s, uint16_t* const* y, bool pdl,
                               cudaStream_t stream) {
    int64_t tot = 0;
    for (int i = 0; i < count; ++i) tot += N[i];
    GsConfig c = gs_config(K, tot);
    // CTAs per matrix in proportion to its rows (at least one each)
    int cta0[kGsMaxGroup + 1];
    cta0[0] = 0;
    int64_t acc = 0;
    for (int i = 0; i < count; ++i) {
        acc += N[i];
        int e = static_cast<int>(acc * c.grid / tot);
        if (e < cta0[i] + 1) e = cta0[i] + 1;
        cta0[i + 1] = e;
    }
    c.grid = cta0[count];
    int rmax = 0;
    for (int i = 0; i < count; ++i) {
        const int nb = cta0[i + 1] - cta0[i];
        const int r = static_cast<int>((N[i] + nb - 1) / nb);
        if (r > rmax) rmax = r;
    }
    c.rows_cta_max = rmax;
    const size_t part_bytes = static_cast<size_t>(rmax) * c.WK * 2 * 4;
    c.smem = 256 + static_cast<size_t>(c.NS) * c.RS * (K / 2 + K / 16) + 1024 + part_bytes;
    if (c.smem < 80 * 1024) c.smem = 80 * 1024;
    if (c.smem > static_cast<size_t>(kGsSmemMax)) return static_cast<int>(cudaErrorInvalidConfiguration);
    for (int64_t t0 = 0; t0 < n; t0 += 2) {
        const int cnt = (n - t0) >= 2 ? 2 : 1;
        GsArgs a{};
        a.x = x + t0 * K;
        a.w = reinterpret_cast<const uint8_t*>(w[0]);
        a.s = reinterpret_cast<const uint8_t*>(s[0]);
        a.y = y[0] + t0 * N[0];
        a.N = N[0];
        a.K = static_cast<int>(K);
        a.G = static_cast<int>(K / kGroup);
        a.WK = c.WK; a.H = c.H; a.RS = c.RS; a.NS = c.NS;
        a.ops = 0;
        a.Nout = N[0];
        a.nmat = count;
        for (int i = 0; i <= count; ++i) a.cta0[i] = cta0[i];
        for (int i = 0; i < count; ++i) {
            a.wgp[i] = reinterpret_cast<const uint8_t*>(w[i]);
            a.sgp[i] = reinterpret_cast<const uint8_t*>(s[i]);
            a.ygp[i] = y[i] + t0 * N[i];
            a.Ngp[i] = N[i];
        }
        a.stage_bytes = static_cast<uint32_t>(c.RS * (K / 2 + K / 16));
        a.rows_cta_max = c.rows_cta_max;
        a.prefetch = gs_prefetch();
        a.trigger = gs_trigger();
        a.l2_prefetch = gs_l2_prefetch();
        a.trace_seq = gs_trace() ? ++g_launch_seq : 0u;
        a.trace_xload = knob_int("RELAX_Q4_TRACE_XLOAD", 0);
        const int rc = cnt == 1 ? launch_gs_z<1, 2>(a, c, pdl, stream) : launch_gs_z<2, 2>(a, c, pdl, stream);
        if (rc != 0) return rc;
    }
    return 0;
}

}  // namespace rq4

#if RQ4_TRACE
extern "C" RELAX_API int relax_debug_trace_read(void* host, size_t max_records, size_t* n_records, int reset) {
    uint32_t n = 0;
    if (cudaMemcpyFromSymbol(&n, rq4::g_trace_n, sizeof n) != cudaSuccess) return RELAX_ERR_CUDA;
    if (n > static_cast<uint32_t>(rq4::kTraceMax)) n = rq4::kTraceMax;
    const size_t m = n < max_records ? n : max_records;
    if (m && cudaMemcpyFromSymbol(host, rq4::g_trace, m * sizeof(rq4::TraceRec)) != cudaSuccess) return RELAX_ERR_CUDA;
    if (n_records) *n_records = m;
    if (reset) {
        const uint32_t z = 0;
        if (cudaMemcpyToSymbol(rq4::g_trace_n, &z, sizeof z) != cudaSuccess) return RELAX_ERR_CUDA;
    }
    return RELAX_OK;
}
#endif
