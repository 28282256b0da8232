// smalln_mma.cu -- the small-batch path (n = 3..8 tokens per launch): a
// streamed q4f16 GEMV whose multiply-accumulate runs on the warp-level tensor
// cores (mma.sync m16n8k16, fp16 x fp16 -> fp32).
//
// y[t][j] = sum_k x[t][k] * W(k, j),  W = (q - 7) * s   (dequant fused
// into the matmul; K, N static per call, n runtime).
//
// Why: at n = 3..16 the tcgen05 kernel needs split-K clusters
// to cover 148 SMs with 128-row tiles and pays their fill/drain per kernel
// (1.6-1.9 TB/s at n = 8); the CUDA-core decode kernel would spend n FHFMA per
// weight.  Here the MMA's N dimension is the token (8 columns), so one
// instruction does 16 rows x 16 k x 8 tokens, the A operand comes straight
// from the unpacked codes in registers, and 16-row tiles need no split-K.
//
// Arithmetic (factored zero point, exact products, as the decode kernel):
//   codes enter the MMA as fp16 subnormals -- w & 0x000F000F and
//   (w >> 8) & 0x000F000F give (q0, q4), (q2, q6) * 2^-24, w & 0x00F000F0 and
//   (w >> 8) & 0x00F000F0 give (q1, q5), (q3, q7) * 2^-20 -- with x / 16 on the
//   odd-code B rows, so per (16 rows x 32-code group)
//       d  = mma(odd, x/16, mma(even, x, 0))       = 2^-24 sum q x
//       dz = the same two MMAs with every code = 7 = 2^-24 sum 7 x
//   and acc += s * (d - dz).  For an all-7 group d and dz are the same
//   operations on the same operands, so the group adds exactly 0
//   (r == 0 => y == +-0, reading 10); y = fp16_RNE(2^24 * acc).
//
// Data movement:
//   * CTA b owns whole 16-row blocks [rb0, rb1) (balanced to +-1 block);
//     stages of (16 rows x 2048 k) = 16 KB codes + 2 KB scales, one 3-D
//     (codes) and one 2-D (scales) TMA tensor load each, 128-B swizzle (the
//     fragment loads below are bank-conflict free); rows past N and k past K
//     are zero-filled by the TMA (zero scale => zero contribution);
//   * stages go chunk-major (every row block of k-chunk 0, then chunk 1 ...),
//     so consumer warp w keeps, for a whole chunk, the B fragments of its 8
//     groups [8w, 8w+8) in registers (loaded from x -- L2/L1 -- and permuted
//     to the code order once per chunk) and their zero-point terms dz;
//   * each lane's D fragment holds 2 rows x 2 tokens, so partial sums need no
//     shuffles: warp w accumulates its (row, token) slots in shared memory
//     over the chunks; the 8 warps are summed in fixed order: deterministic;
//   * PDL: the producer streams weights before griddepcontrol.wait; only the
//     x loads and y stores wait for the previous kernel.
#include <cstdio>
#include <cstring>
#include "internal.h"
#include "relax_q4.h"
#include "ptx.cuh"
#include "knobs.h"

namespace rq4 {

constexpr int kSnRows = 16;                          // MMA M: rows per block
constexpr int kSnChunkG = 64;                        // groups per k-chunk
constexpr int kSnChunkK = kSnChunkG * kGroup;        // 2048 k
constexpr int kSnTok = 8;                            // MMA N: tokens per launch
constexpr int kSnMaxWarps = 16;                      // consumer warps (partial-sum slots sized for it)
constexpr int kSnDefaultWarps = 8;
constexpr uint32_t kSnCodeBytes = kSnRows * kSnChunkK / 2;      // 16 KB
constexpr uint32_t kSnScaleBytes = kSnRows * kSnChunkG * 2;     // 2 KB
constexpr uint32_t kSnStageBytes = kSnCodeBytes + kSnScaleBytes;  // 18 KB (multiple of 1 KB)
// Two CTAs per SM must fit (this kernel and the next one under PDL).
constexpr size_t kSnSmemCap = 113 * 1024;
constexpr size_t kSnSmemMax = 220 * 1024;           // the attribute (experiments may raise the cap; static smem aside)
// experiments build: RELAX_Q4_SN_SMEM_KB raises the shared-memory cap (one CTA per SM above ~114 KB)
static size_t sn_smem_cap() {
    static const size_t v = [] {
        const int kb = knob_int("RELAX_Q4_SN_SMEM_KB", 113);
        return static_cast<size_t>(kb >= 64 && kb <= 220 ? kb : 113) * 1024;
    }();
    return v;
}

constexpr int kSnMaxGroup = 4;                       // matrices per grouped launch

#if RQ4_TRACE
// per-CTA timeline (experiments build, RELAX_Q4_TRACE=1): start, after
// griddepcontrol.wait, first stage's operands ready (x fragments + dz), epilogue
// start, end (globaltimer ns)
constexpr int kSnTraceMax = 1 << 16;
struct SnTraceRec { uint32_t seq, cta, pad0, pad1; uint64_t t0, t_wait, t_first, t_epi, t_end; };
__device__ SnTraceRec g_sn_trace[kSnTraceMax];
__device__ uint32_t g_sn_trace_n;
#endif

struct SnArgs {
    const uint16_t* x;     // [n][K] fp16
    int K, G, n, NS, nkc;
    int rows_max;          // 16 * the most row blocks any CTA owns (partial-sum slots per warp)
    // matrices of the launch (relax_q4_matmul_grouped: q/k/v, gate/up share x):
    // matrix m takes CTAs [cta0[m], cta0[m+1]) and writes ygp[m] [n][Ngp[m]]
    int nmat;
    int cta0[kSnMaxGroup + 1];
    uint16_t* ygp[kSnMaxGroup];
    int64_t Ngp[kSnMaxGroup];
    int64_t nrbgp[kSnMaxGroup];   // 16-row blocks of each matrix
    uint32_t trace_seq;           // experiments build: 0 = no trace, else the launch's sequence number
};

// TMA descriptors of every matrix of the launch (kernel parameter space)
struct alignas(64) SnMaps {
    CUtensorMap w[kSnMaxGroup];   // codes: {32 words, N rows, K/256 chunks}, box {32, 16, 8}
    CUtensorMap s[kSnMaxGroup];   // scales: {K/32, N}, box {64, 16}
};

__device__ __forceinline__ void mma16816_acc(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1,
                                             const float (&c)[4]) {
    asm("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%10,%11,%12,%13};"
        : "=f"(d[0]), "=f"(d[1]), "=f"(d[2]), "=f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1),
          "f"(c[0]), "f"(c[1]), "f"(c[2]), "f"(c[3]));
}

// d = 2^-24 sum_k q x over one 32-code group for rows (g, g+8) and tokens
// (2t, 2t+1): the even-code MMA, then the odd-code MMA accumulating onto it.
__device__ __forceinline__ void group_mma(float (&d)[4], uint32_t wa, uint32_t wb, const uint4& b) {
    const uint32_t wa8 = wa >> 8, wb8 = wb >> 8;
    const uint32_t ae[4] = {wa & 0x000F000Fu, wb & 0x000F000Fu, wa8 & 0x000F000Fu, wb8 & 0x000F000Fu};
    const uint32_t ao[4] = {wa & 0x00F000F0u, wb & 0x00F000F0u, wa8 & 0x00F000F0u, wb8 & 0x00F000F0u};
    const float z[4] = {0.f, 0.f, 0.f, 0.f};
    float e[4];
    mma16816_acc(e, ae, b.x, b.y, z);
    mma16816_acc(d, ao, b.z, b.w, e);
}

// W consumer warps; warp w owns groups [GPW w, GPW (w+1)) of every 64-group chunk.
template <int W>
__global__ void __launch_bounds__((W + 1) * 32, 2)
q4_smalln_mma_kernel(const __grid_constant__ SnMaps maps, const __grid_constant__ SnArgs a) {
    constexpr int kSnWarps = W;
    constexpr int GPW = kSnChunkG / W;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);   // provably warp-uniform
    const int lane = threadIdx.x & 31;
    // [pad to 1 KB][ring NS x 18 KB][barriers 256 B][part]
    uint8_t* ring = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + static_cast<size_t>(a.NS) * kSnStageBytes);
    uint64_t* empty = full + a.NS;
    float* part = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(full) + 256);

    // this CTA's matrix and its share of that matrix's row blocks
    int m = 0;
#pragma unroll 1
    for (int i = 1; i < a.nmat; ++i) if (static_cast<int>(blockIdx.x) >= a.cta0[i]) m = i;
    const int cb = static_cast<int>(blockIdx.x) - a.cta0[m];
    const int nb = a.cta0[m + 1] - a.cta0[m];
    const int64_t Nm = a.Ngp[m];
    uint16_t* const ym = a.ygp[m];
#if RQ4_TRACE
    const uint64_t sn_t0 = a.trace_seq ? globaltimer() : 0;
    __shared__ uint64_t sn_tw, sn_tf;
#endif
    const int64_t rb0 = static_cast<int64_t>(cb) * a.nrbgp[m] / nb;
    const int64_t rb1 = static_cast<int64_t>(cb + 1) * a.nrbgp[m] / nb;
    const int nrb = static_cast<int>(rb1 - rb0);
    const int nst = nrb * a.nkc;

    if (threadIdx.x == 0) {
        for (int i = 0; i < a.NS; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], kSnWarps); }
        fence_mbar_init();
    }
    __syncthreads();
    pdl_launch_dependents();

    if (warp == kSnWarps) {
        // ------------------------------------------------ producer (one thread)
        if (lane == 0) {
            const CUtensorMap* mw = &maps.w[m];
            const CUtensorMap* ms = &maps.s[m];
            tma_prefetch_desc(mw);
            tma_prefetch_desc(ms);
            const uint64_t pol = policy_evict_first();
            int slot = 0, rb = 0, kc = 0;
            uint32_t phase = 0;
            for (int st = 0; st < nst; ++st) {
                mbar_wait(&empty[slot], phase ^ 1);
                uint8_t* stage = ring + static_cast<size_t>(slot) * kSnStageBytes;
                const int32_t r = static_cast<int32_t>((rb0 + rb) * kSnRows);
                mbar_arrive_expect_tx(&full[slot], kSnStageBytes);
                tma_load_3d(stage, mw, &full[slot], 0, r, kc * (kSnChunkK / 256), pol);
                tma_load_2d(stage + kSnCodeBytes, ms, &full[slot], kc * kSnChunkG, r, pol);
                if (++slot == a.NS) { slot = 0; phase ^= 1; }
                if (++rb == nrb) { rb = 0; ++kc; }
            }
        }
    } else {
        // ------------------------------------------------ consumers
        const int g = lane >> 2, t = lane & 3;
        const int w = warp;
        pdl_wait();
#if RQ4_TRACE
        if (a.trace_seq && threadIdx.x == 0) sn_tw = globaltimer();
#endif
        const __half2 sixteenth = __float2half2_rn(0.0625f);
        const uint4 sevens = make_uint4(0x00070007u, 0x00700070u, 0u, 0u);
        uint4 bf[GPW];      // B fragments of the warp's groups of the current chunk (token g)
        float dz[GPW][2];   // zero-point terms 2^-24 sum 7 x (tokens 2t, 2t+1)
        int slot = 0, rb = 0, kc = 0;
        uint32_t phase = 0;
        for (int st = 0; st < nst; ++st) {
            if (rb == 0) {
                // new chunk: this lane's B fragments (token g, codes 8t..8t+7 of each
                // of the warp's groups, permuted to the code order) and dz
#pragma unroll
                for (int j = 0; j < GPW; ++j) {
                    const int jg = kc * kSnChunkG + w * GPW + j;
                    uint4 v = make_uint4(0u, 0u, 0u, 0u);
                    if (g < a.n && jg < a.G)
                        v = *reinterpret_cast<const uint4*>(a.x + static_cast<int64_t>(g) * a.K + jg * 32 + t * 8);
                    bf[j] = make_uint4(prmt(v.x, v.z, 0x5410u), prmt(v.y, v.w, 0x5410u),
                                       h2_as_u32(__hmul2(u32_as_h2(prmt(v.x, v.z, 0x7632u)), sixteenth)),
                                       h2_as_u32(__hmul2(u32_as_h2(prmt(v.y, v.w, 0x7632u)), sixteenth)));
                }
#pragma unroll
                for (int j = 0; j < GPW; ++j) {
                    // every code = 7: words 0x77777777 in both rows
                    float d[4];
                    const uint32_t ae[4] = {sevens.x, sevens.x, sevens.x, sevens.x};
                    const uint32_t ao[4] = {sevens.y, sevens.y, sevens.y, sevens.y};
                    const float z[4] = {0.f, 0.f, 0.f, 0.f};
                    float e[4];
                    mma16816_acc(e, ae, bf[j].x, bf[j].y, z);
                    mma16816_acc(d, ao, bf[j].z, bf[j].w, e);
                    dz[j][0] = d[0];
                    dz[j][1] = d[1];
                }
            }
#if RQ4_TRACE
            if (a.trace_seq && threadIdx.x == 0 && st == 0) sn_tf = globaltimer();
#endif
            if (rb == 0 && kc + 1 < a.nkc && g < a.n) {
                // the next chunk's x is read at the next chunk boundary: pull it into
                // L1 now, so that load does not stall all warps on an L2 round trip
                const uint16_t* xn = a.x + static_cast<int64_t>(g) * a.K + ((kc + 1) * kSnChunkG + w * GPW) * 32 + t * 8;
#pragma unroll 1
                for (int j = 0; j < GPW; ++j)
                    if ((kc + 1) * kSnChunkG + w * GPW + j < a.G) prefetch_l1(xn + j * 32);
            }
            mbar_wait(&full[slot], phase);
            const uint8_t* stage = ring + static_cast<size_t>(slot) * kSnStageBytes;
            // scales of the warp's GPW groups for rows g and g+8 (16-B unit jj / 8 of
            // row r sits at unit (jj / 8) ^ (r % 8); GPW consecutive scales in it)
            const int j0 = w * GPW;
            const uint8_t* srow = stage + kSnCodeBytes + g * 128 + (((j0 >> 3) ^ g) << 4) + (j0 & 7) * 2;
            uint32_t sa[GPW / 2], sb[GPW / 2];
#pragma unroll
            for (int i = 0; i < GPW / 2; ++i) {
                sa[i] = *reinterpret_cast<const uint32_t*>(srow + 4 * i);
                sb[i] = *reinterpret_cast<const uint32_t*>(srow + 1024 + 4 * i);
            }
            uint32_t wa[GPW], wb[GPW];
#pragma unroll
            for (int j = 0; j < GPW; ++j) {
                const int jj = j0 + j;
                const uint8_t* p = stage + (jj >> 3) * 2048 + g * 128 + (((jj & 7) ^ g) << 4) + 4 * t;
                wa[j] = *reinterpret_cast<const uint32_t*>(p);
                wb[j] = *reinterpret_cast<const uint32_t*>(p + 1024);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[slot]);      // operands are in registers
            float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int j = 0; j < GPW; ++j) {
                float d[4];
                group_mma(d, wa[j], wb[j], bf[j]);
                const float fa = __half2float(__ushort_as_half(static_cast<uint16_t>(sa[j >> 1] >> ((j & 1) * 16))));
                const float fb = __half2float(__ushort_as_half(static_cast<uint16_t>(sb[j >> 1] >> ((j & 1) * 16))));
                acc[0] = fmaf(fa, d[0] - dz[j][0], acc[0]);
                acc[1] = fmaf(fa, d[1] - dz[j][1], acc[1]);
                acc[2] = fmaf(fb, d[2] - dz[j][0], acc[2]);
                acc[3] = fmaf(fb, d[3] - dz[j][1], acc[3]);
            }
            // slots [warp][row][token]: only this warp touches its slots; one
            // 8-B access per (row, token pair) -- the 16 lanes of each half-warp
            // hit 16 distinct bank pairs
            float2* p0 = reinterpret_cast<float2*>(part + (static_cast<size_t>(w) * a.rows_max + rb * kSnRows + g) * kSnTok + 2 * t);
            float2* p1 = p0 + 8 * kSnTok / 2;
            if (kc == 0) {
                *p0 = make_float2(acc[0], acc[1]);
                *p1 = make_float2(acc[2], acc[3]);
            } else {
                const float2 u0 = *p0, u1 = *p1;
                *p0 = make_float2(u0.x + acc[0], u0.y + acc[1]);
                *p1 = make_float2(u1.x + acc[2], u1.y + acc[3]);
            }
            if (++slot == a.NS) { slot = 0; phase ^= 1; }
            if (++rb == nrb) { rb = 0; ++kc; }
        }
    }
    __syncthreads();
#if RQ4_TRACE
    const uint64_t sn_te0 = (a.trace_seq && threadIdx.x == 0) ? globaltimer() : 0;
#endif
    // fixed-order sum over the 8 warps; y = fp16_RNE(2^24 * acc)
    const int rows = nrb * kSnRows;
    for (int o = threadIdx.x; o < rows * a.n; o += blockDim.x) {
        const int rl = o / a.n;
        const int tok = o - rl * a.n;
        const int64_t row = rb0 * kSnRows + rl;
        if (row >= Nm) continue;
        float sum = 0.f;
#pragma unroll
        for (int c = 0; c < kSnWarps; ++c) sum += part[(static_cast<size_t>(c) * a.rows_max + rl) * kSnTok + tok];
        ym[static_cast<int64_t>(tok) * Nm + row] = __half_as_ushort(__float2half_rn(sum * 16777216.0f));
    }
#if RQ4_TRACE
    if (a.trace_seq) {
        __syncthreads();
        if (threadIdx.x == 0) {
            const uint64_t te = globaltimer();
            const uint32_t i = atomicAdd(&g_sn_trace_n, 1u);
            if (i < kSnTraceMax) {
                SnTraceRec r;
                r.seq = a.trace_seq; r.cta = blockIdx.x; r.pad0 = 0; r.pad1 = 0;
                r.t0 = sn_t0; r.t_wait = sn_tw; r.t_first = sn_tf; r.t_epi = sn_te0; r.t_end = te;
                g_sn_trace[i] = r;
            }
        }
    }
#endif
}

// consumer warps (8; 16 in the experiments build with RELAX_Q4_SN_WARPS=16)
static int sn_warps() {
    static const int w = knob_int("RELAX_Q4_SN_WARPS", kSnDefaultWarps) == 16 ? 16 : 8;
    return w;
}

struct SnConfig {
    int grid, NS, rows_max;
    int cta0[kSnMaxGroup + 1];
    size_t smem;
    bool ok;
};

// CTAs per matrix in proportion to its 16-row blocks (at least one each),
// grid <= the SM count.
static SnConfig sn_config_group(int64_t K, int count, const int64_t* N) {
    SnConfig c{};
    c.ok = false;
    if (K % 256 != 0 || K <= 0 || count < 1 || count > kSnMaxGroup) return c;
    int64_t tot = 0, nrb[kSnMaxGroup];
    for (int i = 0; i < count; ++i) {
        if (N[i] <= 0 || N[i] >= (int64_t{1} << 30)) return c;
        nrb[i] = (N[i] + kSnRows - 1) / kSnRows;
        tot += nrb[i];
    }
    if (tot < count) return c;
    const int64_t gmax = static_cast<int64_t>(num_sms()) * (knob_int("RELAX_Q4_SN_GRID_MULT", 1) == 2 ? 2 : 1);
    const int grid = static_cast<int>(tot < gmax ? tot : gmax);
    c.cta0[0] = 0;
    int64_t acc = 0, nrb_max = 0;
    for (int i = 0; i < count; ++i) {
        acc += nrb[i];
        int e = static_cast<int>(acc * grid / tot);
        if (e < c.cta0[i] + 1) e = c.cta0[i] + 1;
        if (i == count - 1 && e < grid) e = grid;
        c.cta0[i + 1] = e;
        const int nb = e - c.cta0[i];
        if (nb > nrb[i]) return c;                                   // a CTA without rows
        const int64_t r = (nrb[i] + nb - 1) / nb;
        if (r > nrb_max) nrb_max = r;
    }
    c.grid = c.cta0[count];
    c.rows_max = static_cast<int>(nrb_max * kSnRows);
    const size_t part_bytes = static_cast<size_t>(nrb_max) * kSnRows * sn_warps() * kSnTok * 4;
    const size_t fixed = 1024 + 256 + part_bytes;
    const size_t cap = sn_smem_cap();
    if (fixed + 3 * static_cast<size_t>(kSnStageBytes) > cap) return c;
    const int ns = static_cast<int>((cap - fixed) / kSnStageBytes);
    c.NS = ns > 12 ? 12 : ns;
    c.smem = fixed + static_cast<size_t>(c.NS) * kSnStageBytes;
    c.ok = true;
    return c;
}

bool smalln_mma_ok(int64_t n, int64_t K, int64_t N) {
    return n >= 1 && sn_config_group(K, 1, &N).ok;
}

bool smalln_mma_grouped_ok(int64_t n, int64_t K, int count, const int64_t* N) {
    return n >= 1 && sn_config_group(K, count, N).ok;
}

static int sn_maps(SnMaps* maps, int i, int64_t K, int64_t N, const uint32_t* w, const uint16_t* s) {
    const uint64_t dims[3] = {32, static_cast<uint64_t>(N), static_cast<uint64_t>(K / 256)};
    const uint64_t strides[2] = {static_cast<uint64_t>(K / 2), 128};
    const uint32_t box[3] = {32, kSnRows, kSnChunkK / 256};
    int rc = make_tensor_map(&maps->w[i], CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, w, dims, strides, box,
                             CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) return rc;
    const uint64_t sdims[2] = {static_cast<uint64_t>(K / kGroup), static_cast<uint64_t>(N)};
    const uint64_t sstrides[1] = {static_cast<uint64_t>(K / kGroup) * 2};
    const uint32_t sbox[2] = {kSnChunkG, kSnRows};
    return make_tensor_map(&maps->s[i], CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, s, sdims, sstrides, sbox,
                           CU_TENSOR_MAP_SWIZZLE_128B);
}

// `count` matrices sharing x and K in one launch per 8 tokens (count = 1: the
// plain call).
int launch_smalln_mma_grouped(const uint16_t* x, int64_t n, int64_t K, int count, const int64_t* N,
                              const uint32_t* const* w, const uint16_t* const* s, uint16_t* const* y, bool pdl,
                              cudaStream_t stream) {
    const SnConfig c = sn_config_group(K, count, N);
    if (!c.ok || n < 1) return static_cast<int>(cudaErrorInvalidConfiguration);
    SnMaps maps;
    memset(&maps, 0, sizeof maps);
    for (int i = 0; i < count; ++i) {
        const int rc = sn_maps(&maps, i, K, N[i], w[i], s[i]);
        if (rc) return rc;
    }
    const int W = sn_warps();
    auto kern = W == 16 ? q4_smalln_mma_kernel<16> : q4_smalln_mma_kernel<8>;
    const cudaError_t e = ensure_kernel_attrs(reinterpret_cast<const void*>(kern), static_cast<int>(kSnSmemMax));
    if (e != cudaSuccess) return static_cast<int>(e);
    if (knob_int("RELAX_Q4_GS_PRINT", 0))
        fprintf(stderr, "smalln_mma K=%lld N0=%lld count=%d n=%lld NS=%d grid=%d smem=%zu\n", (long long)K,
                (long long)N[0], count, (long long)n, c.NS, c.grid, c.smem);
    for (int64_t t0 = 0; t0 < n; t0 += kSnTok) {          // 8 tokens (the MMA's N) per launch
        SnArgs a{};
        a.x = x + t0 * K;
        a.K = static_cast<int>(K);
        a.G = static_cast<int>(K / kGroup);
        a.n = static_cast<int>(n - t0 < kSnTok ? n - t0 : kSnTok);
        a.NS = c.NS;
        a.nkc = static_cast<int>((K + kSnChunkK - 1) / kSnChunkK);
        a.rows_max = c.rows_max;
        a.nmat = count;
#if RQ4_TRACE
        static uint32_t sn_seq = 0;
        a.trace_seq = knob_int("RELAX_Q4_TRACE", 0) == 1 ? ++sn_seq : 0u;
#endif
        for (int i = 0; i <= count; ++i) a.cta0[i] = c.cta0[i];
        for (int i = 0; i < count; ++i) {
            a.ygp[i] = y[i] + t0 * N[i];
            a.Ngp[i] = N[i];
            a.nrbgp[i] = (N[i] + kSnRows - 1) / kSnRows;
        }
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(c.grid);
        cfg.blockDim = dim3((W + 1) * 32);
        cfg.dynamicSmemBytes = c.smem;
        cfg.stream = stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        const int rc = static_cast<int>(cudaLaunchKernelEx(&cfg, kern, maps, a));
        if (rc) return rc;
    }
    return 0;
}

int launch_smalln_mma(const uint16_t* x, int64_t n, int64_t K, int64_t N, const uint32_t* w,
                      const uint16_t* s, uint16_t* y, bool pdl, cudaStream_t stream) {
    return launch_smalln_mma_grouped(x, n, K, 1, &N, &w, &s, &y, pdl, stream);
}

// Largest n the automatic dispatch gives this kernel (measured
// crossover with the tcgen05 kernel); RELAX_Q4_SMALLN_MAX_N in the experiments build.
int smalln_max_n() {
    static const int v = [] { const int x = knob_int("RELAX_Q4_SMALLN_MAX_N", 8); return x >= 0 ? x : 8; }();
    return v;
}

}  // namespace rq4

#if RQ4_TRACE
extern "C" RELAX_API int relax_debug_sntrace_read(void* host, size_t max_records, size_t* n_records, int reset) {
    uint32_t n = 0;
    if (cudaMemcpyFromSymbol(&n, rq4::g_sn_trace_n, sizeof n) != cudaSuccess) return RELAX_ERR_CUDA;
    if (n > static_cast<uint32_t>(rq4::kSnTraceMax)) n = rq4::kSnTraceMax;
    const size_t m = n < max_records ? n : max_records;
    if (m && cudaMemcpyFromSymbol(host, rq4::g_sn_trace, m * sizeof(rq4::SnTraceRec)) != cudaSuccess) return RELAX_ERR_CUDA;
    if (n_records) *n_records = m;
    if (reset) {
        const uint32_t z = 0;
        if (cudaMemcpyToSymbol(rq4::g_sn_trace_n, &z, sizeof z) != cudaSuccess) return RELAX_ERR_CUDA;
    }
    return RELAX_OK;
}
#endif
