// decode_chain.cu -- a whole decode step's chain of q4f16 GEMVs (n = 1) in ONE
// persistent launch (relax_q4_chain_*; include/relax_q4.h).
//
// y_m[j] = sum_k x_m[k] * W_m(k, j),  W = (q - 7) * s   (dequant fused
// into the matmul), for ops m = 0 .. count-1 in order; op m may read
// (as x_m) what earlier ops wrote.
//
// Why: launched one by one, even with programmatic dependent launch, each
// decode GEMV leaves HBM idle while it drains, the next one's griddepcontrol
// wait releases and its x arrives (~2 us per kernel): the 7B
// step ran at ~4.5 TB/s for a 6.55 TB/s copy peak.  Here one CTA per SM lives
// for the whole chain and its producer warp streams the weights of op after op
// through a ~200 KB shared-memory ring without ever waiting for activations --
// weights do not depend on them -- so HBM keeps streaming while the consumers
// wait for a dependency: ~4.5 us of look-ahead per SM.
//
// Per CTA (992 threads: 30 consumer warps + 1 producer warp):
//   * op m's rows are split over the CTAs (balanced to +-1 row); the CTA's
//     rows are contiguous bytes in the NK layout, streamed as stages of
//     RS = H * RPW rows (codes, then scales) by 1-D bulk async copies;
//   * consumer warp (h, kw), h < H, kw < WK = ceil(K/1024): lane l owns the
//     32-code group 32 kw + l of every row (x of that group in 16-bit fixed
//     point in registers, decode_math.cuh) and handles rows h*RPW .. of every
//     stage; every consumer warp passes through every stage (the ring's
//     "empty" barrier counts all 30), so the ring protocol does not depend on
//     the op's shape;
//   * at the end of op m the WK partials of each row are summed in fixed order
//     (deterministic), y is stored, and the CTA adds 1 to op m's completion
//     counter (release); an op flagged `after` first waits (acquire) until
//     every CTA has completed every earlier op, then loads its x through L2.
// Counters are monotone across launches: launch generation g (read from the
// workspace) waits for (g + 1) * grid, and the last CTA to finish bumps g.
#include <cstdio>
#include <cstring>
#include <vector>
#include "internal.h"
#include "relax_q4.h"
#include "ptx.cuh"
#include "decode_math.cuh"
#include "knobs.h"

namespace rq4 {

constexpr int kChWarps = 30;                           // consumer warps
constexpr int kChThreads = (kChWarps + 1) * 32;        // + the producer warp
constexpr uint32_t kChSlot = 18432;                    // bytes per ring slot
constexpr int kChSlots = 12;                           // 216 KB ring
constexpr int kChMaxOps = 1024;
constexpr uint32_t kChPartBytes = 8192;                // per-op partial sums [rows][WK] fp32
constexpr size_t kChSmem = 256 + static_cast<size_t>(kChSlots) * kChSlot + kChPartBytes;

struct ChainOpDev {
    const uint16_t* x;
    const uint8_t* w;
    const uint8_t* s;
    uint16_t* y;
    int K, N, after;
    int WK, H, RPW, RS;
    uint32_t cb, sb;        // code / scale bytes per row
    int flags;              // kChReuseX | kChSignal
    int q, rem;             // rows per CTA: q, +1 for the first rem CTAs
};
__device__ __forceinline__ int64_t chain_r0(const ChainOpDev& op, int cta) {
    return static_cast<int64_t>(cta) * op.q + (cta < op.rem ? cta : op.rem);
}
constexpr int kChReuseX = 1;   // same x and K as the op before, no wait: the x registers carry over
constexpr int kChSignal = 2;   // the next op waits on this one: count its completion

struct ChainHdr {
    uint32_t gen;           // launch generation
    uint32_t done;          // CTAs finished (monotone)
    int32_t count;          // ops
    int32_t grid;           // CTAs the counters were set up for
};
// workspace: [ChainHdr, padded to 256][completion counters: count x u32, padded to 256][op table]
__host__ __device__ __forceinline__ size_t chain_ctr_off() { return 256; }
__host__ __device__ __forceinline__ size_t chain_ops_off(int count) { return 256 + ((static_cast<size_t>(count) * 4 + 255) / 256) * 256; }

#if RQ4_TRACE
// per (CTA, op) globaltimer stamps (experiments build): op start, dependency
// satisfied, x in registers, last stage consumed, completion signalled, and
// the producer's first issue of the op
constexpr int kChTrOps = 256;
constexpr int kChTrF = 7;
__device__ uint64_t g_chain_tr[160 * kChTrOps * kChTrF];
#define CH_TR(m, f)                                                                                 \
    do {                                                                                           \
        if ((m) < kChTrOps) g_chain_tr[(static_cast<size_t>(blockIdx.x) * kChTrOps + (m)) * kChTrF + (f)] = globaltimer(); \
    } while (0)
#else
#define CH_TR(m, f) do { } while (0)
#endif

__device__ __forceinline__ void red_release_gpu_add(uint32_t* p, uint32_t v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void consumers_sync() {
    asm volatile("bar.sync 1, %0;" ::"r"(kChWarps * 32) : "memory");
}

// One stage (RPW rows) of op `op` for the warp of K-column kw of the owning group.
template <int RPW>
__device__ __forceinline__ void chain_stage(const uint8_t* stage, const ChainOpDev& op, int nr, int kw, int lane,
                                            bool gv, const uint32_t (&xi)[1][4][4], const int (&sx7)[1],
                                            const float (&xinv)[1], float* part, int row_base) {
    const int g = kw * 32 + lane;
    float acc[RPW];
#pragma unroll
    for (int i = 0; i < RPW; ++i) {
        float o[1] = {0.f};
        if (i < nr && gv) {
            const uint4 cw = *reinterpret_cast<const uint4*>(stage + i * op.cb + g * 16);
            const uint16_t sbits = *reinterpret_cast<const uint16_t*>(stage + RPW * op.cb + i * op.sb + g * 2);
            row_dot_idp<1>(cw, sbits, xi, sx7, xinv, o);
        }
        acc[i] = o[0];
    }
    const float v = reduce_rows<RPW>(acc, lane);
    const int rsel = reduce_row_of_lane<RPW>(lane);
    if ((lane & (32 / RPW - 1)) == 0 && rsel < nr) part[(row_base + rsel) * op.WK + kw] = v;
}

__global__ void __launch_bounds__(kChThreads, 1) q4_decode_chain_kernel(uint8_t* __restrict__ ws) {
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + kChSlots;
    uint8_t* ring = smem + 256;
    float* part = reinterpret_cast<float*>(ring + static_cast<size_t>(kChSlots) * kChSlot);
    ChainHdr* hdr = reinterpret_cast<ChainHdr*>(ws);
    uint32_t* ctr = reinterpret_cast<uint32_t*>(ws + chain_ctr_off());
    const int count = hdr->count;                      // written by relax_q4_chain_init, constant
    const ChainOpDev* ops = reinterpret_cast<const ChainOpDev*>(ws + chain_ops_off(count));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int cta = blockIdx.x, ncta = gridDim.x;   // ncta == the grid the row split was planned for
    if (threadIdx.x == 0) {
        for (int i = 0; i < kChSlots; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
        fence_mbar_init();
    }
    __syncthreads();
    pdl_launch_dependents();

    if (warp == kChWarps) {
        // ------------------------------------------------ producer: every op's rows, back to back
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            int slot = 0;
            uint32_t phase = 0;
            for (int m = 0; m < count; ++m) {
                const ChainOpDev op = ops[m];
                const int64_t r0 = chain_r0(op, cta);
                const int64_t r1 = r0 + op.q + (cta < op.rem ? 1 : 0);
                for (int64_t r = r0; r < r1; r += op.RS) {
                    const uint32_t nr = static_cast<uint32_t>(r1 - r < op.RS ? r1 - r : op.RS);
                    mbar_wait(&empty[slot], phase ^ 1);
                    if (r == r0) CH_TR(m, 5);
                    uint8_t* dst = ring + static_cast<size_t>(slot) * kChSlot;
                    mbar_arrive_expect_tx(&full[slot], nr * (op.cb + op.sb));
                    bulk_load(dst, op.w + r * op.cb, nr * op.cb, &full[slot], pol);
                    bulk_load(dst + op.RPW * op.cb, op.s + r * op.sb, nr * op.sb, &full[slot], pol);
                    if (++slot == kChSlots) { slot = 0; phase ^= 1; }
                }
            }
        }
        return;
    }
    // ---------------------------------------------------- consumers
    pdl_wait();
    const uint32_t gen = *reinterpret_cast<volatile uint32_t*>(&hdr->gen);
    const uint32_t target = (gen + 1u) * static_cast<uint32_t>(ncta);
    uint32_t seq = 0;                                    // stages of earlier ops (this CTA)
    uint32_t xi[1][4][4];
    int sx7[1] = {0};
    float xinv[1] = {1.f};
    // op descriptors staged in shared memory (double-buffered: op m + 1 is
    // loaded before the barrier that ends op m)
    __shared__ ChainOpDev op_s[2];
    if (threadIdx.x < sizeof(ChainOpDev) / 4)
        reinterpret_cast<uint32_t*>(&op_s[0])[threadIdx.x] = reinterpret_cast<const uint32_t*>(&ops[0])[threadIdx.x];
    consumers_sync();
    for (int m = 0; m < count; ++m) {
        const ChainOpDev& op = op_s[m & 1];
        const int64_t r0 = chain_r0(op, cta);
        const int rows = op.q + (cta < op.rem ? 1 : 0);
        const int h = warp / op.WK, kw = warp - h * op.WK;
        const bool active = h < op.H;
        const int G = op.K / kGroup;
        const int g = kw * 32 + lane;
        const bool gv = active && g < G;
        if (threadIdx.x == 0) CH_TR(m, 0);
        if (op.after && m > 0) {
            // every CTA has completed every earlier op (they run in order per CTA)
            if (threadIdx.x == 0) {
                const uint64_t t0 = globaltimer();
                while (static_cast<int32_t>(ld_acquire_gpu_u32(&ctr[m - 1]) - target) < 0)
                    if (globaltimer() - t0 > 10000000000ull) __trap();
            }
            consumers_sync();
        }
        if (threadIdx.x == 0) CH_TR(m, 1);
        // x of the lane's group (it may have been written by other SMs in this
        // launch: the acquire above and the barrier order these loads after
        // those writes), in fixed point; kept for following ops on the same x
        if (!(op.flags & kChReuseX)) {
            uint4 xr[4];
            const uint4* xp = reinterpret_cast<const uint4*>(op.x + g * 32);
#pragma unroll
            for (int q = 0; q < 4; ++q) xr[q] = gv ? xp[q] : make_uint4(0u, 0u, 0u, 0u);
            x_to_fixed(xr, xi[0], sx7[0], xinv[0]);
        }
        if (threadIdx.x == 0) CH_TR(m, 2);
        // stages go round-robin to the H row groups (group h: stages h, h + H, ...),
        // each read by the group's WK warps and released by one arrival after
        // the group's named barrier; H divides the slot count, so a group only
        // ever waits on its own sub-ring
        const int nst = (rows + op.RS - 1) / op.RS;
        if (active && h < nst) {
            const uint32_t sq0 = seq + static_cast<uint32_t>(h);
            int sl = static_cast<int>(sq0 % kChSlots);
            uint32_t ph = (sq0 / kChSlots) & 1u;
            for (int st = h; st < nst; st += op.H) {
                mbar_wait(&full[sl], ph);
                const uint8_t* stage = ring + static_cast<size_t>(sl) * kChSlot;
                const int nr = rows - st * op.RS < op.RS ? rows - st * op.RS : op.RS;
                switch (op.RPW) {
                    case 8: chain_stage<8>(stage, op, nr, kw, lane, gv, xi, sx7, xinv, part, st * op.RS); break;
                    case 4: chain_stage<4>(stage, op, nr, kw, lane, gv, xi, sx7, xinv, part, st * op.RS); break;
                    case 2: chain_stage<2>(stage, op, nr, kw, lane, gv, xi, sx7, xinv, part, st * op.RS); break;
                    default: chain_stage<1>(stage, op, nr, kw, lane, gv, xi, sx7, xinv, part, st * op.RS); break;
                }
                if (op.WK > 1) asm volatile("bar.sync %0, %1;" ::"r"(2 + h), "r"(op.WK * 32) : "memory");
                else __syncwarp();
                if (kw == 0 && lane == 0) mbar_arrive(&empty[sl]);
                sl += op.H;                              // H <= kChSlots
                if (sl >= kChSlots) { sl -= kChSlots; ph ^= 1u; }
            }
        }
        seq += static_cast<uint32_t>(nst);
        consumers_sync();
        if (threadIdx.x == 0) CH_TR(m, 3);
        // fixed-order sum over the WK K-columns; fp32 -> fp16 RNE
        for (int o = threadIdx.x; o < rows; o += kChWarps * 32) {
            float sum = 0.f;
            for (int c = 0; c < op.WK; ++c) sum += part[o * op.WK + c];
            op.y[r0 + o] = __half_as_ushort(__float2half_rn(sum));
        }
        if (m + 1 < count && threadIdx.x < sizeof(ChainOpDev) / 4)
            reinterpret_cast<uint32_t*>(&op_s[(m + 1) & 1])[threadIdx.x] =
                reinterpret_cast<const uint32_t*>(&ops[m + 1])[threadIdx.x];
        consumers_sync();                                // y stored, part free, next op staged
        if ((op.flags & kChSignal) && threadIdx.x == 0) {
            // release: the barrier above ordered every consumer's y stores before it
            red_release_gpu_add(&ctr[m], 1u);
        }
        if (threadIdx.x == 0) CH_TR(m, 4);
    }
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(&hdr->done, 1u) == target - 1u) {
            __threadfence();
            atomicExch(&hdr->gen, gen + 1u);             // the next launch (stream order) reads it
        }
    }
}

// ---------------------------------------------------------------- host side
static bool chain_op_config(int64_t K, int64_t N, ChainOpDev* d) {
    if (K <= 0 || N <= 0 || K % 256 != 0 || N >= (int64_t{1} << 30)) return false;
    const int G = static_cast<int>(K / kGroup);
    const int WK = (G + 31) / 32;
    if (WK > kChWarps) return false;
    const uint32_t cb = static_cast<uint32_t>(K / 2), sb = static_cast<uint32_t>(K / 16);
    // row groups: H divides the slot count, so within an op slot j only ever
    // holds stages of group j % H (a private sub-ring per group: a group never
    // waits on a slot two phases ahead); named barriers 2..15 synchronise a
    // group's WK warps (a one-warp group needs none)
    int H = kChWarps / WK;
    if (H > kChSlots) H = kChSlots;
    while (kChSlots % H != 0) --H;
    if (cb + sb > kChSlot) return false;
    int RPW = 8;
    while (RPW > 1 && static_cast<uint64_t>(RPW) * (cb + sb) > kChSlot) RPW >>= 1;
    const int64_t rows_max = (N + num_sms() - 1) / num_sms();
    if (static_cast<uint64_t>(rows_max) * WK * 4 > kChPartBytes) return false;
    d->K = static_cast<int>(K);
    d->N = static_cast<int>(N);
    d->WK = WK;
    d->H = H;
    d->RPW = RPW;
    d->RS = RPW;
    d->cb = cb;
    d->sb = sb;
    return true;
}

int chain_max_ops() { return kChMaxOps; }

bool chain_op_ok(int64_t K, int64_t N) {
    ChainOpDev d{};
    return chain_op_config(K, N, &d);
}

size_t chain_workspace_bytes(int count) {
    return chain_ops_off(count) + static_cast<size_t>(count) * sizeof(ChainOpDev);
}

int chain_init(const ChainOpHost* ops, int count, void* ws) {
    std::vector<uint8_t> img(chain_workspace_bytes(count), 0);
    ChainHdr* hdr = reinterpret_cast<ChainHdr*>(img.data());
    hdr->gen = 0;
    hdr->done = 0;
    hdr->count = count;
    hdr->grid = num_sms();
    ChainOpDev* d = reinterpret_cast<ChainOpDev*>(img.data() + chain_ops_off(count));
    if (count > kChMaxOps) return static_cast<int>(cudaErrorInvalidValue);
    for (int i = 0; i < count; ++i) {
        if (!chain_op_config(ops[i].K, ops[i].N, &d[i])) return static_cast<int>(cudaErrorInvalidValue);
        d[i].x = ops[i].x;
        d[i].w = reinterpret_cast<const uint8_t*>(ops[i].w);
        d[i].s = reinterpret_cast<const uint8_t*>(ops[i].s);
        d[i].y = ops[i].y;
        d[i].after = ops[i].after ? 1 : 0;
    }
    for (int i = 0; i < count; ++i) {
        d[i].q = static_cast<int>(d[i].N / hdr->grid);
        d[i].rem = static_cast<int>(d[i].N % hdr->grid);
        d[i].flags = 0;
        if (i > 0 && !d[i].after && d[i].x == d[i - 1].x && d[i].K == d[i - 1].K) d[i].flags |= kChReuseX;
        if (i + 1 < count && d[i + 1].after) d[i].flags |= kChSignal;
    }
    const cudaError_t e = cudaMemcpy(ws, img.data(), img.size(), cudaMemcpyHostToDevice);
    return static_cast<int>(e);
}

int launch_chain(void* ws, bool pdl, cudaStream_t stream) {
    const cudaError_t ae = ensure_kernel_attrs(reinterpret_cast<const void*>(q4_decode_chain_kernel),
                                               static_cast<int>(kChSmem));
    if (ae != cudaSuccess) return static_cast<int>(ae);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(num_sms());
    cfg.blockDim = dim3(kChThreads);
    cfg.dynamicSmemBytes = kChSmem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return static_cast<int>(cudaLaunchKernelEx(&cfg, q4_decode_chain_kernel, static_cast<uint8_t*>(ws)));
}

}  // namespace rq4

#if RQ4_TRACE
extern "C" RELAX_API int relax_debug_chain_trace_read(void* host, size_t bytes) {
    const size_t n = sizeof(rq4::g_chain_tr) < bytes ? sizeof(rq4::g_chain_tr) : bytes;
    return cudaMemcpyFromSymbol(host, rq4::g_chain_tr, n) == cudaSuccess ? RELAX_OK : RELAX_ERR_CUDA;
}
#endif
