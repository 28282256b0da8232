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
#include "internal.h"
#include "ptx.cuh"
#include "q4_unpack.cuh"

namespace rq4 {

struct GsArgs {
    const uint16_t* x;     // [NT][K] fp16
    const uint8_t* w;      // [N][K/2] bytes
    const uint8_t* s;      // [N][K/16] bytes (fp16 scales)
    uint16_t* y;           // [NT][N]
    int64_t N;
    int K, G, WK, H, RS, NS;
    uint32_t stage_bytes;  // RS * (K/2 + K/16)
    int rows_cta_max;
};

struct GsConfig {
    int WK, H, RPW, RS, NS, threads, rows_cta_max, grid;
    size_t smem;
};

constexpr int kGsMaxConsumerWarps = 16;   // WK * H <= 16 in the 2-CTA/SM build
constexpr int kGsSmemBudget = 100 * 1024;

__device__ __forceinline__ uint4 lds128(const uint8_t* p) { return *reinterpret_cast<const uint4*>(p); }

// Transposed butterfly: acc[0..R) per lane -> every lane holds, in acc[0],
// the full 32-lane sum of row rsel(lane) = sum_s bit(lane, 4-s) * R >> (s+1).
template <int R>
__device__ __forceinline__ float reduce_rows(float (&acc)[R], int lane) {
    int cnt = R;
    int off = 16;
#pragma unroll
    for (int step = 0; (R >> step) > 1; ++step) {
        const int half = cnt >> 1;
        const bool upper = (lane & off) != 0;
#pragma unroll
        for (int j = 0; j < R / 2; ++j) {
            if (j < half) {
                const float send = upper ? acc[j] : acc[j + half];
                const float keep = upper ? acc[j + half] : acc[j];
                acc[j] = keep + __shfl_xor_sync(0xffffffffu, send, off);
            }
        }
        cnt = half;
        off >>= 1;
    }
#pragma unroll
    for (; off > 0; off >>= 1) acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], off);
    return acc[0];
}

template <int R>
__device__ __forceinline__ int reduce_row_of_lane(int lane) {
    int row = 0, off = 16;
#pragma unroll
    for (int step = 0; (R >> step) > 1; ++step) {
        if (lane & off) row += R >> (step + 1);
        off >>= 1;
    }
    return row;
}

template <int NT, int RPW, int MAXT, int MINB>
__global__ void __launch_bounds__(MAXT, MINB) gemv_stream_kernel(const __grid_constant__ GsArgs a) {
    extern __shared__ __align__(128) uint8_t smem[];
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int nwc = a.WK * a.H;                        // consumer warps
    // [barriers: 2*NS x 8 B, padded to 128][ring: NS stages][partials]
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + a.NS;
    uint8_t* ring = smem + 128;
    float* part = reinterpret_cast<float*>(ring + static_cast<size_t>(a.NS) * a.stage_bytes);

    const int64_t row0 = static_cast<int64_t>(blockIdx.x) * a.N / gridDim.x;
    const int64_t row1 = static_cast<int64_t>(blockIdx.x + 1) * a.N / gridDim.x;
    const int rows = static_cast<int>(row1 - row0);
    const int nst = (rows + a.RS - 1) / a.RS;
    const uint32_t cb_row = static_cast<uint32_t>(a.K / 2);
    const uint32_t sb_row = static_cast<uint32_t>(a.K / 16);
    const uint32_t codes_stage = static_cast<uint32_t>(a.RS) * cb_row;

    if (threadIdx.x == 0) {
        for (int i = 0; i < a.NS; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], nwc); }
        fence_mbar_init();
    }
    __syncthreads();
    pdl_launch_dependents();

    if (warp == nwc) {
        // ------------------------------------------------ producer (one thread)
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            const uint8_t* wsrc = a.w + row0 * cb_row;
            const uint8_t* ssrc = a.s + row0 * sb_row;
            for (int st = 0; st < nst; ++st) {
                const int slot = st % a.NS;
                mbar_wait(&empty[slot], ((st / a.NS) & 1) ^ 1);
                const int r = st * a.RS;
                const int nr = rows - r < a.RS ? rows - r : a.RS;
                const uint32_t bc = static_cast<uint32_t>(nr) * cb_row;
                const uint32_t bs = static_cast<uint32_t>(nr) * sb_row;
                uint8_t* dst = ring + static_cast<size_t>(slot) * a.stage_bytes;
                mbar_arrive_expect_tx(&full[slot], bc + bs);
                bulk_load(dst, wsrc + static_cast<size_t>(r) * cb_row, bc, &full[slot], pol);
                bulk_load(dst + codes_stage, ssrc + static_cast<size_t>(r) * sb_row, bs, &full[slot], pol);
            }
        }
    } else {
        // ------------------------------------------------ consumers
        const int h = warp / a.WK;
        const int kw = warp - h * a.WK;
        const int g = kw * 32 + lane;
        const bool gv = g < a.G;
        pdl_wait();
        uint4 xr[NT][4];
#pragma unroll
        for (int t = 0; t < NT; ++t)
#pragma unroll
            for (int q = 0; q < 4; ++q)
                xr[t][q] = gv ? reinterpret_cast<const uint4*>(a.x + static_cast<int64_t>(t) * a.K + g * 32)[q]
                              : make_uint4(0u, 0u, 0u, 0u);
        const int rsel = reduce_row_of_lane<RPW>(lane);
        for (int st = 0; st < nst; ++st) {
            const int slot = st % a.NS;
            mbar_wait(&full[slot], (st / a.NS) & 1);
            const uint8_t* stage = ring + static_cast<size_t>(slot) * a.stage_bytes;
            const int r_base = st * a.RS;
            const int nr = rows - r_base < a.RS ? rows - r_base : a.RS;
            float acc[NT][RPW];
#pragma unroll
            for (int i = 0; i < RPW; ++i) {
                const int rl = h * RPW + i;
#pragma unroll
                for (int t = 0; t < NT; ++t) acc[t][i] = 0.f;
                if (rl < nr && gv) {
                    const uint4 cw = lds128(stage + static_cast<size_t>(rl) * cb_row + g * 16);
                    const uint16_t sbits = *reinterpret_cast<const uint16_t*>(
                        stage + codes_stage + static_cast<size_t>(rl) * sb_row + g * 2);
                    const uint32_t words[4] = {cw.x, cw.y, cw.z, cw.w};
                    float ga[NT][2];
#pragma unroll
                    for (int t = 0; t < NT; ++t) { ga[t][0] = 0.f; ga[t][1] = 0.f; }
#pragma unroll
                    for (int wi = 0; wi < 4; ++wi) {
                        __half2 cc[4];
                        unpack_centered_interleaved(words[wi], cc);
                        const uint32_t c0 = h2_as_u32(cc[0]), c1 = h2_as_u32(cc[1]);
                        const uint32_t c2 = h2_as_u32(cc[2]), c3 = h2_as_u32(cc[3]);
#pragma unroll
                        for (int t = 0; t < NT; ++t) {
                            const uint4 X = xr[t][wi];    // (k0,k1) (k2,k3) (k4,k5) (k6,k7)
                            float e = ga[t][0], o = ga[t][1];
                            e = fhfma(lo16(c0), lo16(X.x), e);   // k0
                            o = fhfma(lo16(c1), hi16(X.x), o);   // k1
                            e = fhfma(lo16(c2), lo16(X.y), e);   // k2
                            o = fhfma(lo16(c3), hi16(X.y), o);   // k3
                            e = fhfma(hi16(c0), lo16(X.z), e);   // k4
                            o = fhfma(hi16(c1), hi16(X.z), o);   // k5
                            e = fhfma(hi16(c2), lo16(X.w), e);   // k6
                            o = fhfma(hi16(c3), hi16(X.w), o);   // k7
                            ga[t][0] = e;
                            ga[t][1] = o;
                        }
                    }
                    const float sc = __half2float(__ushort_as_half(sbits));
#pragma unroll
                    for (int t = 0; t < NT; ++t) acc[t][i] = sc * (ga[t][0] + ga[t][1]);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[slot]);      // stage bytes fully consumed
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                const float v = reduce_rows<RPW>(acc[t], lane);
                const int rl = h * RPW + rsel;
                if ((lane & (32 / RPW - 1)) == 0 && rl < nr)
                    part[(static_cast<size_t>(r_base + rl) * a.WK + kw) * NT + t] = v;
            }
        }
    }
    __syncthreads();
    // fixed-order sum over the WK K-columns; fp32 -> fp16 RNE
    for (int o = threadIdx.x; o < rows * NT; o += blockDim.x) {
        const int rl = o / NT;
        const int t = o - rl * NT;
        float sum = 0.f;
        for (int c = 0; c < a.WK; ++c) sum += part[(static_cast<size_t>(rl) * a.WK + c) * NT + t];
        a.y[static_cast<int64_t>(t) * a.N + row0 + rl] = __half_as_ushort(__float2half_rn(sum));
    }
}

static GsConfig gs_config(int64_t K, int64_t N) {
    GsConfig c{};
    const int G = static_cast<int>(K / kGroup);
    c.WK = (G + 31) / 32;
    c.H = 1;
    while (c.WK * c.H * 2 <= kGsMaxConsumerWarps && c.H < 16) c.H *= 2;
    const double row_bytes = 0.5625 * static_cast<double>(K);
    int rpw = static_cast<int>(32768.0 / (c.H * row_bytes));
    c.RPW = rpw >= 4 ? 4 : rpw >= 2 ? 2 : 1;
    c.RS = c.H * c.RPW;
    const size_t stage = static_cast<size_t>(c.RS) * (K / 2 + K / 16);
    int ns = static_cast<int>(kGsSmemBudget / stage);
    c.NS = ns < 2 ? 2 : ns > 6 ? 6 : ns;
    c.threads = (c.WK * c.H + 1) * 32;
    c.grid = static_cast<int>(N < kNumSMs ? N : kNumSMs);
    c.rows_cta_max = static_cast<int>((N + c.grid - 1) / c.grid);
    return c;
}

bool gemv_stream_ok(int nt, int64_t K) {
    if (nt < 1 || nt > 2 || K % 256 != 0) return false;
    const int G = static_cast<int>(K / kGroup);
    return (G + 31) / 32 <= 31;   // <= 1024 threads incl. the producer warp
}

template <int NT, int RPW>
static int launch_gs_t(const GsArgs& a, const GsConfig& c, bool pdl, cudaStream_t stream) {
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
    if (c.threads <= 544) {
        auto k = gemv_stream_kernel<NT, RPW, 544, 2>;
        static bool set = false;
        if (!set) {
            cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 113 * 1024);
            if (e != cudaSuccess) return static_cast<int>(e);
            set = true;
        }
        return static_cast<int>(cudaLaunchKernelEx(&cfg, k, a));
    }
    auto k = gemv_stream_kernel<NT, RPW, 1024, 1>;
    static bool set = false;
    if (!set) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        if (e != cudaSuccess) return static_cast<int>(e);
        set = true;
    }
    return static_cast<int>(cudaLaunchKernelEx(&cfg, k, a));
}

int launch_gemv_stream(const uint16_t* x, int64_t n, int64_t K, int64_t N, const uint32_t* w,
                       const uint16_t* s, uint16_t* y, bool pdl, cudaStream_t stream) {
    GsConfig c = gs_config(K, N);
    c.smem = 128 + static_cast<size_t>(c.NS) * c.RS * (K / 2 + K / 16) +
             static_cast<size_t>(c.rows_cta_max) * c.WK * 2 * 4;
    for (int64_t t0 = 0; t0 < n; t0 += 2) {
        const int cnt = (n - t0) >= 2 ? 2 : 1;
        GsArgs a;
        a.x = x + t0 * K;
        a.w = reinterpret_cast<const uint8_t*>(w);
        a.s = reinterpret_cast<const uint8_t*>(s);
        a.y = y + t0 * N;
        a.N = N;
        a.K = static_cast<int>(K);
        a.G = static_cast<int>(K / kGroup);
        a.WK = c.WK; a.H = c.H; a.RS = c.RS; a.NS = c.NS;
        a.stage_bytes = static_cast<uint32_t>(c.RS * (K / 2 + K / 16));
        a.rows_cta_max = c.rows_cta_max;
        int rc;
        if (cnt == 1) {
            rc = c.RPW == 4 ? launch_gs_t<1, 4>(a, c, pdl, stream)
               : c.RPW == 2 ? launch_gs_t<1, 2>(a, c, pdl, stream) : launch_gs_t<1, 1>(a, c, pdl, stream);
        } else {
            rc = c.RPW == 4 ? launch_gs_t<2, 4>(a, c, pdl, stream)
               : c.RPW == 2 ? launch_gs_t<2, 2>(a, c, pdl, stream) : launch_gs_t<2, 1>(a, c, pdl, stream);
        }
        if (rc != 0) return rc;
    }
    return 0;
}

}  // namespace rq4
