// gemv_row.cu -- decode GEMV, "lane = output row" organisation (n = 1).
//
// y[j] = sum_k x[k] * W(k, j), W = (q - 7) * s  (dequant fused into
// the matmul; K, N static, n runtime).
//
// Versus gemv_stream.cu (lane = 32-code group, rows reduced across lanes with
// shuffles) this kernel removes every cross-lane reduction from the inner
// loop: each lane owns one output row of a 32-row block, each warp owns a
// fixed slice of K, and a lane's dot product accumulates in one register.
//   * one producer thread streams the CTA's rows through a shared-memory ring
//     with 1-D bulk async copies (TMA engine, L2 evict-first), one copy per
//     row segment into a padded row slot (stride K_c/2 + 16 B) so that the
//     32 lanes' LDS.128 of 32 different rows are bank-conflict free;
//   * x is copied once per CTA (bulk copy, after griddepcontrol.wait) and read
//     with broadcast LDS.128 (all lanes, same address: one wavefront);
//   * codes stay packed until the FHFMA: masks give fp16 subnormals q * 2^-24
//     (1 SHF + 4 LOP3 per 8 codes) and the zero point is factored per group,
//     sum (q - 7) x = 2^24 (acc_e + acc_o / 16) - 7 * sum x, with the group
//     sums of x computed once per CTA;
//   * the 16 K-slice partials of a row are summed in shared memory in fixed
//     order at the end: deterministic.
#include <cstdlib>
#include "internal.h"
#include "ptx.cuh"
#include "q4_unpack.cuh"

namespace rq4 {

constexpr int kGrWarps = 16;          // consumer warps = K slices
constexpr int kGrGroupsPerWarp = 4;   // 32-code groups per warp per stage
constexpr int kGrChunkGroups = kGrWarps * kGrGroupsPerWarp;   // 64 groups = 2048 k per stage
constexpr int kGrRows = 32;           // rows per block (lanes)
constexpr int kGrCodesStride = kGrChunkGroups * 16 + 16;     // 1040 B per row slot
constexpr int kGrScalesStride = kGrChunkGroups * 2 + 16;     // 144 B per row slot
constexpr int kGrStageBytes = kGrRows * (kGrCodesStride + kGrScalesStride);   // 37,888 B

struct GrArgs {
    const uint16_t* x;
    const uint8_t* w;      // [N][K/2]
    const uint8_t* s;      // [N][K/16]
    uint16_t* y;
    int64_t N;
    int K, G, NS, rows_cta_max;
};

template <int FULLC>
__global__ void __launch_bounds__((kGrWarps + 1) * 32, 2) gemv_row_kernel(const __grid_constant__ GrArgs a) {
    extern __shared__ __align__(128) uint8_t smem[];
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    // [bars 128 B][ring NS stages][x: K fp16][xsum: G f32][part: rows x 16 f32]
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + a.NS;
    uint64_t* xbar = empty + a.NS;
    uint8_t* ring = smem + 128;
    uint16_t* xs = reinterpret_cast<uint16_t*>(ring + static_cast<size_t>(a.NS) * kGrStageBytes);
    float* m7x = reinterpret_cast<float*>(xs + a.K);
    float* part = m7x + ((a.G + 3) & ~3);

    const int64_t row0 = static_cast<int64_t>(blockIdx.x) * a.N / gridDim.x;
    const int64_t row1 = static_cast<int64_t>(blockIdx.x + 1) * a.N / gridDim.x;
    const int rows = static_cast<int>(row1 - row0);
    const int nchunk = (a.G + kGrChunkGroups - 1) / kGrChunkGroups;
    const int nblk = (rows + kGrRows - 1) / kGrRows;
    const int nst = nblk * nchunk;
    const uint32_t cb_row = static_cast<uint32_t>(a.K / 2);
    const uint32_t sb_row = static_cast<uint32_t>(a.K / 16);

    if (threadIdx.x == 0) {
        for (int i = 0; i < a.NS; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], kGrWarps); }
        mbar_init(xbar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    pdl_launch_dependents();

    if (warp == kGrWarps) {
        // ------------------------------------------------ producer (one thread)
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            int slot = 0;
            uint32_t phase = 0;
            bool x_issued = false;
            for (int st = 0; st < nst; ++st) {
                const int blk = st / nchunk;
                const int c = st - blk * nchunk;
                const int r0 = blk * kGrRows;
                const int nr = rows - r0 < kGrRows ? rows - r0 : kGrRows;
                const int g0 = c * kGrChunkGroups;
                const int ng = a.G - g0 < kGrChunkGroups ? a.G - g0 : kGrChunkGroups;
                mbar_wait(&empty[slot], phase ^ 1);
                uint8_t* dst = ring + static_cast<size_t>(slot) * kGrStageBytes;
                uint8_t* sdst = dst + kGrRows * kGrCodesStride;
                mbar_arrive_expect_tx(&full[slot], static_cast<uint32_t>(nr) * static_cast<uint32_t>(ng) * 18u);
                const uint8_t* wsrc = a.w + (row0 + r0) * cb_row + static_cast<size_t>(g0) * 16;
                const uint8_t* ssrc = a.s + (row0 + r0) * sb_row + static_cast<size_t>(g0) * 2;
                for (int r = 0; r < nr; ++r) {
                    bulk_load(dst + r * kGrCodesStride, wsrc + static_cast<size_t>(r) * cb_row,
                              static_cast<uint32_t>(ng) * 16u, &full[slot], pol);
                    bulk_load(sdst + r * kGrScalesStride, ssrc + static_cast<size_t>(r) * sb_row,
                              static_cast<uint32_t>(ng) * 2u, &full[slot], pol);
                }
                if (++slot == a.NS) { slot = 0; phase ^= 1; }
                if (!x_issued && (st + 1 == a.NS || st + 1 == nst)) {
                    // the ring is primed with weights: now wait for x's producer
                    pdl_wait();
                    mbar_arrive_expect_tx(xbar, static_cast<uint32_t>(a.K) * 2u);
                    bulk_load(xs, a.x, static_cast<uint32_t>(a.K) * 2u, xbar, policy_evict_last());
                    x_issued = true;
                }
            }
        }
    } else {
        // ------------------------------------------------ consumers
        mbar_wait(xbar, 0);
        // -7 * sum of x over each 32-group (factored zero point)
        for (int g = threadIdx.x; g < a.G; g += kGrWarps * 32) {
            const uint4* xg = reinterpret_cast<const uint4*>(xs + g * 32);
            float sx = 0.f;
#pragma unroll
            for (int qd = 0; qd < 4; ++qd) {
                const uint4 v = xg[qd];
                const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const float2 f = __half22float2(u32_as_h2(w4[u]));
                    sx += f.x + f.y;
                }
            }
            m7x[g] = -7.0f * sx;
        }
        asm volatile("bar.sync 1, %0;" :: "n"(kGrWarps * 32) : "memory");

        int slot = 0;
        uint32_t phase = 0;
        float acc = 0.f;
        for (int st = 0; st < nst; ++st) {
            const int blk = st / nchunk;
            const int c = st - blk * nchunk;
            mbar_wait(&full[slot], phase);
            const uint8_t* stage = ring + static_cast<size_t>(slot) * kGrStageBytes;
            const uint8_t* crow = stage + lane * kGrCodesStride + warp * (kGrGroupsPerWarp * 16);
            const uint8_t* srow = stage + kGrRows * kGrCodesStride + lane * kGrScalesStride + warp * (kGrGroupsPerWarp * 2);
            const int gbase = c * kGrChunkGroups + warp * kGrGroupsPerWarp;
#pragma unroll
            for (int gi = 0; gi < kGrGroupsPerWarp; ++gi) {
                const int g = gbase + gi;
                if (!FULLC && g >= a.G) break;                      // warp-uniform
                const uint4 cw = *reinterpret_cast<const uint4*>(crow + gi * 16);
                const uint16_t sbits = *reinterpret_cast<const uint16_t*>(srow + gi * 2);
                const uint4* xg = reinterpret_cast<const uint4*>(xs + g * 32);
                const uint32_t words[4] = {cw.x, cw.y, cw.z, cw.w};
                float ge = 0.f, go = 0.f;
#pragma unroll
                for (int wi = 0; wi < 4; ++wi) {
                    const uint4 X = xg[wi];                            // broadcast LDS.128
                    const uint32_t v8 = words[wi] >> 8;
                    const uint32_t c0 = words[wi] & 0x000F000Fu;       // (q0, q4) * 2^-24
                    const uint32_t c1 = words[wi] & 0x00F000F0u;       // (q1, q5) * 2^-20
                    const uint32_t c2 = v8 & 0x000F000Fu;              // (q2, q6) * 2^-24
                    const uint32_t c3 = v8 & 0x00F000F0u;              // (q3, q7) * 2^-20
                    ge = fhfma(lo16(c0), lo16(X.x), ge);
                    go = fhfma(lo16(c1), hi16(X.x), go);
                    ge = fhfma(lo16(c2), lo16(X.y), ge);
                    go = fhfma(lo16(c3), hi16(X.y), go);
                    ge = fhfma(hi16(c0), lo16(X.z), ge);
                    go = fhfma(hi16(c1), hi16(X.z), go);
                    ge = fhfma(hi16(c2), lo16(X.w), ge);
                    go = fhfma(hi16(c3), hi16(X.w), go);
                }
                const float u = fmaf(go, 0.0625f, ge);
                const float sc = __half2float(__ushort_as_half(sbits));
                acc = fmaf(sc, fmaf(u, 16777216.0f, m7x[g]), acc);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[slot]);
            if (++slot == a.NS) { slot = 0; phase ^= 1; }
            if (c == nchunk - 1) {
                const int r = blk * kGrRows + lane;
                if (r < rows) part[r * kGrWarps + warp] = acc;
                acc = 0.f;
            }
        }
    }
    __syncthreads();
    for (int r = threadIdx.x; r < rows; r += blockDim.x) {
        float sum = 0.f;
#pragma unroll
        for (int w = 0; w < kGrWarps; ++w) sum += part[r * kGrWarps + w];
        a.y[row0 + r] = __half_as_ushort(__float2half_rn(sum));
    }
}

bool gemv_row_ok(int64_t K) {
    if (K % 256 != 0) return false;
    // ring + x + sums + partials must fit (2 CTAs per SM for K <= ~12K)
    return static_cast<size_t>(K) * 2 + 2 * kGrStageBytes + 64 * 1024 <= 220 * 1024;
}

int launch_gemv_row(const uint16_t* x, int64_t n, int64_t K, int64_t N, const uint32_t* w,
                    const uint16_t* s, uint16_t* y, bool pdl, cudaStream_t stream) {
    const int grid = static_cast<int>(N < num_sms() ? N : num_sms());
    const int rows_max = static_cast<int>((N + grid - 1) / grid);
    const int G = static_cast<int>(K / kGroup);
    int NS = 2;
    if (const char* e = std::getenv("RELAX_Q4_GR_NS")) { const int v = std::atoi(e); if (v >= 2 && v <= 4) NS = v; }
    const size_t smem = 128 + static_cast<size_t>(NS) * kGrStageBytes + static_cast<size_t>(K) * 2 +
                        static_cast<size_t>((G + 3) & ~3) * 4 + static_cast<size_t>(rows_max) * kGrWarps * 4;
    if (smem > 227 * 1024) return static_cast<int>(cudaErrorInvalidConfiguration);
    const bool fullc = G % kGrChunkGroups == 0;
    for (int64_t t = 0; t < n; ++t) {
        GrArgs a;
        a.x = x + t * K;
        a.w = reinterpret_cast<const uint8_t*>(w);
        a.s = reinterpret_cast<const uint8_t*>(s);
        a.y = y + t * N;
        a.N = N;
        a.K = static_cast<int>(K);
        a.G = G;
        a.NS = NS;
        a.rows_cta_max = rows_max;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3((kGrWarps + 1) * 32);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cudaError_t e;
        if (fullc) {
            static bool set = false;
            if (!set) {
                e = set_kernel_smem(reinterpret_cast<const void*>(gemv_row_kernel<1>), 227 * 1024);
                if (e != cudaSuccess) return static_cast<int>(e);
                set = true;
            }
            e = cudaLaunchKernelEx(&cfg, gemv_row_kernel<1>, a);
        } else {
            static bool set = false;
            if (!set) {
                e = set_kernel_smem(reinterpret_cast<const void*>(gemv_row_kernel<0>), 227 * 1024);
                if (e != cudaSuccess) return static_cast<int>(e);
                set = true;
            }
            e = cudaLaunchKernelEx(&cfg, gemv_row_kernel<0>, a);
        }
        if (e != cudaSuccess) return static_cast<int>(e);
    }
    return 0;
}

}  // namespace rq4
