// internal.h -- host-side declarations shared by the C-ABI (abi.cpp) and the
// kernel translation units.  Not part of the public boundary (include/).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace rq4 {

constexpr int kGroup = 32;          // codes per fp16 scale (reading 2)
constexpr int kB200SMs = 148;       // B200: the SM count the measured tables were taken on

// SM count of the current device, read once per device (std::call_once) and
// cached; kB200SMs when no device is visible (host-only planning).  Every
// schedule decision (grids, split-K, cluster waves) is planned with it.
int num_sms();
// cudaGetDevice, or -1 without a device.
int current_device();
constexpr int kGemvMaxNT = 8;       // tokens per GEMV launch
constexpr int kTcBM = 128;          // tcgen05 tile: weight rows (MMA M)
constexpr int kTcWStageK = 256;     // k per weight (codes+scales) TMA stage
constexpr int kTcXStageK = 64;      // k per x TMA stage / A sub-block (4 MMAs)
constexpr size_t kTicketBytes = 4096;  // split-K tickets: fixed region at workspace offset 0
constexpr int64_t kMaxSplitTiles = kTicketBytes / 4;
constexpr int kMaxClusterSplit = 16;   // non-portable cluster size limit on sm_100

// Per-kernel attributes set once before the first launch: the dynamic
// shared-memory limit, and the maximum shared-memory carveout.  A fixed
// carveout matters under programmatic dependent launch: an SM whose carveout
// was sized for one kernel cannot take a CTA of the next kernel that needs a
// different split until it drains, which serialised the chain and let the
// next kernel pack two CTAs onto half the SMs.
inline cudaError_t set_kernel_smem(const void* fn, int dyn_bytes) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_bytes);
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout,
                                static_cast<int>(cudaSharedmemCarveoutMaxShared));
}
// set_kernel_smem (plus, with `cluster`, the non-portable cluster-size
// attribute) once per (device, kernel): function attributes are per device,
// so a process driving several GPUs sets them on each.  Thread-safe; the
// steady-state cost is one uncontended lock and a hash lookup.
cudaError_t ensure_kernel_attrs(const void* fn, int dyn_bytes, bool cluster = false);

// Tensor-parallel row split with the all-reduce fused into the decode
// kernel's epilogue (relax_q4_matmul_allreduce).  Each rank's
// exchange buffer: [epoch counters: kTpMaxCta u32][words: 2 parities x world
// x 2 tokens x N u64], a word = (epoch << 32) | fp32 bits of one partial.
constexpr int kTpMaxWorld = 8;
constexpr int kTpMaxCta = 1024;
constexpr size_t kTpHdrBytes = static_cast<size_t>(kTpMaxCta) * 4;
constexpr uint32_t kOpTpAllReduce = 1u << 31;     // internal Fusion bit (never in the public ops)
struct TpComm {
    int world = 0;
    int rank = 0;
    uint8_t* bufs[kTpMaxWorld] = {};
};
inline size_t tp_comm_bytes(int world, int64_t N) {
    return kTpHdrBytes + static_cast<size_t>(2) * world * 2 * static_cast<size_t>(N) * 8;
}

// Fused neighbours of one call (include/relax_q4.h RELAX_OP_*); ops == 0: none.
struct Fusion {
    uint32_t ops = 0;
    float eps = 0.f;
    const uint16_t* gamma = nullptr;   // RMSNORM_X, fp16 [K]
    const uint16_t* res = nullptr;     // RESIDUAL, fp16 [n][N_out]
    const TpComm* tp = nullptr;        // kOpTpAllReduce: the exchange buffers
    uint16_t* kc = nullptr;            // KV_APPEND: caches [n][H][Lmax][128], positions, shape
    uint16_t* vc = nullptr;
    const int32_t* kv_pos = nullptr;
    int64_t kv_lmax = 0;
    int kv_heads = 0, kv_row0 = 0;
};

enum Variant : int { kVariantAuto = 0, kVariantGemv = 1, kVariantTc = 2, kVariantSmallN = 3 };

struct Plan {
    int variant = 0;
    int nt = 0;          // GEMV: tokens per launch
    int bn = 0;          // TC: token tile (MMA N)
    int split = 1;       // TC: split-K factor
    int cluster = 0;     // TC: split-K reduced in a thread-block cluster (DSMEM), no workspace
    int persist = 0;     // TC: persistent kernel, double-buffered accumulator (BN = 128 / 256, no split);
                         // 2 = its stream-K schedule (k ranges split over clusters, workspace reduction)
    int64_t rows_a = 0;  // TC two-part schedule (> 0): rows [0, rows_a) as whole 256-token tiles, the
    int split_b = 1;     // rest rows [rows_a, N) in a second launch with split-K split_b (cluster)
    int persist_a = 0;   // two-part: the leading rows on the persistent kernel (1) or as one tile per CTA (0)
    int grid = 0;
    size_t ws_bytes = 0; // workspace bytes this plan needs
};

// Host-pure dispatch (a1): variant, tiles, split-K and workspace for (n,K,N).
// `force_variant` / `force_split` / `force_bn` override (0 = choose).
int make_plan(int64_t n, int64_t K, int64_t N, int force_variant, int force_split,
              int force_bn, Plan* out, bool force_ws, bool no_persist = false, bool allow_sk = true);
size_t tc_workspace_bytes(int64_t n, int64_t N, int bn, int split);
int gemv_max_n();                   // GEMV/TC threshold (env RELAX_Q4_GEMV_MAX_N)
bool gemv_fits(int nt, int64_t K);

// Launchers (return cudaError_t as int).  All asynchronous on `stream`.
int launch_dequant(const uint32_t* w, const uint16_t* s, int64_t K, int64_t N,
                   uint16_t* out, cudaStream_t stream);
int launch_gemv(const uint16_t* x, int64_t n, int64_t K, int64_t N, const uint32_t* w,
                const uint16_t* s, uint16_t* y, int nt, bool pdl, cudaStream_t stream);
int launch_gemv_stream(const uint16_t* x, int64_t n, int64_t K, int64_t N, const uint32_t* w,
                       const uint16_t* s, uint16_t* y, bool pdl, cudaStream_t stream,
                       const Fusion& fu = Fusion());
// Whether the streamed decode kernel can run nt (1, 2) tokens of this shape
// (K % 256 == 0, N < 2^24, its shared-memory footprint within the attribute);
// pair = 2 with the SiLU-mul epilogue (CTAs own whole (gate, up) row pairs).
bool gemv_stream_ok(int nt, int64_t K, int64_t N, int pair = 1);
// CTAs of the decode kernel for this shape (the fused all-reduce keys its
// epoch counters by CTA, so the grid must be <= kTpMaxCta and co-resident).
int gemv_stream_grid(int64_t K, int64_t N);
// Grouped decode launch: up to 4 matrices sharing x and K in one kernel.
bool gemv_stream_grouped_ok(int64_t n, int64_t K, int count, const int64_t* N);
int launch_gemv_stream_grouped(const uint16_t* x, int64_t n, int64_t K, int count, const int64_t* N,
                               const uint32_t* const* w, const uint16_t* const* s, uint16_t* const* y, bool pdl,
                               cudaStream_t stream);
// Small-batch warp-MMA streamed kernel (smalln_mma.cu): any n (8 tokens per
// launch), K % 256 == 0.
bool smalln_mma_ok(int64_t n, int64_t K, int64_t N);
int launch_smalln_mma(const uint16_t* x, int64_t n, int64_t K, int64_t N, const uint32_t* w,
                      const uint16_t* s, uint16_t* y, bool pdl, cudaStream_t stream);
int smalln_max_n();                 // largest n the automatic dispatch sends to it
// Grouped small-batch launch: up to 4 matrices sharing x and K in one kernel
// per 8 tokens (CTAs split in proportion to the matrices' 16-row blocks).
bool smalln_mma_grouped_ok(int64_t n, int64_t K, int count, const int64_t* N);
int launch_smalln_mma_grouped(const uint16_t* x, int64_t n, int64_t K, int count, const int64_t* N,
                              const uint32_t* const* w, const uint16_t* const* s, uint16_t* const* y, bool pdl,
                              cudaStream_t stream);
#ifdef RQ4_EXPERIMENTS
// A chain of n = 1 GEMVs in one persistent launch (experiments/csrc/decode_chain.cu).
struct ChainOpHost {
    const uint16_t* x;
    const uint32_t* w;
    const uint16_t* s;
    uint16_t* y;
    int64_t K, N;
    int after;          // wait for every earlier op before reading x
};
bool chain_op_ok(int64_t K, int64_t N);
int chain_max_ops();
size_t chain_workspace_bytes(int count);
int chain_init(const ChainOpHost* ops, int count, void* ws);     // synchronous (writes the op table)
int launch_chain(void* ws, bool pdl, cudaStream_t stream);
#endif
// Decode attention over a symbolic KV length and the KV append (attention.cu).
size_t attn_workspace_bytes(int64_t batch, int64_t Hq, int64_t Lmax);
int launch_attention_decode(const uint16_t* q, const uint16_t* k, const uint16_t* v, const int32_t* lens,
                            int64_t batch, int64_t Hq, int64_t Hkv, int64_t Lmax, uint16_t* out, void* ws,
                            bool pdl, cudaStream_t st);
int launch_kv_append(const uint16_t* kn, const uint16_t* vn, const int32_t* pos, int64_t batch, int64_t Hkv,
                     int64_t Lmax, uint16_t* kc, uint16_t* vc, bool pdl, cudaStream_t st);
// One-time format conversion into the native layout (repack.cu).
int launch_repack(const uint32_t* src_w, const uint16_t* src_s, int64_t K, int64_t N, int layout, int group,
                  uint32_t* w, uint16_t* s, cudaStream_t stream);
// RMSNorm of fp16 rows into `out` (the TC path's RMSNORM_X prologue; the
// decode GEMV normalises in registers instead).
int launch_rmsnorm(const uint16_t* x, int64_t n, int64_t K, const uint16_t* gamma, float eps,
                   uint16_t* out, bool pdl, cudaStream_t stream);
#ifdef RQ4_EXPERIMENTS
// measured-slower decode variants (experiments/csrc/, experiments build only)
int launch_gemv_mma(const uint16_t* x, int64_t n, int64_t K, int64_t N, const uint32_t* w,
                    const uint16_t* s, uint16_t* y, bool pdl, cudaStream_t stream, bool bd = false);
bool gemv_mma_ok(int nt, int64_t K, int64_t N);
bool gemv_bdmma_ok(int64_t K, int64_t N);
int launch_gemv_row(const uint16_t* x, int64_t n, int64_t K, int64_t N, const uint32_t* w,
                    const uint16_t* s, uint16_t* y, bool pdl, cudaStream_t stream);
bool gemv_row_ok(int64_t K);
#endif
// 2-D tiled map, cached per host thread (gemm_tc.cu)
int make_map_2d(CUtensorMap* m, CUtensorMapDataType dt, const void* base, uint64_t inner,
                uint64_t outer, uint64_t row_bytes, uint32_t box_inner, uint32_t box_outer,
                CUtensorMapSwizzle sw);
// mode: Plan::persist (1 whole tiles, 2 stream-K reduced through `ws` --
// persist_sk_ws_bytes, its ticket region zero before and after the call)
int launch_tc_persist(const uint16_t* x, int64_t n, int64_t K, int64_t N, const uint32_t* w, const uint16_t* s,
                      uint16_t* y, int bn, int mode, void* ws, bool pdl, cudaStream_t stream, int64_t ldy = 0);
size_t persist_sk_ws_bytes(int bn);
int make_tensor_map(CUtensorMap* m, CUtensorMapDataType dt, int rank, const void* base,
                    const uint64_t* dims, const uint64_t* strides, const uint32_t* box,
                    CUtensorMapSwizzle sw);
// ldy: row stride of y for a plain matmul over a range of output rows (0: N)
int launch_tc(const uint16_t* x, int64_t n, int64_t K, int64_t N, const uint32_t* w,
              const uint16_t* s, uint16_t* y, const Plan& plan, void* ws, bool pdl,
              cudaStream_t stream,
              const Fusion& fu = Fusion(), int64_t ldy = 0);

}  // namespace rq4
