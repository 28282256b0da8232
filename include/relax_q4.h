/*
 * relax_q4.h -- C-ABI of the B200-native fused q4f16 dequantize+matmul.
 *
 * The operation (PAPER.md = /root/reference/PAPER.md, arXiv 2311.02103):
 *
 *     y[n, N] = x[n, K] . dequant(Wq[K, N])
 *
 * with "4-bit integer (int4) weight quantization and float16 activations"
 * (P:640), the dequantize step fused into the matmul as one tensor program
 * (FuseOps / FuseTensorIR), n a symbolic token count passed at run
 * time while K and N are static per call site (call_tir "specializes to most
 * static dimensions and only uses dynamic dimensions when necessary (like
 * dimension n)"), called in destination-passing style -- the
 * caller passes input and output memory explicitly (P:394-396,
 * call_dps_library P:415-416) -- with any temporary workspace lifted out of
 * the kernel into caller-planned memory sized from the upper
 * bound of n.
 *
 * Storage format (the paper names int4 only; DESIGN.md §3 readings 1-4):
 *   packed_w  uint32 [N][K/8]   8 unsigned 4-bit codes per word, element k at
 *                               bits 4*(k mod 8) of word k/8 (low nibble first)
 *   scales    fp16   [N][K/32]  one scale per 32 consecutive k
 *   W(k, j) = fp16_RNE((q(k,j) - 7) * scales[j][k/32])      (zero point 7)
 *   x         fp16   [n][K]     row-major
 *   y         fp16   [n][N]     row-major; fp32 accumulation, one RNE rounding
 * Every array is dense, IEEE binary16 where fp16, little-endian.
 *
 * Conventions shared by every entry point:
 *   - Returns an int status (RELAX_OK == 0, codes below); never throws,
 *     never aborts, never prints.
 *   - All pointers except those named "host" are DEVICE pointers owned by
 *     the caller; the library keeps none of them after return.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *     stream).  Work is enqueued asynchronously; the library never
 *     synchronises the host, never allocates or frees device memory, so
 *     every call can be captured into a CUDA graph.
 *   - Inputs are never modified (DPS "inputs unmodified").
 *   - Argument validation is O(1) and happens before any CUDA call; on any
 *     error nothing is launched and y is untouched ("never a wrong answer",
 *     S:629).
 *   - Kernels are compiled for sm_100a (B200) only.
 *   - Reentrant and thread-safe.  The only global state is per device and
 *     initialised once, under std::call_once / a mutex: the SM count every
 *     schedule is planned with, and the kernels' function attributes (set on
 *     each device the process uses).  Tensor maps of the operands are cached
 *     per host thread (keyed by everything they encode), so steady-state
 *     host dispatch is a few hash probes, not a driver encode.
 *   - "Host only" planning calls (relax_plan_workspace*, relax_query_schedule)
 *     launch nothing; they read the current device's SM count when a device
 *     is visible (the plan then matches what a call on that device does) and
 *     assume a B200's 148 SMs otherwise.
 *   - The library reads no environment variable (experiment knobs exist only
 *     in the separate experiments build).
 */
#ifndef RELAX_Q4_H
#define RELAX_Q4_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define RELAX_API __attribute__((visibility("default")))
#else
#define RELAX_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

enum relax_status {
    RELAX_OK = 0,
    RELAX_ERR_INVALID_ARG = 1,       /* NULL pointer with work to do, n < 0, K <= 0, N <= 0 */
    RELAX_ERR_UNSUPPORTED_SHAPE = 2, /* K not a multiple of 32, or a forced variant that cannot run it */
    RELAX_ERR_MISALIGNED = 3,        /* a pointer is not 16-byte aligned */
    RELAX_ERR_ALIAS = 4,             /* y (or w_out) overlaps an input or the workspace */
    RELAX_ERR_WORKSPACE = 5,         /* ws_bytes smaller than the chosen schedule needs */
    RELAX_ERR_DEVICE = 6,            /* no CUDA device, or current device is not sm_100 */
    RELAX_ERR_CUDA = 7               /* a CUDA runtime call or launch failed */
};

/* Variants (the dispatch decision on n, "partial lowering" made at
 * run time).  RELAX_VARIANT_AUTO lets the library choose. */
enum relax_variant {
    RELAX_VARIANT_AUTO = 0,
    RELAX_VARIANT_GEMV = 1,   /* CUDA-core split-free GEMV, 128-bit loads, warp-shuffle reduce */
    RELAX_VARIANT_TC = 2,     /* TMA + tcgen05/TMEM GEMM with in-kernel dequant (K % 256 == 0) */
    RELAX_VARIANT_SMALLN = 3  /* small batches: streamed warp-MMA (mma.sync) GEMV, 8 tokens per
                                 launch, no workspace (K % 256 == 0) */
};

/* Flags for relax_q4_matmul_ex. */
#define RELAX_FLAG_NO_PDL 1u            /* launch without programmatic dependent launch */
#define RELAX_FLAG_SPLIT_WORKSPACE 2u   /* TC split-K through the workspace, not a cluster */
#define RELAX_FLAG_TILE_PER_CTA 4u      /* TC: one tile per CTA, never the persistent
                                           double-buffered-accumulator kernel */

/* Upper-bound workspace plan (lifted workspace P:438-441).
 * Host only, pure: no launch, no allocation.
 *   n_max     largest token count the caller will pass (>= 0)
 *   K, N      static shape of the weight
 *   ws_bytes  out: max over n in [1, n_max] of the bytes the automatic
 *             schedule of relax_q4_matmul_ws needs (0 when no n needs one)
 * Guarantee: every relax_q4_matmul_ws call with n <= n_max and a workspace of
 * at least *ws_bytes bytes succeeds (never RELAX_ERR_WORKSPACE).
 * The workspace must be zero-filled before its first use; every call leaves
 * it zero-filled again (its split-K tickets reset themselves), so one buffer
 * serves any number of sequential calls.  Calls that may run concurrently
 * need separate workspaces.
 * Errors: RELAX_ERR_INVALID_ARG (ws_bytes NULL, n_max < 0, K <= 0, N <= 0),
 *         RELAX_ERR_UNSUPPORTED_SHAPE (K % 32 != 0). */
RELAX_API int relax_plan_workspace(int64_t n_max, int64_t K, int64_t N, size_t* ws_bytes);

/* y = x . dequant(packed_w, scales), no workspace (schedules that need one
 * are replaced by workspace-free ones).  n == 0 is a no-op (RELAX_OK).
 *   x         device fp16 [n][K]
 *   n         runtime token count (>= 0)
 *   K, N      K % 32 == 0
 *   packed_w  device uint32 [N][K/8];  scales device fp16 [N][K/32]
 *   y         device fp16 [n][N] (output; must not overlap any input)
 *   stream    cudaStream_t or NULL */
RELAX_API int relax_q4_matmul(const void* x, int64_t n, int64_t K, int64_t N,
                    const uint32_t* packed_w, const void* scales, void* y, void* stream);

/* As relax_q4_matmul, plus a caller-provided device workspace (DPS: the
 * lifted workspace is an extra output-position argument).
 *   workspace  device memory of ws_bytes bytes, 16-byte aligned, zero-filled
 *              before first use (see relax_plan_workspace); may be NULL when
 *              ws_bytes == 0. */
RELAX_API int relax_q4_matmul_ws(const void* x, int64_t n, int64_t K, int64_t N,
                       const uint32_t* packed_w, const void* scales, void* y,
                       void* workspace, size_t ws_bytes, void* stream);

/* Grouped form: `count` (1..4) linears that read the SAME x (q, k and v of a
 * layer; gate and up), each with its own weights and output:
 *   y[i] = x . dequant(packed_w[i], scales[i]),  y[i] fp16 [n][N[i]].
 * `N`, `packed_w`, `scales`, `y` are HOST arrays of `count` entries (read
 * during the call only) holding device pointers.  For decode (n <= 2) the
 * members run as ONE launch of the streamed decode kernel, its CTAs split
 * among them in proportion to N[i] -- one dependent step of the stream
 * instead of `count` (horizontal fusion of independent operators); small
 * batches (3 <= n <= 8, K % 256 == 0, K <= 16384, sum N[i] >= 2048) run as
 * ONE launch of the small-batch kernel the same way; other n run member by
 * member through relax_q4_matmul.  Results equal `count`
 * separate relax_q4_matmul calls within the tolerance (bitwise for the
 * pinned cases).  No workspace.  Errors as relax_q4_matmul, plus
 * RELAX_ERR_INVALID_ARG for count outside 1..4 and RELAX_ERR_ALIAS when an
 * output overlaps x, any weight, or another output. */
RELAX_API int relax_q4_matmul_grouped(const void* x, int64_t n, int64_t K, int count, const int64_t* N,
                                      const uint32_t* const* packed_w, const void* const* scales,
                                      void* const* y, void* stream);

/* ---- Tensor-parallel row split with the all-reduce fused
 *
 * The row-split (K-split) linears of Megatron TP -- o and down of a Llama
 * block -- end in a sum over the ranks.  The paper fuses a consumer into its
 * producer's kernel so that intermediate results never make a round trip
 * through memory (§3.5 FuseOps / FuseTensorIR: "reduce the overall
 * memory loading cost"); here the consumer is that sum, and it runs
 * in the decode kernel's epilogue over NVLink peer memory instead of a
 * separate NCCL all-reduce.  Each CTA stores the fp32 partial of its output
 * rows (x_r . W_r over this rank's K slice) into every other rank's exchange
 * buffer as 8-byte (epoch, value) words, waits until the same rows' words of
 * every other rank carry the call's epoch, and sums the partials in rank
 * order 0..world-1 (fp32, one fp16 rounding -- DESIGN.md §3 reading 14), so
 * every rank ends with the same y bit for bit:
 *   y[n, N] = fp16( sum_p  x_p[n, K] . dequant(W_p)[K, N] )  (+ residual)
 *
 * relax_tp_comm: bufs[p] is rank p's exchange buffer as mapped on THIS device
 * (e.g. torch symmetric memory's buffer_ptrs), buf_bytes its size (>=
 * relax_tp_comm_bytes(world, N)).  Every buffer must be zero-filled once,
 * before the first call on any rank, and the ranks must then issue the same
 * sequence of relax_q4_matmul_allreduce calls (same N and K per call) -- the
 * per-CTA epoch counters inside the buffers pair up call e of every rank.
 * A rank that never arrives makes the kernel trap after ~10 s (a CUDA error,
 * not a hang). */
#define RELAX_TP_MAX_WORLD 8
typedef struct relax_tp_comm {
    int32_t world;                      /* ranks in the group, 1..RELAX_TP_MAX_WORLD */
    int32_t rank;                       /* this rank, 0..world-1 */
    void* bufs[RELAX_TP_MAX_WORLD];     /* device pointers valid on this device; 16-B aligned */
    size_t buf_bytes;                   /* bytes of every rank's buffer */
} relax_tp_comm;

/* Exchange-buffer bytes per rank for outputs of up to N_max features.
 * Errors: RELAX_ERR_INVALID_ARG (bytes NULL, world outside 1..8, N_max <= 0). */
RELAX_API int relax_tp_comm_bytes(int32_t world, int64_t N_max, size_t* bytes);

/* y[n,N] = fp16(sum over ranks of x_r . W_r) (+ residual[n,N] when residual is
 * non-NULL; it may equal y), for this rank's K slice: x fp16 [n][K], packed_w
 * [N][K/8], scales [N][K/32] (the plain layout of relax_q4_matmul, K = this
 * rank's slice).  n <= 2 (decode; larger n: relax_q4_matmul + an NCCL
 * all-reduce), K % 256 == 0.  Asynchronous on `stream`; CUDA-graph capturable.
 * Errors: RELAX_ERR_INVALID_ARG (comm NULL, world/rank out of range, a NULL
 * buffer, n < 0, K <= 0, N <= 0), RELAX_ERR_WORKSPACE (buf_bytes too small),
 * RELAX_ERR_UNSUPPORTED_SHAPE (n > 2, K % 256 != 0, a shape the decode kernel
 * cannot hold), RELAX_ERR_MISALIGNED, RELAX_ERR_ALIAS (y overlapping x, the
 * weights, this rank's buffer, or partially overlapping residual),
 * RELAX_ERR_DEVICE, RELAX_ERR_CUDA. */
RELAX_API int relax_q4_matmul_allreduce(const relax_tp_comm* comm, const void* x, int64_t n, int64_t K, int64_t N,
                                        const uint32_t* packed_w, const void* scales, const void* residual,
                                        void* y, void* stream);

/* Explicit-schedule form, for parity tests of every variant and for benches.
 *   variant   enum relax_variant (AUTO = same as relax_q4_matmul_ws)
 *   split_k   TC only: split-K factor, 0 = choose; > 1 needs a workspace
 *   bn        TC only: token tile in {16,32,64,128,256}, 0 = choose
 *   flags     RELAX_FLAG_* bits
 * Errors as relax_q4_matmul_ws, plus RELAX_ERR_UNSUPPORTED_SHAPE when the
 * forced variant cannot run this shape (TC needs K % 256 == 0). */
RELAX_API int relax_q4_matmul_ex(const void* x, int64_t n, int64_t K, int64_t N,
                       const uint32_t* packed_w, const void* scales, void* y,
                       void* workspace, size_t ws_bytes, int variant, int split_k,
                       int bn, unsigned flags, void* stream);

/* ---------------------------------------------------------------------------
 * Fused neighbours: the dequant-matmul with the element-wise
 * operators of a Llama decoder block fused into it, the way FuseOps /
 * FuseTensorIR fold element-wise producers and consumers into the tensor
 * program of the matmul ("absorb ... downstream ElementWise",
 * SPEC S:472).  Fusion preserves the semantics of the unfused fp16 program
 * (P:483-494), so each operator is defined exactly as the unfused kernel
 * chain computes it, fp16 at every tensor boundary (DESIGN.md §3 readings
 * 16-18):
 *
 *   RELAX_OP_RMSNORM_X  (prologue on x, Llama RMSNorm)
 *       r_t     = 1 / sqrt(mean_k x[t][k]^2 + eps)          (fp32)
 *       xn[t,k] = fp16_RNE(fp16_RNE(x[t][k] * r_t) * gamma[k])
 *       and the matmul consumes xn instead of x.
 *   RELAX_OP_SILU_MUL   (epilogue, SwiGLU): the weight rows are interleaved
 *       pairs -- row 2j is gate_j, row 2j+1 is up_j (a one-time repack of the
 *       two matrices, F3) -- and with g = fp16_RNE(acc[2j]), u = fp16_RNE(acc[2j+1])
 *       y[t][j] = fp16_RNE(silu(g) * u),  silu(g) = g / (1 + exp(-g))  (fp32)
 *       so y has N/2 columns.
 *   RELAX_OP_RESIDUAL   (epilogue, residual add), applied last:
 *       y[t][j] = fp16_RNE(v + residual[t][j]),  v = the fp16 output so far.
 *   RELAX_OP_KV_APPEND  (epilogue of the fused q/k/v projection at decode, the
 *       consumer relax_kv_append fused into its producer): y is
 *       written as usual and, in addition, its rows kv_row0 + h*128 + d
 *       (h < kv_heads: the new token's keys) and kv_row0 + (kv_heads + h)*128
 *       + d (its values) are stored at k_cache / v_cache[t][h][kv_pos[t]][d]
 *       for token t (= sequence t; caches as relax_attn_decode; positions
 *       outside [0, kv_len_max) store nothing).  Decode only: n <= 2 and a
 *       shape the streamed decode kernel holds (else RELAX_ERR_UNSUPPORTED_SHAPE);
 *       not with SILU_MUL.
 *
 * Combinations are allowed; the order is prologue, matmul, SiLU-mul, residual,
 * KV append.
 */
#define RELAX_OP_RMSNORM_X 1u
#define RELAX_OP_SILU_MUL 2u
#define RELAX_OP_RESIDUAL 4u
#define RELAX_OP_KV_APPEND 8u

typedef struct relax_q4_fusion {
    uint32_t ops;             /* RELAX_OP_* bitmask (0 = plain matmul) */
    float rms_eps;            /* RMSNORM_X: epsilon (>= 0, finite) */
    const void* rms_weight;   /* RMSNORM_X: device fp16 [K] (gamma), 16-byte aligned; a model
                                 parameter: like packed_w/scales it may be read before the
                                 kernel waits on the previous kernel of the stream (PDL) */
    const void* residual;     /* RESIDUAL: device fp16 [n][N_out], 16-byte aligned; may be
                                 exactly y (in-place add) but not partially overlap it */
    /* KV_APPEND (ignored otherwise; zero them) */
    void* k_cache;            /* device fp16 [n][kv_heads][kv_len_max][128], 16-byte aligned */
    void* v_cache;            /* likewise */
    const int32_t* kv_pos;    /* device int32 [n]: the position written for each token */
    int64_t kv_len_max;
    int32_t kv_heads;
    int32_t kv_row0;          /* first key row of y; kv_row0 + 2*kv_heads*128 <= N */
} relax_q4_fusion;

/* Workspace plan of relax_q4_matmul_fused for n <= n_max: the plain plan plus
 * n_max*K*2 bytes for the normalised x when RMSNORM_X is requested and some
 * n <= n_max takes the tensor-core path (the decode GEMV normalises in
 * registers).  The normalised x is written at an offset past the split-K
 * ticket region (>= 4096 B), so a fused workspace may also serve
 * relax_q4_matmul_ex calls with RELAX_FLAG_SPLIT_WORKSPACE.  Same guarantee
 * and zero-fill contract as relax_plan_workspace (the ticket region is left
 * zero; the normalised-x region is scratch).
 * Errors: as relax_plan_workspace, plus RELAX_ERR_INVALID_ARG for unknown ops
 * bits and RELAX_ERR_UNSUPPORTED_SHAPE when ops != 0 and K % 256 != 0 or
 * (SILU_MUL) N is odd. */
RELAX_API int relax_plan_workspace_fused(int64_t n_max, int64_t K, int64_t N, uint32_t ops,
                                         size_t* ws_bytes);

/* y = ops(x, W): the fused form above; with fusion == NULL or ops == 0 it is
 * relax_q4_matmul_ws.
 *   y         device fp16 [n][N_out], N_out = N/2 with SILU_MUL, else N
 *   fusion    host pointer to the descriptor (read during the call only)
 * Errors: as relax_q4_matmul_ws, plus RELAX_ERR_INVALID_ARG (unknown ops bits,
 * missing rms_weight/residual, eps < 0 or not finite), RELAX_ERR_MISALIGNED,
 * RELAX_ERR_ALIAS (residual partially overlapping y, or y overlapping x,
 * gamma, weights), RELAX_ERR_UNSUPPORTED_SHAPE (ops != 0 needs K % 256 == 0;
 * SILU_MUL needs N even). */
RELAX_API int relax_q4_matmul_fused(const void* x, int64_t n, int64_t K, int64_t N,
                                    const uint32_t* packed_w, const void* scales, void* y,
                                    const relax_q4_fusion* fusion, void* workspace,
                                    size_t ws_bytes, void* stream);

/* Host-only report of the schedule relax_q4_matmul_ws would use for (n,K,N):
 * out pointers may be NULL.  variant: enum relax_variant; tile: GEMV / SMALLN
 * tokens per launch or TC token tile; split_k: TC split factor; ws_bytes:
 * bytes needed; persistent: 1 when the TC schedule is the persistent
 * double-buffered-accumulator kernel, 2 for its stream-K schedule (the k
 * ranges of the tiles spread evenly over the CTA pairs, cut tiles reduced
 * through the workspace; experiments build only, and only when the caller's
 * workspace holds it, else the call falls back to another schedule), 3 for
 * the two-part schedule (the full waves of whole 256-token tiles over the
 * leading output rows, the remaining rows in a second launch as split-K
 * clusters; no workspace), 4 for the same with the leading rows on the
 * persistent kernel.
 * Errors: RELAX_ERR_INVALID_ARG, RELAX_ERR_UNSUPPORTED_SHAPE. */
RELAX_API int relax_query_schedule(int64_t n, int64_t K, int64_t N, int* variant, int* tile,
                         int* split_k, size_t* ws_bytes, int* persistent);

/* Bit-exact dequant export: w_out[j][k] = fp16_RNE((q(k,j) - 7) * s), the
 * producer half of the fused op on its own (used to pin the in-kernel
 * dequant).
 *   w_out   device fp16 [N][K] (output; must not overlap the inputs)
 * Errors: as relax_q4_matmul (N == 0 is a no-op). */
RELAX_API int relax_q4_dequant(const uint32_t* packed_w, const void* scales, int64_t K, int64_t N,
                     void* w_out, void* stream);

/* ---------------------------------------------------------------------------
 * Format variants: "lift out quantization and layout
 * transforms in tensor programs to enable pre-computation".  A
 * weight stored in another layout or group size is converted ONCE into the
 * native format above; the converted weight dequantizes to the same W bit for
 * bit (codes move unchanged; every 32-group takes the scale of the G-group
 * that contains it).  Source formats (DESIGN.md §3 readings 19-20):
 *   RELAX_LAYOUT_NK  src_packed uint32 [N][K/8], src_scales fp16 [N][K/G]
 *   RELAX_LAYOUT_KN  src_packed uint32 [K/8][N] (word (k/8, j) holds codes
 *                    k..k+7 of output column j, low nibble first -- the
 *                    per-column packing of GPTQ-style checkpoints),
 *                    src_scales fp16 [K/G][N]
 *   RELAX_LAYOUT_NK3 3-bit codes ("3-bit" Llama-2-7B on the iPhone;
 *                    DESIGN.md reading 20): src_packed uint32 [N][3 K/32],
 *                    the 32 codes of group g of column j at bits 3 i .. 3 i + 2
 *                    of words 3 g .. 3 g + 2 (96 bits, little-endian), zero
 *                    point 3: W(k, j) = fp16_RNE((q3 - 3) * s(k/G, j)); stored
 *                    natively as q4 = q3 + 4 (bit-exact, 4.5 instead of 3.5
 *                    bits per weight in HBM);
 *                    src_scales fp16 [N][K/G]
 *   group G in {32, 64, 128}; W(k, j) = fp16_RNE((q - 7) * s(k/G, j)).
 * Outputs: packed_w uint32 [N][K/8], scales fp16 [N][K/32] (device, caller-
 * owned, must not overlap the inputs).  Asynchronous on `stream`.
 * Errors: RELAX_ERR_INVALID_ARG (unknown layout, NULL, K <= 0, N < 0),
 * RELAX_ERR_UNSUPPORTED_SHAPE (G not in {32, 64, 128} or K % G != 0),
 * RELAX_ERR_MISALIGNED, RELAX_ERR_ALIAS, RELAX_ERR_DEVICE, RELAX_ERR_CUDA.
 * N == 0 is a no-op. */
#define RELAX_LAYOUT_NK 0
#define RELAX_LAYOUT_KN 1
#define RELAX_LAYOUT_NK3 2
RELAX_API int relax_q4_repack(const uint32_t* src_packed, const void* src_scales, int64_t K, int64_t N,
                              int layout, int group, uint32_t* packed_w, void* scales, void* stream);

/* ---------------------------------------------------------------------------
 * Decode attention over a symbolic KV length ("the KV-cache
 * context length" as a dynamic dimension; single-batch decode):
 * the other operator of a decode step, so the whole step runs on this library
 * (bench.py --block fused --kv L).  One query token per sequence, DESIGN.md
 * reading 21:
 *   q        device fp16 [batch][n_heads][head_dim]
 *   k_cache, v_cache  device fp16 [batch][n_kv_heads][kv_len_max][head_dim]
 *   kv_lens  device int32 [batch], 0 <= kv_lens[b] <= kv_len_max: the keys
 *            j < kv_lens[b] of sequence b are attended (the symbolic length;
 *            values outside the range are the caller's error and are clamped
 *            by nothing -- keep them in range)
 *   out      device fp16 [batch][n_heads][head_dim]
 *   s_j = (q . k_j) / sqrt(head_dim), out = softmax(s) . V in fp32, fp16 RNE;
 *   query head h uses kv head h / (n_heads / n_kv_heads) (grouped-query
 *   attention); a sequence with kv_lens[b] == 0 gets out = 0.
 * head_dim must be 128, n_heads / n_kv_heads one of 1, 2, 4, 8, kv_len_max <= 65536.
 * Split over 256-key chunks (flash decoding); the fp32 partials live in a
 * caller-owned workspace of relax_attn_decode_workspace(batch, n_heads,
 * kv_len_max) bytes (no zero-fill needed).  Deterministic.
 * Errors: RELAX_ERR_INVALID_ARG, RELAX_ERR_UNSUPPORTED_SHAPE, RELAX_ERR_MISALIGNED,
 * RELAX_ERR_ALIAS, RELAX_ERR_WORKSPACE, RELAX_ERR_DEVICE, RELAX_ERR_CUDA.
 * relax_kv_append writes k_new, v_new [batch][n_kv_heads][head_dim] at
 * position pos[b] of each sequence's cache (positions outside
 * [0, kv_len_max) write nothing). */
RELAX_API int relax_attn_decode_workspace(int64_t batch, int64_t n_heads, int64_t kv_len_max, size_t* ws_bytes);
RELAX_API int relax_attn_decode(const void* q, const void* k_cache, const void* v_cache, const int32_t* kv_lens,
                                int64_t batch, int64_t n_heads, int64_t n_kv_heads, int64_t head_dim,
                                int64_t kv_len_max, void* out, void* workspace, size_t ws_bytes, void* stream);
RELAX_API int relax_kv_append(const void* k_new, const void* v_new, const int32_t* pos, int64_t batch,
                              int64_t n_kv_heads, int64_t head_dim, int64_t kv_len_max, void* k_cache,
                              void* v_cache, void* stream);

/* Static description of a status code; never NULL. */
RELAX_API const char* relax_status_str(int status);

/* Library version string, e.g. "relax_q4 0.1 sm_100a". */
RELAX_API const char* relax_version(void);

#ifdef __cplusplus
}
#endif

#endif /* RELAX_Q4_H */
