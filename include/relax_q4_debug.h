/* relax_q4_debug.h -- diagnostics, not part of the operator boundary.
 * Exported only by the experiments build (build_exp/librelax_q4_exp.so,
 * `python -m paper_2311_02103_b200.build --experiments`), never by the
 * product library.
 *
 * With RELAX_Q4_TRACE=1 in the environment, every streamed-GEMV CTA records
 * {launch seq, cta, smid, t_start, t_after_griddepcontrol_wait,
 *  t_first_stage_ready, t_end} (globaltimer ns) into a device ring.
 * relax_debug_trace_read copies up to max_records 48-byte records to host
 * memory, reports how many, and optionally resets the ring.  Synchronous. */
#ifndef RELAX_Q4_DEBUG_H
#define RELAX_Q4_DEBUG_H
#include <stddef.h>
#include "relax_q4.h"
#ifdef __cplusplus
extern "C" {
#endif
RELAX_API int relax_debug_trace_read(void* host, size_t max_records, size_t* n_records, int reset);
/* Tensor-core kernel: per-CTA {cta, smid, nsub, pad, t0, t_end (ns), wait
 * cycles of: W producer, x producer, x permuter, transform (W data), transform
 * (A slot), MMA (A ready), MMA (x ready), epilogue} -- 96-byte records. */
RELAX_API int relax_debug_tctrace_read(void* host, size_t max_records, size_t* n_records, int reset);
/* Decode-chain timeline: per (CTA, op) 7 globaltimer stamps (ns). */
RELAX_API int relax_debug_chain_trace_read(void* host, size_t bytes);

/* ---- Decode chain (experiments build only: measured slower than the PDL chain
 * of relax_q4_matmul calls): a whole step's GEMVs (n = 1) in
 * one persistent launch
 *
 * ops[0..count) are matmuls y_m[1][N_m] = x_m[1][K_m] . dequant(W_m), in
 * order, exactly as `count` relax_q4_matmul calls with n = 1 on one stream --
 * an op's x may be an earlier op's y.  One launch runs them all: each SM
 * streams its rows of op after op without waiting for activations (weights
 * do not depend on them), and an op flagged `after` waits until every earlier
 * op has completed before it reads x.  Ops that read the same
 * x as the op before them (q, k, v; gate, up) need no `after`.
 * Set-up once: relax_q4_chain_workspace gives the bytes, relax_q4_chain_init
 * validates the ops and writes the device-side op table and counters into the
 * workspace (synchronous; the pointers are captured, not the data);
 * relax_q4_chain_run then launches the chain (asynchronous, CUDA-graph
 * capturable) as often as wanted, on the device the workspace was set up on.
 * Per op: K % 256 == 0, K <= 30720, N < 2^30, 16-B aligned pointers, y not
 * overlapping the op's x or weights.  Same arithmetic as the decode kernel
 * (within the tolerance of relax_q4_matmul; r == 0 => y == +-0). */
typedef struct relax_q4_chain_op {
    const void* x;                      /* fp16 [K] (device) */
    const uint32_t* packed_w;           /* [N][K/8] */
    const void* scales;                 /* fp16 [N][K/32] */
    void* y;                            /* fp16 [N] */
    int64_t K, N;
    int32_t after;                      /* 1: wait for every earlier op before reading x */
    int32_t reserved;                   /* 0 */
} relax_q4_chain_op;

/* Errors: RELAX_ERR_INVALID_ARG (ws_bytes NULL, count outside 1..1024). */
RELAX_API int relax_q4_chain_workspace(int count, size_t* ws_bytes);
/* Errors: RELAX_ERR_INVALID_ARG (NULL op pointer, count outside 1..1024, reserved != 0,
 * K or N <= 0), RELAX_ERR_UNSUPPORTED_SHAPE (an op the chain kernel cannot
 * hold), RELAX_ERR_MISALIGNED, RELAX_ERR_ALIAS (y over the op's x or
 * weights), RELAX_ERR_WORKSPACE (ws_bytes too small), RELAX_ERR_DEVICE,
 * RELAX_ERR_CUDA. */
RELAX_API int relax_q4_chain_init(const relax_q4_chain_op* ops, int count, void* ws, size_t ws_bytes);
/* Errors: RELAX_ERR_INVALID_ARG (ws NULL), RELAX_ERR_DEVICE, RELAX_ERR_CUDA. */
RELAX_API int relax_q4_chain_run(void* ws, void* stream);


#ifdef __cplusplus
}
#endif
#endif
