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
#ifdef __cplusplus
}
#endif
#endif
