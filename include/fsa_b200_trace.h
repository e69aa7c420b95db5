/* Trace build only (python -m paper_2508_18224_b200.build --trace ->
 * libfsa_b200_trace.so, compiled with -DFSA_TRACE): development hooks that
 * are not part of the product library's ABI. */
#ifndef FSA_B200_TRACE_H
#define FSA_B200_TRACE_H

#include "fsa_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Debugging: record a per-item clock64 timeline of CTA 0 of the next launches
 * of the selected/sliding backward (K8), sliding dQ and window forward kernels
 * into a device int64 buffer (tools/trace_k8.py, trace_dq.py, trace_qo.py);
 * NULL turns it off.  Not for production use. */
void fsa_debug_bwd_trace(void* device_buf);
void fsa_debug_dq_trace(void* device_buf);
void fsa_debug_qo_trace(void* device_buf);
void fsa_debug_sel_fwd_trace(void* device_buf);
/* Debugging: TMA tile::gather4 / tile::scatter4 round trip of n rows (tools/gather4_test.py). */
int fsa_debug_gather4_test(const void* src, int64_t rows, const int32_t* idx, const int32_t* idx2,
                           int n, int box_rows, void* out, void* out2, int64_t rows2, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* FSA_B200_TRACE_H */
