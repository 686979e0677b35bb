/*
 * adaserve_debug.h -- entry points compiled ONLY into libadaserve_debug.so
 * (python -m paper_2501_12162_b200.build --debug).  Tuning instruments, not
 * part of the AdaServe method: the product library libadaserve.so exports
 * none of them.  Same conventions as adaserve.h.
 */
#ifndef ADASERVE_DEBUG_H_
#define ADASERVE_DEBUG_H_

#include "adaserve.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Debug / tuning only: every CTA of `grid` streams chunks (chunk_bytes each, in
 * the order given by `order` [n_chunks] chunk indices) of the device buffer
 * `src` through a shared-memory ring of `stages` slots.  mode 0: one thread
 * issues bulk copies (TMA engine); 1: two issuing threads; 2: 16-byte vector
 * loads by 256 threads.  `sink` [grid] receives a dummy value.  Time it with
 * events to measure achievable HBM streaming bandwidth. */
as_status as_debug_stream_bw(const void* src, const int32_t* order, int32_t n_chunks, int32_t chunk_bytes,
                             int32_t stages, int32_t mode, unsigned long long* sink, int32_t grid, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* ADASERVE_DEBUG_H_ */
