/* jsontape_b200.h — B200 additions to the jsontape C ABI (new exports only;
 * nothing in jsontape.h changes).  They expose the device-resident path the
 * reference has no equivalent for: input already in HBM, outputs left in
 * HBM, caller-chosen CUDA stream. */
#ifndef JSONTAPE_B200_H
#define JSONTAPE_B200_H

#include "jsontape.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Parser-owned device input buffer with room for `len` bytes.  The library
 * keeps >= 64 zero bytes after `len` (the reference's padded_input,
 * proj/src/indexer.h:15-36); the caller writes bytes [0, len) (cudaMemcpy or a
 * kernel) before calling a *_resident entry point.  NULL on allocation
 * failure.  Valid until the next call that changes the capacity. */
void *jt_b200_input_buffer(jt_parser *p, size_t len);

/* Fill the input buffer from host or device memory (cudaMemcpyDefault);
 * 0 on success. */
int jt_b200_copy_in(jt_parser *p, const void *src, size_t len);

/* stage 1 / full parse over the `len` bytes in jt_b200_input_buffer; results
 * stay in device memory (see the accessors below).  Same codes and offsets
 * as jt_stage1 / jt_parse. */
jt_error jt_b200_stage1_resident(jt_parser *p, size_t len, long long *error_offset);
jt_error jt_b200_parse_resident(jt_parser *p, size_t len, long long *error_offset);

/* Asynchronous variant: enqueue the full parse on the parser's stream and
 * return immediately; jt_b200_finish waits and returns the result. */
jt_error jt_b200_parse_async(jt_parser *p, size_t len);
jt_error jt_b200_finish(jt_parser *p, long long *error_offset);

/* Device views of the last results (valid until the next call). */
const uint32_t *jt_b200_device_index(const jt_parser *p, size_t *count);
const uint64_t *jt_b200_device_tape(const jt_parser *p, size_t *words);
const uint8_t *jt_b200_device_strings(const jt_parser *p, size_t *bytes);

/* Materialise the last successful resident parse as a host document. */
jt_error jt_b200_download(jt_parser *p, jt_document **out);

/* Run the parser's work on a caller stream (a cudaStream_t, e.g. torch's
 * current stream) instead of its own; NULL restores the parser's stream. */
void jt_b200_set_stream(jt_parser *p, void *cuda_stream);

/* Number of kernel launches enqueued by the last parse call. */
int jt_b200_last_launches(const jt_parser *p);

/* Per-kernel timing of full parses (events recorded on the parser's
 * stream): jt_b200_kernel_times fills ms[] for the last parse in launch
 * order init, stage1, tokens, slow, tree, struct, final; returns count. */
void jt_b200_profile(jt_parser *p, int enable);
int jt_b200_kernel_times(jt_parser *p, float *ms, int max);

/* CUDA device ordinal the parser was created on. */
int jt_b200_device(const jt_parser *p);

/* Last CUDA error string seen by the parser ("" if none). */
const char *jt_b200_last_error(const jt_parser *p);

#ifdef __cplusplus
}
#endif

#endif /* JSONTAPE_B200_H */
