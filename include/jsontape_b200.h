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
/* jt_stage1 over the resident input without waiting (UTF-8 check + index,
 * the k_index path); jt_b200_finish completes it like jt_stage1 would. */
jt_error jt_b200_stage1_async(jt_parser *p, size_t len);

/* Device views of the last results (valid until the next call). */
const uint32_t *jt_b200_device_index(const jt_parser *p, size_t *count);
const uint64_t *jt_b200_device_tape(const jt_parser *p, size_t *words);
const uint8_t *jt_b200_device_strings(const jt_parser *p, size_t *bytes);

/* Materialise the last successful resident parse as a host document. */
jt_error jt_b200_download(jt_parser *p, jt_document **out);

/* Host views of a document's tape words and string buffer (the reference's
 * parsed_document::tape / ::strings, proj/src/tape.h:49-58; valid until
 * jt_document_free).  Used by the C++ entry points in jsontape.hpp. */
const uint64_t *jt_b200_document_tape(const jt_document *doc, size_t *words);
const uint8_t *jt_b200_document_strings(const jt_document *doc, size_t *bytes);
/* A host document holding a copy of the given tape words and string buffer
 * (free with jt_document_free); NULL on allocation failure.  Lets a C++
 * parsed_document go through jt_document_dump / jt_document_distinct. */
jt_document *jt_b200_document_from(const uint64_t *tape, size_t words, const uint8_t *strings, size_t bytes);

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

/* ---- NDJSON records (BASELINE config C3) ----
 * The len resident bytes are '\n'-separated records (the last one may lack
 * the '\n'); each is parsed as jt_parse(record) would parse it alone
 * (proj/src/capi.cpp:70-93), all in one GPU pass with per-record carries
 * (in-string state and depth reset at every '\n').  Results per record:
 * code, offset relative to the record start, and on JT_OK the record's tape
 * (record-relative indices, root words at both ends) and string buffer,
 * stored back to back on the device. */
typedef struct {
  int32_t code;             /* jt_error */
  int32_t reserved;
  long long offset;         /* relative to the record start, -1 if none */
  uint64_t tape_begin;      /* index of the record's root word in the device tape */
  uint64_t tape_words;      /* root .. root close; 0 unless JT_OK */
  uint64_t string_begin;    /* offset of its strings in the device string buffer */
  uint64_t string_bytes;
} jt_b200_record;
int jt_b200_parse_records(jt_parser *p, size_t len, size_t *n_records);
const void *jt_b200_records(jt_parser *p);        /* host jt_b200_record[n_records], copied on first use */
const void *jt_b200_device_records(const jt_parser *p); /* the same on the device */
void jt_b200_records_size(const jt_parser *p, unsigned long long *out);
int jt_b200_records_download(jt_parser *p, uint64_t *tape, uint8_t *strings);

/* ---- Byte-range sharding of one document across GPUs ----
 * Shard g of G parses bytes [begin, end) of a document whose len bytes are
 * resident in the parser's input buffer (jt_b200_input_buffer /
 * jt_b200_copy_in).  begin is a multiple of 16384; shard 0 starts at 0 and
 * shard G-1 ends at len.  Four phases, each enqueued asynchronously on the
 * parser's stream, write a fixed-size summary (jt_b200_shard_summary_bytes)
 * to a caller device buffer; the caller all-gathers the G summaries of a
 * phase (NCCL all_gather, or device copies when emulating shards on one
 * GPU) and passes them to the next phase.  Replaces, for one document, the
 * single sequential pass of jt_parse (proj/src/capi.cpp:70-93; carries as in
 * blocks.h:31-35 and tape_builder.cpp:140-258). */
size_t jt_b200_shard_summary_bytes(int phase);
int jt_b200_shard_begin(jt_parser *p, size_t len, unsigned g, unsigned G, size_t begin, size_t end);
/* Bytes [lo, hi) of the document are resident on this GPU (hi = 0: all of
 * it, the default); must cover [begin - 64, end + 64) of every later shard.
 * A number that starts in the shard and runs to hi makes the parse fail
 * with JT_CAPACITY, offset -1 (upload a larger halo and parse again). */
int jt_b200_shard_resident(jt_parser *p, size_t lo, size_t hi);
int jt_b200_shard_phase(jt_parser *p, int phase, const void *gathered, void *summary);
/* Document result (same code/offset as jt_parse of the whole document); waits. */
jt_error jt_b200_shard_finish(jt_parser *p, const void *gathered, long long *error_offset);
/* out[7]: document tape index of local word out[1], local words, document
 * string offset of local byte 0, string bytes, first token index, tokens. */
int jt_b200_shard_extent(const jt_parser *p, unsigned long long *out);
/* Enqueue (no wait) a copy of bytes [offset, offset + n) of a host or device
 * document into the same positions of the input buffer (a shard's range). */
int jt_b200_copy_in_range(jt_parser *p, const void *src, size_t offset, size_t n);
/* Copy this shard's tape words and string bytes (sizes from the extent) to host. */
int jt_b200_shard_download(jt_parser *p, uint64_t *tape, uint8_t *strings);

/* CUDA device ordinal the parser was created on. */
int jt_b200_device(const jt_parser *p);
/* Bytes of device memory the parser holds (its grow-only arena). */
size_t jt_b200_device_bytes(const jt_parser *p);

/* Last CUDA error string seen by the parser ("" if none). */
const char *jt_b200_last_error(const jt_parser *p);

/* distinct_values over the last successful parse, on the device ("parse +
 * select"; document.cpp:134-192): the same text as
 * jt_document_distinct on the downloaded document (sorted distinct scalars at
 * a dotted key path, one per line).  Free with jt_string_free; NULL without a
 * successful parse or on a device error. */
char *jt_b200_distinct(jt_parser *p, const char *path);

#ifdef __cplusplus
}
#endif

#endif /* JSONTAPE_B200_H */
