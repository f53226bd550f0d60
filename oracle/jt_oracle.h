/* jt_oracle — CPU restatement of the reference parse path, TEST
 * INFRASTRUCTURE ONLY.
 *
 * This is the parity checker for the B200 parser in paper_1902_08318_b200/.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it, and only as the checker / CPU baseline,
 * never as the thing measured or shipped.  The product library never links
 * it and has no CPU fallback.
 *
 * It restates, one byte / one token at a time, the algorithm of
 * /root/reference/proj (paper arXiv:1902.08318 "Parsing Gigabytes of JSON per
 * Second"): stage 1 = UTF-8 validation + structural index
 * (proj/src/indexer.cpp:29-56, blocks.h:155-194, utf8.cpp:200-243), stage 2 =
 * tape construction (proj/src/tape_builder.cpp:140-258) with the string
 * (stringparse.cpp:143-183) and number (numbers.cpp:52-178) parsers.  Float
 * slow path = glibc strtod, exactly as numbers.cpp:37-48.
 *
 * Parity pinned: tests/test_oracle_golden.py checks it against the
 * reference's own known-answer vectors (proj/tests/*), and
 * tests/test_oracle_vs_ref.py differentially against the compiled reference
 * (oracle/_ref/libjsontape_ref.so built by oracle/build_ref.sh). */
#ifndef JT_ORACLE_H
#define JT_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* same numbering as jt_error (proj/include/jsontape.h:15-24) */
enum {
  JTO_OK = 0,
  JTO_UTF8_ERROR,
  JTO_STRING_ERROR,
  JTO_NUMBER_ERROR,
  JTO_TAPE_ERROR,
  JTO_DEPTH_ERROR,
  JTO_CAPACITY,
  JTO_EMPTY
};

typedef struct jto_result {
  int code;
  long long offset;
  uint32_t *index; /* structural index (valid unless UTF8/CAPACITY) */
  size_t index_count;
  uint64_t *tape; /* tape words (valid on OK) */
  size_t tape_len;
  uint8_t *strings; /* string buffer (valid on OK) */
  size_t strings_len;
} jto_result;

/* first invalid UTF-8 sequence start, or -1 (utf8.cpp:200-243) */
long long jto_utf8_error_offset(const uint8_t *data, size_t len);

/* stage 1 only (indexer.cpp:29-56); fills r->index / index_count */
int jto_stage1(const uint8_t *data, size_t len, jto_result *r);

/* full parse (capi.cpp:73-93 semantics); allocations freed by jto_free */
int jto_parse(const uint8_t *data, size_t len, jto_result *r);
void jto_free(jto_result *r);
/* jt_minify: parse, then minify_pass; out >= len bytes */
int jto_minify(const uint8_t *data, size_t len, uint8_t *out, size_t *out_len, long long *offset);

/* single-token helpers, for the number/string unit vectors */
int jto_parse_number(const uint8_t *buf, size_t len, size_t offset,
                     int *is_integer, uint64_t *bits);
int jto_parse_string(const uint8_t *buf, size_t len, size_t offset,
                     uint8_t *dst, uint32_t *out_len, long long *err_off);

#ifdef __cplusplus
}
#endif

#endif
