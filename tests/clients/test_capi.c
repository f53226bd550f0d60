/* test_capi.c — a plain C client of include/jsontape.h, compiled with gcc and
 * linked against libjsontape_b200.so (tests/test_clients.py).  Restates the
 * reference's own C-ABI tests (proj/tests/test_capi.cpp) case by case, so a C
 * program written against the reference builds and behaves the same against
 * the B200 library.  Exit status 0 = all checks passed. */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "jsontape.h"

static int failures = 0;
#define CHECK(c)                                                      \
  do {                                                                \
    if (!(c)) {                                                       \
      fprintf(stderr, "%s:%d: CHECK failed: %s\n", __FILE__, __LINE__, #c); \
      failures++;                                                     \
    }                                                                 \
  } while (0)
#define REQUIRE(c)                                                    \
  do {                                                                \
    if (!(c)) {                                                       \
      fprintf(stderr, "%s:%d: REQUIRE failed: %s\n", __FILE__, __LINE__, #c); \
      exit(1);                                                        \
    }                                                                 \
  } while (0)

/* test_capi.cpp:24-41 */
static void parse_and_error_codes(void) {
  jt_parser *p = jt_parser_new();
  REQUIRE(p != NULL);
  jt_document *d = NULL, *bad = (jt_document *)1;
  long long off = -2;
  CHECK(jt_parse(p, "{\"a\":1}", 7, &d, &off) == JT_OK);
  CHECK(d != NULL);
  CHECK(off == -1);
  CHECK(jt_parse(p, "{\"a\":1,}", 8, &bad, &off) == JT_TAPE_ERROR);
  CHECK(bad == NULL);
  CHECK(jt_parse(p, "[01]", 4, NULL, &off) == JT_NUMBER_ERROR);
  CHECK(jt_parse(p, "[\"\\q\"]", 6, NULL, &off) == JT_STRING_ERROR);
  CHECK(jt_parse(p, "\"\xff\"", 3, NULL, &off) == JT_UTF8_ERROR);
  CHECK(off == 1);
  CHECK(jt_parse(p, "  ", 2, NULL, &off) == JT_EMPTY);
  CHECK(off == -1);
  CHECK(jt_parse(p, "7", 1, NULL, NULL) == JT_OK); /* out params are optional */
  jt_document_free(d);
  jt_parser_free(p);
}

/* test_capi.cpp:43-51 */
static void error_names(void) {
  CHECK(strcmp(jt_error_name(JT_OK), "OK") == 0);
  CHECK(strcmp(jt_error_name(JT_UTF8_ERROR), "UTF8_ERROR") == 0);
  CHECK(strcmp(jt_error_name(JT_STRING_ERROR), "STRING_ERROR") == 0);
  CHECK(strcmp(jt_error_name(JT_NUMBER_ERROR), "NUMBER_ERROR") == 0);
  CHECK(strcmp(jt_error_name(JT_TAPE_ERROR), "TAPE_ERROR") == 0);
  CHECK(strcmp(jt_error_name(JT_DEPTH_ERROR), "DEPTH_ERROR") == 0);
  CHECK(strcmp(jt_error_name(JT_CAPACITY), "CAPACITY") == 0);
  CHECK(strcmp(jt_error_name(JT_EMPTY), "EMPTY") == 0);
}

/* test_capi.cpp:53-73 */
static void stage1_then_stage2(void) {
  jt_parser *p = jt_parser_new();
  const char *src = "{ \"k\" : [ 1 , 2 ] }";
  long long off = -1;
  REQUIRE(jt_stage1(p, src, strlen(src), &off) == JT_OK);
  size_t n = jt_index_count(p);
  const uint32_t *pos = jt_index_positions(p);
  static const uint32_t expect[] = {0, 2, 6, 8, 10, 12, 14, 16, 18};
  REQUIRE(n == 9);
  CHECK(memcmp(pos, expect, sizeof(expect)) == 0);
  CHECK(jt_stage2(p, NULL, &off) == JT_OK); /* validate-only first, then materialize */
  jt_document *d = NULL, *direct = NULL;
  REQUIRE(jt_stage2(p, &d, &off) == JT_OK);
  REQUIRE(jt_parse(p, src, strlen(src), &direct, &off) == JT_OK);
  CHECK(jt_document_equal(d, direct) == 1);
  jt_document_free(d);
  jt_document_free(direct);
  jt_parser_free(p);
}

/* test_capi.cpp:75-80 */
static void stage1_utf8(void) {
  jt_parser *p = jt_parser_new();
  long long off = -1;
  CHECK(jt_stage1(p, "[\"\xed\xa0\x80\"]", 7, &off) == JT_UTF8_ERROR);
  CHECK(off == 2);
  jt_parser_free(p);
}

/* test_capi.cpp:82-96 */
static void equality_and_dump(void) {
  jt_parser *p = jt_parser_new();
  jt_document *a = NULL, *b = NULL, *c = NULL;
  REQUIRE(jt_parse(p, "[1, 2]", 6, &a, NULL) == JT_OK);
  REQUIRE(jt_parse(p, "[ 1 ,2 ]", 8, &b, NULL) == JT_OK);
  REQUIRE(jt_parse(p, "[1, 3]", 6, &c, NULL) == JT_OK);
  CHECK(jt_document_equal(a, b) == 1);
  CHECK(jt_document_equal(a, c) == 0);
  char *dump = jt_document_dump(a);
  REQUIRE(dump != NULL);
  CHECK(strstr(dump, "integer 2") != NULL);
  jt_string_free(dump);
  jt_document_free(a);
  jt_document_free(b);
  jt_document_free(c);
  jt_parser_free(p);
}

/* test_capi.cpp:98-108 */
static void distinct_values(void) {
  jt_parser *p = jt_parser_new();
  jt_document *d = NULL;
  const char *src = "{\"a\": {\"k\": 2}, \"b\": [{\"k\": 1}, {\"k\": 2}]}";
  REQUIRE(jt_parse(p, src, strlen(src), &d, NULL) == JT_OK);
  char *out = jt_document_distinct(d, "k");
  REQUIRE(out != NULL);
  CHECK(strcmp(out, "1\n2\n") == 0);
  jt_string_free(out);
  jt_document_free(d);
  jt_parser_free(p);
}

/* test_capi.cpp:110-123 */
static void minify(void) {
  jt_parser *p = jt_parser_new();
  const char *src = " { \"a\" : [ 1 , 2 ] } ";
  size_t len = strlen(src), dst_len = 0;
  char dst[64];
  long long off = -1;
  REQUIRE(jt_minify(p, src, len, dst, &dst_len, &off) == JT_OK);
  CHECK(dst_len == 11 && memcmp(dst, "{\"a\":[1,2]}", 11) == 0);
  CHECK(jt_minify(p, "[1,]", 4, dst, &dst_len, &off) == JT_TAPE_ERROR);
  jt_parser_free(p);
}

/* test_capi.cpp:125-140 */
static void stats(void) {
  jt_parser *p = jt_parser_new();
  const char *src = "{\"a\": [1, 2.5], \"b\": null}";
  jt_stats st;
  long long off = -1;
  REQUIRE(jt_compute_stats(p, src, strlen(src), &st, &off) == JT_OK);
  CHECK(st.integers == 1);
  CHECK(st.floats == 1);
  CHECK(st.strings == 2);
  CHECK(st.objects == 1);
  CHECK(st.arrays == 1);
  CHECK(st.nulls == 1);
  CHECK(st.bytes == strlen(src));
  CHECK(st.bytes_per_structural > 0);
  jt_parser_free(p);
}

/* test_capi.cpp:142-146 */
static void oracle_validation(void) {
  CHECK(jt_oracle_validate("[1,2]", 5) == 1);
  CHECK(jt_oracle_validate("[1,2,]", 6) == 0);
  CHECK(jt_oracle_validate("", 0) == 0);
}

/* test_capi.cpp:148-163 exercises jt_generate, the reference's corpus
 * generator: out of scope here, documented to return NULL. */
static void generate_stub(void) {
  size_t len = 7;
  CHECK(jt_generate("numbers", 10, 7, &len) == NULL);
}

/* test_capi.cpp:165-178 */
static void ablation_flags(void) {
  const char *src = "{\"s\": \"a\\u0041\\\\\", \"n\": [1.5, -2, 1e10], \"t\": true}";
  size_t len = strlen(src);
  jt_parser *ref = jt_parser_new();
  jt_document *ref_doc = NULL;
  REQUIRE(jt_parse(ref, src, len, &ref_doc, NULL) == JT_OK);
  for (int mask = 0; mask < 8; mask++) {
    jt_parser *p = jt_parser_new();
    jt_parser_set_flags(p, mask & 1, !!(mask & 2), !!(mask & 4));
    jt_document *d = NULL;
    REQUIRE(jt_parse(p, src, len, &d, NULL) == JT_OK);
    CHECK(jt_document_equal(d, ref_doc) == 1);
    jt_document_free(d);
    jt_parser_free(p);
  }
  jt_document_free(ref_doc);
  jt_parser_free(ref);
}

/* capi.cpp:75-76, 86-89: *out = NULL on any error, and the
 * stale index after a UTF-8 failure (indexer.cpp:35-36) */
static void boundary_semantics(void) {
  jt_parser *p = jt_parser_new();
  long long off = 0;
  REQUIRE(jt_stage1(p, "[1,2]", 5, &off) == JT_OK);
  CHECK(jt_index_count(p) == 5);
  CHECK(jt_stage1(p, "[\xff]", 3, &off) == JT_UTF8_ERROR && off == 1);
  CHECK(jt_index_count(p) == 5); /* not refreshed */
  jt_document *d = (jt_document *)&off;
  CHECK(jt_parse(p, "[", 1, &d, &off) == JT_TAPE_ERROR && d == NULL && off == 1);
  jt_parser_free(p);
}

int main(void) {
  parse_and_error_codes();
  error_names();
  stage1_then_stage2();
  stage1_utf8();
  equality_and_dump();
  distinct_values();
  minify();
  stats();
  oracle_validation();
  generate_stub();
  ablation_flags();
  boundary_semantics();
  if (failures) {
    fprintf(stderr, "%d check(s) failed\n", failures);
    return 1;
  }
  printf("test_capi: all checks passed\n");
  return 0;
}
