// test_cpp_api.cpp — a C++ client of the reference's C++ entry points
// (jt::build_structural_index / jt::build_tape / jt::parse / jt::tape_dump,
// proj/src/indexer.h:55-57, tape.h:62-71) through include/jsontape.hpp, linked
// against libjsontape_b200.so (tests/test_clients.py).  The steady-state loop
// restates the reference's own harness (proj/tests/acceptance.cpp:455-473):
// one padded_input, index and document reused across runs.  Every result is
// checked against the C ABI's jt_parse of the same bytes.  Exit 0 = passed.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "jsontape.hpp"

extern "C" char *jtg_generate(int config, uint64_t target, uint64_t seed, int err_kind, size_t *len_out);
extern "C" void jtg_free(char *p);

static int failures = 0;
#define CHECK(c)                                                              \
  do {                                                                        \
    if (!(c)) {                                                               \
      std::fprintf(stderr, "%s:%d: CHECK failed: %s\n", __FILE__, __LINE__, #c); \
      failures++;                                                             \
    }                                                                         \
  } while (0)

// the C ABI's answer for the same bytes
struct CRef {
  jt_error code;
  long long off;
  std::vector<uint64_t> tape;
  std::vector<uint8_t> strings;
  std::vector<uint32_t> index;
};

static CRef c_parse(const std::string &s) {
  CRef r;
  jt_parser *p = jt_parser_new();
  jt_document *d = nullptr;
  r.code = jt_parse(p, s.data(), s.size(), &d, &r.off);
  size_t n = jt_index_count(p);
  const uint32_t *pos = n ? jt_index_positions(p) : nullptr;
  r.index.assign(pos, pos + n);
  if (d) {
    size_t w = 0, b = 0;
    const uint64_t *t = jt_b200_document_tape(d, &w);
    const uint8_t *st = jt_b200_document_strings(d, &b);
    r.tape.assign(t, t + w);
    r.strings.assign(st, st + b);
  }
  jt_document_free(d);
  jt_parser_free(p);
  return r;
}

static void check_doc(const std::string &s, const char *what) {
  const CRef ref = c_parse(s);
  // acceptance.cpp:455-473 style: padded once, buffers reused
  jt::padded_input input = jt::padded_input::from(s.data(), s.size());
  jt::structural_index idx;
  jt::parsed_document doc;
  for (int run = 0; run < 2; run++) {
    jt::parse_result r = jt::build_structural_index(input, {}, idx);
    if (r.ok()) {
      CHECK(idx.count == ref.index.size());
      CHECK(std::memcmp(idx.positions(), ref.index.data(), 4 * idx.count) == 0);
      r = jt::build_tape(input, idx, doc);
    }
    if ((jt_error)r.code != ref.code || r.offset != ref.off)
      std::fprintf(stderr, "%s: run %d: %s %lld vs C ABI %s %lld\n", what, run, jt::error_name(r.code), r.offset,
                   jt_error_name(ref.code), ref.off);
    CHECK((jt_error)r.code == ref.code && r.offset == ref.off);
    if (r.ok()) {
      CHECK(doc.tape == ref.tape);
      CHECK(doc.strings == ref.strings);
      CHECK(doc.source_length == s.size());
    }
  }
  // jt::parse (tape_builder.cpp:267-275)
  jt::parsed_document doc2;
  jt::parse_result r2 = jt::parse((const uint8_t *)s.data(), s.size(), {}, doc2);
  CHECK((jt_error)r2.code == ref.code && r2.offset == ref.off);
  if (r2.ok()) CHECK(doc2 == doc);
}

int main() {
  const char *docs[] = {
      "{\"a\":1}", "{\"a\":1,}", "[01]", "[\"\\q\"]", "\"\xff\"", "  ", "7", "[1,2",
      "{\"Width\": 800, \"Title\": \"View \\u00e9 \\ud834\\udd1e\", \"a\": [1.5e300, -0.0, true, null]}",
  };
  for (const char *d : docs) check_doc(d, d);
  for (int cfg : {0, 1, 2, 4}) {
    size_t n = 0;
    char *g = jtg_generate(cfg, cfg == 0 ? (1u << 20) : (4u << 20), 7, 0, &n);
    check_doc(std::string(g, n), "generated");
    jtg_free(g);
  }
  // an index built for one input, then build_tape on another input: the
  // document of the input passed to build_tape (the index is a function of it)
  {
    jt::padded_input a = jt::padded_input::from("[1,2]", 5), b = jt::padded_input::from("[3]", 3);
    jt::structural_index idx;
    jt::parsed_document da, db;
    CHECK(jt::build_structural_index(a, {}, idx).ok());
    CHECK(jt::build_tape(b, idx, db).ok());
    CHECK(jt::parse(b.data(), b.size(), {}, da).ok());
    CHECK(da == db);
  }
  // UTF-8 failure leaves the index as it was (indexer.cpp:35-36)
  {
    jt::padded_input ok = jt::padded_input::from("[1,2]", 5), bad = jt::padded_input::from("[\xff]", 3);
    jt::structural_index idx;
    CHECK(jt::build_structural_index(ok, {}, idx).ok());
    jt::parse_result r = jt::build_structural_index(bad, {}, idx);
    CHECK(r.code == jt::error_code::utf8_error && r.offset == 1);
    CHECK(idx.count == 5);
  }
  // tape_dump matches the C ABI's jt_document_dump
  {
    jt::parsed_document d;
    CHECK(jt::parse((const uint8_t *)"[1, 2.5, \"x\"]", 13, {}, d).ok());
    const std::string dump = jt::tape_dump(d);
    CHECK(dump.find("integer 1") != std::string::npos);
    jt_parser *p = jt_parser_new();
    jt_document *cd = nullptr;
    CHECK(jt_parse(p, "[1, 2.5, \"x\"]", 13, &cd, nullptr) == JT_OK);
    char *cdump = jt_document_dump(cd);
    CHECK(cdump && dump == cdump);
    jt_string_free(cdump);
    jt_document_free(cd);
    jt_parser_free(p);
  }
  CHECK(std::string(jt::error_name(jt::error_code::depth_error)) == "DEPTH_ERROR");
  if (failures) {
    std::fprintf(stderr, "%d check(s) failed\n", failures);
    return 1;
  }
  std::printf("test_cpp_api: all checks passed\n");
  return 0;
}
