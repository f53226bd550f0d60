// CPU harness for the device number parser (numparse.cuh compiled with g++):
// the same code path the sm_100a kernels run, checked against the oracle's
// glibc-strtod restatement by tests/test_numbers_cpu.py.
#include <stdint.h>
#include <string.h>

#include "../paper_1902_08318_b200/csrc/numparse.cuh"

using namespace jt;

// returns 0 fail, 1 int, 2 float; *bits the word; *slow whether the exact
// fallback was needed
extern "C" int jt_cpu_number(const uint8_t *buf, uint64_t len, uint64_t *bits, int *slow) {
  auto at = [&](uint64_t i) -> uint32_t { return i < len ? buf[i] : 0; };
  num::NumResult r = num::parse_number(at, len, 0);
  *slow = 0;
  if (r.kind == num::kNumSlow) {
    *slow = 1;
    static num::Decimal dec;
    uint64_t b;
    if (!num::slow_decimal(at, len, 0, dec, &b)) return 0;
    *bits = b;
    return 2;
  }
  *bits = r.bits;
  return r.kind;
}
