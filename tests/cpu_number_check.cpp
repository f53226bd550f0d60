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
  struct At {
    const uint8_t *buf;
    uint64_t len;
    uint32_t operator()(uint64_t i) const { return i < len ? buf[i] : 0; }
    uint64_t load8(uint64_t i) const {
      uint64_t v = 0;
      for (int k = 0; k < 8; k++) v |= (uint64_t)(*this)(i + k) << (8 * k);
      return v;
    }
  } at{buf, len};
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
