// CPU harness for the stage-1 kernel's per-thread bit algebra.
//
// Compiles paper_1902_08318_b200/csrc/stage1_block.cuh with g++ (the
// functions are __host__ __device__) and runs the kernel's decomposition
// sequentially: per 64-byte block, classify -> transfer function -> final
// mask under the carried state, plus the fused UTF-8 check and the exact
// offset pass.  Additionally every block state is recomputed through
// composed transfer functions (the look-back path).  tests/test_stage1_cpu.py
// compares the result with the oracle; no GPU needed.
#include <stdint.h>
#include <string.h>

#include <vector>

#include "../paper_1902_08318_b200/csrc/stage1_block.cuh"

using namespace jt;

extern "C" int jt_cpu_stage1(const uint8_t *data, uint64_t len, uint32_t *out,
                             uint64_t *count, long long *utf8_off) {
  uint64_t nblocks = (len + 63) / 64;
  std::vector<uint8_t> buf(nblocks * 64 + 64, 0);
  if (len) memcpy(buf.data(), data, len);
  auto at = [&](uint64_t i) -> uint32_t { return i < len ? buf[i] : 0; };
  uint32_t state = s1::kInitState;
  uint32_t composed = 0x03020100u;  // identity on (odd, in_string)
  uint64_t n = 0;
  long long bad = -1;
  int mismatch = 0;
  for (uint64_t b = 0; b < nblocks; b++) {
    uint32_t w[16];
    memcpy(w, buf.data() + b * 64, 64);
    s1::Masks m;
    s1::classify64(w, m);
    uint64_t esc0 = s1::escaped_no_carry(m.bs);
    uint64_t tog = s1::carry_toggle(m.bs);
    uint32_t f = s1::block_function(m, esc0, tog);
    uint64_t blk = b * 64;
    uint64_t valid = len - blk >= 64 ? ~0ULL : ((1ULL << (len - blk)) - 1);
    uint64_t fin = s1::final_mask(m, esc0, tog, state, valid);
    while (fin) {
      out[n++] = (uint32_t)(blk + ctz64(fin));
      fin &= fin - 1;
    }
    // UTF-8
    uint32_t prev = 0;
    if (blk >= 4) memcpy(&prev, buf.data() + blk - 4, 4);
    if (s1::utf8_block_error(m.P, prev, blk + 64 >= len)) {
      uint64_t lo = blk >= 3 ? blk - 3 : 0, hi = blk + 64 < len ? blk + 64 : len;
      for (uint64_t i = lo; i < hi; i++)
        if (s1::utf8_flagged(at, i, len)) {
          if (bad < 0 || (long long)i < bad) bad = (long long)i;
          break;
        }
    }
    // sequential carry vs composed function (look-back path)
    uint32_t next = s1::apply(f, state);
    composed = s1::compose(f, composed);
    uint32_t via = s1::apply(composed, s1::kInitState);
    if ((via & 3) != (next & 3) || (b > 0 && via != next)) mismatch = 1;
    state = next;
  }
  *count = n;
  *utf8_off = bad;
  return mismatch;
}
