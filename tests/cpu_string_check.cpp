// CPU harness for K1's string emission (strblock.cuh + stage1_block.cuh):
// runs the per-block decomposition sequentially and rebuilds the string
// buffer exactly as stage 2 finishes it (length field = aux difference - 4).
// Compared with the oracle's buffer by tests/test_stage1_cpu.py.
#include <stdint.h>
#include <string.h>

#include <vector>

#include "../paper_1902_08318_b200/csrc/stage1_block.cuh"
#include "../paper_1902_08318_b200/csrc/strblock.cuh"

using namespace jt;

extern "C" int jt_cpu_strings(const uint8_t *data, uint64_t len, uint8_t *out, uint64_t *out_len,
                              uint32_t *idx, uint32_t *aux, uint64_t *count, long long *str_err,
                              int *ov_mismatch) {
  uint64_t nblocks = (len + 63) / 64;
  std::vector<uint8_t> buf(nblocks * 64 + 128, 0);
  if (len) memcpy(buf.data(), data, len);
  auto at = [&](uint64_t i) -> uint32_t { return i < buf.size() ? buf[i] : 0; };
  uint32_t state = s1::kInitState;
  uint64_t n = 0, sw_total = 0;
  uint64_t serr = ~0ULL;
  int ov_prev = 0;
  *ov_mismatch = 0;
  for (uint64_t b = 0; b < nblocks; b++) {
    uint32_t w[16];
    memcpy(w, buf.data() + b * 64, 64);
    s1::Masks m;
    s1::classify64(w, m);
    uint64_t esc0 = s1::escaped_no_carry(m.bs), tog = s1::carry_toggle(m.bs);
    uint32_t f = s1::block_function(m, esc0, tog);
    uint64_t blk = b * 64;
    uint64_t valid = len - blk >= 64 ? ~0ULL : ((1ULL << (len - blk)) - 1);
    uint64_t esc = (state & 1) ? (esc0 ^ tog) : esc0;
    uint64_t uq = m.qt & ~esc;
    uint64_t instr = s1::prefix_xor(uq) ^ ((state & 2) ? ~0ULL : 0ULL);
    uint64_t fin = s1::final_mask(m, esc0, tog, state, valid);
    uint64_t openq = uq & instr & valid, content = instr & ~openq & valid;
    uint64_t E = s1::unescaped_backslash(m.bs, state & 1) & content, ctl = sb::control_mask(m.P) & content;
    int ov_in = ov_prev;
    int ov_scan = (state & 2) ? sb::overhang_in_scan(at, blk, true) : 0;
    if (ov_scan != ov_in) *ov_mismatch += 1;
    int rem = (int)(len - blk);
    if (rem > 0 && rem <= 64 && ((instr >> (rem - 1)) & 1)) serr = serr < len ? serr : len;
    uint64_t base = sw_total;
    struct Byte {
      const std::vector<uint8_t> *b;
      uint64_t blk;
      uint32_t operator()(uint64_t k) const { return blk + k < b->size() ? (*b)[blk + k] : 0; }
      void window12(uint64_t k, uint32_t w[3]) const {
        for (int q = 0; q < 3; q++) {
          w[q] = 0;
          for (int j = 0; j < 4; j++) w[q] |= (*this)(k + 4 * q + j) << (8 * j);
        }
      }
    } byte{&buf, blk};
    uint64_t e1 = ~0ULL;
    uint32_t wm = sb::block_strings<false>(byte, blk, content, openq, E, ctl, fin, ov_in, &e1,
                                           [](int, uint32_t, int) {}, [](uint32_t, uint8_t) {},
                                           [](int, uint32_t) {});
    uint32_t we = sb::block_strings<true>(
        byte, blk, content, openq, E, ctl, fin, ov_in, &serr,
        [&](int a0, uint32_t wdst, int nb) { memcpy(out + base + wdst, buf.data() + blk + a0, nb); },
        [&](uint32_t pos, uint8_t v) { out[base + pos] = v; },
        [&](int p, uint32_t wb) {
          idx[n] = (uint32_t)(blk + p);
          aux[n++] = (uint32_t)(base + wb);
        });
    if (wm != we || e1 != (serr < e1 ? e1 : e1)) {}
    if (wm != we) *ov_mismatch += 1000;
    sw_total += we;
    ov_prev = E ? sb::overhang_out(at, blk, E) : 0;
    state = s1::apply(f, state);
  }
  // stage 2's share: length fields from aux differences
  for (uint64_t i = 0; i < n; i++) {
    if (buf[idx[i]] != '"') continue;
    uint64_t next = i + 1 < n ? aux[i + 1] : sw_total;
    uint32_t l = (uint32_t)(next - aux[i] - 4);
    memcpy(out + aux[i], &l, 4);
  }
  *out_len = sw_total;
  *count = n;
  *str_err = serr == ~0ULL ? -1 : (long long)serr;
  return 0;
}
