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
  // K1's shared copy of the current 16 KiB tile: escapes are decoded in
  // place there (the global input is never written)
  std::vector<uint8_t> tile(16384);
  for (uint64_t b = 0; b < nblocks; b++) {
    if ((b * 64) % 16384 == 0)
      for (uint64_t k = 0; k < 16384; k++) tile[k] = at(b * 64 + k);
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
    uint32_t spill_bytes = 0;
    int ov_scan = (state & 2) ? sb::overhang_in_scan(at, blk, true, &spill_bytes) : 0;
    if (ov_scan != ov_in) *ov_mismatch += 1;
    int rem = (int)(len - blk);
    if (rem > 0 && rem <= 64 && ((instr >> (rem - 1)) & 1)) serr = serr < len ? serr : len;
    uint64_t base = sw_total;
    struct Byte {  // the tile copy for the block's own bytes, the global input past them
      const std::vector<uint8_t> *b;
      const std::vector<uint8_t> *t;
      uint64_t blk;
      uint32_t operator()(uint64_t k) const {
        const uint64_t rel = blk % 16384 + k;
        if (k < 64 && rel < 16384) return (*t)[rel];
        return blk + k < b->size() ? (*b)[blk + k] : 0;
      }
      void window12(uint64_t k, uint32_t w[3]) const {
        for (int q = 0; q < 3; q++) {
          w[q] = 0;
          for (int j = 0; j < 4; j++) w[q] |= (*this)(k + 4 * q + j) << (8 * j);
        }
      }
    } byte{&buf, &tile, blk};
    const uint64_t local = blk % 16384;
    auto rewrite = [&](int k, uint8_t v) {
      if (local + (uint64_t)k < 16384) tile[local + k] = v;
    };
    // K1's order: step 1 before the previous block's overhang is known
    // (an escape reaching past the block is decoded and written here), ...
    sb::BlockEsc be{};
    if (E) be = sb::block_escapes(m.P, m.qt, m.bs, E, byte, rewrite);
    const int ov_next = E ? be.ov_out : 0;
    const int vin = ov_in >> 8, ov = ov_in & 0xFF;
    if (ctl) {
      uint64_t x = blk + (uint64_t)ctz64(ctl);
      if (x < serr) serr = x;
    }
    // the first block of a tile: the bytes an escape of the previous tile
    // spills into it (that tile drops its rewrites past its end)
    if (local == 0)
      for (int k = 0; k < vin; k++) tile[k] = (uint8_t)(spill_bytes >> (8 * k));
    // ... step 2 with it: weights and errors ...
    uint64_t W = content;
    if (E || ov) {
      W = sb::block_weights(content, be, ov, vin);
      if (be.bad) {
        const uint64_t x = blk + (uint64_t)ctz64(be.bad);
        if (x < serr) serr = x;
      }
      // ... step 3 before the payload copy: the escapes inside the block
      sb::decode_in_place(be.ec.tr, be.bmp, be.pair,
                          [&](uint64_t k, uint32_t w[3]) { byte.window12(k, w); }, byte, rewrite);
    }
    const uint32_t we = 4u * popc64(openq) + popc64(W);
    // the payload: every weighted byte of the tile copy in order, a 4-byte
    // gap for each opening quote
    uint32_t wdst = 0;
    for (uint64_t bits = W | openq; bits; bits &= bits - 1) {
      const int k = ctz64(bits);
      if ((openq >> k) & 1) {
        wdst += 4;
      } else {
        out[base + wdst++] = tile[local + k];
      }
    }
    for (uint64_t fm = fin; fm; fm &= fm - 1) {
      const int p = ctz64(fm);
      const uint64_t below = sb::low_bits(p);
      idx[n] = (uint32_t)(blk + p);
      aux[n++] = (uint32_t)(base + 4u * popc64(openq & below) + popc64(W & below));
    }
    sw_total += we;
    ov_prev = ov_next;
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

// atom_ok8 (register form used by k_scalars) against the byte-at-a-time
// atom_ok, over every literal start in `data` (padded with zeros past len,
// as the device input is); returns the number of disagreements
extern "C" int jt_cpu_atoms(const uint8_t *data, uint64_t len) {
  std::vector<uint8_t> pad(data, data + len);
  pad.resize(len + 16, 0);
  auto at = [&](uint64_t i) -> uint32_t { return pad[i]; };
  int bad = 0;
  for (uint64_t p = 0; p < len; p++) {
    const uint32_t c = pad[p];
    if (c != 't' && c != 'f' && c != 'n') continue;
    uint64_t w = 0;
    for (int k = 7; k >= 0; k--) w = (w << 8) | pad[p + k];
    if (jt::str::atom_ok8(w, len, p, c) != jt::str::atom_ok(at, len, p, c)) bad++;
  }
  return bad;
}

// hex4_swar (the four hex digits of a \\u escape in one word) = hex4w, the
// byte-at-a-time decode, on words [lo, hi); returns the number of mismatches
extern "C" uint64_t jt_cpu_hex4_check(uint64_t lo, uint64_t hi) {
  uint64_t bad = 0;
  for (uint64_t x = lo; x < hi; x++) {
    const uint32_t w = (uint32_t)x;
    if (sb::hex4_swar(w) != sb::hex4w(w & 0xFF, (w >> 8) & 0xFF, (w >> 16) & 0xFF, w >> 24)) bad++;
  }
  return bad;
}
