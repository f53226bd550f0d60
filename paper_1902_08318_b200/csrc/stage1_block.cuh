// stage1_block.cuh — per-thread bit algebra of stage 1 (structural index).
//
// One thread owns one 64-byte block, like the reference's block loop
// (proj/src/indexer.cpp:42-53), but the sequential 3-bit carry
// {odd_backslash, in_string, prev_separator} (blocks.h:31-35) is replaced by
// a per-block TRANSFER FUNCTION that is scanned across threads, warps and
// tiles (decoupled look-back), so no block waits for its predecessor's bytes.
//
// Byte classification does not use the reference's nibble tables
// (blocks.h:90-136).  The 64 loaded bytes are bit-transposed into 8 bit
// planes (plane k bit i = bit k of byte i); every byte predicate (quote,
// backslash, the 6 structurals, the 4 whitespace bytes, the UTF-8 classes)
// is then a handful of LOP3s over 32 bytes at a time.
#pragma once

#include "jt_common.cuh"

namespace jt {
namespace s1 {

constexpr uint64_t kEven = 0x5555555555555555ULL;
constexpr uint64_t kOdd = 0xAAAAAAAAAAAAAAAAULL;

// 32 bytes in 8 little-endian words -> 8 bit planes of 32 bits.
// Step 1 (PRMT, two 4x4 byte transposes): word v[i] = bytes i, i+8, i+16,
// i+24, so bit 8b+k of v[i] is bit k of byte 8b+i.
// Step 2: in every byte lane at once, the 8x8 bit transpose ACROSS the eight
// words (bit k of v[i] <-> bit i of p[k]) as three rounds of pairwise
// exchanges; each exchange is two bit-selects (one LOP3 each) on a shifted
// operand -- 4 operations per pair, the left shifts as multiplies (FMA pipe;
// the ALU pipe, LOP3/SHF/PRMT, is what binds these kernels).  52 ALU + 12 FMA
// operations per 32 bytes (the 8x8-transpose-per-8-bytes form this replaced:
// 80 + 20).
template <uint32_t kMask, int kShift>
JT_HD void plane_exchange(uint32_t &a, uint32_t &b) {
  const uint32_t lo = bit_select(a, b * (1u << kShift), kMask);
  const uint32_t hi = bit_select(a >> kShift, b, kMask);
  a = lo;
  b = hi;
}

JT_HD void transpose32(const uint32_t w[8], uint32_t p[8]) {
  uint32_t tl, th, ul, uh;
  tl = byte_perm(w[0], w[2], 0x5140);
  th = byte_perm(w[0], w[2], 0x7362);
  ul = byte_perm(w[4], w[6], 0x5140);
  uh = byte_perm(w[4], w[6], 0x7362);
  p[0] = byte_perm(tl, ul, 0x5410);
  p[1] = byte_perm(tl, ul, 0x7632);
  p[2] = byte_perm(th, uh, 0x5410);
  p[3] = byte_perm(th, uh, 0x7632);
  tl = byte_perm(w[1], w[3], 0x5140);
  th = byte_perm(w[1], w[3], 0x7362);
  ul = byte_perm(w[5], w[7], 0x5140);
  uh = byte_perm(w[5], w[7], 0x7362);
  p[4] = byte_perm(tl, ul, 0x5410);
  p[5] = byte_perm(tl, ul, 0x7632);
  p[6] = byte_perm(th, uh, 0x5410);
  p[7] = byte_perm(th, uh, 0x7632);
#pragma unroll
  for (int i = 0; i < 4; i++) plane_exchange<0x0F0F0F0Fu, 4>(p[i], p[i + 4]);
#pragma unroll
  for (int i = 0; i < 8; i++)
    if (!(i & 2)) plane_exchange<0x33333333u, 2>(p[i], p[i + 2]);
#pragma unroll
  for (int i = 0; i < 8; i += 2) plane_exchange<0x55555555u, 1>(p[i], p[i + 1]);
}

struct Masks {
  uint64_t bs, qt, st, ws;  // backslash, quote, structural, whitespace
  uint64_t open, close;     // { [   and   } ]
  uint64_t cc;              // , :
  uint64_t num;             // - and digits (number token starts)
  uint64_t P[8];            // bit planes (kept for the UTF-8 check)
};

JT_HD uint64_t join(uint32_t lo, uint32_t hi) { return ((uint64_t)hi << 32) | lo; }

// 64 bytes (16 words) -> planes + the four stage-1 predicates.  The
// predicates are the exact byte sets of the reference's classify_block
// (blocks.h:96-136; equivalence over all 256 bytes: test_bitmask.cpp:102-118).
JT_HD void classify64(const uint32_t w[16], Masks &m) {
  uint32_t a[8], b[8];
  transpose32(w, a);
  transpose32(w + 8, b);
#pragma unroll
  for (int k = 0; k < 8; k++) m.P[k] = join(a[k], b[k]);
  const uint64_t *P = m.P;
  uint64_t n7 = ~P[7], n6 = ~P[6], n5 = ~P[5], n4 = ~P[4];
  uint64_t n3 = ~P[3], n2 = ~P[2], n1 = ~P[1], n0 = ~P[0];
  // 0x22 = 0010 0010
  m.qt = n7 & n6 & P[5] & n4 & n3 & n2 & P[1] & n0;
  // 0x5C = 0101 1100
  m.bs = n7 & P[6] & n5 & P[4] & P[3] & P[2] & n1 & n0;
  // [ ] { } = 01x1 1011 / 01x1 1101
  uint64_t brackets = n7 & P[6] & P[4] & P[3] & P[0] & (P[2] ^ P[1]);
  // , = 0010 1100   : = 0011 1010
  uint64_t hi001 = n7 & n6 & P[5];
  uint64_t comma = hi001 & n4 & P[3] & P[2] & n1 & n0;
  uint64_t colon = hi001 & P[4] & P[3] & n2 & P[1] & n0;
  m.st = brackets | comma | colon;
  m.open = brackets & P[1];   // low nibble 1011
  m.close = brackets & P[2];  // low nibble 1101
  m.cc = comma | colon;
  // '-' = 0010 1101, '0'..'9' = 0011 0000..1001
  m.num = (hi001 & n4 & P[3] & P[2] & n1 & P[0]) | (n7 & n6 & P[5] & P[4] & (n3 | (n2 & n1)));
  // 0x20 = 0010 0000 ; 0x09 0x0A 0x0D = 0000 1001 / 1010 / 1101
  uint64_t hi000 = n7 & n6 & n4;
  uint64_t space = hi000 & P[5] & n3 & n2 & n1 & n0;
  uint64_t ctl = hi000 & n5 & P[3] & ((n2 & (P[1] ^ P[0])) | (P[2] & n1 & P[0]));
  m.ws = space | ctl;
}

// bytes following an odd-length backslash run, assuming no run is carried
// in: the add-carry formulation of blocks.h:58-75 with carry_in = 0.
JT_HD uint64_t escaped_no_carry(uint64_t bs) {
  uint64_t starts = bs & ~(bs << 1);
  uint64_t even_carries = bs + (starts & kEven);
  uint64_t odd_carries = bs + (starts & kOdd);
  return ((even_carries & ~bs) & kOdd) | ((odd_carries & ~bs) & kEven);
}

// With an odd run carried in, only the first non-backslash byte of the block
// changes its escaped status (the leading run grows by an odd length).
JT_HD uint64_t carry_toggle(uint64_t bs) { return ~bs & (bs + 1); }

// Backslashes at an even offset within their run (1st, 3rd, ...): inside a
// string these start an escape sequence.  `odd_in` = the run ending at the
// previous block's last byte has odd length, which makes a run continuing at
// bit 0 behave as if it started at an odd position (blocks.h:58-75 uses the
// same re-classification of its starts).
JT_HD uint64_t unescaped_backslash(uint64_t bs, uint32_t odd_in) {
  uint64_t starts = bs & ~(bs << 1);
  uint64_t em = kEven ^ (uint64_t)odd_in;
  uint64_t runs_e = bs & ~(bs + (starts & em));
  uint64_t runs_o = bs & ~(bs + (starts & ~em));
  return (runs_e & kEven) | (runs_o & kOdd);
}

// Transfer function of one block (or a span of blocks), 4 bytes: byte x,
// x = odd_in | in_string_in << 1, holds odd_out | in_string_out << 1 |
// sep_out << 2, where sep_out is the prev_separator carry (blocks.h:161).
JT_HD uint32_t block_function(const Masks &m, uint64_t esc0, uint64_t tog) {
  uint64_t uq0 = m.qt & ~esc0;
  uint64_t uq1 = m.qt & ~(esc0 ^ tog);
  uint32_t par0 = popc64(uq0) & 1, par1 = popc64(uq1) & 1;
  uint32_t odd_fixed = clz64(~m.bs) & 1;  // parity of the run ending at bit 63
  bool all_bs = m.bs == ~0ULL;
  uint32_t ws63 = (uint32_t)(m.ws >> 63), st63 = (uint32_t)(m.st >> 63);
  uint32_t f = 0;
#pragma unroll
  for (uint32_t x = 0; x < 4; x++) {
    uint32_t o = x & 1, s = x >> 1;
    uint32_t oo = all_bs ? o : odd_fixed;
    uint32_t so = s ^ (o ? par1 : par0);
    uint32_t uq63 = (uint32_t)((o ? uq1 : uq0) >> 63);
    uint32_t sep = ws63 | uq63 | (st63 & (so ^ 1));
    f |= (oo | (so << 1) | (sep << 2)) << (8 * x);
  }
  return f;
}

// '\n' bytes (0x0A = 0000 1010): record separators in NDJSON mode
JT_HD uint64_t newline_mask(const uint64_t P[8]) {
  return ~P[7] & ~P[6] & ~P[5] & ~P[4] & P[3] & ~P[2] & P[1] & ~P[0];
}

// Record (NDJSON) mode: a '\n' ends its record, so the in-string carry out of
// a block with a newline is the quote parity after its last newline, whatever
// came in (a backslash run cannot cross the newline either).
JT_HD uint32_t block_function_rec(const Masks &m, uint64_t esc0, uint64_t tog, uint64_t nl) {
  uint32_t f = block_function(m, esc0, tog);
  if (!nl) return f;
  const int r = 63 - clz64(nl);
  const uint64_t after = r >= 63 ? 0ULL : (~0ULL << (r + 1));
  const uint32_t so = popc64(m.qt & ~esc0 & after) & 1;  // bits > r do not see the carry
  const uint32_t ws63 = (uint32_t)(m.ws >> 63), st63 = (uint32_t)(m.st >> 63);
  const uint32_t uq63 = (uint32_t)(((m.qt & ~esc0) >> 63) & (r < 63 ? 1u : 0u));
  const uint32_t sep = ws63 | uq63 | (st63 & (so ^ 1));
  uint32_t g = 0;
#pragma unroll
  for (uint32_t x = 0; x < 4; x++) {
    const uint32_t oo = (f >> (8 * x)) & 1;  // odd-run carry as before
    g |= (oo | (so << 1) | (sep << 2)) << (8 * x);
  }
  return g;
}

// g after f (f applied first), 5 integer ops
JT_HD uint32_t compose(uint32_t g_later, uint32_t f_earlier) {
  uint32_t v = f_earlier & 0x03030303u;
  uint32_t v2 = v | (v >> 4);
  uint32_t sel = byte_perm(v2, 0, 0x4420);
  return byte_perm(g_later, 0, sel);
}

// state = odd | in_string << 1 | prev_separator << 2
JT_HD uint32_t apply(uint32_t f, uint32_t state) { return (f >> (8 * (state & 3))) & 7; }

constexpr uint32_t kInitState = 4;  // scan_carry{0, 0, 1}, blocks.h:31-35

// inclusive prefix XOR of the bits of a word (bits.h:19-27)
JT_HD uint64_t prefix_xor(uint64_t x) {
  x ^= x << 1;
  x ^= x << 2;
  x ^= x << 4;
  x ^= x << 8;
  x ^= x << 16;
  x ^= x << 32;
  return x;
}

// In-string mask with resets: bits after a newline see only the quotes
// after it; the newline itself is outside every string.
JT_HD uint64_t instr_records(uint64_t uq, uint32_t in_str, uint64_t nl) {
  const uint64_t x = prefix_xor(uq);
  uint64_t instr = x ^ (in_str ? ~0ULL : 0ULL);
  while (nl) {
    const int r = ctz64(nl);
    nl &= nl - 1;
    const uint64_t seg = ~0ULL << r;  // bits >= r
    const uint64_t base = ((x >> r) & 1) ? ~0ULL : 0ULL;  // x at r (the newline is no quote)
    instr = (instr & ~seg) | ((x ^ base) & seg);
  }
  return instr;
}


// final structural mask of a block once its carry-in state is known
// (string_mask blocks.h:79-85 + finalize_structurals blocks.h:155-168)
JT_HD uint64_t final_mask(const Masks &m, uint64_t esc0, uint64_t tog, uint32_t state,
                          uint64_t valid) {
  uint64_t esc = (state & 1) ? (esc0 ^ tog) : esc0;
  uint64_t uq = m.qt & ~esc;
  uint64_t instr = prefix_xor(uq) ^ ((state & 2) ? ~0ULL : 0ULL);
  uint64_t s1 = (m.st & ~instr) | uq;
  uint64_t cand = s1 | m.ws;
  uint64_t pseudo = ((cand << 1) | (uint64_t)(state >> 2)) & ~m.ws & ~instr;
  return (s1 | pseudo) & ~(uq & ~instr) & valid;
}

// ---- UTF-8 (fused; validity only, the offset is a separate scalar pass) --

// Required-continuation spill into a block from its 3 predecessor bytes,
// plus the second-byte range flags of the byte right before the block.
// prev = little-endian word of bytes [blk-4, blk).
JT_HD void utf8_carry_in(uint32_t prev, uint64_t &req_in, uint32_t &range_in) {
  req_in = 0;
  range_in = 0;
#pragma unroll
  for (int d = 1; d <= 3; d++) {
    uint32_t b = (prev >> (8 * (4 - d))) & 0xFF;
    int n = b >= 0xF0 ? 4 : b >= 0xE0 ? 3 : b >= 0xC0 ? 2 : 0;
    int bits = n - 1 - (d - 1);  // positions blk-d+1 .. blk-d+n-1 that are >= blk
    if (bits > 0) req_in |= (1ULL << bits) - 1;
  }
  uint32_t b1 = prev >> 24;
  range_in = (b1 == 0xE0) ? 1 : (b1 == 0xED) ? 2 : (b1 == 0xF0) ? 4 : (b1 == 0xF4) ? 8 : 0;
}

// true if the block (with its carried-in context) breaks UTF-8 somewhere in
// [blk-3, blk+64): continuation structure, forbidden bytes, or the
// second-byte ranges of E0/ED/F0/F4 (Table 2).
JT_HD bool utf8_block_error(const uint64_t P[8], uint32_t prev, bool ends_input) {
  uint64_t req_in;
  uint32_t range_in;
  utf8_carry_in(prev, req_in, range_in);
  uint64_t cont = P[7] & ~P[6];
  uint64_t lead = P[7] & P[6];
  uint64_t l2 = lead & ~P[5];
  uint64_t l34 = lead & P[5];
  uint64_t l4 = l34 & P[4];
  uint64_t l3 = l34 & ~P[4];
  uint64_t anylead = lead;
  uint64_t req = (anylead << 1) | (l34 << 2) | (l4 << 3) | req_in;
  uint64_t bad = (l2 & ~P[4] & ~P[3] & ~P[2] & ~P[1])              // C0 C1
                 | (l4 & (P[3] | (P[2] & (P[1] | P[0]))));          // F5..FF
  uint64_t e0 = l3 & ~P[3] & ~P[2] & ~P[1] & ~P[0];
  uint64_t ed = l3 & P[3] & P[2] & ~P[1] & P[0];
  uint64_t l4x = l4 & ~P[3];
  uint64_t f0 = l4x & ~P[2] & ~P[1] & ~P[0];
  uint64_t f4 = l4x & P[2] & ~P[1] & ~P[0];
  uint64_t lo = cont & ~P[5];          // 80..9F
  uint64_t hi = cont & P[5];           // A0..BF
  uint64_t c80_8f = lo & ~P[4];        // 80..8F
  uint64_t c90_bf = cont & (P[5] | P[4]);
  uint64_t rng = (((e0 << 1) | (range_in & 1)) & lo) |
                 (((ed << 1) | ((range_in >> 1) & 1)) & hi) |
                 (((f0 << 1) | ((range_in >> 2) & 1)) & c80_8f) |
                 (((f4 << 1) | ((range_in >> 3) & 1)) & c90_bf);
  uint64_t spill = (anylead >> 63) | (l34 >> 62) | (l4 >> 61);
  return (req != cont) || bad || rng || (ends_input && spill);
}

// Exact first-error offset (utf8.cpp:200-243 semantics) among positions
// [lo, hi): a byte is flagged if it is an invalid lead, a valid lead whose
// sequence is malformed or truncated, or a continuation byte not covered by a
// valid lead 1..3 bytes before it.  In a valid prefix nothing is flagged and
// the sequential failure point always is, so the global minimum equals the
// reference's offset.  `at(i)` returns byte i, 0 past
// the end (the padding).
template <class At>
JT_HD int seq_len(At at, uint64_t j, uint64_t len) {
  // length of the valid sequence starting at j, 0 if j does not start one
  uint32_t b = at(j);
  if (b < 0x80) return 1;
  int n;
  uint32_t lo = 0x80, hi = 0xBF;
  if (b >= 0xC2 && b <= 0xDF) n = 2;
  else if (b == 0xE0) { n = 3; lo = 0xA0; }
  else if ((b >= 0xE1 && b <= 0xEC) || b == 0xEE || b == 0xEF) n = 3;
  else if (b == 0xED) { n = 3; hi = 0x9F; }
  else if (b == 0xF0) { n = 4; lo = 0x90; }
  else if (b >= 0xF1 && b <= 0xF3) n = 4;
  else if (b == 0xF4) { n = 4; hi = 0x8F; }
  else return 0;
  if (j + (uint64_t)n > len) return 0;
  uint32_t c = at(j + 1);
  if (c < lo || c > hi) return 0;
  for (int k = 2; k < n; k++) {
    c = at(j + k);
    if (c < 0x80 || c > 0xBF) return 0;
  }
  return n;
}

template <class At>
JT_HD bool utf8_flagged(At at, uint64_t i, uint64_t len) {
  uint32_t b = at(i);
  if (b < 0x80) return false;
  if (b <= 0xBF) {  // continuation: covered by a valid lead 1..3 back?
    for (int d = 1; d <= 3; d++) {
      if (i < (uint64_t)d) break;
      uint32_t c = at(i - d);
      if (c >= 0xC0) return seq_len(at, i - d, len) <= d;
      if (c < 0x80) return true;
    }
    return true;
  }
  return seq_len(at, i, len) == 0;
}

}  // namespace s1
}  // namespace jt
