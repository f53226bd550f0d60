// strblock.cuh — string payload emission inside the stage-1 block pass.
//
// Every byte of a 64-byte block gets a WEIGHT = bytes it contributes to the
// string buffer (proj/src/tape.h:51-52 layout, tape_builder.cpp:88-89):
//   opening quote          4  (the u32 length field, filled by stage 2)
//   plain string byte      1  (copied verbatim, stringparse.cpp:176-181)
//   escape start (\ not escaped, inside a string)  1..4  (decoded bytes,
//                          handle_escape stringparse.cpp:73-102); the rest of
//                          the escape sequence weighs 0
//   anything else          0
// The exclusive prefix of weights at a token is its string offset, so a
// string's length is the difference of the prefixes of the token and the
// next token minus 4.  String errors (control byte inside a string, invalid
// escape, unterminated string) are reported as byte positions; the first
// failing string is the one holding the minimum position.
//
// Blocks without escapes or control bytes (the common case) take the mask
// fast path; others run a sequential walker over their bytes.
#pragma once

#include "jt_common.cuh"
#include "strparse.cuh"

namespace jt {
namespace sb {

// control bytes (< 0x20) from the bit planes
JT_HD uint64_t control_mask(const uint64_t P[8]) { return ~P[7] & ~P[6] & ~P[5]; }

// Length of the escape sequence at p (p = backslash) and its decoded bytes;
// 0 if invalid.  Same checks as handle_escape.
template <class At>
JT_HD int escape_len(At at, uint64_t p, uint32_t *cp) {
  return str::escape_at(at, p, cp);
}

JT_HD int encode(uint32_t cp, uint8_t out[4]) {
  if (cp < 0x80) {
    out[0] = (uint8_t)cp;
    return 1;
  }
  if (cp < 0x800) {
    out[0] = (uint8_t)(0xC0 | (cp >> 6));
    out[1] = (uint8_t)(0x80 | (cp & 0x3F));
    return 2;
  }
  if (cp < 0x10000) {
    out[0] = (uint8_t)(0xE0 | (cp >> 12));
    out[1] = (uint8_t)(0x80 | ((cp >> 6) & 0x3F));
    out[2] = (uint8_t)(0x80 | (cp & 0x3F));
    return 3;
  }
  out[0] = (uint8_t)(0xF0 | (cp >> 18));
  out[1] = (uint8_t)(0x80 | ((cp >> 12) & 0x3F));
  out[2] = (uint8_t)(0x80 | ((cp >> 6) & 0x3F));
  out[3] = (uint8_t)(0x80 | (cp & 0x3F));
  return 4;
}

// Bytes of the NEXT block covered by the last escape sequence of this block
// (escape starts E are known for the whole block).  Only a start at bit >= 52
// can overhang, and whether it is consumed as the low half of a surrogate
// pair depends on starts >= 40, so the answer does not depend on the
// block's own incoming overhang (<= 11 bytes).
template <class At>
JT_HD int overhang_out(At at, uint64_t blk, uint64_t E) {
  uint64_t cand = E & (~0ULL << 40);
  if (!(E >> 52)) return 0;
  // walk starts from bit 40 upward, skipping consumed lows
  int p = 40;
  int ov = 0;
  while (p < 64) {
    uint64_t rest = cand >> p;
    if (!rest) break;
    p += ctz64(rest);
    uint32_t cp;
    int L = str::escape_at(at, blk + (uint64_t)p, &cp);
    if (L == 0) L = 2;  // invalid: the document fails anyway; stay bounded
    if (p + L > 64) ov = p + L - 64;
    p += L;
  }
  return ov;
}

// Overhang into block `blk` from the bytes before it, computed without the
// previous block's masks: odd_in = parity of the backslash run ending at
// blk-1, in_str = blk-1 is inside a string.  Used for a tile's first block.
template <class At>
JT_HD int overhang_in_scan(At at, uint64_t blk, bool in_str) {
  if (!in_str || blk == 0) return 0;
  const uint64_t lo = blk >= 12 ? blk - 12 : 0;
  // escape starts among [lo, blk): unescaped backslashes, after the last
  // unescaped quote of the window (the string started after it)
  uint32_t starts = 0;  // bit k = position blk - 12 + k
  uint64_t p = blk;
  while (p > lo) {
    uint64_t q = p - 1;
    uint32_t c = at(q);
    if (c == '\\') {
      // run [r0, q]
      uint64_t r0 = q;
      while (r0 > 0 && at(r0 - 1) == '\\') r0--;
      for (uint64_t s = r0; s <= q; s += 2)
        if (s >= lo) starts |= 1u << (uint32_t)(s - (blk - 12));
      p = r0;
      continue;
    }
    if (c == '"') {
      // escaped iff preceded by an odd run
      uint64_t r = q;
      while (r > 0 && at(r - 1) == '\\') r--;
      if (((q - r) & 1) == 0) {  // unescaped quote: the string began here
        starts &= ~((1u << (uint32_t)(q + 1 - (blk - 12))) - 1);
        break;
      }
    }
    p = q;
  }
  int ov = 0;
  uint64_t s = lo;
  while (starts && s < blk) {
    uint32_t k = (uint32_t)(s - (blk - 12));
    uint32_t rest = starts >> k;
    if (!rest) break;
    s += (uint64_t)ctz32(rest);
    uint32_t cp;
    int L = str::escape_at(at, s, &cp);
    if (L == 0) L = 2;
    if (s + (uint64_t)L > blk) ov = (int)(s + (uint64_t)L - blk);
    s += (uint64_t)L;
  }
  return ov;
}

JT_HD uint64_t low_bits(int n) { return n >= 64 ? ~0ULL : ((1ULL << n) - 1); }

JT_HD int hexv(uint32_t c) {
  uint32_t d = c - '0';
  if (d < 10u) return (int)d;
  uint32_t l = (c | 0x20) - 'a';
  return l < 6u ? (int)(l + 10) : -1;
}

JT_HD int hex4w(uint32_t b0, uint32_t b1, uint32_t b2, uint32_t b3) {
  int a = hexv(b0), b = hexv(b1), c = hexv(b2), d = hexv(b3);
  if ((a | b | c | d) < 0) return -1;
  return (a << 12) | (b << 8) | (c << 4) | d;
}

// handle_escape (stringparse.cpp:73-102) on a 12-byte register window
// starting at the backslash: w[k] holds bytes 4k..4k+3 (little endian).
// Returns the consumed length (2, 6 or 12) and the code point, 0 if invalid.
JT_HD int escape_window(const uint32_t w[3], uint32_t *cp) {
  const uint32_t e = (w[0] >> 8) & 0xFF;
  if (e != 'u') {
    uint32_t d = str::escape_char(e);
    *cp = d;
    return d ? 2 : 0;
  }
  int v = hex4w((w[0] >> 16) & 0xFF, w[0] >> 24, w[1] & 0xFF, (w[1] >> 8) & 0xFF);
  if (v < 0) return 0;
  if (v >= 0xD800 && v <= 0xDBFF) {
    if (((w[1] >> 16) & 0xFF) != '\\' || (w[1] >> 24) != 'u') return 0;
    int lo = hex4w(w[2] & 0xFF, (w[2] >> 8) & 0xFF, (w[2] >> 16) & 0xFF, w[2] >> 24);
    if (lo < 0xDC00 || lo > 0xDFFF) return 0;
    *cp = 0x10000u + ((((uint32_t)v - 0xD800u) << 10) | ((uint32_t)lo - 0xDC00u));
    return 12;
  }
  if (v >= 0xDC00 && v <= 0xDFFF) return 0;
  *cp = (uint32_t)v;
  return 6;
}

// String bytes of one block, by segments between escape starts.  Inside a
// segment the weights are popcounts (4 per opening quote, 1 per string
// byte) and the payload is copied as runs; each escape start is decoded.
// kEmit = false measures only.  `byte(k)` returns block-relative byte k
// (k may run past 63 into the next block), `copy_run(a, w, n)` copies block
// bytes [a, a+n) to payload offset w, `put(w, b)` stores one payload byte,
// `mark(p, w)` records index entry p with string offset w.  *err gets the
// minimum string error position (control byte or invalid escape).
template <bool kEmit, class Byte, class CopyRun, class Put, class Mark>
JT_HD uint32_t block_strings(Byte byte, uint64_t blk, uint64_t content, uint64_t openq,
                             uint64_t E, uint64_t ctl, uint64_t fin, int ov, uint64_t *err,
                             CopyRun copy_run, Put put, Mark mark) {
  uint32_t w = 0;
  if (kEmit && ov > 0) {  // index entries inside the incoming escape (invalid input)
    uint64_t fm = fin & low_bits(ov);
    while (fm) {
      mark(ctz64(fm), 0u);
      fm &= fm - 1;
    }
  }
  int p = ov;
  while (p < 64) {
    const uint64_t from = ~0ULL << p;
    const uint64_t rest = E & from;
    const int e = rest ? ctz64(rest) : 64;
    const uint64_t seg = from & low_bits(e);
    const uint64_t cseg = content & seg, oseg = openq & seg;
    const uint64_t cs = ctl & seg;
    if (cs) {
      uint64_t x = blk + (uint64_t)ctz64(cs);
      if (x < *err) *err = x;
    }
    if (kEmit) {
      uint64_t fm = fin & seg;
      while (fm) {
        int f = ctz64(fm);
        uint64_t below = low_bits(f);
        mark(f, w + 4u * popc64(oseg & below) + popc64(cseg & below));
        fm &= fm - 1;
      }
      uint64_t cm = cseg;
      while (cm) {
        int a0 = ctz64(cm);
        uint64_t sh = cm >> a0;
        int n = ~sh == 0 ? 64 - a0 : ctz64(~sh);
        uint64_t below = low_bits(a0);
        copy_run(a0, w + 4u * popc64(oseg & below) + popc64(cseg & below), n);
        cm &= ~(low_bits(n) << a0);
      }
    }
    w += 4u * popc64(oseg) + popc64(cseg);
    if (e >= 64) break;
    uint32_t cp = 0, win[3];
    byte.window12((uint64_t)e, win);
    int L = escape_window(win, &cp);
    if (L == 0) {  // invalid escape: error at the backslash
      uint64_t x = blk + (uint64_t)e;
      if (x < *err) *err = x;
      p = e + 1;
      continue;
    }
    uint8_t b[4];
    int n = L == 2 ? (b[0] = (uint8_t)cp, 1) : encode(cp, b);
    if (kEmit) {
      for (int k = 0; k < n; k++) put(w + (uint32_t)k, b[k]);
      uint64_t fm = fin & (low_bits(e + L < 64 ? e + L : 64) & ~low_bits(e + 1));
      while (fm) {  // index entries inside an escape (invalid input only)
        mark(ctz64(fm), w + (uint32_t)n);
        fm &= fm - 1;
      }
    }
    w += (uint32_t)n;
    p = e + L;
  }
  return w;
}

// Slow-path walker over one block.  Calls emit(pos_in_block, byte) for each
// payload byte in order and mark(pos_in_block, weight_before) for each index
// entry; returns the block weight.  *err gets the first string error
// position (absolute) or stays ~0.  `content`, `openq`, `E`, `fin` are the
// block masks, `ov` the incoming overhang.
template <class At, class Emit, class Mark>
JT_HD uint32_t walk_block(At at, uint64_t blk, uint64_t content, uint64_t openq, uint64_t E,
                          uint64_t ctl, uint64_t fin, int ov, uint64_t *err, Emit emit,
                          Mark mark) {
  uint32_t w = 0;
  int p = 0;
  // index entries inside the overhang region are impossible in a valid
  // string; still report them (bounded behaviour on invalid input)
  while (p < ov && p < 64) {
    if ((fin >> p) & 1) mark(p, w);
    p++;
  }
  while (p < 64) {
    if ((fin >> p) & 1) mark(p, w);
    uint64_t bit = 1ULL << p;
    if (E & bit) {
      uint32_t cp;
      int L = str::escape_at(at, blk + (uint64_t)p, &cp);
      if (L == 0) {
        uint64_t e = blk + (uint64_t)p;
        if (e < *err) *err = e;
        p++;
        continue;
      }
      uint8_t b[4];
      int n = L == 2 ? (b[0] = (uint8_t)cp, 1) : encode(cp, b);
      for (int k = 0; k < n; k++) emit(w + (uint32_t)k, b[k]);
      w += (uint32_t)n;
      // index entries cannot fall inside an escape of a valid string
      int end = p + L;
      for (int k = p + 1; k < end && k < 64; k++)
        if ((fin >> k) & 1) mark(k, w);
      p = end;
      continue;
    }
    if (content & bit) {
      if (ctl & bit) {
        uint64_t e = blk + (uint64_t)p;
        if (e < *err) *err = e;
      }
      emit(w, (uint8_t)at(blk + (uint64_t)p));
      w++;
    } else if (openq & bit) {
      w += 4;
    }
    p++;
  }
  return w;
}

}  // namespace sb
}  // namespace jt
