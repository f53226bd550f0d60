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
// Blocks with escapes decode them (escape_weights) into a weight mask W so
// that every block uses the same popcount formulas; the decoded bytes are
// written after the plain runs (escape_emit).
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
// Decoded length of a valid escape (L = 2, 6 or 12 input bytes).
JT_HD int out_len(int L, uint32_t cp) {
  return L == 2 ? 1 : cp < 0x80 ? 1 : cp < 0x800 ? 2 : cp < 0x10000 ? 3 : 4;
}

// Returns ov | spill << 8: ov = input bytes, spill = weight bytes (see
// escape_weights) of the last escape that fall into the next block.
template <class At>
JT_HD int overhang_out(At at, uint64_t blk, uint64_t E) {
  uint64_t cand = E & (~0ULL << 40);
  if (!(E >> 52)) return 0;
  // walk starts from bit 40 upward, skipping consumed lows
  int p = 40;
  int ov = 0, spill = 0;
  while (p < 64) {
    uint64_t rest = cand >> p;
    if (!rest) break;
    p += ctz64(rest);
    uint32_t cp;
    int L = str::escape_at(at, blk + (uint64_t)p, &cp);
    int n = L ? out_len(L, cp) : 0;
    if (L == 0) L = 2;  // invalid: the document fails anyway; stay bounded
    if (p + L > 64) {
      ov = p + L - 64;
      spill = p + n > 64 ? p + n - 64 : 0;
    }
    p += L;
  }
  return ov | (spill << 8);
}

// Overhang into block `blk` from the bytes before it (ov | spill << 8 as
// overhang_out; *spill_bytes = the spilled decoded bytes, little endian),
// computed without the previous block's masks: odd_in = parity of the backslash run ending at
// blk-1, in_str = blk-1 is inside a string.  Used for a tile's first block.
template <class At>
JT_HD int overhang_in_scan(At at, uint64_t blk, bool in_str, uint32_t *spill_bytes) {
  *spill_bytes = 0;
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
  int ov = 0, spill = 0;
  uint64_t s = lo;
  while (starts && s < blk) {
    uint32_t k = (uint32_t)(s - (blk - 12));
    uint32_t rest = starts >> k;
    if (!rest) break;
    s += (uint64_t)ctz32(rest);
    uint32_t cp;
    int L = str::escape_at(at, s, &cp);
    int n = L ? out_len(L, cp) : 0;
    if (L == 0) L = 2;
    if (s + (uint64_t)L > blk) {
      ov = (int)(s + (uint64_t)L - blk);
      spill = s + (uint64_t)n > blk ? (int)(s + (uint64_t)n - blk) : 0;
      *spill_bytes = 0;
      if (spill) {  // decoded bytes n - spill .. n-1 land in this block
        uint8_t b[4];
        if (L == 2) b[0] = (uint8_t)cp;
        else encode(cp, b);
        for (int k = 0; k < spill; k++) *spill_bytes |= (uint32_t)b[n - spill + k] << (8 * k);
      }
    }
    s += (uint64_t)L;
  }
  return ov | (spill << 8);
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

// Weight mask of a block with escapes.  Every valid escape sequence
// [p, p+L) is given the weight of its decoded bytes by counting its first n
// positions [p, p+n) (n <= L always); its other bytes weigh 0.  Then every
// block's string-buffer prefix at bit x is 4*popc(openq below x) +
// popc(W below x), the same formula as for blocks without escapes.  ov_in /
// vin = input / weight bytes of an escape begun in the previous block.
// *err gets the minimum invalid-escape position (handle_escape,
// stringparse.cpp:73-102).
template <class Byte>
JT_HD uint64_t escape_weights(Byte byte, uint64_t blk, uint64_t content, uint64_t E, int ov_in,
                              int vin, uint64_t *err) {
  uint64_t cov = low_bits(ov_in), virt = low_bits(vin);
  uint64_t rest = E & ~cov;
  while (rest) {
    const int p = ctz64(rest);
    uint32_t cp = 0, win[3];
    byte.window12((uint64_t)p, win);
    const int L = escape_window(win, &cp);
    int end = p + 1;
    if (L == 0) {
      if (blk + (uint64_t)p < *err) *err = blk + (uint64_t)p;
    } else {
      end = p + L;
      cov |= low_bits(end) & ~low_bits(p);
      virt |= low_bits(p + out_len(L, cp)) & ~low_bits(p);
    }
    rest = E & ~low_bits(end);
  }
  return (content & ~cov) | virt;
}

// Decoded bytes of the block's escapes at their string-buffer offsets
// (`put(w, b)`, w block-relative), after the plain runs were copied.
template <class Byte, class Put>
JT_HD void escape_emit(Byte byte, uint64_t E, int ov_in, uint64_t openq, uint64_t W, Put put) {
  uint64_t rest = E & ~low_bits(ov_in);
  while (rest) {
    const int p = ctz64(rest);
    uint32_t cp = 0, win[3];
    byte.window12((uint64_t)p, win);
    const int L = escape_window(win, &cp);
    int end = p + 1;
    if (L != 0) {
      uint8_t b[4];
      const int n = L == 2 ? (b[0] = (uint8_t)cp, 1) : encode(cp, b);
      const uint64_t below = low_bits(p);
      const uint32_t w = 4u * popc64(openq & below) + popc64(W & below);
      for (int k = 0; k < n; k++) put(w + (uint32_t)k, b[k]);
      end = p + L;
    }
    rest = E & ~low_bits(end);
  }
}

}  // namespace sb
}  // namespace jt
