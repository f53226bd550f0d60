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
// Blocks with escapes turn them into a weight mask W (block_escapes /
// block_weights) so that every block uses the same popcount formulas, and write each escape's
// decoded bytes IN PLACE over its own weight positions of the tile's shared
// copy (n <= L decoded bytes over the L-byte sequence): the string payload of
// a block is then just its weighted bytes in order, one copy, no fix-ups.
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

// The four hex digits of a \uXXXX escape held in one word (first digit in
// byte 0) as their value, or -1 if any is not a hex digit: every byte at once
// (bytes < 0x80, so the byte-wise range tests carry into no neighbour).
// Same result as hex4w on every word (tests/cpu_string_check.cpp
// jt_cpu_hex4_check, all 2^32).
JT_HD int hex4_swar(uint32_t x) {
  if (x & 0x80808080u) return -1;
  const uint32_t l = x | 0x20202020u;                                           // letters lowered
  const uint32_t dig = (x + 0x50505050u) & ~(x + 0x46464646u);                  // 0x30..0x39
  const uint32_t let = (l + 0x1F1F1F1Fu) & ~(l + 0x19191919u);                  // 0x61..0x66
  if (((dig | let) & 0x80808080u) != 0x80808080u) return -1;
  const uint32_t n = (x & 0x0F0F0F0Fu) + ((let >> 7) & 0x01010101u) * 9u;       // nibble values
  const uint32_t q = byte_perm(n, 0, 0x0123);                                   // n3 n2 n1 n0
  const uint32_t r = q | (q >> 4);
  return (int)((r & 0xFFu) | ((r >> 8) & 0xFF00u));
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
  int v = hex4_swar((w[0] >> 16) | (w[1] << 16));
  if (v < 0) return 0;
  if (v >= 0xD800 && v <= 0xDBFF) {
    if (((w[1] >> 16) & 0xFF) != '\\' || (w[1] >> 24) != 'u') return 0;
    int lo = hex4_swar(w[2]);
    if (lo < 0xDC00 || lo > 0xDFFF) return 0;
    *cp = 0x10000u + ((((uint32_t)v - 0xD800u) << 10) | ((uint32_t)lo - 0xDC00u));
    return 12;
  }
  if (v >= 0xDC00 && v <= 0xDFFF) return 0;
  *cp = (uint32_t)v;
  return 6;
}

// Decoded length of a valid escape (L = 2, 6 or 12 input bytes).
JT_HD int out_len(int L, uint32_t cp) {
  return L == 2 ? 1 : cp < 0x80 ? 1 : cp < 0x800 ? 2 : cp < 0x10000 ? 3 : 4;
}

// Weight positions of a valid escape at p (see block_escapes): a two-byte
// escape weighs on its second byte [p+1, p+2), so that \\ \" \/ need no
// rewrite; a \u escape on [p, p+n).  Returns how many of them are >= end.
JT_HD int spill_of(int p, int L, int n, int end) {
  if (n == 0) return 0;  // invalid escape: no weight moves
  const int a = L == 2 ? p + 1 : p, b = a + n;
  return b > end ? b - (a > end ? a : end) : 0;
}

// Overhang into block `blk` from the bytes before it (ov | spill << 8 as
// block_escapes' ov_out; *spill_bytes = the spilled decoded bytes, little endian),
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
      spill = spill_of((int)(s - (blk - 64)), L, n, 64);
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

// Escape starts of a block by the class of the following byte: two-byte
// escapes whose output is that byte (\" \\ \/), two-byte escapes that are
// translated (\b \f \n \r \t), \u escapes, and invalid ones (handle_escape,
// stringparse.cpp:73-102).
struct EscClass {
  uint64_t sim, tr, u, bad;
};

// 0 if c is not a two-byte escape letter, else the decoded byte
JT_HD uint32_t simple_decode(uint32_t c) {
  switch (c) {
    case '"': return '"';
    case '\\': return '\\';
    case '/': return '/';
    case 'b': return 0x08;
    case 'f': return 0x0C;
    case 'n': return 0x0A;
    case 'r': return 0x0D;
    case 't': return 0x09;
    default: return 0;
  }
}

// E = escape starts; c64 = the byte after bit 63 (next block's byte 0).
JT_HD EscClass classify_escapes(const uint64_t P[8], uint64_t qt, uint64_t bs, uint64_t E,
                                uint32_t c64) {
  const uint64_t n7 = ~P[7], n6 = ~P[6], n5 = ~P[5], n4 = ~P[4], n3 = ~P[3], n2 = ~P[2],
                 n1 = ~P[1], n0 = ~P[0];
  const uint64_t slash = n7 & n6 & P[5] & n4 & P[3] & P[2] & P[1] & P[0];  // 0x2F
  const uint64_t h6 = n7 & P[6] & P[5] & n4;                              // 0x6_
  const uint64_t h7 = n7 & P[6] & P[5] & P[4];                            // 0x7_
  const uint64_t lb = h6 & n3 & n2 & P[1] & n0;                           // b 0x62
  const uint64_t lf = h6 & n3 & P[2] & P[1] & n0;                         // f 0x66
  const uint64_t ln = h6 & P[3] & P[2] & P[1] & n0;                       // n 0x6E
  const uint64_t lr = h7 & n3 & n2 & P[1] & n0;                           // r 0x72
  const uint64_t lt = h7 & n3 & P[2] & n1 & n0;                           // t 0x74
  const uint64_t lu = h7 & n3 & P[2] & n1 & P[0];                         // u 0x75
  const uint64_t S = qt | bs | slash, T = lb | lf | ln | lr | lt;
  const uint32_t d64 = simple_decode(c64);
  const uint64_t s64 = (d64 != 0 && (c64 == '"' || c64 == '\\' || c64 == '/')) ? 1 : 0;
  const uint64_t t64 = (d64 != 0 && !s64) ? 1 : 0, u64 = c64 == 'u' ? 1 : 0;
  const uint64_t nS = (S >> 1) | (s64 << 63), nT = (T >> 1) | (t64 << 63),
                 nU = (lu >> 1) | (u64 << 63);
  return EscClass{E & nS, E & nT, E & nU, E & ~(nS | nT | nU)};
}

// ---- \u escapes decided from the bit planes ---------------------------------
// handle_escape's \uXXXX checks (stringparse.cpp:86-101) for every escape
// start of a block at once: hex-digit, 'D', "8..B" and "C..F" byte classes
// from the planes, shifted onto the start's bit.  A start p is decided here
// when every byte it depends on lies in the block (p + 5 <= 63, for the high
// half of a pair p + 11 <= 63); the rest (`und`) are decoded one at a time
// from the bytes (decode_und).  In a prefix without errors the set of valid
// escapes equals the sequential walk's: a start is skipped by the walk iff it
// is the low half of a valid pair (the only backslash a valid escape covers),
// which is `pair << 6` here; after the first error only the minimum matters.
struct UClass {
  uint64_t bmp, pair;  // valid \uXXXX (no surrogate) / \uD8..\uDC.. pairs inside the block
  uint64_t n1, n3;     // bmp escapes that decode to 1 byte / to 3 bytes (else 2)
  uint64_t bad;        // failing starts: a non-hex digit, a lone surrogate half
  uint64_t und;        // starts that need bytes of the next block
};

JT_HD UClass classify_u(const uint64_t P[8], uint64_t U) {
  const uint64_t n7 = ~P[7], n6 = ~P[6], n4 = ~P[4], n3 = ~P[3], n2 = ~P[2], n1 = ~P[1], n0 = ~P[0];
  const uint64_t dig = n7 & n6 & P[5] & P[4] & (n3 | (n2 & n1));               // 0..9
  const uint64_t let = n7 & P[6] & n4 & n3 & (P[2] | P[1] | P[0]) & ~(P[2] & P[1] & P[0]);  // A..F a..f
  const uint64_t hexd = dig | let;
  const uint64_t zero = dig & n3 & n2 & n1 & n0;                                // 0
  const uint64_t lt8 = dig & n3;                                                // 0..7
  const uint64_t isD = let & P[2] & n1 & n0;                                    // D d
  const uint64_t c8B = (dig & P[3]) | (let & n2 & (P[1] ^ P[0]));               // 8 9 A B a b
  const uint64_t cCF = let & (P[2] | (P[1] & P[0]));                            // C..F c..f
  const uint64_t h4 = (hexd >> 2) & (hexd >> 3) & (hexd >> 4) & (hexd >> 5);
  const uint64_t kDec6 = (1ULL << 59) - 1, kDec12 = (1ULL << 53) - 1;
  const uint64_t Ud = U & kDec6;
  const uint64_t ok = Ud & h4;
  const uint64_t d0D = isD >> 2;
  const uint64_t hiS = ok & d0D & (c8B >> 3), loS = ok & d0D & (cCF >> 3);
  UClass r;
  r.bmp = ok & ~(hiS | loS);
  r.pair = hiS & (loS >> 6) & kDec12;
  r.bad = (Ud & ~h4) | (hiS & kDec12 & ~(loS >> 6)) | (loS & ~(r.pair << 6));
  r.und = (U & ~kDec6) | (hiS & ~kDec12);
  const uint64_t t = (zero >> 2) & (lt8 >> 3);  // code point < 0x800
  r.n3 = r.bmp & ~t;
  r.n1 = r.bmp & t & (zero >> 3) & (lt8 >> 4);  // < 0x80
  return r;
}

// bytes the decided escapes cover / the weight positions of their decoded
// bytes (the first n bytes of each sequence, see escape_weights)
JT_HD void u_masks(const UClass &u, uint64_t *cov, uint64_t *virt) {
  const uint64_t a = u.bmp | u.pair;
  const uint64_t h = a | (u.pair << 6);  // six-byte halves
  const uint64_t s2 = h | (h << 1);
  const uint64_t s4 = s2 | (s2 << 2);
  *cov = s4 | (s2 << 4);
  *virt = a | ((a & ~u.n1) << 1) | ((u.n3 | u.pair) << 2) | (u.pair << 3);
}

// four hex digits known to be valid (first digit in byte 0) -> value
JT_HD uint32_t hex4_value(uint32_t x) {
  const uint32_t n = (x & 0x0F0F0F0Fu) + ((x >> 6) & 0x01010101u) * 9u;
  const uint32_t q = byte_perm(n, 0, 0x0123);
  const uint32_t r = q | (q >> 4);
  return (r & 0xFFu) | ((r >> 8) & 0xFF00u);
}

// The undecided starts in order (each reads bytes of the next block through
// `byte`): failing ones go to *bad; returns p | L << 6 | cp << 10 of the last
// valid one (it reaches past the block: at most one in a block), 0 if none.
template <class Byte>
JT_HD uint32_t decode_und(Byte byte, uint64_t und, uint64_t *bad) {
  uint32_t res = 0;
  uint64_t rest = und;
  while (rest) {
    const int p = ctz64(rest);
    uint32_t cp = 0, win[3];
    byte.window12((uint64_t)p, win);
    const int L = escape_window(win, &cp);
    int end = p + 1;
    if (L == 0) {
      *bad |= 1ULL << p;
    } else {
      end = p + L;
      res = (uint32_t)p | ((uint32_t)L << 6) | (cp << 10);
    }
    rest = und & ~low_bits(end);
  }
  return res;
}

// \b \f \n \r \t -> the control byte (a 16 x 4-bit table indexed by bits 1..4
// of the letter: b 1, f 3, n 7, r 9, t 10)
JT_HD uint32_t translate_letter(uint32_t c) {
  const uint32_t k = (c >> 1) & 15;
  const uint32_t lo = 0xA000C080u;  // nibble 1 = 8 (\b), 3 = C (\f), 7 = A (\n)
  const uint32_t hi = 0x000009D0u;  // nibble 9 = D (\r), 10 = 9 (\t)
  return (((k & 8) ? hi : lo) >> (4 * (k & 7))) & 15;
}

JT_HD EscClass restrict_from(const EscClass &c, int ov_in) {
  const uint64_t k = ~low_bits(ov_in);
  return EscClass{c.sim & k, c.tr & k, c.u & k, c.bad & k};
}

// ---- a block's escapes in three steps ---------------------------------------
// Every valid escape sequence [p, p+L) carries the weight of its decoded bytes
// on n of its own positions: the second byte of a two-byte escape (so that
// \\ \" \/ are already right when the weighted bytes are copied), the first n
// bytes of a \u escape; its other bytes weigh 0.  Then every block's
// string-buffer prefix at bit x is 4*popc(openq below x) + popc(W below x),
// the same formula as for blocks without escapes.
//
// 1. block_escapes (needs nothing from other blocks): the escape classes,
//    the coverage / weight masks of the \u escapes, the failing starts, and
//    ov | spill << 8 = input bytes / weight bytes of the last escape that fall
//    into the NEXT block.  An escape that reaches past the block is decoded
//    here and its bytes go to their weight positions right away (rewrite(k, b)
//    with k possibly >= 64: the next block copies them as its first `spill`
//    weighted bytes; the caller drops positions past its tile).
// 2. block_weights, once ov_in / vin (the previous block's ov / spill) are
//    known: the weight mask W and the failing starts outside the overhang.
// 3. decode_in_place, any time before the block's weighted bytes are copied:
//    the decoded bytes of the escapes inside the block over their weight
//    positions (\" \\ \/ decode to their own second byte: nothing to do).
struct BlockEsc {
  EscClass ec;
  uint64_t bmp, pair;    // decided \u escapes (see UClass)
  uint64_t ucov, uvirt;  // bytes covered by / weight positions of the block's \u escapes
  uint64_t bad;          // failing escape starts
  int ov_out;
};

template <class Byte, class Rewrite>
JT_HD BlockEsc block_escapes(const uint64_t P[8], uint64_t qt, uint64_t bs, uint64_t E, Byte byte,
                             Rewrite rewrite) {
  BlockEsc r;
  r.ec = classify_escapes(P, qt, bs, E, (E >> 63) ? byte(64) : 0u);
  r.bmp = r.pair = r.ucov = r.uvirt = 0;
  r.bad = r.ec.bad;
  r.ov_out = 0;
  if (r.ec.u) {
    const UClass uc = classify_u(P, r.ec.u);
    u_masks(uc, &r.ucov, &r.uvirt);
    r.bmp = uc.bmp;
    r.pair = uc.pair;
    r.bad |= uc.bad;
    if (uc.und) {
      const uint32_t res = decode_und(byte, uc.und, &r.bad);
      if (res) {
        const int p = (int)(res & 63), L = (int)((res >> 6) & 15);
        uint8_t b[4];
        const int n = encode(res >> 10, b);
        for (int k = 0; k < n; k++) rewrite(p + k, b[k]);
        if (p + L > 64) r.ov_out = (p + L - 64) | (spill_of(p, L, n, 64) << 8);
        r.ucov |= low_bits(p + L) & ~low_bits(p);
        r.uvirt |= low_bits(p + n) & ~low_bits(p);
      }
    }
  }
  // a two-byte escape at bit 63 covers the next block's byte 0, which also
  // carries its weight
  if ((r.ec.sim | r.ec.tr) >> 63) {
    r.ov_out = 1 | (1 << 8);
    if (r.ec.tr >> 63) rewrite(64, (uint8_t)translate_letter(byte(64)));
  } else if (r.ec.bad >> 63) {
    r.ov_out = 1;
  }
  return r;
}

// ov_in / vin = input / weight bytes of an escape begun in the previous block
JT_HD uint64_t block_weights(uint64_t content, BlockEsc &e, int ov_in, int vin) {
  const uint64_t over = low_bits(ov_in);
  e.bad &= ~over;
  e.bmp &= ~over;
  e.pair &= ~over;
  e.ec.tr &= ~over;
  return (content & ~(over | e.ec.sim | e.ec.tr | e.ucov)) | low_bits(vin) | e.uvirt;
}

// UTF-8 bytes of a code point as a little-endian word (first byte lowest)
JT_HD uint32_t encode4_word(uint32_t cp) {  // cp >= 0x10000
  return 0x808080F0u | (cp >> 18) | (((cp >> 12) & 0x3Fu) << 8) | (((cp >> 6) & 0x3Fu) << 16) |
         ((cp & 0x3Fu) << 24);
}
JT_HD uint32_t encode123_word(uint32_t cp, int *n) {  // cp < 0x10000
  if (cp < 0x80u) {
    *n = 1;
    return cp;
  }
  if (cp < 0x800u) {
    *n = 2;
    return 0x80C0u | (cp >> 6) | ((cp & 0x3Fu) << 8);
  }
  *n = 3;
  return 0x8080E0u | (cp >> 12) | (((cp >> 6) & 0x3Fu) << 8) | ((cp & 0x3Fu) << 16);
}

// window(p, w): 12 bytes from block-relative p (only bytes inside the block
// are used); byte(q): block-relative byte q < 64; put(k, b): decoded byte b to
// block-relative k < 64
template <class Window, class Byte, class Put>
JT_HD void decode_in_place(uint64_t tr, uint64_t bmp, uint64_t pair, Window window, Byte byte, Put put) {
  for (uint64_t t = tr & ~(1ULL << 63); t; t &= t - 1) {
    const int q = ctz64(t) + 1;
    put(q, (uint8_t)translate_letter(byte((uint64_t)q)));
  }
  for (uint64_t r = bmp | pair; r; r &= r - 1) {
    const int p = ctz64(r);
    uint32_t win[3];
    window((uint64_t)p, win);
    const uint32_t v = hex4_value((win[0] >> 16) | (win[1] << 16));
    if ((pair >> p) & 1) {
      const uint32_t lo = hex4_value(win[2]);
      const uint32_t w = encode4_word(0x10000u + (((v - 0xD800u) << 10) | (lo - 0xDC00u)));
      put(p, (uint8_t)w);
      put(p + 1, (uint8_t)(w >> 8));
      put(p + 2, (uint8_t)(w >> 16));
      put(p + 3, (uint8_t)(w >> 24));
    } else {
      int n;
      const uint32_t w = encode123_word(v, &n);
      put(p, (uint8_t)w);
      if (n > 1) put(p + 1, (uint8_t)(w >> 8));
      if (n > 2) put(p + 2, (uint8_t)(w >> 16));
    }
  }
}

}  // namespace sb
}  // namespace jt
