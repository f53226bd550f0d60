// strparse.cuh — string tokens (validate + decoded length, then decode) and
// atoms, bit-exact with the reference.
//
// parse_string (proj/src/stringparse.cpp:143-183) scans 32-byte chunks for
// the first quote / backslash / control byte; handle_escape (73-102) decodes
// \" \\ \/ \b \f \n \r \t and \uXXXX with surrogate pairs.  The first event
// in scan order decides, so a byte-at-a-time scan with the same event order
// is equivalent; end of input reads as NUL (the padding) -> error at len.
// Two passes: string_measure (phase A of the token kernel, before the
// string-buffer offsets are known) and string_decode (phase B).
#pragma once

#include "jt_common.cuh"

namespace jt {
namespace str {

JT_HD int hexval(uint32_t c) {
  if (c - '0' < 10u) return (int)(c - '0');
  uint32_t l = c | 0x20;
  if (l - 'a' < 6u) return (int)(l - 'a' + 10);
  return -1;
}

template <class At>
JT_HD int hex4(At at, uint64_t p) {
  int a = hexval(at(p)), b = hexval(at(p + 1)), c = hexval(at(p + 2)), d = hexval(at(p + 3));
  if ((a | b | c | d) < 0) return -1;
  return (a << 12) | (b << 8) | (c << 4) | d;
}

JT_HD uint32_t escape_char(uint32_t e) {  // kEscapeMap, stringparse.cpp:11-28
  switch (e) {
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

// One escape at p (p points at the backslash).  Returns the number of
// source bytes consumed (2, 6 or 12) and the code point, or 0 on error.
template <class At>
JT_HD int escape_at(At at, uint64_t p, uint32_t *cp) {
  uint32_t e = at(p + 1);
  if (e != 'u') {
    uint32_t d = escape_char(e);
    *cp = d;
    return d ? 2 : 0;
  }
  int v = hex4(at, p + 2);
  if (v < 0) return 0;
  if (v >= 0xD800 && v <= 0xDBFF) {
    if (at(p + 6) != '\\' || at(p + 7) != 'u') return 0;
    int lo = hex4(at, p + 8);
    if (lo < 0xDC00 || lo > 0xDFFF) return 0;
    *cp = 0x10000u + ((((uint32_t)v - 0xD800u) << 10) | ((uint32_t)lo - 0xDC00u));
    return 12;
  }
  if (v >= 0xDC00 && v <= 0xDFFF) return 0;
  *cp = (uint32_t)v;
  return 6;
}

JT_HD uint32_t utf8_len(uint32_t cp) { return cp < 0x80 ? 1 : cp < 0x800 ? 2 : cp < 0x10000 ? 3 : 4; }

struct Measure {
  bool ok;
  uint32_t len;      // decoded payload bytes
  uint64_t err;      // error offset when !ok
};

// Validate the string whose opening quote is at `q` and measure its decoded
// length.
template <class At>
JT_HD Measure string_measure(At at, uint64_t q) {
  Measure m{false, 0, 0};
  uint64_t p = q + 1;
  uint32_t n = 0;
  for (;;) {
    uint32_t c = at(p);
    if (c == '"') {
      m.ok = true;
      m.len = n;
      return m;
    }
    if (c < 0x20) {
      m.err = p;
      return m;
    }
    if (c == '\\') {
      uint32_t cp;
      int k = escape_at(at, p, &cp);
      if (!k) {
        m.err = p;
        return m;
      }
      n += k == 2 ? 1 : utf8_len(cp);
      p += (uint64_t)k;
      continue;
    }
    n++;
    p++;
  }
}

// Decode a validated string into dst (payload only; the caller writes the
// 4-byte length prefix).  `put(i, byte)` stores payload byte i.
template <class At, class Put>
JT_HD void string_decode(At at, uint64_t q, Put put) {
  uint64_t p = q + 1;
  uint32_t n = 0;
  for (;;) {
    uint32_t c = at(p);
    if (c == '"') return;
    if (c == '\\') {
      uint32_t cp;
      int k = escape_at(at, p, &cp);
      if (k == 2) {
        put(n++, (uint8_t)cp);
      } else if (cp < 0x80) {  // encode_utf8, stringparse.cpp:52-69
        put(n++, (uint8_t)cp);
      } else if (cp < 0x800) {
        put(n++, (uint8_t)(0xC0 | (cp >> 6)));
        put(n++, (uint8_t)(0x80 | (cp & 0x3F)));
      } else if (cp < 0x10000) {
        put(n++, (uint8_t)(0xE0 | (cp >> 12)));
        put(n++, (uint8_t)(0x80 | ((cp >> 6) & 0x3F)));
        put(n++, (uint8_t)(0x80 | (cp & 0x3F)));
      } else {
        put(n++, (uint8_t)(0xF0 | (cp >> 18)));
        put(n++, (uint8_t)(0x80 | ((cp >> 12) & 0x3F)));
        put(n++, (uint8_t)(0x80 | ((cp >> 6) & 0x3F)));
        put(n++, (uint8_t)(0x80 | (cp & 0x3F)));
      }
      p += (uint64_t)k;
      continue;
    }
    put(n++, (uint8_t)c);
    p++;
  }
}

JT_HD bool is_sep(uint32_t c) {  // is_separator_byte, tape_builder.cpp:14-30
  return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == ',' || c == ':' ||
         c == '[' || c == ']' || c == '{' || c == '}';
}

// true/false/null: exact literal and a separator, quote or end of input
// next (tape_builder.cpp:92-115, atom_terminated 53-56)
template <class At>
JT_HD bool atom_ok(At at, uint64_t len, uint64_t p, uint32_t c) {
  uint64_t e;
  if (c == 't') {
    if (at(p + 1) != 'r' || at(p + 2) != 'u' || at(p + 3) != 'e') return false;
    e = p + 4;
  } else if (c == 'f') {
    if (at(p + 1) != 'a' || at(p + 2) != 'l' || at(p + 3) != 's' || at(p + 4) != 'e') return false;
    e = p + 5;
  } else {
    if (at(p + 1) != 'u' || at(p + 2) != 'l' || at(p + 3) != 'l') return false;
    e = p + 4;
  }
  if (e >= len) return true;
  uint32_t t = at(e);
  return is_sep(t) || t == '"';
}

// atom_ok on the 8 bytes from p (little endian, w = bytes p..p+7): the
// literal and its terminator in registers, no dependent byte loads
JT_HD bool atom_ok8(uint64_t w, uint64_t len, uint64_t p, uint32_t c) {
  uint64_t e;
  uint32_t t;
  if (c == 't') {
    if ((uint32_t)w != 0x65757274u) return false;  // "true"
    e = p + 4;
    t = (uint32_t)(w >> 32) & 0xFF;
  } else if (c == 'f') {
    if ((w & 0xFFFFFFFFFFULL) != 0x65736c6166ULL) return false;  // "false"
    e = p + 5;
    t = (uint32_t)(w >> 40) & 0xFF;
  } else {
    if ((uint32_t)w != 0x6c6c756eu) return false;  // "null"
    e = p + 4;
    t = (uint32_t)(w >> 32) & 0xFF;
  }
  return e >= len || is_sep(t) || t == '"';
}

}  // namespace str
}  // namespace jt
