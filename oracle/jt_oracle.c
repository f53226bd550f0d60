/* jt_oracle.c — scalar CPU restatement of the reference parse path.
 * TEST INFRASTRUCTURE ONLY (see jt_oracle.h): the parity checker for the
 * B200 kernels, never part of the product path.
 *
 * Every function cites the reference file:line it restates
 * (/root/reference/proj/...).  Byte-at-a-time on purpose: an independent
 * formulation of the SIMD reference, so agreement is evidence. */
#define _GNU_SOURCE
#include "jt_oracle.h"

#include <errno.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#define PADDING 64 /* proj/src/indexer.h:17 */
#define MAX_DEPTH 1024 /* proj/src/tape_builder.cpp:12 */

static uint64_t tape_word(uint8_t tag, uint64_t payload) {
  /* proj/src/tape.h:30-32 */
  return ((uint64_t)tag << 56) | (payload & ((1ULL << 56) - 1));
}

/* ---------------------------------------------------------------- UTF-8 */

/* proj/src/utf8.cpp:200-243: sequential walk, first failing sequence start */
long long jto_utf8_error_offset(const uint8_t *data, size_t len) {
  size_t i = 0;
  while (i < len) {
    uint8_t b = data[i];
    if (b < 0x80) {
      i++;
      continue;
    }
    int n;
    uint8_t lo = 0x80, hi = 0xBF;
    if (b >= 0xC2 && b <= 0xDF) {
      n = 2;
    } else if (b == 0xE0) {
      n = 3;
      lo = 0xA0;
    } else if ((b >= 0xE1 && b <= 0xEC) || b == 0xEE || b == 0xEF) {
      n = 3;
    } else if (b == 0xED) {
      n = 3;
      hi = 0x9F;
    } else if (b == 0xF0) {
      n = 4;
      lo = 0x90;
    } else if (b >= 0xF1 && b <= 0xF3) {
      n = 4;
    } else if (b == 0xF4) {
      n = 4;
      hi = 0x8F;
    } else {
      return (long long)i;
    }
    if (i + (size_t)n > len)
      return (long long)i;
    if (data[i + 1] < lo || data[i + 1] > hi)
      return (long long)i;
    for (int k = 2; k < n; k++)
      if (data[i + k] < 0x80 || data[i + k] > 0xBF)
        return (long long)i;
    i += (size_t)n;
  }
  return -1;
}

/* ------------------------------------------------------------- stage 1 */

static int is_ws(uint8_t c) { /* blocks.h:88-93 table semantics */
  return c == ' ' || c == '\t' || c == '\n' || c == '\r';
}
static int is_structural(uint8_t c) {
  return c == ',' || c == ':' || c == '[' || c == ']' || c == '{' || c == '}';
}

/* proj/src/indexer.cpp:29-56 with the per-block algebra of
 * blocks.h:58-194 restated per byte: escaped = previous backslash run has
 * odd length (odd_backslash_ends, 58-75); in_string = inclusive prefix XOR of
 * unescaped quotes (string_mask, 79-85); final = finalize_structurals
 * (155-168) with prev_separator starting at 1 (scan_carry, 31-35). */
int jto_stage1(const uint8_t *data, size_t len, jto_result *r) {
  r->index = NULL;
  r->index_count = 0;
  if ((uint64_t)len >= (1ULL << 32)) { /* indexer.cpp:33-34 */
    r->code = JTO_CAPACITY;
    r->offset = -1;
    return r->code;
  }
  long long bad = jto_utf8_error_offset(data, len); /* indexer.cpp:35-36 */
  if (bad >= 0) {
    r->code = JTO_UTF8_ERROR;
    r->offset = bad;
    return r->code;
  }
  uint32_t *idx = (uint32_t *)malloc((len + 1) * sizeof(uint32_t));
  size_t n = 0;
  int run_odd = 0, in_string = 0, prev_sep = 1;
  for (size_t i = 0; i < len; i++) {
    uint8_t c = data[i];
    int escaped = run_odd;
    run_odd = c == '\\' ? !run_odd : 0;
    int uq = c == '"' && !escaped;
    if (uq)
      in_string = !in_string;
    int st = is_structural(c), ws = is_ws(c);
    int fin = (st && !in_string) || (uq && in_string) ||
              (prev_sep && !ws && !in_string && !uq);
    if (fin)
      idx[n++] = (uint32_t)i;
    prev_sep = (st && !in_string) || uq || ws;
  }
  r->index = idx;
  r->index_count = n;
  r->code = JTO_OK;
  r->offset = -1;
  return JTO_OK;
}

/* jt_minify (capi.cpp:154-167): full parse, then minify_pass
 * (indexer.cpp:58-75): keep in-string bytes (opening quote included),
 * unescaped quotes (the closing one) and every non-whitespace byte. */
int jto_minify(const uint8_t *data, size_t len, uint8_t *out, size_t *out_len, long long *offset) {
  jto_result r;
  int code = jto_parse(data, len, &r);
  *offset = r.offset;
  jto_free(&r);
  *out_len = 0;
  if (code != JTO_OK) return code;
  size_t n = 0;
  int run_odd = 0, in_string = 0;
  for (size_t i = 0; i < len; i++) {
    uint8_t c = data[i];
    int escaped = run_odd;
    run_odd = c == '\\' ? !run_odd : 0;
    int uq = c == '"' && !escaped;
    if (uq) in_string = !in_string;
    if (in_string || uq || !is_ws(c)) out[n++] = c;
  }
  *out_len = n;
  return JTO_OK;
}

/* ------------------------------------------------------------- strings */

static int hex_value(uint8_t c) { /* stringparse.cpp:30-38 */
  if (c >= '0' && c <= '9')
    return c - '0';
  if (c >= 'a' && c <= 'f')
    return c - 'a' + 10;
  if (c >= 'A' && c <= 'F')
    return c - 'A' + 10;
  return -1;
}

static int parse_hex4(const uint8_t *p) { /* stringparse.cpp:41-50 */
  int v = 0;
  for (int i = 0; i < 4; i++) {
    int h = hex_value(p[i]);
    if (h < 0)
      return -1;
    v = (v << 4) | h;
  }
  return v;
}

static uint8_t *encode_utf8(uint32_t cp, uint8_t *dst) { /* 52-69 */
  if (cp < 0x80) {
    *dst++ = (uint8_t)cp;
  } else if (cp < 0x800) {
    *dst++ = (uint8_t)(0xC0 | (cp >> 6));
    *dst++ = (uint8_t)(0x80 | (cp & 0x3F));
  } else if (cp < 0x10000) {
    *dst++ = (uint8_t)(0xE0 | (cp >> 12));
    *dst++ = (uint8_t)(0x80 | ((cp >> 6) & 0x3F));
    *dst++ = (uint8_t)(0x80 | (cp & 0x3F));
  } else {
    *dst++ = (uint8_t)(0xF0 | (cp >> 18));
    *dst++ = (uint8_t)(0x80 | ((cp >> 12) & 0x3F));
    *dst++ = (uint8_t)(0x80 | ((cp >> 6) & 0x3F));
    *dst++ = (uint8_t)(0x80 | (cp & 0x3F));
  }
  return dst;
}

static uint8_t escape_map(uint8_t e) { /* kEscapeMap, stringparse.cpp:11-28 */
  switch (e) {
  case '"': return '"';
  case '/': return '/';
  case '\\': return '\\';
  case 'b': return 0x08;
  case 'f': return 0x0C;
  case 'n': return 0x0A;
  case 'r': return 0x0D;
  case 't': return 0x09;
  default: return 0;
  }
}

/* handle_escape, stringparse.cpp:73-102 (src points at the backslash) */
static int handle_escape(const uint8_t *buf, size_t *src, uint8_t **dst) {
  size_t p = *src;
  uint8_t esc = buf[p + 1];
  if (esc == 'u') {
    int cp = parse_hex4(buf + p + 2);
    if (cp < 0)
      return 0;
    p += 6;
    if (cp >= 0xD800 && cp <= 0xDBFF) {
      if (buf[p] != '\\' || buf[p + 1] != 'u')
        return 0;
      int low = parse_hex4(buf + p + 2);
      if (low < 0xDC00 || low > 0xDFFF)
        return 0;
      cp = 0x10000 + (((cp - 0xD800) << 10) | (low - 0xDC00));
      p += 6;
    } else if (cp >= 0xDC00 && cp <= 0xDFFF) {
      return 0;
    }
    *dst = encode_utf8((uint32_t)cp, *dst);
  } else {
    uint8_t d = escape_map(esc);
    if (d == 0)
      return 0;
    *(*dst)++ = d;
    p += 2;
  }
  *src = p;
  return 1;
}

/* parse_string, stringparse.cpp:143-183, one byte at a time: the first of
 * {closing quote, backslash, control byte < 0x20} in scan order decides.
 * `buf` must carry >= 64 zero bytes past len (indexer.h:20-25). */
int jto_parse_string(const uint8_t *buf, size_t len, size_t offset,
                     uint8_t *dst, uint32_t *out_len, long long *err_off) {
  (void)len;
  uint8_t *out = dst + 4;
  size_t src = offset + 1;
  for (;;) {
    uint8_t c = buf[src];
    if (c == '"') {
      uint32_t n = (uint32_t)(out - (dst + 4));
      memcpy(dst, &n, 4);
      *out_len = n;
      return 1;
    }
    if (c < 0x20) {
      *err_off = (long long)src;
      return 0;
    }
    if (c == '\\') {
      if (!handle_escape(buf, &src, &out)) {
        *err_off = (long long)src;
        return 0;
      }
      continue;
    }
    *out++ = c;
    src++;
  }
}

/* ------------------------------------------------------------- numbers */

static int is_digit(uint8_t c) { return c >= '0' && c <= '9'; }

static int is_number_terminator(uint8_t c) { /* numbers.cpp:14-30 */
  return is_ws(c) || is_structural(c);
}

static const double kPow10[23] = {1e0,  1e1,  1e2,  1e3,  1e4,  1e5,
                                  1e6,  1e7,  1e8,  1e9,  1e10, 1e11,
                                  1e12, 1e13, 1e14, 1e15, 1e16, 1e17,
                                  1e18, 1e19, 1e20, 1e21, 1e22};

/* slow_float, numbers.cpp:37-48: glibc strtod on the unsigned substring;
 * overflow rejected, underflow accepted */
static int slow_float(const uint8_t *begin, size_t n, double *out) {
  char *token = (char *)malloc(n + 1);
  memcpy(token, begin, n);
  token[n] = 0;
  errno = 0;
  char *end = NULL;
  double d = strtod(token, &end);
  int ok = end == token + n;
  if (errno == ERANGE && (d == HUGE_VAL || d == -HUGE_VAL))
    ok = 0;
  free(token);
  if (ok)
    *out = d;
  return ok;
}

/* parse_number, numbers.cpp:52-178.  The reference's eight-digit SWAR path
 * (numbers.cpp:88-95, 106-113) is the same arithmetic as eight add_digit
 * steps while digits + 8 <= 19, so one digit at a time here. */
int jto_parse_number(const uint8_t *buf, size_t len, size_t offset,
                     int *is_integer, uint64_t *bits) {
  size_t p = offset;
  int negative = 0;
  if (p < len && buf[p] == '-') {
    negative = 1;
    p++;
  }
  if (p >= len || !is_digit(buf[p]))
    return 0;
  uint64_t mant = 0;
  int digits = 0, truncated = 0;
  long long exp10 = 0;
#define ADD_DIGIT(d, frac)                                                   \
  do {                                                                       \
    if (digits < 19) {                                                       \
      mant = mant * 10 + (d);                                                \
      digits++;                                                              \
      if (frac)                                                              \
        exp10--;                                                             \
    } else {                                                                 \
      if ((d) != 0 || !(frac))                                               \
        truncated = 1;                                                       \
      if (!(frac))                                                           \
        exp10++;                                                             \
    }                                                                        \
  } while (0)
  if (buf[p] == '0') { /* numbers.cpp:82-85 */
    p++;
    if (p < len && is_digit(buf[p]))
      return 0;
  } else {
    while (p < len && is_digit(buf[p])) {
      ADD_DIGIT(buf[p] - '0', 0);
      p++;
    }
  }
  int has_frac = 0, has_exp = 0;
  if (p < len && buf[p] == '.') { /* numbers.cpp:99-118 */
    has_frac = 1;
    p++;
    size_t fs = p;
    while (p < len && is_digit(buf[p])) {
      ADD_DIGIT(buf[p] - '0', 1);
      p++;
    }
    if (p == fs)
      return 0;
  }
  if (p < len && (buf[p] == 'e' || buf[p] == 'E')) { /* numbers.cpp:120-138 */
    has_exp = 1;
    p++;
    int eneg = 0;
    if (p < len && (buf[p] == '+' || buf[p] == '-')) {
      eneg = buf[p] == '-';
      p++;
    }
    size_t es = p;
    long long ev = 0;
    while (p < len && is_digit(buf[p])) {
      if (ev < 1000000000)
        ev = ev * 10 + (buf[p] - '0');
      p++;
    }
    if (p == es)
      return 0;
    exp10 += eneg ? -ev : ev;
  }
#undef ADD_DIGIT
  (void)has_exp;
  if (p < len && !is_number_terminator(buf[p])) /* numbers.cpp:140-141 */
    return 0;
  if (!has_frac && !has_exp) { /* numbers.cpp:146-157 */
    if (truncated || exp10 > 0)
      return 0;
    uint64_t limit = negative ? 0x8000000000000000ULL : 0x7FFFFFFFFFFFFFFFULL;
    if (mant > limit)
      return 0;
    *is_integer = 1;
    *bits = negative ? 0ULL - mant : mant;
    return 1;
  }
  double d; /* numbers.cpp:159-177 */
  if (!truncated && mant <= (1ULL << 53) && exp10 >= -22 && exp10 <= 22) {
    d = (double)mant;
    d = exp10 < 0 ? d / kPow10[-exp10] : d * kPow10[exp10];
  } else if (mant == 0 && !truncated) {
    d = 0.0;
  } else if (exp10 > 340) {
    return 0;
  } else if (exp10 < -360 - digits) {
    d = 0.0;
  } else {
    size_t ds = offset + (negative ? 1 : 0);
    if (!slow_float(buf + ds, p - ds, &d))
      return 0;
  }
  if (negative)
    d = -d;
  *is_integer = 0;
  memcpy(bits, &d, 8);
  return 1;
}

/* ------------------------------------------------------------- stage 2 */

static int is_atom_sep(uint8_t c) { /* tape_builder.cpp:14-30 */
  return is_ws(c) || is_structural(c);
}

typedef struct {
  const uint8_t *buf;
  size_t len;
  const uint32_t *pos;
  size_t count;
  uint64_t *tape;
  size_t used;
  uint8_t *strings;
  size_t sused;
  int code;
  long long off;
} builder;

/* tape_builder::emit_scalar, tape_builder.cpp:77-138 */
static int emit_scalar(builder *b, size_t token) {
  size_t off = b->pos[token];
  uint8_t c = b->buf[off];
  const char *lit = NULL;
  size_t ln = 0;
  switch (c) {
  case '"': {
    uint32_t n;
    long long e;
    if (!jto_parse_string(b->buf, b->len, off, b->strings + b->sused, &n, &e)) {
      b->code = JTO_STRING_ERROR;
      b->off = e;
      return 0;
    }
    b->tape[b->used++] = tape_word('"', b->sused);
    b->sused += 4 + n;
    return 1;
  }
  case 't': lit = "true"; ln = 4; break;
  case 'f': lit = "false"; ln = 5; break;
  case 'n': lit = "null"; ln = 4; break;
  default: break;
  }
  if (lit) { /* tape_builder.cpp:92-115, atom_terminated 53-56 */
    size_t e = off + ln;
    if (memcmp(b->buf + off, lit, ln) != 0 ||
        !(e >= b->len || is_atom_sep(b->buf[e]) || b->buf[e] == '"')) {
      b->code = JTO_TAPE_ERROR;
      b->off = (long long)off;
      return 0;
    }
    b->tape[b->used++] = tape_word(c, 0);
    return 1;
  }
  if (c != '-' && !is_digit(c)) {
    b->code = JTO_TAPE_ERROR;
    b->off = (long long)off;
    return 0;
  }
  int is_int;
  uint64_t bits;
  if (!jto_parse_number(b->buf, b->len, off, &is_int, &bits)) {
    b->code = JTO_NUMBER_ERROR;
    b->off = (long long)off;
    return 0;
  }
  b->tape[b->used++] = tape_word(is_int ? 'l' : 'd', 0);
  b->tape[b->used++] = bits;
  return 1;
}

enum { S_VALUE, S_OBJ_FIRST, S_OBJ_KEY, S_ARR_FIRST, S_AFTER, S_CLOSE };

/* tape_builder::run, tape_builder.cpp:140-258 (goto machine as a loop) */
static void build_tape(builder *b) {
  size_t stack_open[MAX_DEPTH];
  uint8_t stack_obj[MAX_DEPTH];
  size_t depth = 0;
  b->code = JTO_OK;
  b->off = -1;
  if (b->count == 0) { /* 144-145 */
    b->code = JTO_EMPTY;
    return;
  }
#define TAPE_FAIL(tok)                                                       \
  do {                                                                       \
    b->code = JTO_TAPE_ERROR;                                                \
    b->off = (tok) < b->count ? (long long)b->pos[tok] : (long long)b->len;  \
    return;                                                                  \
  } while (0)
  b->tape[b->used++] = tape_word('r', 0);
  size_t i = 0;
  int state = S_VALUE;
  for (;;) {
    switch (state) {
    case S_VALUE: { /* 158-181 */
      if (i >= b->count)
        TAPE_FAIL(i);
      uint8_t c = b->buf[b->pos[i]];
      if (c == '{' || c == '[') {
        if (depth == MAX_DEPTH) {
          b->code = JTO_DEPTH_ERROR;
          b->off = (long long)b->pos[i];
          return;
        }
        stack_open[depth] = b->used;
        stack_obj[depth] = c == '{';
        depth++;
        b->tape[b->used++] = tape_word(c, 0);
        i++;
        state = c == '{' ? S_OBJ_FIRST : S_ARR_FIRST;
      } else {
        if (!emit_scalar(b, i))
          return;
        i++;
        state = S_AFTER;
      }
      break;
    }
    case S_OBJ_FIRST: /* 183-188 */
      if (i >= b->count)
        TAPE_FAIL(i);
      state = b->buf[b->pos[i]] == '}' ? S_CLOSE : S_OBJ_KEY;
      break;
    case S_OBJ_KEY: /* 190-199 */
      if (i >= b->count || b->buf[b->pos[i]] != '"')
        TAPE_FAIL(i);
      if (!emit_scalar(b, i))
        return;
      i++;
      if (i >= b->count || b->buf[b->pos[i]] != ':')
        TAPE_FAIL(i);
      i++;
      state = S_VALUE;
      break;
    case S_ARR_FIRST: /* 201-206 */
      if (i >= b->count)
        TAPE_FAIL(i);
      state = b->buf[b->pos[i]] == ']' ? S_CLOSE : S_VALUE;
      break;
    case S_AFTER: { /* 208-238 */
      if (depth == 0) {
        if (i != b->count)
          TAPE_FAIL(i);
        goto finish;
      }
      if (i >= b->count)
        TAPE_FAIL(i);
      uint8_t c = b->buf[b->pos[i]];
      if (c == ',') {
        i++;
        state = stack_obj[depth - 1] ? S_OBJ_KEY : S_VALUE;
      } else if (c == (stack_obj[depth - 1] ? '}' : ']')) {
        state = S_CLOSE;
      } else {
        TAPE_FAIL(i);
      }
      break;
    }
    case S_CLOSE: { /* 240-250 */
      depth--;
      size_t open = stack_open[depth];
      int obj = stack_obj[depth];
      if (b->buf[b->pos[i]] != (obj ? '}' : ']'))
        TAPE_FAIL(i);
      b->tape[b->used++] = tape_word(obj ? '}' : ']', open);
      b->tape[open] = tape_word((uint8_t)(b->tape[open] >> 56), b->used);
      i++;
      state = S_AFTER;
      break;
    }
    }
  }
finish: /* 252-257 */
  b->tape[0] = tape_word('r', b->used);
  b->tape[b->used++] = tape_word('r', 0);
#undef TAPE_FAIL
}

/* jt_parse, capi.cpp:73-93 (padded copy, stage 1, stage 2) */
int jto_parse(const uint8_t *data, size_t len, jto_result *r) {
  memset(r, 0, sizeof(*r));
  uint8_t *buf = (uint8_t *)malloc(len + PADDING);
  if (len)
    memcpy(buf, data, len);
  memset(buf + len, 0, PADDING);
  if (jto_stage1(buf, len, r) != JTO_OK) {
    free(buf);
    return r->code;
  }
  builder b;
  memset(&b, 0, sizeof(b));
  b.buf = buf;
  b.len = len;
  b.pos = r->index;
  b.count = r->index_count;
  b.tape = (uint64_t *)malloc((2 * b.count + 3) * sizeof(uint64_t));
  b.strings = (uint8_t *)malloc(len + 4 * b.count + 64);
  build_tape(&b);
  free(buf);
  r->code = b.code;
  r->offset = b.off;
  if (b.code == JTO_OK) {
    r->tape = b.tape;
    r->tape_len = b.used;
    r->strings = b.strings;
    r->strings_len = b.sused;
  } else {
    free(b.tape);
    free(b.strings);
  }
  return r->code;
}

void jto_free(jto_result *r) {
  free(r->index);
  free(r->tape);
  free(r->strings);
  r->index = NULL;
  r->tape = NULL;
  r->strings = NULL;
}
