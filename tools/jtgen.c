/* jtgen.c — seeded synthetic inputs for the five BASELINE.json configs.
 *
 * These stand in for the paper's public datasets (twitter.json, canada.json,
 * ...), which are not in this container and are not
 * recreated.  Shapes, sizes and value distributions follow BASELINE.json
 * `configs` and SURVEY.md §8(d).  Deterministic: own xoshiro256** RNG, no libc
 * random, so the same (config, size, seed) gives identical bytes here and on
 * the GPU box.
 *
 *   C0  1 MiB minified array of flat 6-key objects (ints, %.17g floats,
 *       atoms, ASCII strings with 5% \" / \\ escapes)
 *   C1  64 MiB pretty-printed (2-space, LF) random tree, branching 1-10,
 *       depth <= 8, 30% non-ASCII string chars, 10% strings with \n \t \uXXXX
 *       (incl. surrogate pairs)
 *   C2  >= 256 MiB of rows [16 numbers]: 90% %.17g floats with decimal
 *       exponent U[-300,300], 10% int64 over the full range
 *   C3  NDJSON, lognormal record sizes (mean 256 B, sigma 1), C0-style
 *       objects with 1-3 nested levels, '\n' terminated
 *   C4  adversarial: strings up to 64 KiB dense in backslash runs (1-9) and
 *       escaped quotes, nesting up to depth 1024, mixed UTF-8; optional
 *       single injected error (see jtg_error_kind)
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  uint64_t s[4];
} rng_t;

static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

static uint64_t next_u64(rng_t *r) { /* xoshiro256** */
  uint64_t *s = r->s;
  uint64_t result = rotl(s[1] * 5, 7) * 9;
  uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl(s[3], 45);
  return result;
}

static void seed_rng(rng_t *r, uint64_t seed) { /* splitmix64 expansion */
  for (int i = 0; i < 4; i++) {
    uint64_t z = (seed += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    r->s[i] = z ^ (z >> 31);
  }
}

static uint64_t uniform(rng_t *r, uint64_t n) { return n ? next_u64(r) % n : 0; }
static double unit(rng_t *r) { return (next_u64(r) >> 11) * (1.0 / 9007199254740992.0); }
static int chance(rng_t *r, double p) { return unit(r) < p; }

typedef struct {
  char *buf;
  size_t len, cap;
} sbuf;

static void reserve(sbuf *b, size_t n) {
  if (b->len + n <= b->cap)
    return;
  size_t nc = b->cap ? b->cap : 1 << 16;
  while (nc < b->len + n)
    nc *= 2;
  b->buf = (char *)realloc(b->buf, nc);
  b->cap = nc;
}
static void put(sbuf *b, const char *s, size_t n) {
  reserve(b, n);
  memcpy(b->buf + b->len, s, n);
  b->len += n;
}
static void putc1(sbuf *b, char c) {
  reserve(b, 1);
  b->buf[b->len++] = c;
}
static void puts0(sbuf *b, const char *s) { put(b, s, strlen(s)); }

/* error kinds for C4 / the error sweep */
enum {
  E_NONE = 0,
  E_UTF8_INVALID = 1,
  E_UTF8_OVERLONG = 2,
  E_BRACKET = 3,
  E_CONTROL = 4,
  E_NUMBER = 5
};

typedef struct {
  rng_t rng;
  sbuf out;
  int pretty;
  int err_kind;      /* pending error kind */
  size_t err_at;     /* inject at the first opportunity past this offset */
  int err_done;
} gen;

static int want_err(gen *g, int kind) {
  return !g->err_done && g->err_kind == kind && g->out.len >= g->err_at;
}

static void newline_indent(gen *g, int depth) {
  if (!g->pretty)
    return;
  putc1(&g->out, '\n');
  reserve(&g->out, 2 * (size_t)depth);
  for (int i = 0; i < depth; i++) {
    g->out.buf[g->out.len++] = ' ';
    g->out.buf[g->out.len++] = ' ';
  }
}

static void put_utf8(sbuf *b, uint32_t cp) {
  char t[4];
  int n;
  if (cp < 0x80) {
    t[0] = (char)cp;
    n = 1;
  } else if (cp < 0x800) {
    t[0] = (char)(0xC0 | (cp >> 6));
    t[1] = (char)(0x80 | (cp & 0x3F));
    n = 2;
  } else if (cp < 0x10000) {
    t[0] = (char)(0xE0 | (cp >> 12));
    t[1] = (char)(0x80 | ((cp >> 6) & 0x3F));
    t[2] = (char)(0x80 | (cp & 0x3F));
    n = 3;
  } else {
    t[0] = (char)(0xF0 | (cp >> 18));
    t[1] = (char)(0x80 | ((cp >> 12) & 0x3F));
    t[2] = (char)(0x80 | ((cp >> 6) & 0x3F));
    t[3] = (char)(0x80 | (cp & 0x3F));
    n = 4;
  }
  put(b, t, (size_t)n);
}

/* valid non-ASCII code point: length 2/3/4 uniform, then uniform within the
 * length's range, surrogates excluded */
static uint32_t rand_non_ascii(rng_t *r) {
  switch (uniform(r, 3)) {
  case 0:
    return 0x80 + (uint32_t)uniform(r, 0x800 - 0x80);
  case 1: {
    uint32_t cp;
    do
      cp = 0x800 + (uint32_t)uniform(r, 0x10000 - 0x800);
    while (cp >= 0xD800 && cp <= 0xDFFF);
    return cp;
  }
  default:
    return 0x10000 + (uint32_t)uniform(r, 0x110000 - 0x10000);
  }
}

static char rand_ascii_text(rng_t *r) {
  static const char pool[] =
      "abcdefghijklmnopqrstuvwxyzABCDEFGHIJKLMNOPQRSTUVWXYZ0123456789 .,:;-_!?()[]{}/@#$%&*+=<>'";
  return pool[uniform(r, sizeof(pool) - 1)];
}

static void put_hex4(sbuf *b, uint32_t v) {
  char t[8];
  snprintf(t, sizeof(t), "\\u%04X", v & 0xFFFF);
  put(b, t, 6);
}

/* lowercase ASCII key of 4..12 chars */
static void put_key(gen *g) {
  int n = 4 + (int)uniform(&g->rng, 9);
  putc1(&g->out, '"');
  for (int i = 0; i < n; i++)
    putc1(&g->out, (char)('a' + uniform(&g->rng, 26)));
  putc1(&g->out, '"');
}

/* injected string-level errors, inside an otherwise normal string body */
static void maybe_string_error(gen *g) {
  if (want_err(g, E_CONTROL)) {
    putc1(&g->out, (char)(1 + uniform(&g->rng, 31)));
    g->err_done = 1;
  } else if (want_err(g, E_UTF8_INVALID)) {
    static const char bad[][3] = {{(char)0xFF, 0, 1}, {(char)0x80, 0, 1},
                                  {(char)0xED, (char)0xA0, 2},
                                  {(char)0xF5, 0, 1}};
    int k = (int)uniform(&g->rng, 4);
    if (k == 2) {
      put(&g->out, "\xED\xA0\x80", 3); /* encoded surrogate */
    } else {
      putc1(&g->out, bad[k][0]);
    }
    g->err_done = 1;
  } else if (want_err(g, E_UTF8_OVERLONG)) {
    if (uniform(&g->rng, 2))
      put(&g->out, "\xC0\xAF", 2);
    else
      put(&g->out, "\xE0\x80\xAF", 3);
    g->err_done = 1;
  }
}

/* C0 ASCII string 8..32 chars, 5% with \" or \\ */
static void put_c0_string(gen *g) {
  int n = 8 + (int)uniform(&g->rng, 25);
  int esc = chance(&g->rng, 0.05);
  int at = esc ? (int)uniform(&g->rng, (uint64_t)n) : -1;
  putc1(&g->out, '"');
  for (int i = 0; i < n; i++) {
    if (i == at)
      puts0(&g->out, uniform(&g->rng, 2) ? "\\\"" : "\\\\");
    char c = rand_ascii_text(&g->rng);
    putc1(&g->out, c);
  }
  maybe_string_error(g);
  putc1(&g->out, '"');
}

/* C1 string: 30% non-ASCII chars; 10% of strings carry \n \t \uXXXX escapes */
static void put_c1_string(gen *g, int maxlen) {
  int n = 1 + (int)uniform(&g->rng, (uint64_t)maxlen);
  int esc = chance(&g->rng, 0.10);
  putc1(&g->out, '"');
  for (int i = 0; i < n; i++) {
    if (esc && uniform(&g->rng, (uint64_t)n) < 2) {
      switch (uniform(&g->rng, 4)) {
      case 0: puts0(&g->out, "\\n"); break;
      case 1: puts0(&g->out, "\\t"); break;
      case 2: {
        uint32_t cp;
        do
          cp = (uint32_t)uniform(&g->rng, 0x10000);
        while (cp >= 0xD800 && cp <= 0xDFFF);
        put_hex4(&g->out, cp);
        break;
      }
      default: {
        uint32_t cp = 0x10000 + (uint32_t)uniform(&g->rng, 0x100000);
        cp -= 0x10000;
        put_hex4(&g->out, 0xD800 + (cp >> 10));
        put_hex4(&g->out, 0xDC00 + (cp & 0x3FF));
        break;
      }
      }
      continue;
    }
    if (chance(&g->rng, 0.30))
      put_utf8(&g->out, rand_non_ascii(&g->rng));
    else
      putc1(&g->out, rand_ascii_text(&g->rng));
  }
  maybe_string_error(g);
  putc1(&g->out, '"');
}

/* %.17g float; ".0" appended when the text has neither '.' nor 'e' so the
 * token stays a float */
static void put_float17(gen *g, double v) {
  char t[40];
  int n = snprintf(t, sizeof(t), "%.17g", v);
  if (!strchr(t, '.') && !strchr(t, 'e') && !strchr(t, 'n') && !strchr(t, 'i')) {
    t[n++] = '.';
    t[n++] = '0';
    t[n] = 0;
  }
  put(&g->out, t, (size_t)n);
}

static void put_int(gen *g, long long v) {
  char t[32];
  int n = snprintf(t, sizeof(t), "%lld", v);
  put(&g->out, t, (size_t)n);
}

static int maybe_number_error(gen *g) {
  if (!want_err(g, E_NUMBER))
    return 0;
  static const char *bad[] = {"01", "1.", "-", "1.5e", "--2", "0x1F", "1e+", "-.5"};
  puts0(&g->out, bad[uniform(&g->rng, 8)]);
  g->err_done = 1;
  return 1;
}

/* random double with a 17-significant-digit mantissa and the given decimal
 * exponent range */
static double rand_decimal(gen *g, int emin, int emax) {
  char t[48];
  int p = 0;
  if (uniform(&g->rng, 2))
    t[p++] = '-';
  t[p++] = (char)('1' + uniform(&g->rng, 9));
  t[p++] = '.';
  for (int i = 0; i < 16; i++)
    t[p++] = (char)('0' + uniform(&g->rng, 10));
  p += snprintf(t + p, 12, "e%d", emin + (int)uniform(&g->rng, (uint64_t)(emax - emin + 1)));
  t[p] = 0;
  return strtod(t, NULL);
}

static void put_c0_value(gen *g) {
  if (maybe_number_error(g))
    return;
  switch (uniform(&g->rng, 6)) {
  case 0: put_int(g, (long long)uniform(&g->rng, 2000000001ULL) - 1000000000LL); break;
  case 1: put_float17(g, rand_decimal(g, -8, 8)); break;
  case 2: puts0(&g->out, uniform(&g->rng, 2) ? "true" : "false"); break;
  case 3: puts0(&g->out, "null"); break;
  default: put_c0_string(g); break;
  }
}

static void put_close(gen *g, char c) {
  if (want_err(g, E_BRACKET)) {
    /* wrong kind, or a dropped closer */
    if (uniform(&g->rng, 2))
      putc1(&g->out, c == ']' ? '}' : ']');
    g->err_done = 1;
    return;
  }
  putc1(&g->out, c);
}

/* C0 flat object: 6 keys */
static void put_c0_object(gen *g) {
  putc1(&g->out, '{');
  for (int k = 0; k < 6; k++) {
    if (k)
      putc1(&g->out, ',');
    put_key(g);
    putc1(&g->out, ':');
    put_c0_value(g);
  }
  put_close(g, '}');
}

static void gen_c0(gen *g, uint64_t target) {
  putc1(&g->out, '[');
  int first = 1;
  while (g->out.len + 2 < target) {
    if (!first)
      putc1(&g->out, ',');
    first = 0;
    put_c0_object(g);
  }
  put_close(g, ']');
}

/* ---- C1: pretty random tree ---- */

static void put_c1_scalar(gen *g) {
  if (maybe_number_error(g))
    return;
  switch (uniform(&g->rng, 8)) {
  case 0: put_int(g, (long long)(next_u64(&g->rng) >> (1 + uniform(&g->rng, 63))) *
                         (uniform(&g->rng, 2) ? 1 : -1)); break;
  case 1: put_float17(g, rand_decimal(g, -30, 30)); break;
  case 2: puts0(&g->out, uniform(&g->rng, 2) ? "true" : "false"); break;
  case 3: puts0(&g->out, "null"); break;
  default: put_c1_string(g, 40); break;
  }
}

static void put_c1_node(gen *g, int depth, int maxdepth) {
  /* containers more likely near the top; depth <= maxdepth */
  int container = depth < maxdepth && chance(&g->rng, depth == 0 ? 1.0 : 0.45 / depth + 0.1);
  if (!container) {
    put_c1_scalar(g);
    return;
  }
  int obj = uniform(&g->rng, 2);
  int n = 1 + (int)uniform(&g->rng, 10);
  putc1(&g->out, obj ? '{' : '[');
  for (int i = 0; i < n; i++) {
    if (i)
      putc1(&g->out, ',');
    newline_indent(g, depth + 1);
    if (obj) {
      put_c1_string(g, 16);
      put(&g->out, g->pretty ? ": " : ":", g->pretty ? 2 : 1);
    }
    put_c1_node(g, depth + 1, maxdepth);
  }
  newline_indent(g, depth);
  put_close(g, obj ? '}' : ']');
}

static void gen_c1(gen *g, uint64_t target) {
  putc1(&g->out, '[');
  int first = 1;
  while (g->out.len + 4 < target) {
    if (!first)
      putc1(&g->out, ',');
    first = 0;
    newline_indent(g, 1);
    put_c1_node(g, 1, 8);
  }
  newline_indent(g, 0);
  put_close(g, ']');
  putc1(&g->out, '\n');
}

/* ---- C2: rows of 16 numbers ---- */

static void gen_c2(gen *g, uint64_t target) {
  putc1(&g->out, '[');
  int first = 1;
  while (g->out.len + 2 < target) {
    if (!first)
      putc1(&g->out, ',');
    first = 0;
    putc1(&g->out, '[');
    for (int k = 0; k < 16; k++) {
      if (k)
        putc1(&g->out, ',');
      if (maybe_number_error(g))
        continue;
      if (chance(&g->rng, 0.9))
        put_float17(g, rand_decimal(g, -300, 300));
      else
        put_int(g, (long long)next_u64(&g->rng));
    }
    put_close(g, ']');
  }
  put_close(g, ']');
}

/* ---- C3: NDJSON ---- */

static double rand_normal(rng_t *r) {
  double u1 = unit(r), u2 = unit(r);
  if (u1 < 1e-300)
    u1 = 1e-300;
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}

static void put_c3_object(gen *g, size_t record_end, int depth, int maxdepth) {
  putc1(&g->out, '{');
  int k = 0;
  do {
    if (k++)
      putc1(&g->out, ',');
    put_key(g);
    putc1(&g->out, ':');
    if (depth < maxdepth && chance(&g->rng, 0.25)) {
      if (uniform(&g->rng, 2)) {
        put_c3_object(g, g->out.len + (record_end > g->out.len ? (record_end - g->out.len) / 3 : 8),
                      depth + 1, maxdepth);
      } else {
        putc1(&g->out, '[');
        int n = 1 + (int)uniform(&g->rng, 4);
        for (int i = 0; i < n; i++) {
          if (i)
            putc1(&g->out, ',');
          put_c0_value(g);
        }
        put_close(g, ']');
      }
    } else {
      put_c0_value(g);
    }
  } while (g->out.len < record_end);
  put_close(g, '}');
}

static void gen_c3(gen *g, uint64_t target) {
  const double mu = log(256.0) - 0.5, sigma = 1.0;
  while (g->out.len < target) {
    double s = exp(mu + sigma * rand_normal(&g->rng));
    if (s < 16)
      s = 16;
    if (s > 65536)
      s = 65536;
    int levels = 1 + (int)uniform(&g->rng, 3);
    put_c3_object(g, g->out.len + (size_t)s, 1, levels);
    putc1(&g->out, '\n');
  }
}

/* ---- C4: adversarial ---- */

static void put_c4_string(gen *g) {
  /* mostly short, some long (up to 64 KiB), dense in backslash runs */
  size_t n = chance(&g->rng, 0.02) ? 1024 + uniform(&g->rng, 65536 - 1024)
                                   : 1 + uniform(&g->rng, 64);
  size_t start = g->out.len;
  putc1(&g->out, '"');
  while (g->out.len - start < n) {
    uint64_t r = uniform(&g->rng, 10);
    if (r < 3) {
      int k = 1 + (int)uniform(&g->rng, 9); /* backslash run of 1..9 */
      reserve(&g->out, (size_t)k);
      for (int i = 0; i < k; i++)
        g->out.buf[g->out.len++] = '\\';
      if (k & 1) { /* odd run: the next byte is escaped */
        static const char esc[] = "\"\\/bfnrt";
        char c = esc[uniform(&g->rng, 8)];
        putc1(&g->out, c);
      }
    } else if (r < 4) {
      puts0(&g->out, "\\\""); /* embedded quote */
    } else if (r < 6) {
      put_utf8(&g->out, rand_non_ascii(&g->rng));
    } else if (r < 7) {
      uint32_t cp = (uint32_t)uniform(&g->rng, 0x100000);
      put_hex4(&g->out, 0xD800 + (cp >> 10));
      put_hex4(&g->out, 0xDC00 + (cp & 0x3FF));
    } else {
      putc1(&g->out, rand_ascii_text(&g->rng));
    }
    if (g->out.len - start > n / 2)
      maybe_string_error(g);
  }
  putc1(&g->out, '"');
}

static void put_c4_scalar(gen *g) {
  if (maybe_number_error(g))
    return;
  switch (uniform(&g->rng, 6)) {
  case 0: put_int(g, (long long)next_u64(&g->rng)); break;
  case 1: put_float17(g, rand_decimal(g, -300, 300)); break;
  case 2: puts0(&g->out, uniform(&g->rng, 2) ? "true" : "false"); break;
  case 3: puts0(&g->out, "null"); break;
  default: put_c4_string(g); break;
  }
}

static void put_c4_node(gen *g, int depth) {
  /* occasional deep chain toward the 1024 limit */
  if (depth < 1000 && chance(&g->rng, 0.002)) {
    int chain = (int)uniform(&g->rng, (uint64_t)(1025 - depth));
    int kinds[1024];
    for (int i = 0; i < chain; i++) {
      kinds[i] = (int)uniform(&g->rng, 2);
      if (kinds[i]) {
        putc1(&g->out, '{');
        put_key(g);
        putc1(&g->out, ':');
      } else {
        putc1(&g->out, '[');
      }
    }
    put_c4_scalar(g);
    for (int i = chain - 1; i >= 0; i--)
      put_close(g, kinds[i] ? '}' : ']');
    return;
  }
  int container = depth < 12 && chance(&g->rng, 0.3);
  if (!container) {
    put_c4_scalar(g);
    return;
  }
  int obj = uniform(&g->rng, 2);
  int n = (int)uniform(&g->rng, 8);
  putc1(&g->out, obj ? '{' : '[');
  for (int i = 0; i < n; i++) {
    if (i)
      putc1(&g->out, ',');
    if (obj) {
      if (uniform(&g->rng, 4) == 0)
        put_c4_string(g);
      else
        put_key(g);
      putc1(&g->out, ':');
    }
    put_c4_node(g, depth + 1);
  }
  put_close(g, obj ? '}' : ']');
}

static void gen_c4(gen *g, uint64_t target) {
  putc1(&g->out, '[');
  int first = 1;
  while (g->out.len + 2 < target) {
    if (!first)
      putc1(&g->out, ',');
    first = 0;
    put_c4_node(g, 1);
  }
  put_close(g, ']');
}

/* Generate config `config` (0..4) of about `target` bytes from `seed`.
 * err_kind (C4 and the error sweep, any config): 0 none, 1 invalid UTF-8,
 * 2 overlong UTF-8, 3 unbalanced/mismatched bracket, 4 raw control char in a
 * string, 5 bad number; injected at the first opportunity past a seeded
 * offset.  Returns a malloc'd buffer (free with jtg_free). */
/* was the requested error actually injected? (small docs may end first) */
int jtg_error_injected_last = 0;

char *jtg_generate(int config, uint64_t target, uint64_t seed, int err_kind,
                   size_t *len_out) {
  gen g;
  memset(&g, 0, sizeof(g));
  seed_rng(&g.rng, seed * 0x100000001B3ULL + (uint64_t)config);
  g.pretty = config == 1;
  g.err_kind = err_kind;
  if (err_kind) {
    rng_t er;
    seed_rng(&er, seed ^ 0xE77E77E7ULL);
    g.err_at = (size_t)(unit(&er) * 0.9 * (double)target);
  }
  reserve(&g.out, (size_t)target + 4096);
  switch (config) {
  case 0: gen_c0(&g, target); break;
  case 1: gen_c1(&g, target); break;
  case 2: gen_c2(&g, target); break;
  case 3: gen_c3(&g, target); break;
  case 4: gen_c4(&g, target); break;
  default:
    free(g.out.buf);
    return NULL;
  }
  *len_out = g.out.len;
  jtg_error_injected_last = g.err_done;
  return g.out.buf;
}

void jtg_free(char *p) { free(p); }
