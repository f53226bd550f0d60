/* ref_driver.c — multi-threaded timing driver for the UNMODIFIED reference
 * (oracle/_ref/libjsontape_ref.so) — BASELINE / TEST INFRASTRUCTURE ONLY.
 *
 * bench.py's cpu_baseline leg and `--impl reference` time the reference's own
 * public entry point jt_parse (proj/include/jsontape.h:37-41,
 * proj/src/capi.cpp:73-93) on all host cores.  Driving it from Python
 * threads would serialise the per-record calls on the GIL (C3 has ~4M
 * records of ~256 B, about as long as a ctypes round trip), so the loops live
 * here, one pthread per core, each with its own jt_parser (the reference is
 * thread-compatible, jsontape.h:1-4):
 *
 *   jtref_parse_many     every thread jt_parse()s the whole document `reps`
 *                        times (the reference cannot split one document);
 *   jtref_parse_records  NDJSON: the records ('\n'-separated, as bench.py's
 *                        record split) are dealt to the threads in contiguous
 *                        slices and each record is jt_parse()d on its own
 *                        (what jt_b200_parse_records computes per record).
 *
 * Both return the wall time in seconds of the timed loops (after one untimed
 * warm-up pass per thread), or a negative value on failure.  Linked against
 * the reference library only; never against the product.
 */
#define _GNU_SOURCE
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include "jsontape.h"

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec + ts.tv_nsec * 1e-9;
}

typedef struct {
  const char *buf;
  size_t len;     /* whole document, or this thread's slice of records */
  int reps;
  int records;    /* 1: parse each '\n'-separated record on its own */
  pthread_barrier_t *bar;
  size_t n_records, n_ok;
  int first_code; /* document mode: the code of the last parse */
  int fail;
} work_t;

static void run_once(work_t *w, jt_parser *p, int count) {
  if (!w->records) {
    jt_document *doc = NULL;
    long long off = -1;
    w->first_code = (int)jt_parse(p, w->buf, w->len, &doc, &off);
    if (doc) jt_document_free(doc);
    return;
  }
  const char *s = w->buf, *end = w->buf + w->len;
  while (s < end) {
    const char *nl = memchr(s, '\n', (size_t)(end - s));
    const char *e = nl ? nl : end;
    jt_document *doc = NULL;
    long long off = -1;
    jt_error c = jt_parse(p, s, (size_t)(e - s), &doc, &off);
    if (doc) jt_document_free(doc);
    if (count) {
      w->n_records++;
      w->n_ok += c == JT_OK;
    }
    s = e + 1;
  }
}

static void *worker(void *arg) {
  work_t *w = (work_t *)arg;
  jt_parser *p = jt_parser_new();
  if (!p) w->fail = 1;
  if (p) run_once(w, p, 0); /* warm-up: page in the parser's buffers */
  pthread_barrier_wait(w->bar);
  for (int r = 0; p && r < w->reps; r++) run_once(w, p, r == 0);
  pthread_barrier_wait(w->bar);
  if (p) jt_parser_free(p);
  return NULL;
}

static double run(work_t *ws, int threads) {
  pthread_barrier_t bar;
  pthread_barrier_init(&bar, NULL, (unsigned)threads + 1);
  pthread_t *th = (pthread_t *)calloc((size_t)threads, sizeof(pthread_t));
  for (int t = 0; t < threads; t++) {
    ws[t].bar = &bar;
    pthread_create(&th[t], NULL, worker, &ws[t]);
  }
  pthread_barrier_wait(&bar);
  double t0 = now_s();
  pthread_barrier_wait(&bar);
  double dt = now_s() - t0;
  for (int t = 0; t < threads; t++) pthread_join(th[t], NULL);
  pthread_barrier_destroy(&bar);
  free(th);
  for (int t = 0; t < threads; t++)
    if (ws[t].fail) return -1.0;
  return dt;
}

double jtref_parse_many(const char *buf, size_t len, int threads, int reps, int *code_out) {
  if (threads < 1 || reps < 1) return -1.0;
  work_t *ws = (work_t *)calloc((size_t)threads, sizeof(work_t));
  for (int t = 0; t < threads; t++) {
    ws[t].buf = buf;
    ws[t].len = len;
    ws[t].reps = reps;
  }
  double dt = run(ws, threads);
  if (code_out) *code_out = ws[0].first_code;
  free(ws);
  return dt;
}

double jtref_parse_records(const char *buf, size_t len, int threads, int reps, size_t *n_records,
                           size_t *n_ok) {
  if (threads < 1 || reps < 1) return -1.0;
  work_t *ws = (work_t *)calloc((size_t)threads, sizeof(work_t));
  /* slice t starts after the first '\n' at or after t/threads of the bytes */
  size_t prev = 0;
  for (int t = 0; t < threads; t++) {
    size_t cut = len;
    if (t + 1 < threads) {
      size_t at = len / (size_t)threads * (size_t)(t + 1);
      if (at < prev) at = prev;
      const char *nl = at < len ? memchr(buf + at, '\n', len - at) : NULL;
      cut = nl ? (size_t)(nl - buf) + 1 : len;
    }
    ws[t].buf = buf + prev;
    ws[t].len = cut - prev;
    ws[t].reps = reps;
    ws[t].records = 1;
    prev = cut;
  }
  double dt = run(ws, threads);
  size_t nr = 0, ok = 0;
  for (int t = 0; t < threads; t++) {
    nr += ws[t].n_records;
    ok += ws[t].n_ok;
  }
  if (n_records) *n_records = nr;
  if (n_ok) *n_ok = ok;
  free(ws);
  return dt;
}
