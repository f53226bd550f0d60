// stage2.h — host-side interface of the stage-2 (tape) kernels.
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "shard.h"

namespace jt {

constexpr int kTokPerThread = 16;                       // one "chunk"
constexpr int kS2Threads = 128;
constexpr int kTokPerTile = kTokPerThread * kS2Threads;  // 2048 tokens
constexpr int kStructTok = 8;                           // tokens per k_struct thread
// depth min-tree over the tokens, fan-out 16: level 0 = token records,
// level 1 = per 16 tokens (m1), 2 = per 256 (m2), 3 = per 4096 (m3, int32
// encoded 0x7FFF - min for atomicMax), levels 4..7 = mhi (int16)
constexpr int kTreeLevels = 8;

// Device control block, zeroed before every parse (utf8_pos / err_key set
// to ~0 by the init kernel).
struct Ctrl {
  uint32_t s1_tile_counter;
  uint32_t s2_tile_counter;
  unsigned long long utf8_pos;  // min invalid UTF-8 offset (~0 = none)
  uint64_t S;                   // structural index count
  unsigned long long err_key;   // (token << 8) | code, min wins (~0 = none)
  uint32_t slow_count;          // numbers needing the exact fallback
  uint32_t num_count;           // number tokens queued for k_numbers
  int32_t max_depth;            // max depth_after over all tokens (clamped)
  uint32_t stk_tile_counter;    // k_stack tile claims
  uint64_t tape_words;          // E = 1 + sum of token widths (root close index)
  uint64_t string_bytes;        // string buffer size (stage 1)
  unsigned long long str_err;   // min string error position (~0 = none)
  int64_t depth_total;          // depth change over the (shard's) tokens
  uint64_t n_newlines;          // record mode: '\n' bytes (K0)
  // results written by the finalize kernel
  int32_t code;
  int32_t redo;                 // streamed pieces: a later piece's summary was needed before it existed
  long long offset;
  uint64_t tape_len;            // E + 1 on success
};

// one NDJSON record's result (include/jsontape_b200.h jt_b200_record)
struct RecordResult {
  int32_t code;
  int32_t reserved;
  long long offset;        // relative to the record start, -1 if none
  uint64_t tape_begin;     // tape index of the record's root word
  uint64_t tape_words;     // root .. root close, 0 on error
  uint64_t string_begin;   // string-buffer offset of the record's strings
  uint64_t string_bytes;
};

// A partial stage 2 over the tokens [lo, hi) (streamed jt_parse runs stage 2
// on the document's first tokens while the rest is still uploading; a second
// range finishes it).  lo and hi are multiples of 4096 (the k_stack / k_struct
// tile and the min-tree level-3 group) except the final hi = S; `avail`
// tokens exist (the token after hi is readable); numbers / slow floats from
// list entry num_lo / slow_lo; opener words below patch_lim (already copied to
// the host) written by this range are also recorded in Stage2Args.patch.
struct TokRange {
  uint64_t lo, hi, avail;
  uint32_t num_lo, slow_lo;
  uint64_t fin;        // 1: the document's last range (end-of-document checks)
  uint64_t patch_lim;
  uint64_t tape_end;   // first tape word not final after this range (range A)
};

struct Stage2Args {
  const uint8_t *in;
  uint64_t len;
  const uint32_t *idx;
  const uint32_t *aux;  // per index entry: string-buffer prefix (stage 1)
  Ctrl *ctrl;
  uint32_t *tok;        // per token: c | fail << 8 | (int16 depth_before) << 16 (stage 1 + scalars)
  const uint32_t *tape_idx;  // per token: tape word index (stage 1)
  const uint32_t *tile_flags;  // per stage-1 tile: 1 = string lengths not written
  int16_t *m1;          // tree level 1 (per 16 tokens)
  int16_t *m2;          // tree level 2 (per 256 tokens)
  int32_t *m3;          // tree level 3 (per 4096 tokens), encoded, zeroed by init
  int16_t *mhi;         // tree levels 4..7, at offsets hi_off[0..3]
  uint64_t hi_off[4];
  uint32_t *slow;       // slow-number token list
  uint32_t *numlist;    // number tokens (compacted by k_scalars)
  uint32_t *scopebits;  // bit i: innermost container of token i is an object
  uint64_t *stk_rec;    // k_scalars look-back records (4 words per 256 tokens), zeroed
  uint64_t *tape;       // tape_cap words: writes at or past it are dropped (only a failing
  uint64_t tape_cap;    // document's tape can be longer, engine.cu ensure_stage2)
  uint8_t *strings;     // >= len + 4 * cap + 64 bytes
  uint64_t cap_tokens;  // capacity bound on S (for grid sizing)
  int num_sms;
  // byte-range sharding (shard.h); sh == nullptr: unsharded
  Shard *sh;
  uint64_t *bound;      // kBoundMax: containers open at the shard start (kind << 56 | tape)
  Sum3 *sum3;           // phase-3 summary (error, cross-shard bracket patches)
  // record (NDJSON) mode (records == true): see stage1.h
  bool records;
  const uint32_t *rec_of, *rec_start, *rec_kend, *rec_tend, *rec_send, *rec_utf8, *rec_serr;
  unsigned long long *rec_err;  // per record: (token << 8) | code, ~0 = none
  uint32_t *rec_end_err;        // per record: error at the record's end (0 = none)
  RecordResult *results;        // per record (k_final_records)
  // partial stage 2 (nullptr: all tokens)
  const TokRange *range;
  unsigned long long *patch;    // [0] = count, then (tape index, word) pairs
};

// distinct_values query over the device-resident result of the last parse
// (document.cpp:134-192): matched scalar tokens, then their values.
constexpr int kDistinctMaxKeys = 32;
struct DistinctQuery {
  const uint8_t *key_bytes;   // the path's keys, concatenated
  uint32_t key_off[kDistinctMaxKeys + 1];
  int nkeys;
};
struct DistinctVal {          // one matched scalar
  uint64_t bits;              // int64 / float64 bits; string: byte offset in the compact buffer
  uint32_t len;               // string bytes
  uint32_t tag;               // tape tag
};
// k_distinct_match: S tokens -> match[] (token indices, unordered), *count
cudaError_t distinct_match_launch(const Stage2Args &a, const DistinctQuery &q, uint32_t *match,
                                  uint32_t *count, cudaStream_t stream);
// values of count matches; string lengths into len[] (for the caller's scan)
cudaError_t distinct_values_launch(const Stage2Args &a, const uint32_t *match, uint32_t count,
                                   DistinctVal *vals, uint32_t *len, cudaStream_t stream);
// exclusive prefix sum of n u32 values (one CTA; the distinct string offsets)
cudaError_t scan_u32_launch(const uint32_t *in, uint32_t *out, uint32_t n, cudaStream_t stream);
// string bytes of the matches to out at the scanned offsets off[]
cudaError_t distinct_strings_launch(const Stage2Args &a, const DistinctVal *vals, const uint32_t *off,
                                    uint32_t count, uint8_t *out, cudaStream_t stream);

// words of look-back records / tree nodes needed for up to `cap` tokens
struct Stage2Sizes {
  uint64_t chunks, tiles, n1, n2, n3, nhi;
  uint64_t hi_off[4];
};
Stage2Sizes stage2_sizes(uint64_t cap_tokens);

// Enqueue the whole stage 2 (tokens, slow numbers, tree, structure,
// finalize); returns the number of kernel launches via *launches.
// `ev` (optional, 5 events) is recorded after each of the 5 kernels.
// `fork` (optional, without `ev`): {side stream, fork event, join event} --
// the container-kind stack (k_stack) runs on the side stream next to the
// scalar / number / tree kernels, which it does not depend on.
struct Stage2Fork {
  cudaStream_t side;
  cudaEvent_t fork, join;
};
cudaError_t stage2_launch(const Stage2Args &a, cudaStream_t stream, int *launches,
                          cudaEvent_t *ev = nullptr, const Stage2Fork *fork = nullptr);

// Streamed jt_parse, stage 2 in token ranges.  range_a_launch: the next
// range = [prev.hi (or 0), hi) with hi the last multiple of 4096 below the
// tokens stage 1 has produced so far (*known), written to `r` (with the tape
// words it finalises up to r->tape_end); then the range's stage 2 (no root
// words, no end checks).  range_b_launch: the last range = [prev.hi, S)
// after the whole stage 1, then the document's finalize.  Openers a range
// writes below its patch_lim (earlier ranges' words, already on their way to
// the host) are recorded as patches.
constexpr uint64_t kPatchMax = 8192;  // containers open at the range boundaries (<= kMaxDepth + 1 each)
cudaError_t range_a_launch(const Stage2Args &a, const uint64_t *known, const TokRange *prev, TokRange *r,
                           TokRange *host, cudaStream_t stream, int *launches,
                           const Stage2Fork *fork = nullptr);  // host: pinned copy (or null)
cudaError_t range_b_launch(const Stage2Args &a, const TokRange *ra, TokRange *rb, cudaStream_t stream,
                           int *launches, const Stage2Fork *fork = nullptr);

// Record mode: per-record error slots, then the whole stage 2 with
// per-record grammar, and one result per record.
cudaError_t records_init_launch(const Stage2Args &a, cudaStream_t stream);
cudaError_t records_stage2_launch(const Stage2Args &a, cudaStream_t stream, int *launches,
                                  const Stage2Fork *fork = nullptr);

// Sharded stage 2 (shard.h).  phase 2: bases from the gathered Sum1s, then
// scalars / numbers / depth tree and this shard's open containers (Sum2);
// phase 3: the container stack at the shard start from the gathered Sum2s,
// then stack scan, structure and the local first error (Sum3).
cudaError_t shard_sum1_launch(const Stage2Args &a, Sum1 *out, cudaStream_t stream);
cudaError_t shard_phase2_launch(const Stage2Args &a, const Sum1 *gathered, Sum2 *out,
                                cudaStream_t stream, int *launches);
cudaError_t shard_phase3_launch(const Stage2Args &a, const Sum2 *gathered, cudaStream_t stream,
                                int *launches);
// global first error and the bracket patches that land in this shard
cudaError_t shard_finish_launch(const Stage2Args &a, const Sum3 *gathered, cudaStream_t stream);

// jt_compute_stats after a successful parse: 9 counters in jt_stats order
// (integers, floats, strings, non_ascii_bytes, objects, arrays, nulls, trues,
// falses), zeroed by the caller
cudaError_t stats_launch(const Stage2Args &a, unsigned long long *cnt, cudaStream_t stream);

// Reset kernel for the control block + look-back records.
cudaError_t init_launch(Ctrl *ctrl, uint64_t *s1rec, uint64_t s1words, uint64_t *s2rec,
                        uint64_t s2words, cudaStream_t stream);

// Stage-1-only finalize: copies utf8 verdict into ctrl->code / offset.
cudaError_t stage1_finalize_launch(Ctrl *ctrl, cudaStream_t stream);

}  // namespace jt
