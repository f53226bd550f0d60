// stage1.h — host-side interface of the K1 stage-1 kernel.
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace jt {

#ifndef JT_K1_THREADS
#define JT_K1_THREADS 256
#endif
constexpr int kStage1Threads = JT_K1_THREADS;
constexpr int kStage1Tile = kStage1Threads * 64;  // bytes per CTA tile
// shared-memory staging capacities per tile (larger tiles spill to direct
// global stores)
constexpr int kStageIdx = 16 * kStage1Threads;     // index entries
#ifndef JT_STAGE_PAY
#define JT_STAGE_PAY (80 * JT_K1_THREADS)
#endif
constexpr int kStagePay = JT_STAGE_PAY;  // string-buffer bytes

struct Stage1Args {
  const uint8_t *in;   // padded: readable and zero from len up to the tile end + 64
  uint64_t len;
  uint32_t *idx;       // >= len + 1 entries
  uint32_t *aux;       // per index entry: string-buffer prefix (low 32 bits)
  uint8_t *strings;    // string buffer (payload; length fields left to stage 2)
  uint32_t *tokrec;    // per index entry: byte | clamped depth_before << 16
  uint32_t *tape_idx;  // per index entry: tape word index
  uint32_t *tile_flags; // per tile: 1 = string lengths left to stage 2 (spill mode)
  uint32_t *fn;        // ntiles carry transfer functions (K0a)
  uint32_t *carry;     // ntiles carry-in states (K0b)
  uint64_t *rec_count; // 8 * ntiles look-back words (count, strings, tape, depth), zeroed
  uint32_t *tile_counter;         // zeroed
  unsigned long long *utf8_pos;   // ~0 initially; min flagged offset
  unsigned long long *str_err;    // ~0 initially; min string error offset
  uint64_t *total;                // S
  uint64_t *total_strings;        // string buffer bytes
  uint64_t *tape_words;           // 1 + sum of token widths
  int64_t *depth_total;           // depth change over the range
  uint64_t begin, end;            // byte range [begin, end): a shard, or [0, len)
  // streaming (one document in chunks): the range's first tile in the
  // document's look-back records / tile flags, and the document's last tile
  // (writes the totals); 0 and ~0 = the range is the whole record space
  uint64_t rec_tile0;
  uint64_t last_tile;
  const uint32_t *init_state;     // carry state before the range (nullptr = initial)
  uint32_t *out_state;            // carry state after the range (optional)
  // streamed jt_parse: string-buffer bytes up to the end of the range,
  // written to host-mapped memory by the range's last tile (optional), and
  // the host copy of the string buffer that k_tile_lengths also patches
  uint64_t *sb_out;
  uint64_t *tok_out;     // streamed pieces: index entries up to the range's last tile (device)
  uint8_t *strings_host;
  // record (NDJSON) mode: '\n'-separated records parsed independently
  bool records;
  uint32_t *nl_count, *nl_base;   // per tile: newlines, newlines before it (K0)
  uint64_t *nl_total;             // newlines of the range
  uint32_t *rec_start;            // per record: first byte (rec_start[0] = 0)
  uint32_t *rec_kend, *rec_tend, *rec_send;  // per '\n': token / tape / string prefix at it
  uint32_t *rec_utf8, *rec_serr;  // per record: first UTF-8 / string error position (~0 = none)
  uint32_t *rec_of;               // per index entry: its record
  uint64_t ntiles;                // filled by the launchers
};

// number of tiles for `len` (look-back records: 1 + 8 words per tile)
size_t stage1_records(uint64_t len);

constexpr int kStage1Launches = 3;  // K0a carry functions, K0b carry scan, K1
cudaError_t stage1_launch(const Stage1Args &args, cudaStream_t stream);
// one piece of a streamed document (rec_tile0 / last_tile / init_state /
// out_state set) in two launches: K0a + K0b over the piece's tiles, then K1
// over a tile range (streamed jt_parse runs K1 one tile behind the piece
// boundary)
cudaError_t stage1_chunk_carry(const Stage1Args &args, cudaStream_t stream);
cudaError_t stage1_chunk_main(const Stage1Args &args, cudaStream_t stream);
// after a streamed stage 1: the string length fields K1 left to stage 2
cudaError_t stage1_lengths_launch(const Stage1Args &args, uint64_t ntiles, cudaStream_t stream);

// record (NDJSON) mode, split so the caller can size the per-record arrays
// from the newline count: K0 (carries + newline counts), then K1
cudaError_t stage1_records_count(const Stage1Args &args, cudaStream_t stream);
cudaError_t stage1_records_main(const Stage1Args &args, cudaStream_t stream);

// index-only stage 1 (jt_stage1): K0a, K0b, k_index -> idx, total, utf8_pos
// (rec_count used as ntiles u62 look-back words, zeroed)
constexpr int kIndexLaunches = 1;
cudaError_t index_launch(const Stage1Args &args, cudaStream_t stream);

// jt_minify after a successful parse of the same resident input (the
// carry-ins are K0b's); rec and tile_counter zeroed, ntiles words / 1 word
struct MinifyArgs {
  const uint8_t *in;
  uint64_t len;
  const uint32_t *carry;
  uint8_t *out;
  uint64_t *rec;
  uint32_t *tile_counter;
  uint64_t *total;
  uint64_t ntiles;
};
cudaError_t minify_launch(const MinifyArgs &args, cudaStream_t stream);

struct Sum0;
// sharded stage 1 (shard.h): phase 0 = K0a + the shard's composed carry
// function; phase 1 = carry-in from all shards' functions, K0b, K1
cudaError_t stage1_shard_phase0(const Stage1Args &args, Sum0 *out, cudaStream_t stream);
cudaError_t stage1_shard_phase1(const Stage1Args &args, const Sum0 *gathered, uint32_t g,
                                cudaStream_t stream);

// one-time kernel attributes (dynamic shared memory); call outside capture
cudaError_t stage1_configure();

#ifdef JT_TIMELINE
cudaError_t stage1_timeline(unsigned long long *host, size_t n);
#endif

}  // namespace jt
