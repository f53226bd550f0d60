// shard.h — byte-range sharding of one document across GPUs.
//
// Shard g of G parses bytes [begin, end) of a document of which the GPU holds
// [begin - 64, end + halo) (jt_b200_shard_resident; default: all of it).  A
// token crossing `end` is read from the halo: strings, escapes and atoms need
// at most 64 bytes of it; a number longer than the halo is detected (its digit
// run reaches the resident end) and the parse fails loudly with CAPACITY
// instead of reading bytes the GPU does not hold.  Tokens belong to the shard where
// they start.  Four small all-gathers connect the shards; each phase writes a
// fixed-size summary that the caller all-gathers (NCCL, or a local copy when
// emulating G shards on one GPU) and hands to the next phase:
//   phase 0  K0a + K0b-reduce           -> Sum0: the shard's carry function
//   phase 1  K0b (carry-in from Sum0s) + K1
//                                       -> Sum1: counts, depth, first errors,
//                                          first / last tokens
//   phase 2  bases from Sum1s; scalars, numbers, depth tree; open containers
//                                       -> Sum2: unmatched closers, openers
//   phase 3  container stack at the shard start from Sum2s; stack, structure
//                                       -> Sum3: first error, bracket patches
//   finish   global first error (Sum3s), patches into this shard's tape
// Unsharded parses use the same kernels with G = 0 (bases 0, no exchange).
#pragma once

#include <stdint.h>

namespace jt {

constexpr int kBoundMax = 2048;  // open containers exchanged per shard (> kMaxDepth + 1)

struct Shard {
  // layout (host)
  uint32_t g, G;          // G = 0: unsharded
  uint64_t begin, end;    // byte range; begin % kStage1Tile == 0
  uint64_t len;           // document length
  // from the phase-1 exchange
  uint64_t token_base, tape_base, string_base;
  int64_t depth_base;
  uint64_t S_total;       // tokens of the document
  uint64_t E_total;       // root close index (1 + sum of widths)
  uint64_t sb_total;      // string-buffer bytes of the document
  uint64_t next_pos;      // first token position of the next non-empty shard, or len + 1
  uint64_t next_aux;      // its string offset relative to this shard's string base
  uint32_t prev[2];       // bytes of the two tokens before the shard (prev[0] = nearest)
  uint32_t prev_n;        // how many exist
  uint32_t is_last;
  // from the phase-2 exchange: containers open at the shard start
  uint64_t S0;            // kinds as a shift register (bit 0 = innermost, 1 = object)
  int32_t open_n;         // how many (<= kBoundMax)
  uint32_t patch_n;       // cross-shard bracket patches recorded by k_struct
  uint32_t streamed;      // pieces of one streamed parse: only summaries up to g + 1 are final
                          // when phase 2 runs (later ones may be being written)
  uint32_t last_tok;      // this shard holds the document's last token (end-of-input check)
  uint32_t pad0;
  uint64_t res_hi;        // end of the bytes resident on this GPU (0: the whole document); a
                          // number that starts in the shard and runs to res_hi fails CAPACITY
};

// phase summaries (all-gathered as raw bytes)
struct Sum0 {
  uint32_t fn;  // composed carry function of the shard's tiles
  uint32_t pad[3];
};

struct Sum1 {
  uint64_t S, sb, T;        // tokens, string bytes, tape words (sum of widths)
  int64_t dtotal;           // depth change over the shard
  uint64_t utf8_pos;        // first invalid UTF-8 offset, ~0 = none
  uint64_t str_err;         // min string error position, ~0 = none
  uint64_t first_pos;       // position of the first token
  uint64_t first_aux;       // its string offset (shard-relative)
  uint32_t last[2];         // bytes of the last two tokens (last[0] = last)
  uint32_t pad[2];
};

struct Sum2 {
  int32_t unmatched;        // closers that pop containers opened before the shard
  int32_t n;                // containers still open at the shard end (opened here)
  uint64_t pad;
  uint64_t open[kBoundMax]; // kind << 56 | global tape index, outermost first
};

struct Sum3 {
  unsigned long long err_key;  // (global token << 8) | code, ~0 = none
  long long offset;            // its byte offset
  uint32_t patch_n;
  uint32_t pad[3];
  uint64_t patch[2 * kBoundMax];  // (global tape index, tape word) pairs
};

}  // namespace jt
