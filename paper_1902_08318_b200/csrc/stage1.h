// stage1.h — host-side interface of the K1 stage-1 kernel.
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace jt {

constexpr int kStage1Threads = 256;
constexpr int kStage1Tile = kStage1Threads * 64;  // bytes per CTA tile

struct Stage1Args {
  const uint8_t *in;   // padded: readable and zero from len up to the tile end + 64
  uint64_t len;
  uint32_t *idx;       // >= len + 1 entries
  uint64_t *rec_state; // ntiles look-back records, zeroed
  uint64_t *rec_count; // ntiles look-back records, zeroed
  uint32_t *tile_counter;         // zeroed
  unsigned long long *utf8_pos;   // ~0 initially; min flagged offset
  uint64_t *total;                // S
  uint64_t ntiles;                // filled by stage1_launch
};

// bytes of look-back records needed for `len`
size_t stage1_records(uint64_t len);

cudaError_t stage1_launch(const Stage1Args &args, cudaStream_t stream);

}  // namespace jt
