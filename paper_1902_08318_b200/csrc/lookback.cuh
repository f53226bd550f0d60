// lookback.cuh — decoupled look-back primitives (single-pass scans).
//
// A tile publishes one 64-bit record per channel: bits 63:62 = flag
// (0 empty, 1 aggregate, 2 inclusive prefix), bits 61:0 = payload.  Flag and
// payload travel in ONE aligned 64-bit relaxed store, so readers need no
// fence (and no gpu-scope fence means no L1 invalidation, B300_MICROARCH
// "L1D flush trigger").  Tiles take their ids from an atomic counter, so every
// predecessor of a tile is already resident or finished: spinning on it is
// deadlock-free.
#pragma once

#include <stdint.h>

namespace jt {

constexpr uint64_t kFlagAgg = 1ULL << 62;
constexpr uint64_t kFlagIncl = 2ULL << 62;
constexpr uint64_t kPayload = (1ULL << 62) - 1;

__device__ __forceinline__ void lb_store(uint64_t *p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint64_t lb_load(const uint64_t *p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// spin until the record is non-empty
__device__ __forceinline__ uint64_t lb_wait(const uint64_t *p) {
  uint64_t v = lb_load(p);
  while ((v >> 62) == 0) {
    __nanosleep(32);
    v = lb_load(p);
  }
  return v;
}

// Sum look-back for a u62 counter channel, executed by one full warp.
// Returns the exclusive prefix of tile `tile` (> 0) to all lanes.
__device__ __forceinline__ uint64_t lb_sum_exclusive(const uint64_t *rec, int64_t tile) {
  const int lane = threadIdx.x & 31;
  uint64_t acc = 0;
  int64_t base = tile - 1;
  for (;;) {
    int64_t pred = base - lane;
    uint64_t v = pred >= 0 ? lb_wait(rec + pred) : kFlagIncl;
    uint32_t incl = __ballot_sync(0xffffffffu, (v >> 62) == 2);
    uint64_t pay = v & kPayload;
    if (incl) {
      int k = __ffs(incl) - 1;
      if (lane > k) pay = 0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) pay += __shfl_xor_sync(0xffffffffu, pay, o);
      return acc + pay;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) pay += __shfl_xor_sync(0xffffffffu, pay, o);
    acc += pay;
    base -= 32;
  }
}

}  // namespace jt
