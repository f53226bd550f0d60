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

// JT_TIMELINE (instrumented builds only, never the product library): per-tile
// %globaltimer stamps and look-back counters, read back with
// jt_b200_timeline().  Slot k of tile t is g_tl[16 t + k].
#ifdef JT_TIMELINE
namespace jt {
constexpr int kTlTiles = 1 << 17;
static __device__ unsigned long long g_tl[kTlTiles * 16];  // per TU; stage1.cu reads its copy
__device__ __forceinline__ unsigned long long tl_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
}  // namespace jt
#define JT_TL(tile, k) \
  do { if ((tile) < jt::kTlTiles) jt::g_tl[(tile) * 16 + (k)] = jt::tl_now(); } while (0)
#define JT_TLV(tile, k, v) \
  do { if ((tile) < jt::kTlTiles) jt::g_tl[(tile) * 16 + (k)] = (v); } while (0)
#define JT_TLADD(tile, k, v) \
  do { if ((tile) < jt::kTlTiles && (v)) atomicAdd(&jt::g_tl[(tile) * 16 + (k)], (unsigned long long)(v)); } while (0)
#else
#define JT_TL(tile, k) do { } while (0)
#define JT_TLV(tile, k, v) do { } while (0)
#define JT_TLADD(tile, k, v) do { } while (0)
#endif

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

namespace jt {

// Two-counter channel: each tile owns 4 words, [0..1] aggregate (a, b) and
// [2..3] inclusive (a, b); bit 63 of every word = valid.  A reader trusts a
// pair only when both of its words are valid (each word is written once).
struct Pair {
  unsigned long long a, b;
};

constexpr uint64_t kPairValid = 1ULL << 63;

__device__ __forceinline__ void pair_publish(uint64_t *rec, int64_t tile, int slot, Pair v) {
  uint64_t *r = rec + 4 * tile + 2 * slot;
  lb_store(r, kPairValid | v.a);
  lb_store(r + 1, kPairValid | v.b);
}

__device__ __forceinline__ int pair_read(const uint64_t *rec, int64_t tile, Pair &v) {
  const uint64_t *r = rec + 4 * tile;
  uint64_t x = lb_load(r + 2), y = lb_load(r + 3);
  if ((x & y) >> 63) {
    v.a = x & ~kPairValid;
    v.b = y & ~kPairValid;
    return 2;
  }
  x = lb_load(r), y = lb_load(r + 1);
  if ((x & y) >> 63) {
    v.a = x & ~kPairValid;
    v.b = y & ~kPairValid;
    return 1;
  }
  return 0;
}

// exclusive prefix of tile `tile` (> 0), one full warp
__device__ __forceinline__ Pair pair_lookback(const uint64_t *rec, int64_t tile) {
  const int lane = threadIdx.x & 31;
  Pair acc{0, 0};
  int64_t base = tile - 1;
  for (;;) {
    int64_t pred = base - lane;
    Pair v{0, 0};
    int st = 2;
    if (pred >= 0)
      while ((st = pair_read(rec, pred, v)) == 0) __nanosleep(32);
    uint32_t incl = __ballot_sync(0xffffffffu, st == 2);
    int stop = incl ? __ffs(incl) - 1 : 31;
    if (lane > stop) v = Pair{0, 0};
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      v.a += __shfl_xor_sync(0xffffffffu, v.a, o);
      v.b += __shfl_xor_sync(0xffffffffu, v.b, o);
    }
    acc.a += v.a;
    acc.b += v.b;
    if (incl) return acc;
    base -= 32;
  }
}

}  // namespace jt

namespace jt {

// Four-counter channel (8 words per tile: [0] the packed aggregate, [4..7]
// the inclusive prefix; bit 63 = valid).  Signed counters travel as 63-bit two's
// complement and are sign-extended by the reader (sext63).
struct Quad {
  unsigned long long v[4];
};

constexpr uint64_t kQuadMask = (1ULL << 63) - 1;

__device__ __forceinline__ long long sext63(uint64_t v) { return (long long)(v << 1) >> 1; }

__device__ __forceinline__ void quad_publish(uint64_t *rec, int64_t tile, int slot, const Quad &q) {
  uint64_t *r = rec + 8 * tile + 4 * slot;
#pragma unroll
  for (int k = 0; k < 4; k++) lb_store(r + k, kPairValid | (q.v[k] & kQuadMask));
}

// A tile's AGGREGATE travels as one word (slot 0, word 0): bit 63 valid, bit 62
// the segment flag of the depth counter (record mode), then the tile's depth
// change (16 bits, signed), string-buffer bytes (16), tape words (15) and index
// entries (15) -- a 16 KiB tile has at most 16384 entries, 24576 tape words
// ("[1" is 3 words in 2 bytes), 32768 + 3 string bytes ('""' is 4 in 2 bytes)
// and a depth change within +-16384.  The INCLUSIVE prefix keeps four words
// (slot 1, words 4..7).  A look-back round costs its L2 requests: one 8-byte
// and two 16-byte loads per predecessor (eight 8-byte loads before).
__device__ __forceinline__ uint64_t quad_pack_agg(uint32_t total, uint32_t stotal, uint32_t ttotal,
                                                  int depth, bool seg) {
  return (1ULL << 63) | (seg ? (1ULL << 62) : 0ULL) | ((uint64_t)(uint16_t)depth << 46) |
         ((uint64_t)(stotal & 0xFFFFu) << 30) | ((uint64_t)(ttotal & 0x7FFFu) << 15) | (uint64_t)(total & 0x7FFFu);
}
__device__ __forceinline__ void quad_publish_agg(uint64_t *rec, int64_t tile, uint64_t packed) {
  lb_store(rec + 8 * tile, packed);
}

__device__ __forceinline__ void lb_load2(const uint64_t *p, uint64_t &x, uint64_t &y) {
  asm volatile("ld.relaxed.gpu.global.v2.b64 {%0, %1}, [%2];" : "=l"(x), "=l"(y) : "l"(p) : "memory");
}

// Window of the look-back: each lane reads kQuadPer predecessor records per
// round, so one round covers 32 * kQuadPer tiles.  All loads of a round are
// issued before any is waited on; only records still empty are re-polled.
// A/B on C4 (stage 1): 1 record per lane 2.65 ms, 2 -> 2.98, 3 -> 3.15, 4 -> 3.40: the
// round's cost is its L2 requests, not the number of rounds
#ifndef JT_QUAD_PER
#define JT_QUAD_PER 1
#endif
constexpr int kQuadPer = JT_QUAD_PER;
constexpr int kLbPer = 4;
// x[0] = the aggregate word, x[1..4] = the inclusive words
__device__ __forceinline__ void quad_issue(const uint64_t *rec, int64_t tile, uint64_t x[5]) {
  const uint64_t *r = rec + 8 * tile;
  x[0] = lb_load(r);
  lb_load2(r + 4, x[1], x[2]);
  lb_load2(r + 6, x[3], x[4]);
}
// Segmented counter (record mode depth): bit 62 = the span contains a
// reset, bits 61:0 = the change since its last reset (62-bit two's
// complement).  seg_combine(earlier, later).
constexpr uint64_t kSegFlag = 1ULL << 62;
constexpr uint64_t kSegMask = kSegFlag - 1;
__device__ __forceinline__ uint64_t seg_combine(uint64_t e, uint64_t l) {
  return (l & kSegFlag) ? l : ((e & kSegFlag) | ((e + l) & kSegMask));
}
__device__ __forceinline__ long long seg_value(uint64_t v) { return (long long)(v << 2) >> 2; }

// 2 = the inclusive prefix, 1 = the aggregate (unpacked into the counters'
// sum form), 0 = nothing published yet
template <bool kSeg3>
__device__ __forceinline__ int quad_decode(const uint64_t x[5], Quad &q) {
  if ((x[1] & x[2] & x[3] & x[4]) >> 63) {
#pragma unroll
    for (int k = 0; k < 4; k++) q.v[k] = x[1 + k] & kQuadMask;
    return 2;
  }
  const uint64_t a = x[0];
  if (a >> 63) {
    q.v[0] = a & 0x7FFFu;
    q.v[2] = (a >> 15) & 0x7FFFu;
    q.v[1] = (a >> 30) & 0xFFFFu;
    const long long d = (long long)(int16_t)(uint16_t)(a >> 46);
    q.v[3] = kSeg3 ? ((a & kSegFlag) | ((uint64_t)d & kSegMask)) : ((uint64_t)d & kQuadMask);
    return 1;
  }
  return 0;
}

// exclusive prefix (mod 2^63 per counter) of tile `tile` > 0, one full warp;
// kSeg3: counter 3 is a segmented counter (seg_combine) instead of a sum
template <bool kSeg3 = false>
__device__ __forceinline__ Quad quad_lookback(const uint64_t *rec, int64_t tile) {
  const int lane = threadIdx.x & 31;
  Quad acc{{0, 0, 0, 0}};
  int64_t base = tile - 1;
  for (;;) {
    // lane l owns predecessors base - kQuadPer*l - j, j = 0 (nearest) .. kQuadPer-1
    Quad q[kQuadPer];
    int st[kQuadPer];
    uint64_t x[kQuadPer][5];
#pragma unroll
    for (int j = 0; j < kQuadPer; j++) {
      int64_t pred = base - (int64_t)kQuadPer * lane - j;
      if (pred >= 0) quad_issue(rec, pred, x[j]);
    }
#pragma unroll
    for (int j = 0; j < kQuadPer; j++) {
      int64_t pred = base - (int64_t)kQuadPer * lane - j;
      q[j] = Quad{{0, 0, 0, 0}};
      st[j] = 2;
      if (pred >= 0) {
        while ((st[j] = quad_decode<kSeg3>(x[j], q[j])) == 0) {
          __nanosleep(32);
          quad_issue(rec, pred, x[j]);
          JT_TLADD(tile, 12, 1);
        }
      }
    }
    JT_TLADD(tile, 11, lane == 0);
    // per lane: sum from the nearest up to and including its first inclusive
    Quad mine{{0, 0, 0, 0}};
    bool has_incl = false;
#pragma unroll
    for (int j = 0; j < kQuadPer; j++) {
      if (!has_incl) {
#pragma unroll
        for (int k = 0; k < 3; k++) mine.v[k] += q[j].v[k];
        mine.v[3] = kSeg3 ? seg_combine(q[j].v[3], mine.v[3]) : mine.v[3] + q[j].v[3];
        has_incl = st[j] == 2;
      }
    }
    uint32_t incl = __ballot_sync(0xffffffffu, has_incl);
    int stop = incl ? __ffs(incl) - 1 : 31;
    int stop3 = stop;
    if (kSeg3) {  // a reset makes everything before it irrelevant for counter 3
      const uint32_t fl = __ballot_sync(0xffffffffu, lane <= stop && (mine.v[3] & kSegFlag));
      if (fl) stop3 = __ffs(fl) - 1;
    }
#pragma unroll
    for (int k = 0; k < 4; k++) {
      const int lim = k == 3 ? stop3 : stop;
      unsigned long long x = lane > lim ? 0ULL : (mine.v[k] & (kSeg3 && k == 3 ? kSegMask : kQuadMask));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      if (kSeg3 && k == 3) {
        const bool fl = stop3 < stop || (__shfl_sync(0xffffffffu, mine.v[3], stop3) & kSegFlag);
        acc.v[3] = seg_combine((fl ? kSegFlag : 0) | (x & kSegMask), acc.v[3]);
      } else {
        acc.v[k] = (acc.v[k] + x) & kQuadMask;
      }
    }
    if (incl) return acc;
    base -= 32 * kQuadPer;
  }
}
}  // namespace jt
