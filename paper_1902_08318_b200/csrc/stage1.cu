// stage1.cu — K1: fused UTF-8 validation + structural index, one HBM pass.
//
// Replaces build_structural_index (proj/src/indexer.cpp:29-56) and
// validate_utf8 (proj/src/utf8.cpp:127-158).  Layout: a CTA owns a 16 KiB tile
// (256 threads x 64-byte blocks), tiles are claimed in order through an
// atomic counter.  Per thread: 2 x 256-bit loads -> bit planes -> masks ->
// block transfer function.  Carries {odd_backslash, in_string,
// prev_separator} are resolved by a warp scan of transfer functions, a CTA
// scan, and a decoupled look-back across tiles (channel 1).  Index counts
// then go through a second look-back (channel 2) and the tile's offsets are
// staged in shared memory as u16 and written out coalesced.
#include <cuda_runtime.h>
#include <mutex>

#include "lookback.cuh"
#include "stage1.h"
#include "stage1_block.cuh"

namespace jt {

namespace {

constexpr int kThreads = kStage1Threads;
constexpr int kWarps = kThreads / 32;

__device__ __forceinline__ void ld256(const uint8_t *p, uint32_t *w) {
  asm volatile("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]),
                 "=r"(w[6]), "=r"(w[7])
               : "l"(p));
}

// state look-back (channel 1), one full warp; returns the tile's carry-in
__device__ uint32_t lookback_state(const uint64_t *rec, int64_t tile) {
  const int lane = threadIdx.x & 31;
  uint32_t G = 0;
  bool haveG = false;
  int64_t base = tile - 1;
  for (;;) {
    int64_t pred = base - lane;
    uint64_t v = pred >= 0 ? lb_wait(rec + pred) : (kFlagIncl | s1::kInitState);
    uint32_t incl = __ballot_sync(0xffffffffu, (v >> 62) == 2);
    uint32_t pay = (uint32_t)v;
    if (incl) {
      int k = __ffs(incl) - 1;
      uint32_t s = __shfl_sync(0xffffffffu, pay, k);
      for (int l = k - 1; l >= 0; --l) s = s1::apply(__shfl_sync(0xffffffffu, pay, l), s);
      if (haveG) s = s1::apply(G, s);
      return s;
    }
    uint32_t H = __shfl_sync(0xffffffffu, pay, 31);
    for (int l = 30; l >= 0; --l) H = s1::compose(__shfl_sync(0xffffffffu, pay, l), H);
    G = haveG ? s1::compose(G, H) : H;
    haveG = true;
    base -= 32;
  }
}

__global__ void __launch_bounds__(kThreads, 3) k_stage1(Stage1Args a) {
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_warp_f[kWarps];
  __shared__ uint32_t s_warp_state[kWarps];
  __shared__ uint32_t s_warp_cnt[kWarps];
  __shared__ uint64_t s_base;
  extern __shared__ uint16_t s_stage[];

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_tile = atomicAdd(a.tile_counter, 1u);
  __syncthreads();
  const int64_t tile = s_tile;
  const uint64_t tile_base = (uint64_t)tile * kStage1Tile;
  const uint64_t blk = tile_base + (uint64_t)threadIdx.x * 64;

  uint32_t w[16];
  ld256(a.in + blk, w);
  ld256(a.in + blk + 32, w + 8);

  s1::Masks m;
  s1::classify64(w, m);
  const uint64_t esc0 = s1::escaped_no_carry(m.bs);
  const uint64_t tog = s1::carry_toggle(m.bs);
  const uint32_t f = s1::block_function(m, esc0, tog);

  // warp inclusive scan of transfer functions
  uint32_t inc = f;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) inc = s1::compose(inc, o);
  }
  const uint32_t excl = __shfl_up_sync(0xffffffffu, inc, 1);
  if (lane == 31) s_warp_f[warp] = inc;

  // fused UTF-8 validity: needs only the 3 bytes before the block
  uint32_t prev = __shfl_up_sync(0xffffffffu, w[15], 1);
  if (lane == 0) prev = blk >= 4 ? *(const uint32_t *)(a.in + blk - 4) : 0u;
  if ((m.P[7] | (uint64_t)(prev & 0x80808000u)) != 0 && blk < a.len + 3) {
    if (s1::utf8_block_error(m.P, prev, blk + 64 >= a.len)) {
      const uint8_t *in = a.in;
      const uint64_t len = a.len;
      auto at = [in, len](uint64_t i) -> uint32_t { return i < len ? in[i] : 0u; };
      uint64_t lo = blk >= 3 ? blk - 3 : 0, hi = blk + 64 < len ? blk + 64 : len;
      for (uint64_t i = lo; i < hi; i++)
        if (s1::utf8_flagged(at, i, len)) {
          atomicMin(a.utf8_pos, (unsigned long long)i);
          break;
        }
    }
  }
  __syncthreads();

  // tile aggregate, look-back for the carry-in, warp carry states
  if (warp == 0) {
    uint32_t agg = s_warp_f[0];
#pragma unroll
    for (int k = 1; k < kWarps; k++) agg = s1::compose(s_warp_f[k], agg);
    uint32_t carry;
    if (tile == 0) {
      carry = s1::kInitState;
    } else {
      if (lane == 0) lb_store(a.rec_state + tile, kFlagAgg | agg);
      carry = lookback_state(a.rec_state, tile);
    }
    if (lane == 0) {
      lb_store(a.rec_state + tile, kFlagIncl | s1::apply(agg, carry));
      uint32_t c = carry;
      for (int k = 0; k < kWarps; k++) {
        s_warp_state[k] = c;
        c = s1::apply(s_warp_f[k], c);
      }
    }
  }
  __syncthreads();

  uint32_t state = s_warp_state[warp];
  if (lane > 0) state = s1::apply(excl, state);
  int64_t rem = (int64_t)a.len - (int64_t)blk;
  uint64_t valid = rem >= 64 ? ~0ULL : rem <= 0 ? 0ULL : ((1ULL << rem) - 1);
  uint64_t fin = s1::final_mask(m, esc0, tog, state, valid);
  uint32_t cnt = popc64(fin);

  // CTA exclusive scan of counts
  uint32_t ci = cnt;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    uint32_t o = __shfl_up_sync(0xffffffffu, ci, d);
    if (lane >= d) ci += o;
  }
  if (lane == 31) s_warp_cnt[warp] = ci;
  __syncthreads();
  uint32_t woff = 0, total = 0;
#pragma unroll
  for (int k = 0; k < kWarps; k++) {
    uint32_t c = s_warp_cnt[k];
    woff += k < warp ? c : 0;
    total += c;
  }
  uint32_t off = woff + ci - cnt;

  // stage tile-local offsets (u16) in shared memory
  uint32_t local = threadIdx.x * 64;
  while (fin) {
    s_stage[off++] = (uint16_t)(local + ctz64(fin));
    fin &= fin - 1;
  }

  if (warp == 0) {
    uint64_t base;
    if (tile == 0) {
      base = 0;
    } else {
      if (lane == 0) lb_store(a.rec_count + tile, kFlagAgg | total);
      base = lb_sum_exclusive(a.rec_count, tile);
    }
    if (lane == 0) {
      lb_store(a.rec_count + tile, kFlagIncl | (base + total));
      s_base = base;
      if (tile == (int64_t)a.ntiles - 1) *a.total = base + total;
    }
  }
  __syncthreads();

  uint32_t *dst = a.idx + s_base;
  const uint32_t tb = (uint32_t)tile_base;
  for (uint32_t k = threadIdx.x; k < total; k += kThreads) dst[k] = tb + s_stage[k];
}

}  // namespace

size_t stage1_records(uint64_t len) {
  uint64_t ntiles = (len + kStage1Tile - 1) / kStage1Tile;
  return (size_t)(ntiles == 0 ? 1 : ntiles);
}

cudaError_t stage1_launch(const Stage1Args &args_in, cudaStream_t stream) {
  Stage1Args a = args_in;
  uint64_t ntiles = (a.len + kStage1Tile - 1) / kStage1Tile;
  if (ntiles == 0) ntiles = 1;
  a.ntiles = ntiles;
  const int smem = kStage1Tile * 2;
  static const cudaError_t configured =
      cudaFuncSetAttribute(k_stage1, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (configured != cudaSuccess) return configured;
  k_stage1<<<(unsigned)ntiles, kThreads, smem, stream>>>(a);
  return cudaGetLastError();
}

}  // namespace jt
