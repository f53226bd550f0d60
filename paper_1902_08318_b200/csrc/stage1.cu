// stage1.cu — K1: fused UTF-8 validation + structural index + string
// payload, one HBM pass over the input.
//
// Replaces build_structural_index (proj/src/indexer.cpp:29-56), validate_utf8
// (proj/src/utf8.cpp:127-158) and the byte work of parse_string
// (stringparse.cpp:143-183).  A CTA owns a 16 KiB tile (256 threads x
// 64-byte blocks); tiles are claimed in order through an atomic counter.
// Per thread: 2 x 256-bit loads -> bit planes -> masks -> block transfer
// function.  The carries {odd_backslash, in_string, prev_separator} are
// resolved by a warp scan of transfer functions, a CTA scan and a decoupled
// look-back across tiles (channel 1).  Then every block knows its strings:
// its index entries and string-buffer bytes (weights, strblock.cuh) go
// through a second look-back (channel 2: index count, string bytes), and the
// tile's index, per-entry string offsets (aux) and string payload are staged
// in shared memory and written out coalesced.
#include <cuda_runtime.h>

#include <mutex>

#include "lookback.cuh"
#include "shard.h"
#include "stage1.h"
#include "stage1_block.cuh"
#include "strblock.cuh"

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


// A 16-byte chunk of a block's payload copy: every byte is stored at the
// running shared-memory address d if its weight bit (ww) is set; d += 1 for a
// weight bit, += 4 for an opening quote (ow: the length field).  Written as
// predicated instructions on one address register: the arithmetic form
// (d += bit + 4 * quote bit, address = base + d) was 8 instructions per byte.
#define JT_PB(BIT, WORD, SH)                                                                        \
  "and.b32 t, %5, " #BIT ";\n\tsetp.ne.u32 p, t, 0;\n\tand.b32 t, %6, " #BIT ";\n\tsetp.ne.u32 q, t, 0;\n\t" \
  "shr.u32 v, " WORD ", " #SH ";\n\t@p st.shared.u8 [%0], v;\n\t@p add.u32 %0, %0, 1;\n\t@q add.u32 %0, %0, 4;\n\t"
#define JT_PW(B0, B1, B2, B3, WORD) JT_PB(B0, WORD, 0) JT_PB(B1, WORD, 8) JT_PB(B2, WORD, 16) JT_PB(B3, WORD, 24)
__device__ __forceinline__ void pay_chunk(uint32_t &d, const uint4 v, uint32_t ww, uint32_t ow) {
  asm volatile(
      "{\n\t"
      ".reg .pred p, q;\n\t"
      ".reg .b32 t, v;\n\t"
      JT_PW(1, 2, 4, 8, "%1") JT_PW(16, 32, 64, 128, "%2") JT_PW(256, 512, 1024, 2048, "%3")
      JT_PW(4096, 8192, 16384, 32768, "%4")
      "}"
      : "+r"(d)
      : "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(ww), "r"(ow)
      : "memory");
}
#undef JT_PW
#undef JT_PB

// byte run copy inside shared memory (offsets from the dynamic smem base):
// head bytes to align the destination, then funnel-shifted words
__device__ __forceinline__ void smem_copy(uint8_t *base, uint32_t dst, uint32_t src, int n) {
  while (n > 0 && (dst & 3)) {
    base[dst++] = base[src++];
    n--;
  }
  const uint32_t *s4 = (const uint32_t *)base;
  uint32_t *d4 = (uint32_t *)base;
  const uint32_t sh = (src & 3) * 8;
  uint32_t si = src >> 2, di = dst >> 2;
  int nw = n >> 2;
  uint32_t lo = nw ? s4[si] : 0;
  for (int k = 0; k < nw; k++) {
    uint32_t hi = s4[si + k + 1];
    d4[di + k] = __funnelshift_r(lo, hi, sh);
    lo = hi;
  }
  dst += 4 * nw;
  src += 4 * nw;
  n -= 4 * nw;
  while (n > 0) {
    base[dst++] = base[src++];
    n--;
  }
}

// Block-relative bytes: the tile's shared copy for the block's own 64 bytes,
// the (never written) global input past them.  Escapes are decoded in place
// in the shared copy, so a window reaching into the NEXT block must not read
// it there: that block may already have rewritten an escape of its own (a
// decoded byte can turn an invalid escape of this block into a valid one).
// window12 loads 12 bytes at once (aligned 32-bit loads + funnel shifts).
struct TileBytes {
  const uint8_t *s;    // shared tile copy
  const uint8_t *g;    // global tile base (4-byte aligned)
  uint32_t local;      // block offset in the tile
  __device__ __forceinline__ uint32_t operator()(uint64_t k) const {
    const uint64_t rel = local + k;
    return k < 64 ? (uint32_t)s[rel] : (uint32_t)g[rel];
  }
  // 12 bytes from block-relative k out of the shared copy only (for escapes
  // that lie inside the block: bytes past it are loaded but not used)
  __device__ __forceinline__ void window_own(uint64_t k, uint32_t w[3]) const {
    const uint32_t rel = (uint32_t)(local + k);
    const uint32_t sh = (rel & 3) * 8;
    const uint32_t *s4 = (const uint32_t *)s + (rel >> 2);
    const uint32_t a0 = s4[0], a1 = s4[1], a2 = s4[2], a3 = s4[3];
    w[0] = __funnelshift_r(a0, a1, sh);
    w[1] = __funnelshift_r(a1, a2, sh);
    w[2] = __funnelshift_r(a2, a3, sh);
  }
  __device__ __forceinline__ void window12(uint64_t k, uint32_t w[3]) const {
    const uint32_t rel = (uint32_t)(local + k);
    const uint32_t sh = (rel & 3) * 8;
    uint32_t a0, a1, a2, a3;
    if ((k & ~3ULL) + 16 <= 64) {
      const uint32_t *s4 = (const uint32_t *)s + (rel >> 2);
      a0 = s4[0], a1 = s4[1], a2 = s4[2], a3 = s4[3];
    } else {
      const uint32_t *g4 = (const uint32_t *)g + (rel >> 2);
      a0 = g4[0], a1 = g4[1], a2 = g4[2], a3 = g4[3];
    }
    w[0] = __funnelshift_r(a0, a1, sh);
    w[1] = __funnelshift_r(a1, a2, sh);
    w[2] = __funnelshift_r(a2, a3, sh);
  }
};

// shared memory layout (dynamic)
constexpr int kSmemIn = kStage1Tile;            // tile input bytes
constexpr int kSmemIdx = kStageIdx * 2;         // u16 positions
// per-block record for the copy-out: masks of the block's tokens and the
// block's tile-relative offsets (index entries get their string offset, tape
// index and depth from popcounts below their bit; W = string weight mask,
// strblock.cuh escape_weights)
struct BlockRec {
  uint64_t W, openq, w1, w2, op, cl;
  uint32_t soff, toff;
  int32_t doff;
  uint32_t pad;
};
constexpr int kSmemBlk = kThreads * (int)sizeof(BlockRec);
constexpr int kSmemPay = kStagePay;             // payload bytes (last: word over-read)
constexpr int kOffBlk = kSmemIn + kSmemIdx;
constexpr int kOffPay = kOffBlk + kSmemBlk;
constexpr int kSmemBytes = kOffPay + kSmemPay + 16;
// record (NDJSON) mode: per-block newline data for the copy-out
struct RecBlk {
  uint64_t fin, nl;  // index entries, '\n' bytes
  uint32_t off;      // tile-relative index slot of the block
  uint32_t rid;      // record id at the block start (newlines before it)
};
constexpr int kOffRec = (kSmemBytes + 15) & ~15;
constexpr int kSmemBytesRec = kOffRec + kThreads * (int)sizeof(RecBlk);

// depth_before, relative to the range start (a shard adds its base in stage
// 2); clamped where the document has already failed (|d| > kMaxDepth + base)
__device__ __forceinline__ int clamp16(long long d) { return d < -8192 ? -8192 : d > 8192 ? 8192 : (int)d; }

// ---- K0: carry-in of every tile (reduce-then-scan) --------------------------
// The tile carry (odd backslash run, in-string, previous byte a separator;
// blocks.h:31-35) is a 3-bit state whose per-block transfer functions compose
// (stage1_block.cuh).  K0a reduces each 16 KiB tile to one function, K0b scans
// the functions in one CTA, and K1 reads its carry-in at start: no chained
// look-back on this channel.

// K0a: transfer function of each tile.  128 threads x 2 blocks per tile, all
// four 32-byte loads of a thread issued together.
constexpr int kFnThreads = kStage1Tile / 128;
// It also leaves, per tile, the escape overhang INTO the tile (strblock.cuh
// overhang_in_scan: input / weight bytes of an escape begun before the tile
// that reach into it, and the decoded bytes that spill) for the case that the
// tile starts inside a string -- K1's first block needs it, and there the
// scan would be a chain of dependent byte reads by one thread with its CTA
// waiting at a barrier.  tile_ov[t] = ov | spill << 4 | spill bytes << 8.
struct AbsAt {
  const uint8_t *in;
  __device__ __forceinline__ uint32_t operator()(uint64_t i) const { return in[i]; }
};

template <bool kRec>
__global__ void __launch_bounds__(kFnThreads) k_carry_fn(const uint8_t *in0, uint64_t begin, uint32_t *fn,
                                                          uint32_t *nl_count, uint32_t *tile_ov) {
  __shared__ uint32_t s_f[kFnThreads / 32];
  __shared__ uint32_t s_nl;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (kRec && threadIdx.x == 0) s_nl = 0;
  const uint8_t *in = in0 + begin;
  const uint64_t blk = (uint64_t)blockIdx.x * kStage1Tile + (uint64_t)threadIdx.x * 128;
  uint32_t w[32];
  ld256(in + blk, w);
  ld256(in + blk + 32, w + 8);
  ld256(in + blk + 64, w + 16);
  ld256(in + blk + 96, w + 24);
  // the 16 bytes before the tile, for the overhang scan at the end
  const uint64_t tb = begin + (uint64_t)blockIdx.x * kStage1Tile;  // document offset of the tile
  uint4 before = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == kFnThreads - 1 && tb >= 16) before = *(const uint4 *)(in0 + tb - 16);
  uint32_t f2[2];
  uint32_t nlc = 0;
#pragma unroll
  for (int h = 0; h < 2; h++) {
    s1::Masks m;
    s1::classify64(w + 16 * h, m);
    if constexpr (kRec) {
      const uint64_t nl = s1::newline_mask(m.P);  // bytes past len are 0, never newlines
      nlc += popc64(nl);
      f2[h] = s1::block_function_rec(m, s1::escaped_no_carry(m.bs), s1::carry_toggle(m.bs), nl);
    } else {
      f2[h] = s1::block_function(m, s1::escaped_no_carry(m.bs), s1::carry_toggle(m.bs));
    }
  }
  uint32_t inc = s1::compose(f2[1], f2[0]);
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) inc = s1::compose(inc, o);
  }
  if (lane == 31) s_f[warp] = inc;
  if constexpr (kRec) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nlc += __shfl_xor_sync(0xffffffffu, nlc, o);
  }
  __syncthreads();
  if (kRec && lane == 0) atomicAdd(&s_nl, nlc);
  if (kRec) __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t agg = s_f[0];
#pragma unroll
    for (int k = 1; k < kFnThreads / 32; k++) agg = s1::compose(s_f[k], agg);
    fn[blockIdx.x] = agg;
    if (kRec) nl_count[blockIdx.x] = s_nl;
  }
  // after the CTA's barrier: nobody waits for this chain of byte reads
  if (threadIdx.x == kFnThreads - 1) {
    uint32_t packed = 0;
    if (tb >= 16) {
      // no backslash among the 12 bytes before the tile: no escape reaches in
      const uint4 q = before;
      const uint32_t x1 = q.y ^ 0x5C5C5C5Cu, x2 = q.z ^ 0x5C5C5C5Cu, x3 = q.w ^ 0x5C5C5C5Cu;
      const uint32_t z = ((x1 - 0x01010101u) & ~x1) | ((x2 - 0x01010101u) & ~x2) | ((x3 - 0x01010101u) & ~x3);
      if (z & 0x80808080u) {
        uint32_t spill_bytes = 0;
        const int r = sb::overhang_in_scan(AbsAt{in0}, tb, true, &spill_bytes);
        packed = (uint32_t)(r & 15) | ((uint32_t)(r >> 8) << 4) | (spill_bytes << 8);
      }
    }
    tile_ov[blockIdx.x] = packed;
  }
}

// K0b: carry-in of every tile = (f[t-1] o ... o f[0])(init); one CTA.  init =
// kInitState, or for shard g the state after shards 0..g-1 (their composed
// functions, `gathered`).  With carry == nullptr it only writes the
// composition of all tiles (*total).
// The tiles go through shared memory in chunks of kScanChunk: loaded and
// stored coalesced (one 4-byte word per lane, any alignment of fn / carry),
// each thread scanning kScanPer contiguous tiles of the chunk out of shared
// memory (padded: conflict-free).  The next chunk's loads are in flight while
// the current one is scanned.  (Thread-contiguous global chunks were 8 scalar
// requests per 32-byte sector: 62 us on C4's 65,539 tiles.)
constexpr int kScanThreads = 1024;
constexpr int kScanPer = 8;
constexpr int kScanChunk = kScanThreads * kScanPer;
__device__ __forceinline__ uint32_t scan_pad(uint32_t i) { return i + (i >> 3); }
__global__ void __launch_bounds__(kScanThreads) k_carry_scan(const uint32_t *fn, uint32_t *carry,
                                                             uint64_t ntiles, const Sum0 *gathered,
                                                             uint32_t g, Sum0 *total,
                                                             const uint32_t *nl_count,
                                                             uint32_t *nl_base, uint64_t *nl_total,
                                                             const uint32_t *init_state = nullptr,
                                                             uint32_t *out_state = nullptr) {
  __shared__ uint32_t s_v[kScanChunk + kScanChunk / 8];
  __shared__ uint32_t s_agg[kScanThreads / 32];
  __shared__ uint32_t s_has[kScanThreads / 32];
  __shared__ uint32_t s_nlw[kScanThreads / 32];
  __shared__ uint32_t s_run;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // state before the range: earlier shards' functions applied to the initial state
  uint32_t run = init_state ? *init_state : s1::kInitState;
  if (gathered)
    for (uint32_t h = 0; h < g; h++) run = s1::apply(gathered[h].fn, run);
  uint32_t tot = 0;  // carry == nullptr: composition of the tiles so far (thread 0)
  bool tot_has = false;
  uint32_t nv[kScanPer];
#pragma unroll
  for (int j = 0; j < kScanPer; j++) {
    const uint64_t t = (uint64_t)j * kScanThreads + threadIdx.x;
    nv[j] = t < ntiles ? __ldg(fn + t) : 0u;
  }
  for (uint64_t c0 = 0; c0 < ntiles; c0 += kScanChunk) {
#pragma unroll
    for (int j = 0; j < kScanPer; j++) s_v[scan_pad(j * kScanThreads + threadIdx.x)] = nv[j];
    __syncthreads();
    // the next chunk's words, in flight during this chunk's scan
#pragma unroll
    for (int j = 0; j < kScanPer; j++) {
      const uint64_t t = c0 + kScanChunk + (uint64_t)j * kScanThreads + threadIdx.x;
      nv[j] = t < ntiles ? __ldg(fn + t) : 0u;
    }
    const uint64_t first = c0 + (uint64_t)threadIdx.x * kScanPer;
    const int cnt = first >= ntiles ? 0 : ntiles - first >= (uint64_t)kScanPer ? kScanPer : (int)(ntiles - first);
    uint32_t v[kScanPer];
#pragma unroll
    for (int j = 0; j < kScanPer; j++) v[j] = s_v[scan_pad(threadIdx.x * kScanPer + j)];
    uint32_t acc = v[0];
#pragma unroll
    for (int j = 1; j < kScanPer; j++)
      if (j < cnt) acc = s1::compose(v[j], acc);
    bool has = cnt > 0;
    // warp inclusive scan over (has, acc)
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      uint32_t o = __shfl_up_sync(0xffffffffu, acc, d);
      uint32_t oh = __shfl_up_sync(0xffffffffu, has ? 1u : 0u, d);
      if (lane >= d && oh) {
        acc = has ? s1::compose(acc, o) : o;
        has = true;
      }
    }
    if (lane == 31) {
      s_agg[warp] = acc;
      s_has[warp] = has;
    }
    __syncthreads();
    if (carry == nullptr) {
      if (threadIdx.x == 0) {
        for (int k = 0; k < kScanThreads / 32; k++)
          if (s_has[k]) {
            tot = tot_has ? s1::compose(s_agg[k], tot) : s_agg[k];
            tot_has = true;
          }
      }
      __syncthreads();  // s_v / s_agg are rewritten by the next chunk
      continue;
    }
    // exclusive prefix state of this thread: the chunks before, earlier warps,
    // then earlier lanes
    uint32_t state = run;
    for (int k = 0; k < warp; k++)
      if (s_has[k]) state = s1::apply(s_agg[k], state);
    uint32_t ex = __shfl_up_sync(0xffffffffu, acc, 1);
    uint32_t exh = __shfl_up_sync(0xffffffffu, has ? 1u : 0u, 1);
    if (lane > 0 && exh) state = s1::apply(ex, state);
#pragma unroll
    for (int j = 0; j < kScanPer; j++)
      if (j < cnt) {
        s_v[scan_pad(threadIdx.x * kScanPer + j)] = state;
        state = s1::apply(v[j], state);
      }
    // the last thread ends where the chunk ends (with or without tiles of its own)
    if (threadIdx.x == kScanThreads - 1) s_run = state;
    __syncthreads();
    run = s_run;
#pragma unroll
    for (int j = 0; j < kScanPer; j++) {
      const uint64_t t = c0 + (uint64_t)j * kScanThreads + threadIdx.x;
      if (t < ntiles) carry[t] = s_v[scan_pad(j * kScanThreads + threadIdx.x)];
    }
    __syncthreads();  // s_v is rewritten by the next chunk
  }
  if (carry == nullptr) {
    if (threadIdx.x == 0) total->fn = tot;  // a range has at least one tile
    return;
  }
  if (out_state && threadIdx.x == 0) *out_state = run;  // state after the last tile
  if (nl_count == nullptr) return;
  // record mode: exclusive prefix of the tiles' newline counts (record ids),
  // each thread a contiguous chunk of tiles
  const uint64_t per = (ntiles + kScanThreads - 1) / kScanThreads;
  const uint64_t lo = threadIdx.x * per;
  const uint64_t hi = lo + per < ntiles ? lo + per : ntiles;
  uint32_t mine = 0;
  for (uint64_t t = lo; t < hi; t++) mine += nl_count[t];
  uint32_t incl = mine;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    uint32_t o = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += o;
  }
  if (lane == 31) s_nlw[warp] = incl;
  __syncthreads();
  uint32_t nrun = incl - mine;
  for (int k = 0; k < warp; k++) nrun += s_nlw[k];
  for (uint64_t t = lo; t < hi; t++) {
    nl_base[t] = nrun;
    nrun += nl_count[t];
  }
  if (threadIdx.x == kScanThreads - 1) *nl_total = nrun;
}

// record mode: per-record error slots (~0 = none), first record start
__global__ void k_rec_init(Stage1Args a) {
  const uint64_t n = *a.nl_total + 1;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < n; k += stride) {
    a.rec_utf8[k] = ~0u;
    a.rec_serr[k] = ~0u;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) a.rec_start[0] = 0;
}

#ifndef JT_K1_MINB
#define JT_K1_MINB 3
#endif
template <bool kRec>
__global__ void __launch_bounds__(kThreads, JT_K1_MINB) k_stage1(Stage1Args a) {
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_warp_nl[kWarps];
  __shared__ uint32_t s_warp_tdf[kWarps];
  __shared__ __align__(16) uint32_t s_warp_f[kWarps];
  static_assert(kWarps == 8, "the per-warp totals are read as two 16-byte words");
  __shared__ __align__(16) uint32_t s_warp_cnt[kWarps];
  __shared__ __align__(16) uint32_t s_warp_sw[kWarps];
  __shared__ __align__(16) uint32_t s_warp_tw[kWarps];
  __shared__ __align__(16) int s_warp_td[kWarps];
  __shared__ int s_warp_ov[kWarps];
  __shared__ unsigned long long s_base, s_sbase, s_tbase;
  __shared__ uint32_t s_lb_claim;  // the first warp done staging resolves the tile's counts
  __shared__ long long s_dbase;
  extern __shared__ __align__(16) uint8_t smem[];
  uint8_t *s_in = smem;
  uint16_t *s_idx = (uint16_t *)(smem + kSmemIn);
  BlockRec *s_blk = (BlockRec *)(smem + kOffBlk);
  uint8_t *s_pay = smem + kOffPay;
  RecBlk *s_rec = (RecBlk *)(smem + kOffRec);  // record mode only

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#ifdef JT_K1_TMA
  // A/B build (tools/ab_bench.sh): the tile arrives in shared memory by one
  // bulk async copy (TMA, cp.async.bulk + mbarrier) issued by thread 0 as soon
  // as it has claimed the tile; every thread then reads its 64 bytes back
  // from shared memory instead of loading them and storing the copy.
  __shared__ __align__(8) unsigned long long s_mbar;
  const uint32_t mbar = (uint32_t)__cvta_generic_to_shared(&s_mbar);
#endif
  if (threadIdx.x == 0) {
#ifdef JT_K1_TMA
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
#endif
    s_tile = atomicAdd(a.tile_counter, 1u);
    s_lb_claim = 0;
#ifdef JT_K1_TMA
    {
      const uint8_t *src = a.in + a.begin + (uint64_t)s_tile * kStage1Tile;
      const uint32_t dst = (uint32_t)__cvta_generic_to_shared(smem);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"((uint32_t)kStage1Tile)
                   : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
          "l"(src), "r"((uint32_t)kStage1Tile), "r"(mbar)
          : "memory");
    }
#endif
  }
  __syncthreads();
  const int64_t tile = s_tile;  // tile of the range; byte offset below is global
  if (threadIdx.x == 0) {
    JT_TL(tile, 0);
  }
  const uint64_t tile_base = a.begin + (uint64_t)tile * kStage1Tile;
  const uint64_t blk = tile_base + (uint64_t)threadIdx.x * 64;
  const uint32_t local = threadIdx.x * 64;

  const uint32_t carry_in = a.carry[tile];  // K0b output, read early
  // K0a: the escape overhang into the tile if it starts inside a string
  // (the slot becomes the tile's flag when the tile is done)
  const uint32_t tile_ov = threadIdx.x == 0 ? a.tile_flags[a.rec_tile0 + tile] : 0u;
  uint32_t w[16];
#ifdef JT_K1_TMA
  {
    uint32_t ok;
    do {
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(ok)
          : "r"(mbar)
          : "memory");
    } while (!ok);
    const uint4 *q = (const uint4 *)(s_in + threadIdx.x * 64);
    const uint4 q0 = q[0], q1 = q[1], q2 = q[2], q3 = q[3];
    w[0] = q0.x, w[1] = q0.y, w[2] = q0.z, w[3] = q0.w, w[4] = q1.x, w[5] = q1.y, w[6] = q1.z, w[7] = q1.w;
    w[8] = q2.x, w[9] = q2.y, w[10] = q2.z, w[11] = q2.w, w[12] = q3.x, w[13] = q3.y, w[14] = q3.z, w[15] = q3.w;
  }
#else
  ld256(a.in + blk, w);
  ld256(a.in + blk + 32, w + 8);
  {
    uint4 *d = (uint4 *)(s_in + threadIdx.x * 64);
    d[0] = make_uint4(w[0], w[1], w[2], w[3]);
    d[1] = make_uint4(w[4], w[5], w[6], w[7]);
    d[2] = make_uint4(w[8], w[9], w[10], w[11]);
    d[3] = make_uint4(w[12], w[13], w[14], w[15]);
  }
#endif

  s1::Masks m;
  s1::classify64(w, m);
  const uint64_t esc0 = s1::escaped_no_carry(m.bs);
  const uint64_t tog = s1::carry_toggle(m.bs);
  uint64_t nl = 0;  // record mode: '\n' bytes end records
  uint32_t f;
  if constexpr (kRec) {
    nl = s1::newline_mask(m.P);
    f = s1::block_function_rec(m, esc0, tog, nl);
  } else {
    f = s1::block_function(m, esc0, tog);
  }
  const uint32_t nlc = popc64(nl);
  uint32_t nli = nlc;
  if constexpr (kRec) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      uint32_t o = __shfl_up_sync(0xffffffffu, nli, d);
      if (lane >= d) nli += o;
    }
    if (lane == 31) s_warp_nl[warp] = nli;
  }

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
  if (!kRec && (m.P[7] | (uint64_t)(prev & 0x80808000u)) != 0 && blk < a.len + 3) {
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

  // record mode: record id at the block start; UTF-8 errors per record
  uint32_t rid_blk = 0;
  if constexpr (kRec) {
    rid_blk = a.nl_base[tile] + nli - nlc;
    for (int k = 0; k < warp; k++) rid_blk += s_warp_nl[k];
    if ((m.P[7] | (uint64_t)(prev & 0x80808000u)) != 0 && blk < a.len + 3 &&
        s1::utf8_block_error(m.P, prev, blk + 64 >= a.len)) {
      const uint8_t *in = a.in;
      const uint64_t len = a.len;
      auto at = [in, len](uint64_t i) -> uint32_t { return i < len ? in[i] : 0u; };
      uint64_t lo = blk >= 3 ? blk - 3 : 0, hi = blk + 64 < len ? blk + 64 : len;
      for (uint64_t i = lo; i < hi; i++)
        if (s1::utf8_flagged(at, i, len)) {
          uint32_t rid = rid_blk;
          if (i >= blk) {
            rid += popc64(nl & sb::low_bits((int)(i - blk)));
          } else {
            for (uint64_t j = i; j < blk; j++) rid -= in[j] == '\n';
          }
          atomicMin(a.rec_utf8 + rid, (uint32_t)i);
        }
    }
  }

  // this warp's carry state: the tile's carry-in (K0 pre-pass, no look-back)
  // through the earlier warps' functions, folded by every warp itself (no
  // second barrier)
  uint32_t state = carry_in;
  {
    // all eight functions loaded at once: the chain below is register-only
    const uint4 f03 = *(const uint4 *)&s_warp_f[0], f47 = *(const uint4 *)&s_warp_f[4];
    const uint32_t wf[kWarps] = {f03.x, f03.y, f03.z, f03.w, f47.x, f47.y, f47.z, f47.w};
#pragma unroll
    for (int k = 0; k < kWarps - 1; k++)
      if (k < warp) state = s1::apply(wf[k], state);
  }
  if (lane > 0) state = s1::apply(excl, state);
  int64_t rem = (int64_t)a.len - (int64_t)blk;
  const uint64_t valid = rem >= 64 ? ~0ULL : rem <= 0 ? 0ULL : ((1ULL << rem) - 1);

  // masks under the resolved carry (string_mask + finalize_structurals)
  const uint64_t esc = (state & 1) ? (esc0 ^ tog) : esc0;
  const uint64_t uq = m.qt & ~esc;
  const uint64_t instr = kRec ? s1::instr_records(uq, state & 2, nl)
                              : s1::prefix_xor(uq) ^ ((state & 2) ? ~0ULL : 0ULL);
  uint64_t fin;
  {
    uint64_t st1 = (m.st & ~instr) | uq;
    uint64_t cand = st1 | m.ws;
    uint64_t pseudo = ((cand << 1) | (uint64_t)(state >> 2)) & ~m.ws & ~instr;
    fin = (st1 | pseudo) & ~(uq & ~instr) & valid;
  }
  const uint32_t cnt = popc64(fin);
  // token widths (A.4: 0 for , :  2 for numbers, else 1) and depth changes
  // as masks, so every sum below is a popcount
  const uint64_t w1m = fin & ~m.cc, w2m = fin & m.num;
  const uint64_t opm = fin & m.open, clm = fin & m.close;
  const uint32_t tw = popc64(w1m) + popc64(w2m);
  int td = popc64(opm) - popc64(clm);
  uint32_t tdf = 0;  // record mode: the block resets the depth (a newline)
  if constexpr (kRec) {
    if (nl) {
      const int last = 63 - clz64(nl);
      const uint64_t above = last >= 63 ? 0ULL : (~0ULL << (last + 1));
      td = popc64(opm & above) - popc64(clm & above);
      tdf = 1;
    }
  }

  // strings in this block
  const uint64_t openq = uq & instr & valid;
  const uint64_t content = instr & ~openq & valid;
  const uint64_t E = s1::unescaped_backslash(m.bs, state & 1) & content;
  const uint64_t ctl = sb::control_mask(m.P) & content;
  const TileBytes tbyte{s_in, a.in + tile_base, local};
  // decoded escape bytes go in place over their weight positions of the tile
  // copy (strblock.cuh); an escape straddling the tile end leaves its spilled
  // bytes to the next tile's first block
  auto rewrite = [&](int k, uint8_t b) {
    const uint32_t r = local + (uint32_t)k;
    if (r < (uint32_t)kStage1Tile) s_in[r] = b;
  };
  // step 1 (strblock.cuh): classes, \u masks, failing starts; an escape
  // reaching into the next block is decoded and written now: ov | spill << 8
  sb::BlockEsc be;
  be.ec = sb::EscClass{0, 0, 0, 0};
  be.bmp = be.pair = be.ucov = be.uvirt = be.bad = 0;
  be.ov_out = 0;
  if (E) be = sb::block_escapes(m.P, m.qt, m.bs, E, tbyte, rewrite);
  const int ov_out = be.ov_out;
  int ov_in = __shfl_up_sync(0xffffffffu, ov_out, 1);
  if (lane == 31) s_warp_ov[warp] = ov_out;
  // unterminated string: the reference reads the NUL padding at len (in
  // record mode: at the record's end, a newline or len)
  if constexpr (kRec) {
    for (uint64_t q = nl; q; q &= q - 1) {
      const int r = ctz64(q);
      const uint32_t before = r > 0 ? (uint32_t)((instr >> (r - 1)) & 1) : ((state >> 1) & 1);
      if (before) atomicMin(a.rec_serr + rid_blk + popc64(nl & sb::low_bits(r)), (uint32_t)(blk + r));
    }
    if (rem > 0 && rem <= 64 && ((instr >> (rem - 1)) & 1))
      atomicMin(a.rec_serr + rid_blk + popc64(nl & sb::low_bits((int)rem)), (uint32_t)a.len);
  } else {
    if (rem > 0 && rem <= 64 && ((instr >> (rem - 1)) & 1)) atomicMin(a.str_err, (unsigned long long)a.len);
  }

  // CTA exclusive scan of (index count, string bytes); the block weight of a
  // slow block needs ov_in, which for lane 0 comes from the previous warp
  uint32_t ci = cnt;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    uint32_t o = __shfl_up_sync(0xffffffffu, ci, d);
    if (lane >= d) ci += o;
  }
  if (lane == 31) s_warp_cnt[warp] = ci;
  __syncthreads();
  if (threadIdx.x == 0) JT_TL(tile, 1);
  // the tile's first block also gets the decoded bytes an escape of the
  // previous tile spills into it (that tile's staging drops them)
  uint32_t spill_bytes = 0;
  if (lane == 0) {
    if (warp > 0) ov_in = s_warp_ov[warp - 1];
    else if (state & 2) {
      ov_in = (int)((tile_ov & 15) | (((tile_ov >> 4) & 15) << 8));
      spill_bytes = tile_ov >> 8;
    } else {
      ov_in = 0;
    }
  }
  const int vin = ov_in >> 8;
  ov_in &= 0xFF;
  // the tile's first block: the decoded bytes an escape of the previous tile
  // spills into it go to their weight positions of the tile copy (the copy
  // below takes every weighted byte in order)
  for (int k = 0; k < vin && threadIdx.x == 0; k++) s_in[k] = (uint8_t)(spill_bytes >> (8 * k));
  // step 2: the string weight mask -- the plain string bytes, or for blocks
  // with escapes the weight positions of each escape (strblock.cuh)
  const bool esc_work = (E | (uint64_t)ov_in) != 0;
  uint64_t W = content;
  {
    uint64_t em = ctl;  // every error candidate of the block
    if (esc_work) {
      W = sb::block_weights(content, be, ov_in, vin);
      em |= be.bad;
    }
    if constexpr (kRec) {
      while (em) {  // the first error of each record in the block
        const int q = ctz64(em);
        atomicMin(a.rec_serr + rid_blk + popc64(nl & sb::low_bits(q)), (uint32_t)(blk + q));
        const uint64_t nxt = nl & ~sb::low_bits(q + 1);
        em = nxt ? em & ~sb::low_bits(ctz64(nxt) + 1) : 0;
      }
    } else if (em) {
      atomicMin(a.str_err, (unsigned long long)(blk + (uint64_t)ctz64(em)));
    }
  }
  // step 3 (the escapes inside the block, decoded in place) waits until the
  // tile's counts are published: only this block's payload copy needs it
  const uint64_t dec_tr = be.ec.tr, dec_bmp = be.bmp, dec_pair = be.pair;
  const uint32_t sw = 4u * popc64(openq) + popc64(W);
  uint32_t si = sw;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    uint32_t o = __shfl_up_sync(0xffffffffu, si, d);
    if (lane >= d) si += o;
  }
  uint32_t ti = tw;
  int di = td;
  uint32_t df = tdf;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    uint32_t o = __shfl_up_sync(0xffffffffu, ti, d);
    int od = __shfl_up_sync(0xffffffffu, di, d);
    uint32_t of = kRec ? __shfl_up_sync(0xffffffffu, df, d) : 0u;
    if (lane >= d) {
      ti += o;
      if (!df) di += od;  // segmented (record mode); df == 0 otherwise
      df |= of;
    }
  }
  // block-exclusive depth (record mode: segmented) from the previous lane
  int dex = __shfl_up_sync(0xffffffffu, di, 1);
  uint32_t dexf = kRec ? __shfl_up_sync(0xffffffffu, df, 1) : 0u;
  if (lane == 0) dex = 0, dexf = 0;
  if (lane == 31) {
    s_warp_sw[warp] = si;
    s_warp_tw[warp] = ti;
    s_warp_td[warp] = di;
    s_warp_tdf[warp] = df;
  }
  __syncthreads();
  if (threadIdx.x == 0) JT_TL(tile, 2);
  uint32_t woff = 0, total = 0, wsoff = 0, stotal = 0, wtoff = 0, ttotal = 0;
  int wdoff = 0, dtotal = 0;
  uint32_t wdf = 0, dtf = 0;  // record mode: resets before this warp / in the tile
  uint32_t wc8[kWarps], ws8[kWarps], wt8[kWarps], wd8[kWarps];
  {
    auto ld8 = [](const void *p, uint32_t v[kWarps]) {
      const uint4 lo = ((const uint4 *)p)[0], hi = ((const uint4 *)p)[1];
      v[0] = lo.x, v[1] = lo.y, v[2] = lo.z, v[3] = lo.w, v[4] = hi.x, v[5] = hi.y, v[6] = hi.z, v[7] = hi.w;
    };
    ld8(s_warp_cnt, wc8);
    ld8(s_warp_sw, ws8);
    ld8(s_warp_tw, wt8);
    ld8(s_warp_td, wd8);
  }
#pragma unroll
  for (int k = 0; k < kWarps; k++) {
    uint32_t c = wc8[k], s = ws8[k], t = wt8[k];
    int dd = (int)wd8[k];
    const uint32_t fk = kRec ? s_warp_tdf[k] : 0u;
    woff += k < warp ? c : 0;
    wsoff += k < warp ? s : 0;
    wtoff += k < warp ? t : 0;
    if (k < warp) {
      wdoff = fk ? dd : wdoff + dd;
      wdf |= fk;
    }
    total += c;
    stotal += s;
    ttotal += t;
    dtotal = fk ? dd : dtotal + dd;
    dtf |= fk;
  }
  const uint32_t toff = wtoff + ti - tw;  // tile-relative tape words
  // tile-relative depth at the block start (segmented in record mode:
  // doff_f = a reset lies between the tile start and the block)
  const int doff = dexf ? dex : wdoff + dex;
  const uint32_t doff_f = wdf | dexf;
  const uint32_t off = woff + ci - cnt;   // tile-relative index slot
  const uint32_t soff = wsoff + si - sw;  // tile-relative string byte

  // Look-back 2.  The aggregate goes out now; the prefix is only needed by
  // the copy-out (staging below is tile-relative), so warp 0 emits its own
  // blocks first and looks back afterwards, when the predecessors have most
  // likely published their inclusive prefixes (one round trip, no polling).
  // Tiles that overflow the staging write to global directly and resolve
  // first.
  const bool idx_direct = total > (uint32_t)kStageIdx;
  const bool pay_direct = stotal > (uint32_t)kStagePay;
  const bool direct = idx_direct || pay_direct;  // CTA-uniform
  const uint64_t tdepth = kRec ? ((dtf ? kSegFlag : 0ULL) | ((uint64_t)(long long)dtotal & kSegMask))
                                : ((unsigned long long)(long long)dtotal & kQuadMask);
  const Quad tot{{total, stotal, ttotal, tdepth}};
  const int64_t gt = (int64_t)a.rec_tile0 + tile;  // tile in the document's records
  const int64_t last_tile = a.last_tile == ~0ULL ? (int64_t)a.ntiles - 1 : (int64_t)a.last_tile;
  auto resolve_counts = [&]() {  // one full warp
    Quad base{{0, 0, 0, 0}};
    if (gt > 0) base = quad_lookback<kRec>(a.rec_count, gt);
    if (lane == 0) {
      JT_TL(tile, 5);
      Quad inc;
#pragma unroll
      for (int k = 0; k < 3; k++) inc.v[k] = (base.v[k] + tot.v[k]) & kQuadMask;
      inc.v[3] = kRec ? seg_combine(base.v[3], tot.v[3]) : ((base.v[3] + tot.v[3]) & kQuadMask);
      quad_publish(a.rec_count, gt, 1, inc);
      s_base = base.v[0];
      s_sbase = base.v[1];
      s_tbase = base.v[2];
      s_dbase = kRec ? seg_value(base.v[3]) : sext63(base.v[3]);
      if (a.sb_out && tile == (int64_t)a.ntiles - 1) *a.sb_out = inc.v[1];  // host-mapped
      if (a.tok_out && tile == (int64_t)a.ntiles - 1) *a.tok_out = inc.v[0];
      if (gt == last_tile) {
        *a.total = inc.v[0];
        *a.total_strings = inc.v[1];
        *a.tape_words = 1 + inc.v[2];
        *a.depth_total = kRec ? seg_value(inc.v[3]) : sext63(inc.v[3]);
      }
    }
  };
  if (threadIdx.x == 0 && gt > 0) {
    JT_TL(tile, 4);
    quad_publish_agg(a.rec_count, gt, quad_pack_agg(total, stotal, ttotal, dtotal, kRec && dtf));
  }
  if (direct && warp == 0) resolve_counts();
  if (threadIdx.x == 0) JT_TL(tile, 6);
  s_blk[threadIdx.x] = BlockRec{W, openq, w1m, w2m, opm, clm, soff, toff, doff, doff_f};
  if constexpr (kRec) s_rec[threadIdx.x] = RecBlk{fin, nl, off, rid_blk};
  // stage positions (+ string offsets of slow blocks) and the string
  // payload; spill to global when the tile is larger than the staging
  if (direct) __syncthreads();  // s_base/s_sbase needed now
  const uint64_t gbase = direct ? s_base : 0;
  const uint64_t gsbase = direct ? s_sbase : 0;
  const uint64_t gtbase = idx_direct ? s_tbase : 0;
  const long long gdbase = idx_direct ? s_dbase : 0;
  auto direct_entry = [&](uint32_t slot, int p, uint32_t wb) {
    const uint64_t below = sb::low_bits(p);
    const uint32_t c = s_in[local + p];
    const uint32_t t = toff + popc64(w1m & below) + popc64(w2m & below);
    long long d = (doff_f ? 0 : gdbase) + doff + popc64(opm & below) - popc64(clm & below);
    uint32_t rid = 0;
    if constexpr (kRec) {
      const uint64_t nb = nl & below;
      rid = rid_blk + popc64(nb);
      if (nb) {  // depth since this record's start, inside the block
        const uint64_t since = below & ~sb::low_bits(64 - clz64(nb));
        d = popc64(opm & since) - popc64(clm & since);
      }
      a.rec_of[gbase + slot] = rid;
    }
    a.idx[gbase + slot] = (uint32_t)(tile_base + local + p);
    a.aux[gbase + slot] = (uint32_t)(gsbase + soff + wb);
    a.tokrec[gbase + slot] = c | ((uint32_t)(uint16_t)clamp16(d) << 16);
    a.tape_idx[gbase + slot] = (uint32_t)(1 + gtbase + t + 2 * rid);
  };
  {
    // the weighted bytes in order (escapes already decoded in place; the
    // first vin bits are the spill of the previous block's escape)
    uint64_t cm = W;
    if (dec_tr | dec_bmp | dec_pair)
      sb::decode_in_place(dec_tr, dec_bmp, dec_pair,
                          [&](uint64_t k, uint32_t w3[3]) { tbyte.window_own(k, w3); }, tbyte,
                          [&](int k, uint8_t b) { s_in[local + (uint32_t)k] = b; });
    if (!pay_direct) {
      // each lane copies its own block into the staging buffer, bytes in
      // order with a running destination (+1 per weight bit, +4 per opening
      // quote: the length field, filled by the copy-out); fully unrolled and
      // predicated, 16-byte chunks without string bytes skipped
      if (cm) {
        const uint4 *src = reinterpret_cast<const uint4 *>(s_in + local);
        uint32_t d = (uint32_t)__cvta_generic_to_shared(s_pay) + soff;  // shared-window address
#pragma unroll
        for (int c = 0; c < 4; c++) {
          const uint32_t ww = (uint32_t)(W >> (16 * c)) & 0xFFFFu;
          const uint32_t ow = (uint32_t)(openq >> (16 * c)) & 0xFFFFu;
          if (ww == 0) {
            d += 4u * (uint32_t)__popc(ow);
            continue;
          }
          const uint4 v = src[c];
          pay_chunk(d, v, ww, ow);
        }
      }
      cm = 0;
    }
    // direct (spilled) tiles: warp-uniform choice by the slowest lane's estimated cost (a warp runs
    // the union of its lanes' paths): ~6 instructions per byte for the byte
    // loop, ~35 per run plus a word copy per 4 bytes for the run loop
    const int nruns = popc64(cm & ~(cm << 1));
    int cost_byte = 6 * popc64(cm | openq), cost_run = 35 * nruns + popc64(cm) / 2;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      cost_byte = max(cost_byte, __shfl_xor_sync(0xffffffffu, cost_byte, o));
      cost_run = max(cost_run, __shfl_xor_sync(0xffffffffu, cost_run, o));
    }
    if (cost_byte < cost_run) {
      // fragmented (escape-dense) block: byte by byte, destinations counted
      // as the bits go by (an opening quote adds its 4-byte length field)
      uint64_t bits = cm | openq;
      uint32_t wdst = 0;
      while (bits) {
        const int k = ctz64(bits);
        bits &= bits - 1;
        if ((openq >> k) & 1) {
          wdst += 4;
        } else {
          const uint8_t b = s_in[local + k];
          if (pay_direct) a.strings[gsbase + soff + wdst] = b;
          else s_pay[soff + wdst] = b;
          wdst++;
        }
      }
      cm = 0;
    }
    while (cm) {  // string runs, 4-byte gaps before each run opened here
      const int a0 = ctz64(cm);
      const uint64_t sh = cm >> a0;
      const int n = ~sh == 0 ? 64 - a0 : ctz64(~sh);
      const uint64_t below = sb::low_bits(a0);
      const uint32_t wdst = 4u * popc64(openq & below) + popc64(W & below);
      if (pay_direct) {
        for (int k = 0; k < n; k++) a.strings[gsbase + soff + wdst + k] = s_in[local + a0 + k];
      } else {
        smem_copy(smem, kOffPay + soff + wdst, local + a0, n);
      }
      cm &= ~(sb::low_bits(n) << a0);
    }
    uint64_t fm = fin;
    uint32_t slot = off;
    while (fm) {
      const int p = ctz64(fm);
      fm &= fm - 1;
      if (idx_direct) {
        const uint64_t below = sb::low_bits(p);
        direct_entry(slot, p, 4u * popc64(openq & below) + popc64(W & below));
      } else {
        s_idx[slot] = (uint16_t)(local + p);
      }
      slot++;
    }
  }
  if (threadIdx.x == 0) JT_TL(tile, 8);  // warp 0's own staging done
  if (lane == 0 && warp < 6) JT_TL(tile, 10 + warp);  // each warp's staging done
  if (!direct) {
    // the look-back waits on predecessors: the first warp done with its own
    // staging runs it, not always warp 0
    uint32_t won = 0;
    if (lane == 0) won = atomicCAS(&s_lb_claim, 0u, 1u) == 0u;
    if (__shfl_sync(0xffffffffu, won, 0)) resolve_counts();
  }
  __syncthreads();
  if (threadIdx.x == 0) JT_TL(tile, 3);

  const uint32_t tb = (uint32_t)tile_base;
  const uint64_t gb2 = s_base, gsb2 = s_sbase;  // published before the last barrier
  if (!idx_direct) {
    // one thread per index entry: offsets from the block record's masks
    uint32_t *dst = a.idx + gb2;
    uint32_t *dax = a.aux + gb2;
    uint32_t *drc = a.tokrec + gb2;
    uint32_t *dtp = a.tape_idx + gb2;
    const uint32_t sb32 = (uint32_t)gsb2;
    const uint32_t tb32 = (uint32_t)(1 + s_tbase);
    const long long db = s_dbase;
    for (uint32_t k = threadIdx.x; k < total; k += kThreads) {
      const uint32_t pos = s_idx[k];
      const BlockRec &r = s_blk[pos >> 6];
      const uint64_t below = sb::low_bits((int)(pos & 63));
      const uint32_t aux = r.soff + 4u * popc64(r.openq & below) + popc64(r.W & below);
      uint32_t t = r.toff + popc64(r.w1 & below) + popc64(r.w2 & below);
      long long d = (r.pad ? 0 : db) + r.doff + popc64(r.op & below) - popc64(r.cl & below);
      if constexpr (kRec) {
        const RecBlk &x = s_rec[pos >> 6];
        const uint64_t nb = x.nl & below;
        const uint32_t rid = x.rid + popc64(nb);
        if (nb) {
          const uint64_t since = below & ~sb::low_bits(64 - clz64(nb));
          d = popc64(r.op & since) - popc64(r.cl & since);
        }
        t += 2 * rid;  // every record owns two root words
        a.rec_of[gb2 + k] = rid;
      }
      const uint32_t c = s_in[pos];
      dst[k] = tb + pos;
      dax[k] = sb32 + aux;
      drc[k] = c | ((uint32_t)(uint16_t)clamp16(d) << 16);
      dtp[k] = tb32 + t;
      if (c == '"' && k + 1 < total && !pay_direct) {
        // string length = next entry's string offset - this one - 4 (the
        // string buffer is contiguous in token order); the last entry of a
        // tile is left to k_scalars
        const uint32_t p2 = s_idx[k + 1];
        const BlockRec &r2 = s_blk[p2 >> 6];
        const uint64_t b2 = sb::low_bits((int)(p2 & 63));
        const uint32_t aux2 = r2.soff + 4u * popc64(r2.openq & b2) + popc64(r2.W & b2);
        const uint32_t len = aux2 - aux - 4;
        s_pay[aux] = (uint8_t)len;
        s_pay[aux + 1] = (uint8_t)(len >> 8);
        s_pay[aux + 2] = (uint8_t)(len >> 16);
        s_pay[aux + 3] = (uint8_t)(len >> 24);
      }
    }
  }
  if (threadIdx.x == 0) a.tile_flags[gt] = (idx_direct || pay_direct) ? 1u : 0u;
  if constexpr (kRec) {
    // the record each newline ends: where the next one starts, and the
    // token / tape / string-buffer prefixes at its end
    for (uint64_t q = nl; q; q &= q - 1) {
      const int r = ctz64(q);
      const uint64_t below = sb::low_bits(r);
      const uint32_t rid = rid_blk + popc64(nl & below);
      a.rec_start[rid + 1] = (uint32_t)(blk + r + 1);
      a.rec_kend[rid] = (uint32_t)(gb2 + off + popc64(fin & below));
      a.rec_tend[rid] = (uint32_t)(1 + s_tbase + toff + popc64(w1m & below) + popc64(w2m & below) + 2 * rid);
      a.rec_send[rid] = (uint32_t)(gsb2 + soff + 4u * popc64(openq & below) + popc64(W & below));
    }
  }
  __syncthreads();  // length fields staged before the payload copy-out
  if (threadIdx.x == 0) JT_TL(tile, 9);
  if (!pay_direct && stotal) {
    uint8_t *dst = a.strings + gsb2;
    const uint32_t head = (uint32_t)((4 - ((uintptr_t)dst & 3)) & 3) < stotal
                              ? (uint32_t)((4 - ((uintptr_t)dst & 3)) & 3)
                              : stotal;
    if (threadIdx.x < head) dst[threadIdx.x] = s_pay[threadIdx.x];
    const uint32_t nw = (stotal - head) / 4;
    uint32_t *dw = (uint32_t *)(dst + head);
    const uint32_t *sp = (const uint32_t *)s_pay;
    const uint32_t sh = head * 8;
    // words up to the destination's 16-byte alignment, then 16 bytes per
    // thread and round (five staged words funnel-shifted into one store)
    const uint32_t pre = nw < (uint32_t)((4 - (((uintptr_t)dw >> 2) & 3)) & 3)
                             ? nw
                             : (uint32_t)((4 - (((uintptr_t)dw >> 2) & 3)) & 3);
    if (threadIdx.x < pre) dw[threadIdx.x] = __funnelshift_r(sp[threadIdx.x], sp[threadIdx.x + 1], sh);
    const uint32_t nq = (nw - pre) / 4;
    uint4 *dq = (uint4 *)(dw + pre);
    for (uint32_t k = threadIdx.x; k < nq; k += kThreads) {
      const uint32_t o = pre + 4 * k;
      const uint32_t x0 = sp[o], x1 = sp[o + 1], x2 = sp[o + 2], x3 = sp[o + 3], x4 = sp[o + 4];
      dq[k] = make_uint4(__funnelshift_r(x0, x1, sh), __funnelshift_r(x1, x2, sh), __funnelshift_r(x2, x3, sh),
                         __funnelshift_r(x3, x4, sh));
    }
    for (uint32_t k = pre + 4 * nq + threadIdx.x; k < nw; k += kThreads)
      dw[k] = __funnelshift_r(sp[k], sp[k + 1], sh);
    for (uint32_t k = head + 4 * nw + threadIdx.x; k < stotal; k += kThreads) dst[k] = s_pay[k];
  }
  if (threadIdx.x == 0) JT_TL(tile, 7);
}

// ---- index-only stage 1 (jt_stage1: build_structural_index, indexer.cpp:29-56)
// The reference's stage 1 is UTF-8 validation + the structural index; K1
// also produces what stage 2 needs (string payload, token records, tape
// indices).  k_index does only the former, in ONE pass over the input: no
// carry pre-pass.  A tile's structural count depends on its entry state
// (odd backslash run, in string, previous separator), so every tile counts
// its positions for all four (odd, in_string) entry states and publishes
//   IdxAgg = (carry transfer function f, counts c[4], sep delta d[4])
// -- d[x]: one more position when a separator precedes the tile (bit 0 of
// the tile becomes a pseudo-structural start).  IdxAgg composes
// associatively, so one decoupled look-back over the predecessors' IdxAggs
// yields both the tile's entry state and its index base; the tile then picks
// the final mask of its actual entry state (kept in registers).
struct IdxAgg {
  uint32_t f;     // 4 bytes: state_out (odd | ins << 1 | sep << 2) for x = odd | ins << 1
  uint32_t c[4];  // positions for entry x (separator-free entry)
  uint32_t d;     // bit x: +1 position with a separator before the tile
  bool id;        // the neutral element (no tiles)
};

__device__ __forceinline__ uint32_t pick4(const uint32_t c[4], uint32_t x) {
  const uint32_t lo = (x & 1) ? c[1] : c[0], hi = (x & 1) ? c[3] : c[2];
  return (x & 2) ? hi : lo;
}

// `e` (earlier tiles) followed by `l` (later tiles)
__device__ __forceinline__ IdxAgg idx_combine(const IdxAgg &e, const IdxAgg &l) {
  if (e.id) return l;
  if (l.id) return e;
  IdxAgg r;
  r.id = false;
  r.f = s1::compose(l.f, e.f);
  r.d = e.d;
#pragma unroll
  for (uint32_t x = 0; x < 4; x++) {
    const uint32_t y = (e.f >> (8 * x)) & 7;
    r.c[x] = e.c[x] + pick4(l.c, y & 3) + ((y >> 2) & (l.d >> (y & 3)) & 1u);
  }
  return r;
}

__device__ __forceinline__ IdxAgg idx_shfl_down(const IdxAgg &v, int d) {
  IdxAgg o;
  o.f = __shfl_down_sync(0xffffffffu, v.f, d);
#pragma unroll
  for (int k = 0; k < 4; k++) o.c[k] = __shfl_down_sync(0xffffffffu, v.c[k], d);
  o.d = __shfl_down_sync(0xffffffffu, v.d, d);
  o.id = __shfl_down_sync(0xffffffffu, (uint32_t)v.id, d) != 0;
  return o;
}

// record layout per tile: agg words 2t, 2t+1 and the inclusive word at
// 2 * ntiles + t; bit 63 = written.  agg0 = c0 | f << 16 | d << 48,
// agg1 = c1 | c2 << 16 | c3 << 32 (a tile's counts are <= 16384);
// incl = base | state << 48.
constexpr uint64_t kIdxValid = 1ULL << 63;

// Look-back of tile `tile` (> 0) by one full warp: entry state and base.
// Each round covers 64 predecessors (2 per lane, nearest first), all 6
// record words of a lane loaded together: one L2 round trip per round.  A
// persistent k_index resolves tiles in waves of ~G = #CTAs, so a tile may
// sit up to G tiles past the last inclusive record.  A/B (jt_stage1, C4 / C2):
// 4 per lane 0.894 / 0.229 ms, 2 -> 0.858 / 0.216, 1 -> 0.880 / 0.220.
#ifndef JT_IDX_LB_PER
#define JT_IDX_LB_PER 2
#endif
constexpr int kLbPer = JT_IDX_LB_PER;
__device__ __forceinline__ void idx_lookback(const uint64_t *agg, const uint64_t *incl, int64_t tile,
                                             uint32_t &state, uint64_t &base) {
  const int lane = threadIdx.x & 31;
  IdxAgg acc;
  acc.id = true;
  int64_t j0 = tile - 1;
  for (;;) {
    uint64_t iv[kLbPer], a0[kLbPer], a1[kLbPer];
    int kq;
    for (;;) {
#pragma unroll
      for (int q = 0; q < kLbPer; q++) {
        const int64_t j = j0 - kLbPer * lane - q;
        if (j >= 0) {
          iv[q] = lb_load(incl + j);
          a0[q] = lb_load(agg + 2 * j);
          a1[q] = lb_load(agg + 2 * j + 1);
        } else {  // before tile 0: the initial state, base 0
          iv[q] = kIdxValid | ((uint64_t)s1::kInitState << 48);
          a0[q] = a1[q] = 0;
        }
      }
      // nearest inclusive record of this lane, and whether every nearer
      // tile has published its aggregate
      kq = kLbPer;
      bool ok = true;
#pragma unroll
      for (int q = kLbPer - 1; q >= 0; q--) {
        if (iv[q] & kIdxValid) {
          kq = q;
          ok = true;
        } else if (!(a0[q] & a1[q] & kIdxValid)) {
          ok = false;
        }
      }
      const uint32_t hits = __ballot_sync(0xffffffffu, kq < kLbPer);
      const int L = hits ? __ffs(hits) - 1 : 32;
      const bool need = lane <= L;
      if (__all_sync(0xffffffffu, ok || !need)) break;
      JT_TLADD(tile, 12, lane == 0);
      __nanosleep(64);
    }
    const uint32_t hits = __ballot_sync(0xffffffffu, kq < kLbPer);
    const int L = hits ? __ffs(hits) - 1 : 32;
    // this lane's tiles after the inclusive one, earliest first
    IdxAgg v;
    v.id = true;
    if (lane <= L) {
#pragma unroll
      for (int q = kLbPer - 1; q >= 0; q--) {
        if (lane == L && q >= kq) continue;
        IdxAgg t;
        t.id = false;
        t.c[0] = (uint32_t)(a0[q] & 0xFFFF);
        t.f = (uint32_t)(a0[q] >> 16);
        t.d = (uint32_t)(a0[q] >> 48) & 15u;
        t.c[1] = (uint32_t)(a1[q] & 0xFFFF);
        t.c[2] = (uint32_t)((a1[q] >> 16) & 0xFFFF);
        t.c[3] = (uint32_t)((a1[q] >> 32) & 0xFFFF);
        v = idx_combine(v, t);
      }
    }
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      IdxAgg o = idx_shfl_down(v, d);
      if (lane + d < 32) v = idx_combine(o, v);
    }
    if (lane == 0) acc = idx_combine(v, acc);
    if (hits) {
      uint64_t mine = iv[0];
#pragma unroll
      for (int q = 1; q < kLbPer; q++)
        if (kq == q) mine = iv[q];
      const uint64_t ik = __shfl_sync(0xffffffffu, mine, L);
      if (lane == 0) {
        const uint32_t s = (uint32_t)(ik >> 48) & 7u;
        uint64_t b = ik & ((1ULL << 48) - 1);
        if (acc.id) {
          state = s;
        } else {
          b += pick4(acc.c, s & 3) + ((s >> 2) & (acc.d >> (s & 3)) & 1u);
          state = (acc.f >> (8 * (s & 3))) & 7u;
        }
        base = b;
      }
      return;
    }
    JT_TLADD(tile, 11, lane == 0);
    j0 -= 32 * kLbPer;
  }
}

// final structural mask of a block for entry state s (s1::final_mask with the
// odd-run variants of uq and its prefix XOR shared across the four states)
__device__ __forceinline__ uint64_t idx_fin(const s1::Masks &m, uint64_t uq0, uint64_t uq1,
                                            uint64_t px0, uint64_t px1, uint32_t s,
                                            uint64_t valid) {
  const uint64_t uq = (s & 1) ? uq1 : uq0;
  const uint64_t instr = ((s & 1) ? px1 : px0) ^ ((s & 2) ? ~0ULL : 0ULL);
  const uint64_t s1v = (m.st & ~instr) | uq;
  const uint64_t pseudo = (((s1v | m.ws) << 1) | (uint64_t)(s >> 2)) & ~m.ws & ~instr;
  return (s1v | pseudo) & ~(uq & ~instr) & valid;
}

// Persistent, warp-specialised k_index.  8 compute warps own a 16 KiB tile
// (64 bytes per thread, as K1) and publish its IdxAgg as soon as it is
// counted; a 9th warp (the look-back warp) resolves the look-backs of the
// CTA's tiles in order.  Counted tiles wait in a ring of kIdxRing slots
// (final masks per entry state + slot offsets) until their look-back is
// done; the compute warps extract every resolved tile after each tile they
// count and block only when the ring is full.  So a tile's compute never
// waits on an earlier tile's look-back, aggregates appear in claim order,
// and look-backs find their predecessors published (the first persistent
// version, which waited on the previous tile's look-back before counting
// the next, fed look-back latency back into aggregate latency: 10 us
// look-backs, 7 us behind the predecessors' aggregates).
// Hand-off through shared-memory sequence numbers: `ready` (compute ->
// look-back warp, ring slot filled) and `done` (look-back warp -> compute,
// entry state + base written).
constexpr int kIdxCompute = kThreads;       // 256 compute threads
constexpr int kIdxThreads = kThreads + 32;  // + look-back warp
#ifndef JT_IDX_MINB
#define JT_IDX_MINB 3
#endif
#ifndef JT_IDX_RING
#define JT_IDX_RING 4
#endif
constexpr int kIdxMinBlocks = JT_IDX_MINB;
constexpr int kIdxRing = JT_IDX_RING;

template <int kId, int kN>
__device__ __forceinline__ void bar_sync() {
  asm volatile("bar.sync %0, %1;" ::"n"(kId), "n"(kN) : "memory");
}

struct IdxSlot {
  uint64_t fin[4][kIdxCompute];  // final masks per entry state (per block)
  uint64_t off[kIdxCompute];     // 4 x 16-bit tile-relative slot per entry state
  unsigned long long tc;         // tile counts (4 x 16 bit)
  unsigned long long base;       // from the look-back warp
  uint32_t tile, tf, d, sel, two;
};

struct IdxSmem {
  IdxSlot slot[kIdxRing];
  unsigned long long wc[kWarps];
  uint32_t wf[kWarps];
  uint32_t claim, snap, two;
  volatile uint32_t ready, done;  // sequence numbers
  volatile uint32_t end_seq;      // no tile at this sequence number: the CTA is done
  alignas(16) uint32_t pos[kStageIdx + 8];  // absolute positions, shifted to the output's 16-byte phase
};

__global__ void __launch_bounds__(kIdxThreads, kIdxMinBlocks) k_index(Stage1Args a) {
  extern __shared__ __align__(16) uint8_t idx_smem_raw[];
  IdxSmem &S = *reinterpret_cast<IdxSmem *>(idx_smem_raw);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t ntiles = (uint32_t)a.ntiles;
  if (threadIdx.x == 0) {
    S.claim = atomicAdd(a.tile_counter, 1u);
    S.ready = 0;
    S.done = 0;
    S.end_seq = ~0u;
  }
  __syncthreads();

  if (warp == kWarps) {  // ---- look-back warp
    const uint64_t *agg = a.rec_count;
    uint64_t *incl = a.rec_count + 2 * a.ntiles;
    for (uint32_t seq = 0;; seq++) {
      IdxSlot &R = S.slot[seq % kIdxRing];
      while (S.ready <= seq) __nanosleep(32);
      if (seq == S.end_seq) return;
      const uint32_t tile = R.tile;
      if (lane == 0) JT_TL(tile, 2);
      const uint64_t tile_c = R.tc;
      const uint32_t tile_f = R.tf, d = R.d;
      uint32_t state = s1::kInitState;
      uint64_t base = 0;
      if (tile > 0) idx_lookback(agg, incl, tile, state, base);
      if (lane == 0) {
        const uint32_t x = state & 3, sep = (state >> 2) & (d >> x) & 1u;
        const uint64_t out = base + ((tile_c >> (16 * x)) & 0xFFFF) + sep;
        lb_store(incl + tile, kIdxValid | ((uint64_t)((tile_f >> (8 * x)) & 7u) << 48) | out);
        if (tile == ntiles - 1) *a.total = out;
        R.base = base;
        R.sel = x | (sep << 2);
        JT_TL(tile, 3);
        __threadfence_block();
        S.done = seq + 1;
      }
      __syncwarp();
    }
  }

  // ---- compute warps
  const bool vec_ok = ((uintptr_t)a.idx & 15) == 0;
  // positions of a resolved tile: entry state and base from the look-back
  // warp, final mask from its ring slot, staged then written as 16-byte
  // vectors
  auto extract = [&](uint32_t seq) {
    IdxSlot &R = S.slot[seq % kIdxRing];
    bar_sync<1, kIdxCompute>();  // S.pos free, R.sel / R.base visible
    const uint32_t ptile = R.tile;
    if (threadIdx.x == 0) JT_TL(ptile, 5);
    const uint32_t sel = R.sel, x = sel & 3, sep = sel >> 2;
    const uint64_t base = R.base;
    const uint64_t tc = R.tc;
    uint64_t f = R.fin[R.two ? x : (x & 2)][threadIdx.x];
    if (threadIdx.x == 0) f |= sep;
    const uint32_t off = (uint32_t)((R.off[threadIdx.x] >> (16 * x)) & 0xFFFF) + (threadIdx.x ? sep : 0u);
    const uint32_t total = (uint32_t)((tc >> (16 * x)) & 0xFFFF) + sep;
    const uint32_t blk = ptile * (uint32_t)kStage1Tile + threadIdx.x * 64u;
    if (total > (uint32_t)kStageIdx) {  // CTA-uniform: direct stores
      uint32_t slot = off;
      for (uint64_t fm = f; fm; fm &= fm - 1) a.idx[base + slot++] = blk + (uint32_t)ctz64(fm);
      return;
    }
    const uint32_t shift = vec_ok ? (uint32_t)(base & 3) : 0u;
    uint32_t slot = off + shift;
    uint32_t lo = (uint32_t)f, hi = (uint32_t)(f >> 32);
    while (lo) {
      S.pos[slot++] = blk + (uint32_t)(__ffs(lo) - 1);
      lo &= lo - 1;
    }
    while (hi) {
      S.pos[slot++] = blk + 32u + (uint32_t)(__ffs(hi) - 1);
      hi &= hi - 1;
    }
    bar_sync<1, kIdxCompute>();
    uint32_t *dst = a.idx + (base - shift);  // 16-byte aligned when vec_ok
    const uint32_t end = total + shift;
    if (vec_ok) {
      for (uint32_t q = threadIdx.x; 4 * q < end; q += kIdxCompute) {
        const uint32_t j = 4 * q;
        if (j >= shift && j + 4 <= end) {
          *reinterpret_cast<uint4 *>(dst + j) = *reinterpret_cast<const uint4 *>(&S.pos[j]);
        } else {
          for (uint32_t k = j; k < j + 4; k++)
            if (k >= shift && k < end) dst[k] = S.pos[k];
        }
      }
    } else {
      for (uint32_t k = threadIdx.x; k < total; k += kIdxCompute) dst[k] = S.pos[k];
    }
    if (threadIdx.x == 0) JT_TL(ptile, 6);
  };
  // block until the look-back of pending tile `seq` is done
  auto wait_done = [&](uint32_t seq) {
    if (threadIdx.x == 0) {
      JT_TL(S.slot[seq % kIdxRing].tile, 4);
      while (S.done <= seq) __nanosleep(64);
    }
  };

  uint32_t tile = S.claim;
  uint32_t w[16];
  if (tile < ntiles) {
    const uint64_t blk = (uint64_t)tile * kStage1Tile + (uint64_t)threadIdx.x * 64;
    ld256(a.in + blk, w);
    ld256(a.in + blk + 32, w + 8);
  }
  uint32_t head = 0, tail = 0;  // pending tiles: sequence numbers [head, tail)
  for (;;) {
    if (tile >= ntiles) {
      if (threadIdx.x == 0) {
        S.end_seq = tail;
        __threadfence_block();
        S.ready = tail + 1;
      }
      while (head < tail) {
        wait_done(head);
        extract(head++);
      }
      return;
    }
    if (tail - head == kIdxRing) {  // ring full: the oldest must go first
      wait_done(head);
      extract(head++);
    }
    IdxSlot &R = S.slot[tail % kIdxRing];
    const uint64_t blk = (uint64_t)tile * kStage1Tile + (uint64_t)threadIdx.x * 64;
    if (threadIdx.x == 0) {
      JT_TL(tile, 0);
#ifdef JT_TIMELINE
      uint32_t smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      JT_TLV(tile, 8, smid | ((uint64_t)blockIdx.x << 16));
#endif
    }
    s1::Masks m;
    s1::classify64(w, m);
    const uint64_t esc0 = s1::escaped_no_carry(m.bs), tog = s1::carry_toggle(m.bs);
    uint32_t inc = s1::block_function(m, esc0, tog);
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
      if (lane >= d) inc = s1::compose(inc, o);
    }
    const uint32_t excl = __shfl_up_sync(0xffffffffu, inc, 1);
    if (lane == 31) S.wf[warp] = inc;
    const uint64_t uq0 = m.qt & ~esc0, tq = m.qt & tog;
    // the odd-backslash carry into the tile changes nothing unless block 0's
    // first non-backslash byte is a quote (or block 0 is all backslashes):
    // otherwise only the two in-string entry states are counted
    if (threadIdx.x == 0) S.two = (tq != 0 || m.bs == ~0ULL) ? 1u : 0u;
    // UTF-8 validity (as K1)
    uint32_t prev = __shfl_up_sync(0xffffffffu, w[15], 1);
    if (lane == 0) prev = blk >= 4 ? *(const uint32_t *)(a.in + blk - 4) : 0u;
    if ((m.P[7] | (uint64_t)(prev & 0x80808000u)) != 0 && blk < a.len + 3 &&
        s1::utf8_block_error(m.P, prev, blk + 64 >= a.len)) {
      const uint8_t *in = a.in;
      const uint64_t len = a.len;
      auto at = [in, len](uint64_t k) -> uint32_t { return k < len ? in[k] : 0u; };
      uint64_t lo = blk >= 3 ? blk - 3 : 0, hi = blk + 64 < len ? blk + 64 : len;
      for (uint64_t k = lo; k < hi; k++)
        if (s1::utf8_flagged(at, k, len)) {
          atomicMin(a.utf8_pos, (unsigned long long)k);
          break;
        }
    }
    const int64_t rem = (int64_t)a.len - (int64_t)blk;
    const uint64_t valid = rem >= 64 ? ~0ULL : rem <= 0 ? 0ULL : ((1ULL << rem) - 1);
    const uint64_t uq1 = uq0 ^ tq;
    const uint64_t px0 = s1::prefix_xor(uq0), px1 = px0 ^ (0ULL - tq);
    bar_sync<1, kIdxCompute>();
    // the next tile is claimed here, after the classification (claim order ~
    // aggregate order), but its round trip runs under the counting below
    // instead of in front of the next barrier
    uint32_t claimed = 0;
    if (threadIdx.x == 0) claimed = atomicAdd(a.tile_counter, 1u);
    const bool four = S.two != 0;  // CTA-uniform
    // G: tile entry -> this block's entry
    uint32_t wf = lane < kWarps ? S.wf[lane] : 0u;
#pragma unroll
    for (int d = 1; d < kWarps; d <<= 1) {
      uint32_t o = __shfl_up_sync(0xffffffffu, wf, d);
      if (lane >= d) wf = s1::compose(wf, o);
    }
    const uint32_t tile_f = __shfl_sync(0xffffffffu, wf, kWarps - 1);
    const uint32_t wpre = __shfl_sync(0xffffffffu, wf, warp > 0 ? warp - 1 : 0);
    uint32_t G;
    if (warp == 0)
      G = lane == 0 ? 0x03020100u : excl;
    else
      G = lane == 0 ? wpre : s1::compose(excl, wpre);
    const uint64_t fin0 = idx_fin(m, uq0, uq1, px0, px1, G & 7u, valid);
    const uint64_t fin2 = idx_fin(m, uq0, uq1, px0, px1, (G >> 16) & 7u, valid);
    R.fin[0][threadIdx.x] = fin0;
    R.fin[2][threadIdx.x] = fin2;
    uint64_t fin1 = fin0, fin3 = fin2;
    uint32_t c1 = popc64(fin0), c3 = popc64(fin2);
    const uint32_t c0 = c1, c2 = c3;
    if (four) {
      fin1 = idx_fin(m, uq0, uq1, px0, px1, (G >> 8) & 7u, valid);
      fin3 = idx_fin(m, uq0, uq1, px0, px1, (G >> 24) & 7u, valid);
      R.fin[1][threadIdx.x] = fin1;
      R.fin[3][threadIdx.x] = fin3;
      c1 = popc64(fin1);
      c3 = popc64(fin3);
    }
    // a separator before the tile only adds the pseudo-structural start at
    // the tile's byte 0: bit x = byte 0 is no structural, quote or whitespace
    // byte and lies outside a string for entry x (idx_fin's terms at bit 0;
    // thread 0's own masks -- the other threads' value is not used)
    uint32_t dsep = 0;
    {
      const uint32_t plain0 = (uint32_t)(~m.st & ~m.ws & valid) & 1u;
      const uint32_t o0 = (uint32_t)(~uq0 & ~px0) & 1u;  // entry odd = 0: no quote, outside
      const uint32_t o1 = (uint32_t)(~uq1 & ~px1) & 1u;
      const uint32_t i0 = (uint32_t)(~uq0 & px0) & 1u;   // in_string entry flips instr
      const uint32_t i1 = (uint32_t)(~uq1 & px1) & 1u;
      dsep = plain0 ? (o0 | (o1 << 1) | (i0 << 2) | (i1 << 3)) : 0u;
    }
    const uint64_t cnt = (uint64_t)c0 | ((uint64_t)c1 << 16) | ((uint64_t)c2 << 32) | ((uint64_t)c3 << 48);
    uint64_t ci = cnt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      uint64_t o = __shfl_up_sync(0xffffffffu, ci, d);
      if (lane >= d) ci += o;
    }
    if (lane == 31) S.wc[warp] = ci;
    if (threadIdx.x == 0) {
      S.claim = claimed;
      JT_TL(claimed, 7);
      S.snap = S.done;       // look-backs finished so far (extracted below)
    }
    bar_sync<1, kIdxCompute>();
    const uint32_t next = S.claim;
    const uint32_t snap = S.snap;
    uint64_t wc = lane < kWarps ? S.wc[lane] : 0ULL;
#pragma unroll
    for (int d = 1; d < kWarps; d <<= 1) {
      uint64_t o = __shfl_up_sync(0xffffffffu, wc, d);
      if (lane >= d) wc += o;
    }
    const uint64_t cpre = warp > 0 ? __shfl_sync(0xffffffffu, wc, warp > 0 ? warp - 1 : 0) : 0ULL;
    const uint64_t tile_c = __shfl_sync(0xffffffffu, wc, kWarps - 1);
    R.off[threadIdx.x] = cpre + ci - cnt;
    if (threadIdx.x == 0) {
      // publish the aggregate, then hand the slot to the look-back warp
      if (tile > 0) {
        uint64_t *agg = a.rec_count;
        lb_store(agg + 2 * tile, kIdxValid | (tile_c & 0xFFFF) | ((uint64_t)tile_f << 16) |
                                     ((uint64_t)dsep << 48));
        lb_store(agg + 2 * tile + 1, kIdxValid | (tile_c >> 16));
      }
      R.tc = tile_c;
      R.tf = tile_f;
      R.d = dsep;
      R.two = four ? 1u : 0u;
      R.tile = tile;
      JT_TL(tile, 1);
      __threadfence_block();
      S.ready = tail + 1;
    }
    tail++;
    // next tile's bytes in flight while resolved tiles are written out
    if (next < ntiles) {
      const uint64_t nb = (uint64_t)next * kStage1Tile + (uint64_t)threadIdx.x * 64;
      ld256(a.in + nb, w);
      ld256(a.in + nb + 32, w + 8);
    }
    while (head < snap) extract(head++);
    tile = next;
  }
}

// ---- jt_minify (capi.cpp:154-167, minify_pass indexer.cpp:58-75) -----------
// After a successful parse: keep in-string bytes, unescaped quotes and every
// non-whitespace byte.  One CTA per 16 KiB tile; the carry-in is K0b's from
// the parse; kept bytes are staged in shared memory and written coalesced at
// the tile's output offset (decoupled look-back over the kept counts).
__global__ void __launch_bounds__(kThreads) k_minify(MinifyArgs a) {
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_warp_f[kWarps], s_warp_state[kWarps], s_warp_cnt[kWarps];
  __shared__ unsigned long long s_base;
  extern __shared__ __align__(16) uint8_t smem[];  // input tile | kept bytes
  uint8_t *s_out = smem + kStage1Tile;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_tile = atomicAdd(a.tile_counter, 1u);
  __syncthreads();
  const int64_t tile = s_tile;
  const uint64_t blk = (uint64_t)tile * kStage1Tile + (uint64_t)threadIdx.x * 64;
  const uint32_t local = threadIdx.x * 64;
  uint32_t w[16];
  ld256(a.in + blk, w);
  ld256(a.in + blk + 32, w + 8);
  {
    uint4 *d = (uint4 *)(smem + local);
    d[0] = make_uint4(w[0], w[1], w[2], w[3]);
    d[1] = make_uint4(w[4], w[5], w[6], w[7]);
    d[2] = make_uint4(w[8], w[9], w[10], w[11]);
    d[3] = make_uint4(w[12], w[13], w[14], w[15]);
  }
  s1::Masks m;
  s1::classify64(w, m);
  const uint64_t esc0 = s1::escaped_no_carry(m.bs), tog = s1::carry_toggle(m.bs);
  uint32_t inc = s1::block_function(m, esc0, tog);
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) inc = s1::compose(inc, o);
  }
  const uint32_t excl = __shfl_up_sync(0xffffffffu, inc, 1);
  if (lane == 31) s_warp_f[warp] = inc;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t c = a.carry[tile];
    for (int k = 0; k < kWarps; k++) {
      s_warp_state[k] = c;
      c = s1::apply(s_warp_f[k], c);
    }
  }
  __syncthreads();
  uint32_t state = s_warp_state[warp];
  if (lane > 0) state = s1::apply(excl, state);
  const int64_t rem = (int64_t)a.len - (int64_t)blk;
  const uint64_t valid = rem >= 64 ? ~0ULL : rem <= 0 ? 0ULL : ((1ULL << rem) - 1);
  const uint64_t esc = (state & 1) ? (esc0 ^ tog) : esc0;
  const uint64_t uq = m.qt & ~esc;
  const uint64_t instr = s1::prefix_xor(uq) ^ ((state & 2) ? ~0ULL : 0ULL);
  const uint64_t keep = (instr | uq | ~m.ws) & valid;
  const uint32_t cnt = popc64(keep);
  uint32_t ci = cnt;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    uint32_t o = __shfl_up_sync(0xffffffffu, ci, d);
    if (lane >= d) ci += o;
  }
  if (lane == 31) s_warp_cnt[warp] = ci;
  __syncthreads();
  uint32_t off = ci - cnt, total = 0;
  for (int k = 0; k < kWarps; k++) {
    off += k < warp ? s_warp_cnt[k] : 0;
    total += s_warp_cnt[k];
  }
  // kept runs into the staging buffer
  for (uint64_t cm = keep; cm;) {
    const int a0 = ctz64(cm);
    const uint64_t sh = cm >> a0;
    const int n = ~sh == 0 ? 64 - a0 : ctz64(~sh);
    smem_copy(smem, kStage1Tile + off + popc64(keep & sb::low_bits(a0)), local + a0, n);
    cm &= ~(sb::low_bits(n) << a0);
  }
  if (warp == 0) {
    unsigned long long base = 0;
    if (tile > 0) {
      if (lane == 0) lb_store(a.rec + tile, kFlagAgg | total);
      base = lb_sum_exclusive(a.rec, tile);
    }
    if (lane == 0) {
      lb_store(a.rec + tile, kFlagIncl | (base + total));
      s_base = base;
      if (tile == (int64_t)a.ntiles - 1) *a.total = base + total;
    }
  }
  __syncthreads();
  if (total) {
    uint8_t *dst = a.out + s_base;
    const uint32_t head = (uint32_t)((4 - ((uintptr_t)dst & 3)) & 3) < total
                              ? (uint32_t)((4 - ((uintptr_t)dst & 3)) & 3)
                              : total;
    if (threadIdx.x < head) dst[threadIdx.x] = s_out[threadIdx.x];
    const uint32_t nw = (total - head) / 4;
    uint32_t *dw = (uint32_t *)(dst + head);
    const uint32_t *sp = (const uint32_t *)s_out;
    const uint32_t sh = head * 8;
    for (uint32_t k = threadIdx.x; k < nw; k += kThreads) dw[k] = __funnelshift_r(sp[k], sp[k + 1], sh);
    for (uint32_t k = head + 4 * nw + threadIdx.x; k < total; k += kThreads) dst[k] = s_out[k];
  }
}

}  // namespace

// Kernel attributes (dynamic shared memory limits) and occupancy-derived grid
// sizes are per device: cached per device ordinal, set on first use there.
constexpr int kMaxDevices = 64;
template <class T, class F>
T per_device(std::once_flag (&once)[kMaxDevices], T (&val)[kMaxDevices], F f) {
  int dev = 0;
  cudaGetDevice(&dev);
  dev = dev < 0 ? 0 : dev % kMaxDevices;
  std::call_once(once[dev], [&] { val[dev] = f(); });
  return val[dev];
}

cudaError_t minify_launch(const MinifyArgs &args, cudaStream_t stream) {
  constexpr int kSmemMin = 2 * kStage1Tile + 16;
  static std::once_flag once[kMaxDevices];
  static cudaError_t val[kMaxDevices];
  const cudaError_t configured = per_device(once, val, [] {
    return cudaFuncSetAttribute(k_minify, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMin);
  });
  if (configured != cudaSuccess) return configured;
  k_minify<<<(unsigned)args.ntiles, kThreads, kSmemMin, stream>>>(args);
  return cudaGetLastError();
}

#ifdef JT_TIMELINE
// copy (and clear) the K1 timeline; instrumented builds only
cudaError_t stage1_timeline(unsigned long long *host, size_t n) {
  if (n > (size_t)kTlTiles * 16) n = (size_t)kTlTiles * 16;
  cudaError_t e = cudaMemcpyFromSymbol(host, g_tl, n * sizeof(unsigned long long));
  if (e != cudaSuccess) return e;
  static unsigned long long zero[4096];
  for (size_t off = 0; off < (size_t)kTlTiles * 16; off += 4096)
    if ((e = cudaMemcpyToSymbol(g_tl, zero, sizeof(zero), off * sizeof(unsigned long long))) != cudaSuccess)
      return e;
  return cudaSuccess;
}
#endif

size_t stage1_records(uint64_t len) {
  uint64_t ntiles = (len + kStage1Tile - 1) / kStage1Tile;
  return (size_t)(ntiles == 0 ? 1 : ntiles);
}

cudaError_t stage1_configure() {
  static std::once_flag once[kMaxDevices];
  static cudaError_t val[kMaxDevices];
  return per_device(once, val, [] {
    cudaError_t e = cudaFuncSetAttribute(k_stage1<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         kSmemBytes);
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(k_stage1<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                kSmemBytesRec);
  });
}

static Stage1Args with_tiles(const Stage1Args &args_in) {
  Stage1Args a = args_in;
  uint64_t ntiles = (a.end - a.begin + kStage1Tile - 1) / kStage1Tile;
  if (ntiles == 0) ntiles = 1;
  a.ntiles = ntiles;
  return a;
}

cudaError_t stage1_launch(const Stage1Args &args_in, cudaStream_t stream) {
  const Stage1Args a = with_tiles(args_in);
  const cudaError_t configured = stage1_configure();
  if (configured != cudaSuccess) return configured;
  if (a.records) {
    k_carry_fn<true><<<(unsigned)a.ntiles, kFnThreads, 0, stream>>>(a.in, a.begin, a.fn, a.nl_count, a.tile_flags + a.rec_tile0);
    k_carry_scan<<<1, kScanThreads, 0, stream>>>(a.fn, a.carry, a.ntiles, nullptr, 0, nullptr,
                                                 a.nl_count, a.nl_base, a.nl_total);
    k_rec_init<<<1184, 256, 0, stream>>>(a);
    k_stage1<true><<<(unsigned)a.ntiles, kThreads, kSmemBytesRec, stream>>>(a);
  } else {
    k_carry_fn<false><<<(unsigned)a.ntiles, kFnThreads, 0, stream>>>(a.in, a.begin, a.fn, nullptr, a.tile_flags + a.rec_tile0);
    k_carry_scan<<<1, kScanThreads, 0, stream>>>(a.fn, a.carry, a.ntiles, nullptr, 0, nullptr,
                                                 nullptr, nullptr, nullptr);
    k_stage1<false><<<(unsigned)a.ntiles, kThreads, kSmemBytes, stream>>>(a);
  }
  return cudaGetLastError();
}

// Length fields K1 leaves to stage 2 (a string whose next token is in another
// tile, or any string of a spilled tile), written right after stage 1 so the
// string buffer is final before the tape exists (streamed jt_parse).  One
// thread per tile; counts from the tiles' inclusive look-back records.
__global__ void k_tile_lengths(Stage1Args a, uint64_t ntiles) {
  // one warp per tile: a spilled tile (string-dense text) leaves all its
  // lengths, up to thousands of tokens
  const uint64_t t = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  if (t >= ntiles) return;
  const uint64_t S = *a.total, SB = *a.total_strings;
  auto incl = [&](uint64_t k) { return a.rec_count[8 * k + 4] & kQuadMask; };
  const uint64_t hi = incl(t), lo = t ? incl(t - 1) : 0;
  if (hi == lo) return;
  const uint64_t from = a.tile_flags[t] ? lo : hi - 1;
  for (uint64_t k = from + lane; k < hi; k += 32) {
    if ((a.tokrec[k] & 0xFF) != '"') continue;
    const uint32_t so = a.aux[k];
    const uint32_t nx = k + 1 < S ? a.aux[k + 1] : (uint32_t)SB;
    const uint32_t len = nx - so - 4;
    uint8_t *f = a.strings + so;
    f[0] = (uint8_t)len;
    f[1] = (uint8_t)(len >> 8);
    f[2] = (uint8_t)(len >> 16);
    f[3] = (uint8_t)(len >> 24);
    if (a.strings_host) {  // the host copy already holds the rest of the buffer
      uint8_t *h = a.strings_host + so;
      h[0] = (uint8_t)len;
      h[1] = (uint8_t)(len >> 8);
      h[2] = (uint8_t)(len >> 16);
      h[3] = (uint8_t)(len >> 24);
    }
  }
}

cudaError_t stage1_lengths_launch(const Stage1Args &a, uint64_t ntiles, cudaStream_t stream) {
  k_tile_lengths<<<(unsigned)((ntiles * 32 + 255) / 256), 256, 0, stream>>>(a, ntiles);
  return cudaGetLastError();
}

cudaError_t stage1_chunk_carry(const Stage1Args &args_in, cudaStream_t stream) {
  const Stage1Args a = with_tiles(args_in);
  k_carry_fn<false><<<(unsigned)a.ntiles, kFnThreads, 0, stream>>>(a.in, a.begin, a.fn, nullptr, a.tile_flags + a.rec_tile0);
  k_carry_scan<<<1, kScanThreads, 0, stream>>>(a.fn, a.carry, a.ntiles, nullptr, 0, nullptr, nullptr, nullptr,
                                               nullptr, a.init_state, a.out_state);
  return cudaGetLastError();
}

cudaError_t stage1_chunk_main(const Stage1Args &args_in, cudaStream_t stream) {
  const Stage1Args a = with_tiles(args_in);
  const cudaError_t configured = stage1_configure();
  if (configured != cudaSuccess) return configured;
  k_stage1<false><<<(unsigned)a.ntiles, kThreads, kSmemBytes, stream>>>(a);
  return cudaGetLastError();
}

cudaError_t index_launch(const Stage1Args &args_in, cudaStream_t stream) {
  const Stage1Args a = with_tiles(args_in);
  static std::once_flag once[kMaxDevices];
  static unsigned val[kMaxDevices];
  const unsigned grid_max = per_device(once, val, [] {
    int dev = 0, sms = 148, occ = kIdxMinBlocks;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(k_index, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(IdxSmem));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_index, kIdxThreads, sizeof(IdxSmem));
    return (unsigned)(sms * (occ > 0 ? occ : 1));
  });
  const unsigned grid = a.ntiles < grid_max ? (unsigned)a.ntiles : grid_max;
  k_index<<<grid, kIdxThreads, sizeof(IdxSmem), stream>>>(a);
  return cudaGetLastError();
}

cudaError_t stage1_records_count(const Stage1Args &args_in, cudaStream_t stream) {
  const Stage1Args a = with_tiles(args_in);
  k_carry_fn<true><<<(unsigned)a.ntiles, kFnThreads, 0, stream>>>(a.in, a.begin, a.fn, a.nl_count, a.tile_flags + a.rec_tile0);
  k_carry_scan<<<1, kScanThreads, 0, stream>>>(a.fn, a.carry, a.ntiles, nullptr, 0, nullptr,
                                               a.nl_count, a.nl_base, a.nl_total);
  return cudaGetLastError();
}

cudaError_t stage1_records_main(const Stage1Args &args_in, cudaStream_t stream) {
  const Stage1Args a = with_tiles(args_in);
  const cudaError_t configured = stage1_configure();
  if (configured != cudaSuccess) return configured;
  k_rec_init<<<1184, 256, 0, stream>>>(a);
  k_stage1<true><<<(unsigned)a.ntiles, kThreads, kSmemBytesRec, stream>>>(a);
  return cudaGetLastError();
}

cudaError_t stage1_shard_phase0(const Stage1Args &args_in, Sum0 *out, cudaStream_t stream) {
  const Stage1Args a = with_tiles(args_in);
  k_carry_fn<false><<<(unsigned)a.ntiles, kFnThreads, 0, stream>>>(a.in, a.begin, a.fn, nullptr, a.tile_flags + a.rec_tile0);
  k_carry_scan<<<1, kScanThreads, 0, stream>>>(a.fn, nullptr, a.ntiles, nullptr, 0, out, nullptr,
                                               nullptr, nullptr);
  return cudaGetLastError();
}

cudaError_t stage1_shard_phase1(const Stage1Args &args_in, const Sum0 *gathered, uint32_t g,
                                cudaStream_t stream) {
  const Stage1Args a = with_tiles(args_in);
  const cudaError_t configured = stage1_configure();
  if (configured != cudaSuccess) return configured;
  k_carry_scan<<<1, kScanThreads, 0, stream>>>(a.fn, a.carry, a.ntiles, gathered, g, nullptr,
                                               nullptr, nullptr, nullptr);
  k_stage1<false><<<(unsigned)a.ntiles, kThreads, kSmemBytes, stream>>>(a);
  return cudaGetLastError();
}

}  // namespace jt
