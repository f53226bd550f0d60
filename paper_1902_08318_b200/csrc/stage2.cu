// stage2.cu — tape construction as data-parallel passes.
//
// Replaces tape_builder::run (proj/src/tape_builder.cpp:140-258), a
// sequential goto machine, by:
//   K2 k_tokens   one thread per 16-token chunk, 128 chunks per tile.
//                 Phase A classifies tokens and validates/measures every
//                 scalar (strings, numbers, atoms); a 3-channel decoupled
//                 look-back gives each chunk its tape index (sum of token
//                 widths), depth (sum of +1/-1) and string-buffer offset
//                 (sum of 4 + decoded length).  Phase B writes scalar tape
//                 words and decoded strings, and the per-token record
//                 {byte, scalar-failed, depth_before} used below.
//   K2S k_slow    exact decimal->binary64 for the few numbers Eisel-Lemire
//                 cannot settle (numparse.cuh).
//   KT  k_tree    min-depth summaries over 64 tiles and 64^2 tiles.
//   K3 k_struct   one thread per chunk runs the reference's state machine
//                 over its 16 tokens.  Its entry state is derived from the
//                 two previous tokens; an enclosing container outside the
//                 chunk is found as the previous token with a smaller depth
//                 (a previous-smaller-value query over the depth min-tree).
//                 Grammar errors go to an atomicMin keyed by token index
//                 (first error in walk order wins);
//                 matched brackets write both tape words (App. A.6).
//   K4 k_final    error code/offset (string errors re-measured), root words.
#include <cuda_runtime.h>

#include "lookback.cuh"
#include "numparse.cuh"
#include "stage1.h"
#include "stage2.h"
#include "strparse.cuh"

namespace jt {

namespace {

constexpr int kWarps2 = kS2Threads / 32;

struct InAt {
  const uint8_t *in;
  __device__ __forceinline__ uint32_t operator()(uint64_t i) const { return in[i]; }
  // eight bytes from i: two aligned 8-byte loads (the padded input is
  // readable well past len)
  __device__ __forceinline__ uint64_t load8(uint64_t i) const {
    const uint64_t *q = (const uint64_t *)(in + (i & ~7ULL));
    const uint64_t lo = q[0], hi = q[1];
    const uint32_t sh = (uint32_t)(i & 7) * 8;
    return sh ? (lo >> sh) | (hi << (64 - sh)) : lo;
  }
};

__device__ __forceinline__ int tok_width(uint32_t c) {
  if (c == ',' || c == ':') return 0;
  if (c == '-' || (c - '0') < 10u) return 2;
  return 1;
}

__device__ __forceinline__ int tok_delta(uint32_t c) {
  return (c == '{' || c == '[') ? 1 : (c == '}' || c == ']') ? -1 : 0;
}

__device__ __forceinline__ int clamp16(long long d) {
  return d < -2 ? -2 : d > 1026 ? 1026 : (int)d;
}

__device__ __forceinline__ int tok_depth(uint32_t v) { return (int)(int16_t)(v >> 16); }

__device__ __forceinline__ long long sext63(uint64_t v) { return (long long)(v << 1) >> 1; }

// This shard's place in the document (shard.h); the whole document when
// unsharded.  Token / tape / string indices inside the kernels stay local;
// the bases turn them into document values where they are written.
struct View {
  bool sharded, is_last, last_tok;
  uint64_t begin, token_base, tape_base, string_base, S_total, next_pos, next_aux;
  int64_t depth_base;
  uint32_t prev[2], prev_n;
  uint64_t S0;
  int open_n;
};

__device__ View view_of(const Stage2Args &a) {
  View v{};
  const Ctrl *c = a.ctrl;
  if (a.sh != nullptr && a.sh->G > 0) {
    const Shard *h = a.sh;
    v.sharded = true;
    v.is_last = h->is_last != 0;
    v.last_tok = h->last_tok != 0;
    v.begin = h->begin;
    v.token_base = h->token_base;
    v.tape_base = h->tape_base;
    v.string_base = h->string_base;
    v.S_total = h->S_total;
    v.next_pos = h->next_pos;
    v.next_aux = h->next_aux;
    v.depth_base = h->depth_base;
    v.prev[0] = h->prev[0];
    v.prev[1] = h->prev[1];
    v.prev_n = h->prev_n;
    v.S0 = h->S0;
    v.open_n = h->open_n;
  } else {
    v.is_last = true;
    v.last_tok = true;
    v.S_total = c->S;
    v.next_pos = a.len + 1;
    v.next_aux = c->string_bytes;
  }
  return v;
}

// Tokens of this launch: all of them, or a partial range (TokRange).
struct Rng {
  uint64_t lo, hi, avail;
  bool fin;
};
__device__ __forceinline__ Rng rng_of(const Stage2Args &a, const Ctrl *c) {
  if (!a.range) {
    const uint64_t S = c->S;
    return Rng{0, S, S, true};
  }
  return Rng{a.range->lo, a.range->hi, a.range->avail, a.range->fin != 0};
}

// an opener's tape word; below a partial range's patch_lim it is on the host
// already and goes to the patch list too
__device__ __forceinline__ void put_opener(const Stage2Args &a, uint64_t at, uint64_t w) {
  if (at >= a.tape_cap) return;  // a failing document's tape (ensure_stage2)
  a.tape[at] = w;
  if (a.range && at < a.range->patch_lim) {
    const unsigned long long k = atomicAdd(a.patch, 1ULL);
    if (k < kPatchMax) {
      a.patch[2 + 2 * k] = at;
      a.patch[3 + 2 * k] = w;
    }
  }
}

// ---- K2: scalars, one thread per token ---------------------------------

// Stack of container kinds as a 64-bit shift register: bit 0 = innermost
// open container (1 = object).  A token range acts on it as "pop k, then
// push m kinds P" (P bit 0 = last push); these transfers compose without
// knowing the absolute depth, so a scan gives every token the kind of its
// enclosing container.  Exact while the document's depth stays <= 64.
struct StackT {
  uint64_t P;
  uint32_t k, m;
};

__device__ __forceinline__ uint64_t shl64(uint64_t x, uint32_t n) { return n >= 64 ? 0 : x << n; }
__device__ __forceinline__ uint64_t shr64(uint64_t x, uint32_t n) { return n >= 64 ? 0 : x >> n; }

// t2 after t1
__device__ __forceinline__ StackT stack_compose(const StackT &t2, const StackT &t1) {
  StackT r;
  if (t2.k <= t1.m) {
    r.k = t1.k;
    r.m = t1.m - t2.k + t2.m;
    r.P = shl64(shr64(t1.P, t2.k), t2.m) | t2.P;
  } else {
    r.k = t1.k + t2.k - t1.m;
    r.m = t2.m;
    r.P = t2.P;
  }
  return r;
}

__device__ __forceinline__ uint64_t stack_apply(const StackT &t, uint64_t S) {
  return shl64(shr64(S, t.k), t.m) | t.P;
}

constexpr uint64_t kV = 1ULL << 63;

// ---- K2K: container-kind stack scan -----------------------------------------
// 4096 tokens per CTA (16 per thread); per token the kind of its innermost
// open container (scopebits, 16 bits per thread) and the max depth.
constexpr int kStkTok = 16;

// kPass 0: each tile's stack transfer (reduce); kPass 1: scope bits from the
// tile's carry-in (scan).  k_stack_scan runs between them: no chained
// look-back, so no CTA waits on another.  Records: stk_rec[4t] = P,
// [4t+1] = k | m << 32, [4t+2] = carry-in register.
template <int kPass>
__global__ void __launch_bounds__(256) k_stack(Stage2Args a) {
  __shared__ StackT s_wt[8];
  __shared__ uint64_t s_wS[8];
  Ctrl *ctrl = a.ctrl;
  if (ctrl->utf8_pos != ~0ULL) return;
  // deeper than the 64-kind register (pass 0 left the maximum): nobody reads
  // the scope bits (k_struct's `shallow`; max_depth only grows)
  if (kPass == 1 && ctrl->max_depth > 64) return;
  const Rng R = rng_of(a, ctrl);
  const uint64_t S = R.hi;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t ntiles = (S + 256 * kStkTok - 1) / (256 * kStkTok);
  const View vw = view_of(a);
  for (uint64_t tile = R.lo / (256 * kStkTok) + blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const uint64_t i0 = (tile * 256 + threadIdx.x) * kStkTok;
    uint32_t recs[kStkTok];
    if (i0 + kStkTok <= S) {
      const uint4 *rp = (const uint4 *)(a.tok + i0);
#pragma unroll
      for (int q = 0; q < kStkTok / 4; q++) {
        uint4 r = rp[q];
        recs[4 * q] = r.x, recs[4 * q + 1] = r.y, recs[4 * q + 2] = r.z, recs[4 * q + 3] = r.w;
      }
    } else {
#pragma unroll
      for (int k = 0; k < kStkTok; k++) recs[k] = i0 + k < S ? a.tok[i0 + k] : (uint32_t)' ';
    }
    // thread transfer over its 16 tokens (scope bits need the incoming stack)
    StackT tt{0, 0, 0};
    int dmax = 0;
#pragma unroll
    for (int k = 0; k < kStkTok; k++) {
      const uint32_t c = recs[k] & 0xFF;
      if (c == '{' || c == '[') {
        tt = stack_compose(StackT{c == '{' ? 1ULL : 0ULL, 0, 1}, tt);
        dmax = max(dmax, (int)(int16_t)(recs[k] >> 16) + 1);
      } else if (c == '}' || c == ']') {
        tt = stack_compose(StackT{0, 1, 0}, tt);
      }
    }
    StackT inc = tt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      StackT o;
      o.P = __shfl_up_sync(0xffffffffu, inc.P, d);
      o.k = __shfl_up_sync(0xffffffffu, inc.k, d);
      o.m = __shfl_up_sync(0xffffffffu, inc.m, d);
      if (lane >= d) inc = stack_compose(inc, o);
    }
    if (lane == 31) s_wt[warp] = inc;
    if (kPass == 0) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) dmax = max(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
      if (lane == 0 && dmax > 0) atomicMax(&ctrl->max_depth, dmax + (int)vw.depth_base);
      // a shard starts inside depth_base open containers: the 64-kind
      // register is exact only if that depth fits too (closers at the shard
      // start pop below the carried-in kinds)
      if (threadIdx.x == 0 && blockIdx.x == 0 && tile == R.lo / (256 * kStkTok) && vw.depth_base > 0)
        atomicMax(&ctrl->max_depth, (int)min(vw.depth_base, (int64_t)1 << 20));
      __syncthreads();
      if (threadIdx.x == 0) {
        StackT agg = s_wt[0];
        for (int k = 1; k < 8; k++) agg = stack_compose(s_wt[k], agg);
        a.stk_rec[4 * tile] = agg.P;
        a.stk_rec[4 * tile + 1] = (uint64_t)agg.k | ((uint64_t)agg.m << 32);
      }
      __syncthreads();
      continue;
    }
    StackT ex;
    ex.P = __shfl_up_sync(0xffffffffu, inc.P, 1);
    ex.k = __shfl_up_sync(0xffffffffu, inc.k, 1);
    ex.m = __shfl_up_sync(0xffffffffu, inc.m, 1);
    if (lane == 0) ex = StackT{0, 0, 0};
    __syncthreads();
    if (threadIdx.x == 0) {
      uint64_t sw = a.stk_rec[4 * tile + 2];  // carry-in (k_stack_scan)
      for (int k = 0; k < 8; k++) {
        s_wS[k] = sw;
        sw = stack_apply(s_wt[k], sw);
      }
    }
    __syncthreads();
    uint64_t St = stack_apply(ex, s_wS[warp]);
    uint32_t bits = 0;
#pragma unroll
    for (int k = 0; k < kStkTok; k++) {
      const uint32_t c = recs[k] & 0xFF;
      bits |= (uint32_t)(St & 1) << k;
      if (c == '{' || c == '[') St = (St << 1) | (c == '{' ? 1ULL : 0ULL);
      else if (c == '}' || c == ']') St >>= 1;
    }
    if (i0 < S) ((uint16_t *)a.scopebits)[i0 / kStkTok] = (uint16_t)bits;
    __syncthreads();
  }
}

// carry-in register of every k_stack tile: one CTA, each thread a contiguous
// chunk of tiles; starts from the shard's incoming stack (0 unsharded)
constexpr int kStkScan = 1024;
__global__ void __launch_bounds__(kStkScan) k_stack_scan(Stage2Args a) {
  __shared__ StackT s_w[kStkScan / 32];
  Ctrl *ctrl = a.ctrl;
  if (ctrl->utf8_pos != ~0ULL) return;
  if (ctrl->max_depth > 64) return;  // the scope bits are not used (k_stack pass 1)
  const uint64_t S = rng_of(a, ctrl).hi;  // a partial range rescans all tiles below its end
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t ntiles = (S + 256 * kStkTok - 1) / (256 * kStkTok);
  const uint64_t per = (ntiles + kStkScan - 1) / kStkScan;
  const uint64_t lo = threadIdx.x * per, hi = lo + per < ntiles ? lo + per : ntiles;
  auto tile_t = [&](uint64_t t) {
    const uint64_t km = a.stk_rec[4 * t + 1];
    return StackT{a.stk_rec[4 * t], (uint32_t)km, (uint32_t)(km >> 32)};
  };
  StackT acc{0, 0, 0};
  for (uint64_t t = lo; t < hi; t++) acc = stack_compose(tile_t(t), acc);
  StackT inc = acc;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    StackT o;
    o.P = __shfl_up_sync(0xffffffffu, inc.P, d);
    o.k = __shfl_up_sync(0xffffffffu, inc.k, d);
    o.m = __shfl_up_sync(0xffffffffu, inc.m, d);
    if (lane >= d) inc = stack_compose(inc, o);
  }
  if (lane == 31) s_w[warp] = inc;
  __syncthreads();
  uint64_t St = view_of(a).S0;
  for (int k = 0; k < warp; k++) St = stack_apply(s_w[k], St);
  StackT ex;
  ex.P = __shfl_up_sync(0xffffffffu, inc.P, 1);
  ex.k = __shfl_up_sync(0xffffffffu, inc.k, 1);
  ex.m = __shfl_up_sync(0xffffffffu, inc.m, 1);
  if (lane > 0) St = stack_apply(ex, St);
  for (uint64_t t = lo; t < hi; t++) {
    a.stk_rec[4 * t + 2] = St;
    St = stack_apply(tile_t(t), St);
  }
}

// 4 consecutive tokens per thread (1024 per CTA pass): the token records and
// their index / string-offset / tape-index words arrive as 16-byte vector
// loads, all issued before any is used; the next token's index and string
// offset come from the neighbouring lane.
constexpr int kScTok = 4;

__device__ __forceinline__ void ld4(const uint32_t *p, uint64_t i, uint64_t S, uint32_t v[4]) {
  if (i + 4 <= S) {
    const uint4 x = *(const uint4 *)(p + i);
    v[0] = x.x, v[1] = x.y, v[2] = x.z, v[3] = x.w;
  } else {
#pragma unroll
    for (int k = 0; k < 4; k++) v[k] = i + k < S ? p[i + k] : 0u;
  }
}

__global__ void __launch_bounds__(256) k_scalars(Stage2Args a) {
  // warp minima of the current pass, double-buffered by pass parity: a pair of
  // warps (256 tokens) meets at its own 64-thread barrier once per pass
  // instead of the CTA at two
  __shared__ int s_wmin[2][8];
  int par = 0;
  Ctrl *ctrl = a.ctrl;
  if (ctrl->utf8_pos != ~0ULL) return;
  // tokens [R.lo, S); the next token is readable below R.avail
  const Rng R = rng_of(a, ctrl);
  const uint64_t S = R.hi, Sa = R.avail;
  const unsigned long long str_err = ctrl->str_err;
  const View vw = view_of(a);
  const InAt at{a.in};
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr uint64_t kPass = 256 * kScTok;
  const uint64_t stride = (uint64_t)gridDim.x * kPass;
  for (uint64_t base = R.lo + (uint64_t)blockIdx.x * kPass; base < S; base += stride) {
    const uint64_t i0 = base + (uint64_t)threadIdx.x * kScTok;
    uint32_t rec[4], pos[4], so[4], ti[4];
    ld4(a.tok, i0, S, rec);
    ld4(a.idx, i0, Sa, pos);
    ld4(a.aux, i0, Sa, so);
    ld4(a.tape_idx, i0, S, ti);
    // the token after this thread's four: the next lane's first, or memory
    uint32_t npos = __shfl_down_sync(0xffffffffu, pos[0], 1);
    uint32_t nso = __shfl_down_sync(0xffffffffu, so[0], 1);
    if (lane == 31 && i0 + 4 < Sa) {
      npos = a.idx[i0 + 4];
      nso = a.aux[i0 + 4];
    }
    // depth min-tree levels 1 (16 tokens), 2 (256), 3 (4096)
    int m = 0x7FFF;
#pragma unroll
    for (int k = 0; k < 4; k++)
      if (i0 + k < S) m = min(m, (int)(int16_t)(rec[k] >> 16));
    m = min(m, __shfl_xor_sync(0xffffffffu, m, 1));
    m = min(m, __shfl_xor_sync(0xffffffffu, m, 2));
    if ((lane & 3) == 0 && i0 < S) a.m1[i0 >> 4] = (int16_t)m;
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) s_wmin[par][warp] = m;  // 128 tokens
    // every load that depends on the four positions goes out before any of
    // them is used: the string's stage-1 tile flag, and the 8 bytes of an
    // atom (atom_ok8), instead of a chain of dependent byte loads
    uint32_t tflag[4];
    uint64_t aw[4];
#pragma unroll
    for (int k = 0; k < 4; k++) {
      const uint32_t c = rec[k] & 0xFF;
      const bool live = i0 + k < S;
      const uint64_t lt = ((uint64_t)pos[k] - vw.begin) / (uint64_t)jt::kStage1Tile;
      tflag[k] = live && c == '"' && !a.records ? __ldg(a.tile_flags + lt) : 0u;
      aw[k] = live && (c == 't' || c == 'f' || c == 'n') ? at.load8(pos[k]) : 0ULL;
    }
    uint32_t nummask = 0;
#pragma unroll
    for (int k = 0; k < 4; k++) {
      const uint64_t i = i0 + k;
      if (i >= S) break;
      const uint32_t c = rec[k] & 0xFF;
      if (c == '-' || (c - '0') < 10u) nummask |= 1u << k;
      uint32_t fail = 0;
      if (c == '"') {
        const uint32_t p = pos[k];
        const uint32_t p_next = k < 3 ? pos[k + 1] : npos;
        const uint32_t so_next = k < 3 ? so[k + 1] : nso;
        const unsigned long long end = i + 1 < Sa ? p_next : vw.next_pos;
        uint32_t sbase = 0;  // record mode: offsets within the record's string buffer
        if (a.records) {
          const uint32_t r = a.rec_of[i];
          const uint32_t se = a.rec_serr[r];
          fail = se != ~0u && se >= p && se < end;
          sbase = r ? a.rec_send[r - 1] : 0u;
        } else {
          fail = str_err >= p && str_err < end;  // the failing string holds the minimum
        }
        if (!fail) {
          // stage 1 wrote the length unless the next token is in another
          // stage-1 tile or that tile spilled (kStage1Tile = 16 KiB)
          const uint64_t lt = (p - vw.begin) / (uint64_t)jt::kStage1Tile;
          if (end > a.len || lt != ((end - vw.begin) / (uint64_t)jt::kStage1Tile) || (a.records ? a.tile_flags[lt] : tflag[k])) {
            const uint32_t nx = i + 1 < Sa ? so_next : (uint32_t)vw.next_aux;
            const uint32_t len = nx - so[k] - 4;
            uint8_t *f = a.strings + so[k];
            f[0] = (uint8_t)len;
            f[1] = (uint8_t)(len >> 8);
            f[2] = (uint8_t)(len >> 16);
            f[3] = (uint8_t)(len >> 24);
          }
          if (ti[k] < a.tape_cap) a.tape[ti[k]] = tape_word('"', vw.string_base + so[k] - sbase);
        }
      } else if (c == 't' || c == 'f' || c == 'n') {
        fail = !str::atom_ok8(aw[k], a.len, pos[k], c);
        if (!fail && ti[k] < a.tape_cap) a.tape[ti[k]] = (uint64_t)c << 56;
      }
      if (fail) a.tok[i] = rec[k] | 0x100u;
    }
    // number tokens go to a compacted list: parsed by one thread each in k_numbers
    {
      const uint32_t n = __popc(nummask);
      uint32_t incl = n;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t o = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += o;
      }
      const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
      uint32_t basep = 0;
      if (tot) {
        if (lane == 31) basep = atomicAdd(&ctrl->num_count, tot);
        basep = __shfl_sync(0xffffffffu, basep, 31) + incl - n;
        for (uint32_t q = nummask; q; q &= q - 1) a.numlist[basep++] = (uint32_t)(i0 + __ffs(q) - 1);
      }
    }
    switch (warp >> 1) {  // constant barrier ids: the kernel reserves 5, not all 16
      case 0: asm volatile("bar.sync 1, 64;" ::: "memory"); break;
      case 1: asm volatile("bar.sync 2, 64;" ::: "memory"); break;
      case 2: asm volatile("bar.sync 3, 64;" ::: "memory"); break;
      default: asm volatile("bar.sync 4, 64;" ::: "memory"); break;
    }
    if (lane == 0 && !(warp & 1)) {  // m2 = 256 tokens = 2 warps
      const int mm = min(s_wmin[par][warp], s_wmin[par][warp + 1]);
      const uint64_t g2 = (base >> 8) + (warp >> 1);
      if ((g2 << 8) < S) {
        a.m2[g2] = (int16_t)mm;
        atomicMax(&a.m3[g2 >> 4], 0x7FFF - mm);
      }
    }
    par ^= 1;
  }
}

// ---- K2N: number tokens (compacted list) ----------------------------------

__global__ void __launch_bounds__(256) k_numbers(Stage2Args a) {
  Ctrl *ctrl = a.ctrl;
  if (ctrl->utf8_pos != ~0ULL) return;
  const uint32_t n = ctrl->num_count, k0 = a.range ? a.range->num_lo : 0u;
  const InAt at{a.in};
  for (uint32_t k = k0 + blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const uint32_t i = a.numlist[k];
    const uint32_t p = a.idx[i];
    const uint32_t t = a.tape_idx[i];
    num::NumResult r = num::parse_number(at, a.len, p);
    if (a.sh != nullptr && a.sh->G > 0 && a.sh->res_hi != 0 && i + 1 == ctrl->S) {
      // a shard's last token may run past its end into the halo: a digit run
      // reaching the resident end read bytes this GPU does not hold
      const uint64_t rh = a.sh->res_hi;
      uint64_t q = p;
      while (q < rh) {
        const uint32_t ch = a.in[q];
        if (!((ch - '0') < 10u || ch == '-' || ch == '+' || ch == '.' || ch == 'e' || ch == 'E')) break;
        q++;
      }
      if (q >= rh) {  // not NUMBER_ERROR at this token: its bytes are not all here
        atomicMin(&ctrl->err_key, ((unsigned long long)(a.sh->token_base + i) << 8) | kCapacity);
        continue;
      }
    }
    if (r.kind == num::kNumFail) {
      atomicOr(&a.tok[i], 0x100u);
    } else if (t + 1 >= a.tape_cap) {
      // a failing document's tape (ensure_stage2): nothing to write
    } else if (r.kind == num::kNumSlow) {
      a.tape[t] = (uint64_t)'d' << 56;
      a.slow[atomicAdd(&ctrl->slow_count, 1u)] = i;  // its tape slot is tape_idx[i]
    } else {
      a.tape[t] = (uint64_t)(r.kind == num::kNumInt ? 'l' : 'd') << 56;
      a.tape[t + 1] = r.bits;
    }
  }
}

// ---- K2S: exact fallback for hard floats ----------------------------------

__global__ void __launch_bounds__(128) k_slow(Stage2Args a) {
  Ctrl *ctrl = a.ctrl;
  if (ctrl->utf8_pos != ~0ULL) return;
  const uint32_t n = ctrl->slow_count, k0 = a.range ? a.range->slow_lo : 0u;
  const InAt at{a.in};
  for (uint32_t k = k0 + blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const uint32_t tokn = a.slow[k], slot = a.tape_idx[tokn];
    num::Decimal dec;
    uint64_t bits;
    if (num::slow_decimal(at, a.len, a.idx[tokn], dec, &bits)) a.tape[slot + 1] = bits;
    else atomicOr(&a.tok[tokn], 1u << 8);  // binary64 overflow -> NUMBER_ERROR
  }
}

// ---- KT: depth min-tree above the chunks --------------------------------

__global__ void __launch_bounds__(1024) k_tree(Stage2Args a) {
  Ctrl *ctrl = a.ctrl;
  if (ctrl->utf8_pos != ~0ULL) return;
  const uint64_t S = rng_of(a, ctrl).hi;  // a partial range rebuilds the levels below its end
  uint64_t n = (S + 4095) / 4096;  // level-3 entries
  uint64_t n4 = (n + 15) / 16;
  int16_t *l4 = a.mhi + a.hi_off[0];
  for (uint64_t e = threadIdx.x; e < n4; e += blockDim.x) {
    int m = 0x7FFF;
    uint64_t end = min(16 * e + 16, n);
    for (uint64_t c = 16 * e; c < end; c++) m = min(m, 0x7FFF - a.m3[c]);
    l4[e] = (int16_t)m;
  }
  n = n4;
  for (int lv = 1; lv < 4; lv++) {
    __syncthreads();
    const int16_t *src = a.mhi + a.hi_off[lv - 1];
    int16_t *dst = a.mhi + a.hi_off[lv];
    uint64_t nn = (n + 15) / 16;
    for (uint64_t e = threadIdx.x; e < nn; e += blockDim.x) {
      int m = 0x7FFF;
      uint64_t end = min(16 * e + 16, n);
      for (uint64_t c = 16 * e; c < end; c++) m = min(m, (int)src[c]);
      dst[e] = (int16_t)m;
    }
    n = nn;
  }
}

// ---- K3: structure --------------------------------------------------------

// 16 values of one group at tree level `lv` (group g = elements 16g..16g+15)
__device__ __forceinline__ void load_group(const Stage2Args &a, int lv, int64_t g, int v[16]) {
  if (lv == 0) {
    const uint4 *p = (const uint4 *)(a.tok + 16 * g);
#pragma unroll
    for (int q = 0; q < 4; q++) {
      uint4 x = p[q];
      v[4 * q] = tok_depth(x.x);
      v[4 * q + 1] = tok_depth(x.y);
      v[4 * q + 2] = tok_depth(x.z);
      v[4 * q + 3] = tok_depth(x.w);
    }
  } else if (lv == 3) {
    const int4 *p = (const int4 *)(a.m3 + 16 * g);
#pragma unroll
    for (int q = 0; q < 4; q++) {
      int4 x = p[q];
      v[4 * q] = 0x7FFF - x.x;
      v[4 * q + 1] = 0x7FFF - x.y;
      v[4 * q + 2] = 0x7FFF - x.z;
      v[4 * q + 3] = 0x7FFF - x.w;
    }
  } else {
    const int16_t *base = lv == 1 ? a.m1 : lv == 2 ? a.m2 : a.mhi + a.hi_off[lv - 4];
    const uint4 *p = (const uint4 *)(base + 16 * g);
#pragma unroll
    for (int q = 0; q < 2; q++) {
      uint4 x = p[q];
      uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
      for (int k = 0; k < 4; k++) {
        v[8 * q + 2 * k] = (int)(int16_t)(w[k] & 0xFFFF);
        v[8 * q + 2 * k + 1] = (int)(int16_t)(w[k] >> 16);
      }
    }
  }
}

// nearest j < i whose depth_before <= L (the innermost container open at i
// when L = depth_before(i) - 1), or -1: climb the fan-out-16 min-tree until a
// group left of the path holds a value <= L, then descend to its last such
// leaf.  One vector load per level.
__device__ int64_t psv(const Stage2Args &a, int64_t i, int L) {
  if (i <= 0) return -1;
  int64_t x = i - 1;
  int lv = 0;
  int v[16];
  for (;;) {
    const int64_t g = x >> 4;
    const int hi = (int)(x & 15);
    load_group(a, lv, g, v);
    int found = -1;
#pragma unroll
    for (int k = 0; k < 16; k++)
      if (k <= hi && v[k] <= L) found = k;
    if (found >= 0) {
      x = (g << 4) + found;
      break;
    }
    if (g == 0 || lv == kTreeLevels - 1) return -1;
    x = g - 1;
    lv++;
  }
  while (lv > 0) {
    lv--;
    load_group(a, lv, x, v);
    int found = 0;
#pragma unroll
    for (int k = 0; k < 16; k++)
      if (v[k] <= L) found = k;
    x = (x << 4) + found;
  }
  return x;
}

// tape index of token j (chunk start + widths of the tokens before it)
__device__ __forceinline__ uint32_t tape_of(const Stage2Args &a, int64_t j) { return a.tape_idx[j]; }

enum : int { M_V = 0, M_OF, M_AF, M_K, M_C, M_A };

__device__ __forceinline__ void report(Ctrl *ctrl, uint64_t tokn, int code) {
  atomicMin(&ctrl->err_key, ((unsigned long long)tokn << 8) | (unsigned)code);
}

// K3 works on 4096-token tiles: token records plus a 3-level min-depth tree
// (16 / 256 / 4096) in shared memory, so the enclosing-container search
// (psv) only leaves the tile when the container opened before it.
constexpr int kK3Tok = 16;
constexpr int kK3Tile = 256 * kK3Tok;

struct TileTree {
  const uint32_t *tok;  // shared: 4096 records
  const int16_t *l1;    // shared: 256 group minima
  const int16_t *l2;    // shared: 16 group minima
  int64_t base;
  // shared, per level: the opener of the container open at the tile start
  // (psv from the tile base; kOpenUnknown = not looked up yet, kOpenNone = -1).
  // Every chunk of a tile inside a container opened before it needs the
  // same few of these, and each is a global depth-tree walk.
  uint32_t *open;
};

// 16-bit masks "depth <= L" of one group from vector loads (the records
// hold depth_before in their high half; the tree levels are int16)
__device__ __forceinline__ uint32_t tok_mask_le(const uint32_t *g16, int L) {
  const uint4 *q = (const uint4 *)g16;
  uint32_t m = 0;
#pragma unroll
  for (int h = 0; h < 4; h++) {
    const uint4 x = q[h];
    m |= (uint32_t)(tok_depth(x.x) <= L) << (4 * h);
    m |= (uint32_t)(tok_depth(x.y) <= L) << (4 * h + 1);
    m |= (uint32_t)(tok_depth(x.z) <= L) << (4 * h + 2);
    m |= (uint32_t)(tok_depth(x.w) <= L) << (4 * h + 3);
  }
  return m;
}

__device__ __forceinline__ uint32_t i16_mask_le(const int16_t *g16, int L) {
  const uint4 *q = (const uint4 *)g16;
  uint32_t m = 0;
#pragma unroll
  for (int h = 0; h < 2; h++) {
    const uint4 x = q[h];
    const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int k = 0; k < 4; k++) {
      m |= (uint32_t)((int)(int16_t)(w[k] & 0xFFFF) <= L) << (8 * h + 2 * k);
      m |= (uint32_t)((int)(int16_t)(w[k] >> 16) <= L) << (8 * h + 2 * k + 1);
    }
  }
  return m;
}

__device__ __forceinline__ int last_bit(uint32_t m) { return 31 - __clz(m); }

// Deep documents (containers span many groups): one masked step per tree
// level instead of scanning entries one at a time.
constexpr uint32_t kOpenUnknown = 0xFFFFFFFFu, kOpenNone = 0xFFFFFFFEu;
constexpr int kOpenLevels = kMaxDepth + 4;

__device__ __forceinline__ int64_t psv_below(const Stage2Args &a, const TileTree &T, int L) {
  if (L < 0 || L >= kOpenLevels) return psv(a, T.base, L);
  const uint32_t c = T.open[L];
  if (c != kOpenUnknown) return c == kOpenNone ? -1 : (int64_t)c;
  const int64_t j = psv(a, T.base, L);
  T.open[L] = j < 0 ? kOpenNone : (uint32_t)j;  // racing writers store the same value
  return j;
}

__device__ int64_t psv_tile_masked(const Stage2Args &a, const TileTree &T, int64_t i, int L) {
  const int64_t x = i - 1 - T.base;
  if (x >= 0) {
    const int g = (int)(x >> 4), G = g >> 4;
    uint32_t m = tok_mask_le(T.tok + g * 16, L) & ((2u << (x & 15)) - 1);
    if (m) return T.base + g * 16 + last_bit(m);
    int h = -1;
    const uint32_t mh = i16_mask_le(T.l1 + G * 16, L) & ((1u << (g & 15)) - 1);
    if (mh) {
      h = G * 16 + last_bit(mh);
    } else {
      const uint32_t m2 = i16_mask_le(T.l2, L) & ((1u << G) - 1);
      if (m2) {
        const int H = last_bit(m2);
        h = H * 16 + last_bit(i16_mask_le(T.l1 + H * 16, L));
      }
    }
    if (h >= 0) return T.base + h * 16 + last_bit(tok_mask_le(T.tok + h * 16, L));
  }
  return psv_below(a, T, L);
}

// nearest j < i (j >= tile base) with depth_before <= L inside the tile, or
// the global search below the tile
__device__ int64_t psv_tile(const Stage2Args &a, const TileTree &T, int64_t i, int L) {
  const int64_t x = i - 1 - T.base;
  if (x >= 0) {
    const int g = (int)(x >> 4);
    for (int k = (int)(x & 15); k >= 0; --k)
      if (tok_depth(T.tok[g * 16 + k]) <= L) return T.base + g * 16 + k;
    int hit = -1;
    const int G = g >> 4;
    for (int h = g - 1; h >= G * 16; --h)
      if (T.l1[h] <= L) {
        hit = h;
        break;
      }
    if (hit < 0) {
      for (int H = G - 1; H >= 0 && hit < 0; --H)
        if (T.l2[H] <= L)
          for (int h = H * 16 + 15; h >= H * 16; --h)
            if (T.l1[h] <= L) {
              hit = h;
              break;
            }
    }
    if (hit >= 0)
      for (int k = 15; k >= 0; --k)
        if (tok_depth(T.tok[hit * 16 + k]) <= L) return T.base + hit * 16 + k;
  }
  return psv_below(a, T, L);
}

// previous 32-token chunks of the tile a closer's opener is searched in by
// warp ballots before the tile tree takes over (A/B: tools/ab_bench.sh)
#ifndef JT_STRUCT_BACK
#define JT_STRUCT_BACK 8
#endif
// Token-parallel grammar check for one document no deeper than 64 (the
// scope bits are exact): the state in which token i arrives follows from the
// two tokens before it and their innermost containers' kinds (SURVEY.md
// App. A.5; the goto machine of tape_builder.cpp:140-258 restated as
// adjacent-token transitions), so every token is checked on its own.  A
// closer finds its opener as the previous token with depth_before <= D - 1
// (psv) and writes both bracket words.  Errors: atomicMin of (token, code);
// only the first one is reported, so checks of tokens after an error (whose
// arrival state assumed a valid prefix) are harmless.
__device__ __forceinline__ bool scope_bit(const Stage2Args &a, uint64_t j) {
  return (a.scopebits[j >> 5] >> (j & 31)) & 1;
}

// token classes and the transition table of struct_tokens
enum : uint32_t { C_OBR = 0, C_ABR, C_OCL, C_ACL, C_COM, C_COL, C_STR, C_ATOM, C_NUM, C_BAD, kNCls };
__device__ __forceinline__ uint32_t token_class(uint32_t c) {
  switch (c) {
    case '{': return C_OBR;
    case '[': return C_ABR;
    case '}': return C_OCL;
    case ']': return C_ACL;
    case ',': return C_COM;
    case ':': return C_COL;
    case '"': return C_STR;
    case 't': case 'f': case 'n': return C_ATOM;
    default: return (c == '-' || (c - '0') < 10u) ? C_NUM : C_BAD;
  }
}
// entry for (arrival state, class): bits 0-2 error, 3-5 error when the token
// failed its own parse, 6-8 state after, 9 closes a container, 10 opens one
// (depth check), 11 comma after a value (next state from the scope bit),
// 12 closer after a value (kind from the scope bit)
constexpr uint32_t kTrClose = 1u << 9, kTrOpen = 1u << 10, kTrComma = 1u << 11, kTrKind = 1u << 12;
__host__ __device__ constexpr uint32_t tr_entry(int mode, uint32_t cl) {
  // value position (M_V, and M_AF / M_OF fall-throughs)
  return (mode == M_OF && cl == C_OCL) || (mode == M_AF && cl == C_ACL)
             ? (kTrClose | (M_A << 6))
         : (mode == M_V || mode == M_AF)
             ? (cl == C_OBR ? (kTrOpen | (M_OF << 6))
                : cl == C_ABR ? (kTrOpen | (M_AF << 6))
                : cl == C_STR ? ((kStringError << 3) | (M_A << 6))
                : cl == C_ATOM ? ((kTapeError << 3) | (M_A << 6))
                : cl == C_NUM ? ((kNumberError << 3) | (M_A << 6))
                              : (kTapeError | (kTapeError << 3)))
         : (mode == M_K || mode == M_OF)
             ? (cl == C_STR ? ((kStringError << 3) | (M_C << 6)) : (kTapeError | (kTapeError << 3)))
         : mode == M_C ? (cl == C_COL ? (M_V << 6) : (kTapeError | (kTapeError << 3)))
                       // M_A
                       : (cl == C_COM ? kTrComma
                          : (cl == C_OCL || cl == C_ACL) ? (kTrClose | kTrKind | (M_A << 6))
                                                         : (kTapeError | (kTapeError << 3)));
}

// state in which a token arrives after a token of class cl1 whose innermost
// container is an object (sc1); a key string (M_C) is decided by the caller
__host__ __device__ constexpr int arrival_state(uint32_t cl1, uint32_t sc1) {
  return cl1 == C_OBR ? M_OF : cl1 == C_ABR ? M_AF : cl1 == C_COL ? M_V : cl1 == C_COM ? (sc1 ? M_K : M_V) : M_A;
}

// A byte-range shard's place in the document (shard.h) for struct_tokens:
// depth / tape / token bases, the two tokens before the shard and the
// containers open at its start (a.bound).  Unsharded: all zero, is_last.
struct ShardPos {
  int db;             // depth at the shard start
  uint32_t tb;        // tape base: document tape index = tb + local index
  uint64_t token_base;
  uint32_t prev0, prev1;  // bytes of the tokens before the shard (prev0 nearest)
  int64_t before;     // how many exist (<= 2)
  int open_n;         // containers open at the shard start
  bool is_last;
};

template <bool kShard, class Tree>
__device__ __forceinline__ void struct_tokens(const Stage2Args &a, Ctrl *ctrl, uint64_t S, const Tree &T,
                                              uint64_t tbase, uint64_t tend, const uint16_t *s_tr,
                                              const uint8_t *s_cls, const uint8_t *s_arr, const ShardPos &sp,
                                              uint64_t cstart) {
  const int lane = threadIdx.x & 31;
  const bool bound_obj = kShard && sp.open_n > 0 && (a.bound[sp.open_n - 1] >> 56) == '{';
  // tokens before the shard: their bytes, and the innermost container open
  // at the boundary for their scope bit (only read for , and key strings)
  auto rec = [&](int64_t j) -> uint32_t {
    if (j >= (int64_t)tbase) return T.tok[j - tbase];
    if (!kShard || j >= 0) return a.tok[j];
    return j == -1 ? sp.prev0 : sp.prev1;
  };
  // one warp per 32 consecutive tokens (lane = token), so the two previous
  // tokens, the scope bits and most bracket partners are a shuffle away
  for (uint64_t cb = cstart + 32 * (threadIdx.x >> 5); cb < tend; cb += blockDim.x) {
    const uint64_t i = cb + lane;
    const bool live = i < tend;
    const uint32_t v = live ? T.tok[i - tbase] : (uint32_t)'x';
    const uint32_t c = v & 0xFF;
    const uint32_t cl = s_cls[c];
    const bool fail = (v >> 8) & 1;
    const int D = tok_depth(v);
    const uint32_t sw = a.scopebits[cb >> 5];             // bit l: token cb + l in an object
    const uint32_t swp = cb ? a.scopebits[(cb >> 5) - 1] : (bound_obj ? ~0u : 0u);
    const uint64_t sw2 = ((uint64_t)sw << 32) | swp;     // bit 32 + l - k: token i - k
    const uint32_t sc0 = (sw >> lane) & 1, sc1 = (uint32_t)(sw2 >> (31 + lane)) & 1,
                   sc2 = (uint32_t)(sw2 >> (30 + lane)) & 1;
    uint32_t cl1 = __shfl_up_sync(0xffffffffu, cl, 1), cl2 = __shfl_up_sync(0xffffffffu, cl, 2);
    if (lane < 2) {
      const int64_t gi = (int64_t)i + (kShard ? sp.before : 0);  // tokens before i in the document
      if (lane == 0) cl1 = gi >= 1 ? s_cls[rec((int64_t)i - 1) & 0xFF] : C_BAD;
      cl2 = gi >= 2 ? s_cls[rec((int64_t)i - 2) & 0xFF] : C_BAD;
    }
    const uint32_t ti = live ? a.tape_idx[i] : 0u;
    // arrival state from the two previous tokens (App. A.5)
    const bool key1 = cl1 == C_STR && (cl2 == C_OBR || (cl2 == C_COM && sc2));  // i-1 was a key
    int mode = key1 ? M_C : (int)s_arr[2 * cl1 + sc1];
    if (i == 0 && (!kShard || sp.token_base == 0)) mode = M_V;
    const uint32_t e = s_tr[mode * kNCls + cl];
    int err = (int)((fail ? e >> 3 : e) & 7);
    const int Dd = D + (kShard ? sp.db : 0);  // document depth
    if ((e & kTrOpen) && Dd >= kMaxDepth && !err) err = kDepthError;
    if (mode == M_A && Dd <= 0) err = kTapeError;
    if ((e & kTrKind) && sc0 != (cl == C_OCL ? 1u : 0u)) err = kTapeError;
    const int after = (e & kTrComma) ? (sc0 ? M_K : M_V) : (int)((e >> 6) & 7);
    // bracket partners: the opener is the previous token with depth <= D - 1;
    // inside the warp by ballots (one per distinct depth), else the tile tree
    const bool need = live && (e & kTrClose) && !err;
    int64_t j = -1;
    uint32_t pending = __ballot_sync(0xffffffffu, need);
    while (pending) {
      const int leader = __ffs(pending) - 1;
      const int L = __shfl_sync(0xffffffffu, D - 1, leader);
      const uint32_t m = __ballot_sync(0xffffffffu, live && D <= L);
      const bool mine = need && D - 1 == L;
      if (mine) {
        const uint32_t below = m & ((1u << lane) - 1u);
        j = below ? (int64_t)(cb + 31 - __clz(below)) : -2;  // -2: before this warp
      }
      pending &= ~__ballot_sync(0xffffffffu, mine);
    }
    const int src = j >= 0 ? (int)(j - cb) : lane;
    const uint32_t tj_w = __shfl_sync(0xffffffffu, ti, src);
    // openers before this warp's tokens: the previous chunks of the tile by
    // ballots as well (up to 8), then the tile tree
    uint64_t pb = cb;
    for (int step = 0; step < JT_STRUCT_BACK; step++) {
      uint32_t rem = __ballot_sync(0xffffffffu, need && j == -2);
      if (!rem || pb == tbase) break;
      pb -= 32;
      const int dl = tok_depth(T.tok[pb - tbase + lane]);
      while (rem) {
        const int leader = __ffs(rem) - 1;
        const int L = __shfl_sync(0xffffffffu, D - 1, leader);
        const uint32_t m = __ballot_sync(0xffffffffu, dl <= L);
        const bool mine = need && j == -2 && D - 1 == L;
        if (mine && m) j = (int64_t)(pb + 31 - __clz(m));
        rem &= ~__ballot_sync(0xffffffffu, mine);
      }
    }
    if (need) {
      uint32_t tj = tj_w;
      if (j == -2) j = psv_tile_masked(a, T, (int64_t)pb, D - 1);
      if (j >= 0 && (j < (int64_t)cb)) tj = a.tape_idx[j];
      const uint64_t ow = tape_word(cl == C_OCL ? '{' : '[', (kShard ? sp.tb : 0u) + ti + 1);
      if (j >= 0) {
        if (ti < a.tape_cap) a.tape[ti] = tape_word((uint8_t)c, (kShard ? sp.tb : 0u) + tj);
        put_opener(a, tj, ow);
      } else if (kShard && Dd - 1 >= 0 && Dd - 1 < sp.open_n) {
        // the opener lives in an earlier shard: patched after the last exchange
        const uint64_t at = a.bound[Dd - 1] & ((1ULL << 56) - 1);
        if (ti < a.tape_cap) a.tape[ti] = tape_word((uint8_t)c, at);
        const uint32_t k = atomicAdd(&a.sum3->patch_n, 1u);
        if (k < (uint32_t)kBoundMax) {
          a.sum3->patch[2 * k] = at;
          a.sum3->patch[2 * k + 1] = ow;
        }
      } else {
        err = kTapeError;
      }
    }
    const uint64_t tokbase = kShard ? sp.token_base : 0;
    if (err && live) {
      report(ctrl, tokbase + i, err);
    } else if (live && i == S - 1 && sp.is_last) {  // the root value must be complete (last range)
      const int depth_after = Dd + (cl <= C_ABR ? 1 : cl <= C_ACL ? -1 : 0);
      if (!(after == M_A && depth_after == 0)) report(ctrl, tokbase + S, kTapeError);
    }
  }
}

// 4 CTAs (32 warps) per SM: the token-parallel path is latency-bound, so
// occupancy beats registers (79 -> 64 registers, no spills)
#ifndef JT_STRUCT_MINB
#define JT_STRUCT_MINB 4
#endif
// kMode: 0 one document, 1 a byte-range shard (shard.h), 2 NDJSON records.
// kDeep: the instance for documents deeper than 64 (masked tree search); for
// one document both instances are launched and the other one returns.
template <int kMode, bool kDeep = false>
__global__ void __launch_bounds__(256, JT_STRUCT_MINB) k_struct(Stage2Args a) {
  constexpr bool kShard = kMode == 1, kRecs = kMode == 2;
  __shared__ __align__(16) uint32_t s_tok[kK3Tile];
  __shared__ __align__(16) int16_t s_l1[256];
  __shared__ __align__(16) int16_t s_l2[16];
  __shared__ uint16_t s_tr[6 * kNCls];
  __shared__ uint8_t s_cls[256];
  __shared__ uint8_t s_arr[2 * kNCls];
  __shared__ uint32_t s_open[kOpenLevels];
  if (kMode <= 1) {
    s_cls[threadIdx.x] = (uint8_t)token_class(threadIdx.x);
    if (threadIdx.x < 2 * kNCls) s_arr[threadIdx.x] = (uint8_t)arrival_state(threadIdx.x >> 1, threadIdx.x & 1);
    if (threadIdx.x < 6 * kNCls) s_tr[threadIdx.x] = (uint16_t)tr_entry(threadIdx.x / kNCls, threadIdx.x % kNCls);
    __syncthreads();
  }
  Ctrl *ctrl = a.ctrl;
  if (ctrl->utf8_pos != ~0ULL) return;
  const Rng R = rng_of(a, ctrl);
  const uint64_t S = R.hi;
  const uint64_t ntiles = (S + kK3Tile - 1) / kK3Tile, tile0 = R.lo / kK3Tile;
  const bool shallow = ctrl->max_depth <= 64;  // scope bits exact (k_stack)
  const bool deep = !shallow;

  // this shard's place in the document, as scalars (a View captured by the
  // lambdas below would live in local memory)
  // (tape indices fit 32 bits: tape_idx is u32)
  constexpr bool sharded = kShard;
  bool is_last = R.fin;
  int db = 0, open_n = 0;
  uint32_t tb = 0;
  uint64_t token_base = 0;
  uint32_t prev0 = 0, prev1 = 0;
  int64_t before = 0;
  if (kShard) {
    const View vw = view_of(a);
    is_last = vw.last_tok && R.fin;  // the end-of-input check: the shard with the last token
    db = (int)vw.depth_base;
    open_n = vw.open_n;
    tb = (uint32_t)vw.tape_base;
    token_base = vw.token_base;
    prev0 = vw.prev[0];
    prev1 = vw.prev[1];
    before = (int64_t)vw.prev_n;  // tokens before the shard
  }
  // container open at document level L before this shard (shard.h)
  auto bound_at = [&](int L, uint32_t *tape, bool *obj) -> bool {
    if (!sharded || L < 0 || L >= open_n) return false;
    const uint64_t e = a.bound[L];
    *tape = (uint32_t)(e & ((1ULL << 56) - 1));
    *obj = (e >> 56) == '{';
    return true;
  };
  auto scope_obj = [&](int64_t j) -> bool {  // innermost container of token j is an object
    if (j < 0) {  // a token of an earlier shard: the innermost container at the boundary
      uint32_t tp;
      bool ob = false;
      return bound_at(open_n - 1, &tp, &ob) && ob;
    }
    if (shallow) return (a.scopebits[j >> 5] >> (j & 31)) & 1;  // 16-bit words, same bit order
    const int D = tok_depth(a.tok[j]);
    int64_t o = psv(a, j, D - 1);
    if (o < 0) {
      uint32_t tp;
      bool ob = false;
      return bound_at(D + db - 1, &tp, &ob) && ob;
    }
    return (a.tok[o] & 0xFF) == '{';
  };
  // token j's record; j < 0: the tokens before the shard (byte only)
  auto rec_at = [&](int64_t j, uint64_t tbase) -> uint32_t {
    if (j >= (int64_t)tbase) return s_tok[j - tbase];
    if (j >= 0) return a.tok[j];
    return j == -1 ? prev0 : prev1;
  };
  // token-parallel path on few tiles (a streamed piece, a small document):
  // kSplit CTAs share a tile (each loads it for the tree, checks a quarter),
  // so the per-tile latency of 16 chunk rounds per warp is spread out
  const uint32_t split = (kMode <= 1 && shallow && 2 * (ntiles - tile0) <= (uint64_t)gridDim.x) ? 4u : 1u;
  for (uint64_t work = blockIdx.x; work < (ntiles - tile0) * split; work += gridDim.x) {
    const uint64_t tile = tile0 + work / split;
    const uint64_t tbase = tile * kK3Tile;
    {
      const uint64_t i0 = tbase + threadIdx.x * kK3Tok;
      uint4 *d = (uint4 *)(s_tok + threadIdx.x * kK3Tok);
      int m = 0x7FFF;
      if (i0 + kK3Tok <= S) {
        const uint4 *rp = (const uint4 *)(a.tok + i0);
#pragma unroll
        for (int q = 0; q < kK3Tok / 4; q++) {
          uint4 r = rp[q];
          d[q] = r;
          m = min(m, min(min(tok_depth(r.x), tok_depth(r.y)), min(tok_depth(r.z), tok_depth(r.w))));
        }
      } else {
        for (int k = 0; k < kK3Tok; k++) {
          uint32_t r = i0 + k < S ? a.tok[i0 + k] : 0x7FFF0000u;
          s_tok[threadIdx.x * kK3Tok + k] = r;
          m = min(m, tok_depth(r));
        }
      }
      s_l1[threadIdx.x] = (int16_t)m;
      for (int k = threadIdx.x; k < kOpenLevels; k += blockDim.x) s_open[k] = kOpenUnknown;
    }
    __syncthreads();
    if (threadIdx.x < 16) {
      int m = 0x7FFF;
      for (int k = 0; k < 16; k++) m = min(m, (int)s_l1[threadIdx.x * 16 + k]);
      s_l2[threadIdx.x] = (int16_t)m;
    }
    __syncthreads();
    const TileTree T{s_tok, s_l1, s_l2, (int64_t)tbase, s_open};
    if (kMode <= 1 && shallow) {  // token-parallel grammar check
      const ShardPos sp{db, tb, token_base, prev0, prev1, before, open_n, is_last};
      const uint64_t part = kK3Tile / split, c0 = tbase + (work % split) * part;
      struct_tokens<kShard>(a, ctrl, S, T, tbase, min(c0 + part, S), s_tr, s_cls, s_arr, sp, c0);
      __syncthreads();
      continue;
    }
    const uint64_t i0 = tbase + threadIdx.x * kK3Tok;
    const uint64_t i1 = min(i0 + kK3Tok, S);
    // innermost container of token j is an object -- for a token of this tile
    // in a deep document through the tile's shared tree (scope_obj walks the
    // global one: a chain of dependent loads at every chunk entry)
    auto scope_obj_tile = [&](int64_t j) -> bool {
      if (shallow || j < (int64_t)tbase) return scope_obj(j);
      const int D = tok_depth(s_tok[j - (int64_t)tbase]);
      const int64_t o = psv_tile_masked(a, T, j, D - 1);
      if (o < 0) {
        uint32_t tp;
        bool ob = false;
        return bound_at(D + db - 1, &tp, &ob) && ob;
      }
      return ((o >= (int64_t)tbase ? s_tok[o - (int64_t)tbase] : a.tok[o]) & 0xFF) == '{';
    };
    if (i0 < S) do {
    const uint32_t *recs = s_tok + threadIdx.x * kK3Tok;
    uint32_t t = a.tape_idx[i0];  // local tape index (document index = tb + t)
    // record mode: the chunk's current record, its root word (payloads are
    // record-relative) and how many of the previous tokens belong to it
    uint32_t rcur = 0, rtb = 0;
    int64_t rbefore = (int64_t)i0 + before;
    // record mode: the chunk's record ids (and the next chunk's first) up front
    uint32_t rids[kK3Tok + 1];
    if (kRecs) {
      if (i0 + kK3Tok <= S) {
        const uint4 *rp = (const uint4 *)(a.rec_of + i0);
#pragma unroll
        for (int q = 0; q < kK3Tok / 4; q++) {
          const uint4 r = rp[q];
          rids[4 * q] = r.x, rids[4 * q + 1] = r.y, rids[4 * q + 2] = r.z, rids[4 * q + 3] = r.w;
        }
      } else {
#pragma unroll
        for (int k = 0; k < kK3Tok; k++) rids[k] = i0 + k < S ? a.rec_of[i0 + k] : ~0u;
      }
      rids[kK3Tok] = i0 + kK3Tok < S ? a.rec_of[i0 + kK3Tok] : ~0u;
      rcur = rids[0];
      rtb = rcur ? a.rec_tend[rcur - 1] + 1 : 0u;
      rbefore = (i0 >= 1 && a.rec_of[i0 - 1] == rcur) ? ((i0 >= 2 && a.rec_of[i0 - 2] == rcur) ? 2 : 1) : 0;
    }
    // entry state from the two previous tokens (A.5 arrival rules)
    int mode = M_V;
    if (rbefore > 0) {
      uint32_t v1 = rec_at((int64_t)i0 - 1, tbase);
      uint32_t c1 = v1 & 0xFF;
      if (c1 == '{') mode = M_OF;
      else if (c1 == '[') mode = M_AF;
      else if (c1 == ':') mode = M_V;
      else if (c1 == ',') {
        mode = scope_obj_tile((int64_t)i0 - 1) ? M_K : M_V;
      } else if (c1 == '"') {
        mode = M_A;
        if (rbefore >= 2) {
          uint32_t v2 = rec_at((int64_t)i0 - 2, tbase);
          uint32_t c2 = v2 & 0xFF;
          if (c2 == '{') mode = M_C;
          else if (c2 == ',') {
            if (scope_obj_tile((int64_t)i0 - 2)) mode = M_C;
          }
        }
      } else {
        mode = M_A;
      }
    }

    uint32_t stk[kK3Tok];  // local openers: local tape index | is_object << 31
    int sp = 0;
    int far_level = -100;  // cache of the last far container lookup
    uint32_t far_tape = 0;  // document tape index
    bool far_obj = false;
    // The opener of the last far container this chunk closed: every later
    // far lookup of the chunk is for a container enclosing it, so the search
    // starts there instead of at the token (a run of closers ]]]] of a deep
    // chain finds each opener next to the previous one's).
    int64_t far_j = -1, hint = -1;
    int err = 0;
    bool dead = false;  // record mode: the current record already failed
    uint64_t i = i0;
    int depth_after = 0;
    if (!kRecs) {
      // one document / shard: every token is one lookup in the (state,
      // class) table of the token-parallel path; only a comma or closer after
      // a value needs its enclosing container (this chunk's stack, the scope
      // bits, or the far search)
      for (int k = 0; k < kK3Tok; k++) {
        if (i >= i1) break;
        const uint32_t v = recs[k];
        const uint32_t c = v & 0xFF;
        const int D = tok_depth(v) + db;  // document depth
        const uint32_t e = s_tr[mode * kNCls + s_cls[c]];
        err = (int)((((v >> 8) & 1) ? e >> 3 : e) & 7);
        if ((e & kTrOpen) && D >= kMaxDepth && !err) err = kDepthError;
        if (mode == M_A && D <= 0) err = kTapeError;
        if (err) break;
        depth_after = D + tok_delta(c);
        int next = (int)((e >> 6) & 7);
        bool close = false, top_obj = false, top_local = false;
        uint32_t top_tape = 0;  // document tape index of the enclosing opener
        if (e & kTrOpen) {
          stk[sp++] = t | (c == '{' ? 0x80000000u : 0u);
        } else if (e & (kTrComma | kTrKind)) {  // a comma or closer after a value
          if (sp > 0) {
            top_local = true;
            top_tape = tb + (stk[sp - 1] & 0x7FFFFFFFu);
            top_obj = stk[sp - 1] >> 31;
          } else if (shallow && c == ',') {
            top_obj = (a.scopebits[i >> 5] >> (i & 31)) & 1;  // no opener needed
          } else {
            if (far_level != D - 1) {
              const int64_t from = hint >= 0 ? hint : (int64_t)i;
              const int L = D - 1 - db;
              // after a far close the next enclosing opener usually sits right
              // before the last one ("[[[" or "{ key : {" of a deep chain):
              // probe the three tokens before it, then search
              int64_t j = -2;
              if (hint >= 0 && from - 3 >= (int64_t)tbase) {
                const uint32_t *q = s_tok + (from - (int64_t)tbase);
                if (tok_depth(q[-1]) <= L) j = from - 1;
                else if (tok_depth(q[-2]) <= L) j = from - 2;
                else if (tok_depth(q[-3]) <= L) j = from - 3;
              }
              if (j == -2)
                j = from < (int64_t)tbase ? psv(a, from, L)
                    : deep                ? psv_tile_masked(a, T, from, L)
                                          : psv_tile(a, T, from, L);
              far_j = j;
              if (j >= 0) {
                far_obj = ((j >= (int64_t)tbase ? s_tok[j - tbase] : a.tok[j]) & 0xFF) == '{';
                far_tape = tb + tape_of(a, j);
              } else if (!bound_at(D - 1, &far_tape, &far_obj)) {
                err = kTapeError;
                break;
              }
              far_level = D - 1;
            }
            top_tape = far_tape;
            top_obj = far_obj;
          }
          if (e & kTrComma) {
            next = top_obj ? M_K : M_V;
          } else if ((c == '}') != top_obj) {
            err = kTapeError;
            break;
          } else {
            close = true;
          }
        } else if (e & kTrClose) {  // an empty container: the opener is the previous token
          close = true;
          top_obj = mode == M_OF;
          if (sp > 0) {
            top_local = true;
            top_tape = tb + (stk[sp - 1] & 0x7FFFFFFFu);
          } else {
            top_tape = tb + t - 1;
          }
        }
        if (close) {
          if (top_local) {
            sp--;
          } else if (e & kTrKind) {  // the far container: later searches start at its opener
            far_level = -100;
            hint = far_j;
          }
          if (t < a.tape_cap) a.tape[t] = tape_word((uint8_t)c, top_tape);
          const uint64_t ow = tape_word(top_obj ? '{' : '[', tb + t + 1);
          if (!kShard || top_tape > tb) {
            put_opener(a, top_tape - tb, ow);
          } else {  // the opener lives in an earlier shard: patched after the last exchange
            const uint32_t q = atomicAdd(&a.sum3->patch_n, 1u);
            if (q < (uint32_t)kBoundMax) {
              a.sum3->patch[2 * q] = top_tape;
              a.sum3->patch[2 * q + 1] = ow;
            }
          }
          next = M_A;
        }
        mode = next;
        t += tok_width(c);
        i++;
      }
      if (err) {
        report(ctrl, token_base + i, err);
        break;
      }
      if (i1 == S && is_last && !(mode == M_A && depth_after == 0))
        report(ctrl, token_base + S, kTapeError);
      break;
    }
    for (int k = 0; k < kK3Tok; k++) {
      if (i >= i1) break;
      if (kRecs) {
        const uint32_t r = rids[k];
        if (r != rcur) {  // a new record: a new root value
          rcur = r;
          rtb = a.rec_tend[r - 1] + 1;
          t = a.tape_idx[i];
          mode = M_V;
          sp = 0;
          far_level = -100;
          hint = -1;
          dead = false;
        }
        if (dead) {
          i++;
          continue;
        }
      }
      const uint32_t v = recs[k];
      const uint32_t c = v & 0xFF;
      const bool fail = (v >> 8) & 1;
      const int D = tok_depth(v) + db;  // document depth
      depth_after = D + tok_delta(c);
      bool again;
      do {
        again = false;
        bool close = false, have_top = false, top_obj = false;
        uint32_t top_tape = 0;  // document tape index of the enclosing opener
        bool top_local = false;
        switch (mode) {
          case M_V:
            if (c == '{' || c == '[') {
              if (D >= kMaxDepth) {
                err = kDepthError;
                break;
              }
              stk[sp++] = t | (c == '{' ? 0x80000000u : 0u);
              mode = c == '{' ? M_OF : M_AF;
            } else {
              if (c == '"') err = fail ? kStringError : 0;
              else if (c == 't' || c == 'f' || c == 'n') err = fail ? kTapeError : 0;
              else if (c == '-' || (c - '0') < 10u) err = fail ? kNumberError : 0;
              else err = kTapeError;
              mode = M_A;
            }
            break;
          case M_OF:
          case M_AF: {
            const uint32_t want = mode == M_OF ? '}' : ']';
            if (c == want) {
              close = true;
              have_top = true;
              top_obj = mode == M_OF;
              if (sp > 0) {
                top_local = true;
                top_tape = tb + (stk[sp - 1] & 0x7FFFFFFFu);
              } else {
                top_tape = tb + t - 1;  // the opener is the previous token
              }
            } else {
              mode = mode == M_OF ? M_K : M_V;
              again = true;
            }
            break;
          }
          case M_K:
            if (c != '"') err = kTapeError;
            else if (fail) err = kStringError;
            else mode = M_C;
            break;
          case M_C:
            if (c != ':') err = kTapeError;
            else mode = M_V;
            break;
          case M_A: {
            if (D <= 0) {
              err = kTapeError;
              break;
            }
            if (sp > 0) {
              top_local = true;
              top_tape = tb + (stk[sp - 1] & 0x7FFFFFFFu);
              top_obj = stk[sp - 1] >> 31;
            } else if (shallow && c == ',') {
              top_obj = (a.scopebits[i >> 5] >> (i & 31)) & 1;  // no opener needed
            } else {
              if (far_level != D - 1) {
                const int64_t from = hint >= 0 ? hint : (int64_t)i;
                int64_t j = from < (int64_t)tbase ? psv(a, from, D - 1 - db)
                            : deep                ? psv_tile_masked(a, T, from, D - 1 - db)
                                                  : psv_tile(a, T, from, D - 1 - db);
                far_j = j;
                if (j >= 0) {
                  far_obj = ((j >= (int64_t)tbase ? s_tok[j - tbase] : a.tok[j]) & 0xFF) == '{';
                  far_tape = tb + tape_of(a, j);
                } else if (!bound_at(D - 1, &far_tape, &far_obj)) {
                  err = kTapeError;
                  break;
                }
                far_level = D - 1;
              }
              top_tape = far_tape;
              top_obj = far_obj;
            }
            have_top = true;
            if (c == ',') mode = top_obj ? M_K : M_V;
            else if (c == (top_obj ? '}' : ']')) close = true;
            else err = kTapeError;
            break;
          }
        }
        if (close && have_top) {
          if (top_local) {
            sp--;
          } else {
            far_level = -100;
            hint = far_j;
          }
          if (t < a.tape_cap) a.tape[t] = tape_word((uint8_t)c, top_tape - rtb);
          const uint64_t ow = tape_word(top_obj ? '{' : '[', tb + t + 1 - rtb);
          if (!kShard || top_tape > tb) {
            put_opener(a, top_tape - tb, ow);
          } else {  // the opener lives in an earlier shard: patched after the last exchange
            const uint32_t k = atomicAdd(&a.sum3->patch_n, 1u);
            if (k < (uint32_t)kBoundMax) {
              a.sum3->patch[2 * k] = top_tape;
              a.sum3->patch[2 * k + 1] = ow;
            }
          }
          mode = M_A;
        }
      } while (again && !err);
      if (kRecs) {
        if (err) {  // first error of this record; skip to the next record
          atomicMin(&a.rec_err[rcur], ((unsigned long long)i << 8) | (unsigned)err);
          err = 0;
          dead = true;
          i++;
          continue;
        }
        t += tok_width(c);
        i++;
        // the record's last token: it must close the root value
        if ((i >= S || rids[k + 1] != rcur) && !(mode == M_A && depth_after == 0))
          a.rec_end_err[rcur] = kTapeError;
        continue;
      }
      if (err) break;
      t += tok_width(c);
      i++;
    }
    if (kRecs) break;
    if (err) {
      report(ctrl, token_base + i, err);
      break;
    }
    if (i1 == S && is_last && !(mode == M_A && depth_after == 0))
      report(ctrl, token_base + S, kTapeError);
    } while (false);
    __syncthreads();
  }
}

// ---- K4: finalize ----------------------------------------------------------

__global__ void k_final(Stage2Args a) {
  Ctrl *c = a.ctrl;
  if (c->utf8_pos != ~0ULL) {
    c->code = kUtf8Error;
    c->offset = (long long)c->utf8_pos;
    return;
  }
  const uint64_t S = c->S;
  if (S == 0) {
    c->code = kEmpty;
    c->offset = -1;
    return;
  }
  if (c->err_key != ~0ULL) {
    uint64_t i = c->err_key >> 8;
    int code = (int)(c->err_key & 0xFF);
    c->code = code;
    if (i >= S) {
      c->offset = (long long)a.len;
    } else if (code == kStringError) {
      c->offset = (long long)c->str_err;  // the failing string holds the minimum
    } else {
      c->offset = (long long)a.idx[i];
    }
    return;
  }
  const uint64_t E = c->tape_words;
  a.tape[0] = tape_word(kTagRoot, E);
  a.tape[E] = tape_word(kTagRoot, 0);
  c->tape_len = E + 1;
  c->code = kOk;
  c->offset = -1;
}

__global__ void k_init(Ctrl *ctrl, uint64_t *s1rec, uint64_t s1words, uint64_t *s2rec,
                       uint64_t s2words) {
  uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t k = g; k < s1words; k += stride) s1rec[k] = 0;
  for (uint64_t k = g; k < s2words; k += stride) s2rec[k] = 0;
  if (g == 0 && ctrl) {
    Ctrl z{};
    z.utf8_pos = ~0ULL;
    z.str_err = ~0ULL;
    z.err_key = ~0ULL;
    z.code = -1;
    z.offset = -1;
    *ctrl = z;
  }
}

// ---- jt_compute_stats (stats.cpp:5-47, capi.cpp:169-191) --------------------
// After a successful parse: node counts from the token records (a number's
// int/float from its tape tag) and the input's non-ASCII bytes, as warp-
// aggregated atomics.  cnt: integers, floats, strings, non_ascii, objects,
// arrays, nulls, trues, falses (jt_stats order).
__global__ void __launch_bounds__(256) k_stats(Stage2Args a, unsigned long long *cnt) {
  const uint64_t S = a.ctrl->S;
  const int lane = threadIdx.x & 31;
  unsigned long long loc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < S; i += stride) {
    const uint32_t c = a.tok[i] & 0xFF;
    switch (c) {
      case '"': loc[2]++; break;
      case '{': loc[4]++; break;
      case '[': loc[5]++; break;
      case 'n': loc[6]++; break;
      case 't': loc[7]++; break;
      case 'f': loc[8]++; break;
      default:
        if (c == '-' || (c - '0') < 10u) loc[(a.tape[a.tape_idx[i]] >> 56) == 'l' ? 0 : 1]++;
    }
  }
  const uint64_t words = (a.len + 3) / 4;  // the zero tail counts nothing
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < words; k += stride)
    loc[3] += __popc(((const uint32_t *)a.in)[k] & 0x80808080u);
#pragma unroll
  for (int q = 0; q < 9; q++) {
    unsigned long long v = loc[q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0 && v) atomicAdd(cnt + q, v);
  }
}

// ---- NDJSON records ---------------------------------------------------------

__device__ __forceinline__ uint64_t n_records(const Stage2Args &a) {
  const uint64_t nl = a.ctrl->n_newlines;
  // a record after the last '\n' exists unless the input ends with it
  return nl + ((a.len > 0 && a.in[a.len - 1] != '\n') ? 1 : 0);
}

__global__ void k_records_init(Stage2Args a) {
  const uint64_t n = a.ctrl->n_newlines + 1;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < n; k += stride) {
    a.rec_err[k] = ~0ULL;
    a.rec_end_err[k] = 0;
  }
}

// one thread per record: code and record-relative offset as jt_parse of the
// record alone (App. A.1 order: UTF-8, EMPTY, first grammar error in walk
// order, OK), and on success its root words
__global__ void k_final_records(Stage2Args a) {
  const Ctrl *c = a.ctrl;
  const uint64_t n = n_records(a), nl = c->n_newlines, S = c->S;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n; r += stride) {
    const uint64_t start = a.rec_start[r];
    const uint64_t end = r < nl ? (uint64_t)a.rec_start[r + 1] - 1 : a.len;
    const uint64_t k0 = r ? a.rec_kend[r - 1] : 0, k1 = r < nl ? a.rec_kend[r] : S;
    RecordResult out{};
    out.offset = -1;
    if (a.rec_utf8[r] != ~0u) {
      out.code = kUtf8Error;
      out.offset = (long long)(a.rec_utf8[r] - start);
    } else if (k1 == k0) {
      out.code = kEmpty;
    } else if (a.rec_err[r] != ~0ULL) {
      const uint64_t i = a.rec_err[r] >> 8;
      out.code = (int)(a.rec_err[r] & 0xFF);
      out.offset = out.code == kStringError ? (long long)(a.rec_serr[r] - start) : (long long)(a.idx[i] - start);
    } else if (a.rec_end_err[r]) {
      out.code = (int)a.rec_end_err[r];
      out.offset = (long long)(end - start);
    } else {
      const uint64_t tb = r ? (uint64_t)a.rec_tend[r - 1] + 1 : 0;
      const uint64_t te = r < nl ? (uint64_t)a.rec_tend[r] : c->tape_words + 2 * r;
      const uint64_t sb = r ? a.rec_send[r - 1] : 0, se = r < nl ? a.rec_send[r] : c->string_bytes;
      a.tape[tb] = tape_word(kTagRoot, te - tb);
      a.tape[te] = tape_word(kTagRoot, 0);
      out.code = kOk;
      out.tape_begin = tb;
      out.tape_words = te - tb + 1;
      out.string_begin = sb;
      out.string_bytes = se - sb;
    }
    a.results[r] = out;
  }
}

// ---- shards (shard.h) -------------------------------------------------------

// phase-1 summary of this shard (after K1)
__global__ void k_sum1(Stage2Args a, Sum1 *out) {
  const Ctrl *c = a.ctrl;
  Sum1 r{};
  r.S = c->S;
  r.sb = c->string_bytes;
  r.T = c->tape_words - 1;
  r.dtotal = c->depth_total;
  r.utf8_pos = c->utf8_pos;
  r.str_err = c->str_err;
  r.first_pos = r.S ? a.idx[0] : 0;
  r.first_aux = r.S ? a.aux[0] : 0;
  r.last[0] = r.S >= 1 ? (a.tok[r.S - 1] & 0xFF) : 0;
  r.last[1] = r.S >= 2 ? (a.tok[r.S - 2] & 0xFF) : 0;
  r.pad[0] = 1;  // written (a streamed parse gathers the summaries as they appear)
  *out = r;
}

// bases of shard g from all phase-1 summaries; document-wide first UTF-8
// and string errors into the control block (stage 2 reads them there)
__global__ void k_apply1(Stage2Args a, const Sum1 *gs) {
  Shard *h = a.sh;
  Ctrl *c = a.ctrl;
  const uint32_t g = h->g, G = h->G;
  uint64_t tok = 0, tape = 0, str = 0, S = 0, T = 0, sb = 0;
  int64_t dep = 0;
  unsigned long long u8 = ~0ULL, se = ~0ULL;
  // streamed pieces: summaries past g + 1 may still be in flight (phase 1
  // of later pieces runs concurrently); only earlier ones decide this shard
  const uint32_t kmax = h->streamed && g + 2 < G ? g + 2 : G;
  for (uint32_t k = 0; k < kmax; k++) {
    if (k == g) {
      h->token_base = tok;
      h->tape_base = tape;
      h->string_base = str;
      h->depth_base = dep;
    }
    tok += gs[k].S;
    tape += gs[k].T;
    str += gs[k].sb;
    dep += gs[k].dtotal;
    S += gs[k].S;
    T += gs[k].T;
    sb += gs[k].sb;
    if (gs[k].utf8_pos < u8) u8 = gs[k].utf8_pos;
    if (gs[k].str_err < se) se = gs[k].str_err;
  }
  h->S_total = S;
  h->E_total = 1 + T;
  h->sb_total = sb;
  h->is_last = g + 1 == G;
  // the next shard that has a token
  h->next_pos = h->len + 1;
  h->next_aux = sb - h->string_base;
  uint64_t run = 0;
  for (uint32_t k = g; k < G; k++) {
    if (k > g && (k >= kmax || gs[k].pad[0] == 0)) {  // not parsed yet (streamed pieces): the caller redoes the parse
      c->redo = 1;
      break;
    }
    if (k > g && gs[k].S > 0) {
      h->next_pos = gs[k].first_pos;
      h->next_aux = run + gs[k].first_aux;
      break;
    }
    run += gs[k].sb;
  }
  // no later shard has a token: this one ends the document (a trailing
  // shard can lie inside the last token, e.g. a number cut by the shard end)
  h->last_tok = (gs[g].S > 0 && h->next_pos == h->len + 1) ? 1u : 0u;
  // the two tokens before the shard
  uint32_t n = 0;
  h->prev[0] = h->prev[1] = 0;
  for (int k = (int)g - 1; k >= 0 && n < 2; --k) {
    if (gs[k].S >= 1 && n < 2) h->prev[n++] = gs[k].last[0];
    if (gs[k].S >= 2 && n < 2) h->prev[n++] = gs[k].last[1];
  }
  h->prev_n = n;
  c->utf8_pos = u8;
  c->str_err = se;
}

// containers opened in this shard and still open at its end (outermost
// first), and how many closers pop containers opened before it
__global__ void __launch_bounds__(1024) k_bound(Stage2Args a, Sum2 *out) {
  __shared__ int s_min;
  const Ctrl *c = a.ctrl;
  const uint64_t S = c->S;
  const View vw = view_of(a);
  const int fin = (int)c->depth_total;
  if (threadIdx.x == 0) s_min = fin < 0 ? fin : 0;  // depth_before of token 0 is 0
  __syncthreads();
  if (c->utf8_pos == ~0ULL && S > 0) {
    const uint64_t n3 = (S + 4095) / 4096;
    int m = 0x7FFF;
    for (uint64_t k = threadIdx.x; k < n3; k += blockDim.x) m = min(m, 0x7FFF - a.m3[k]);
    atomicMin(&s_min, m);
  }
  __syncthreads();
  const int mn = s_min;
  int n = fin - mn;
  if (n > kBoundMax) n = kBoundMax;  // deeper than kMaxDepth: the document fails anyway
  if (c->utf8_pos != ~0ULL) n = 0;
  if (threadIdx.x == 0) {
    out->unmatched = -mn;
    out->n = n;
  }
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    const int64_t j = psv(a, (int64_t)S, mn + k);
    uint64_t e = 0;
    if (j >= 0) e = ((uint64_t)(a.tok[j] & 0xFF) << 56) | (vw.tape_base + a.tape_idx[j]);
    out->open[k] = e;
  }
}

// containers open at the start of shard g: walking the earlier shards
// backwards, each keeps the openers that later closers do not pop
__global__ void __launch_bounds__(1024) k_apply2(Stage2Args a, const Sum2 *gs) {
  __shared__ int s_keep[64], s_at[64];
  __shared__ int s_n;
  Shard *h = a.sh;
  const uint32_t g = h->g;
  if (threadIdx.x == 0) {
    long long pop = 0;
    for (int k = (int)g - 1; k >= 0; --k) {
      const long long nk = gs[k].n;
      const long long keep = nk > pop ? nk - pop : 0;
      pop = (pop > nk ? pop - nk : 0) + gs[k].unmatched;
      if (k < 64) s_keep[k] = (int)keep;
    }
    int at = 0;
    for (uint32_t k = 0; k < g && k < 64; k++) {
      s_at[k] = at;
      at += s_keep[k];
    }
    s_n = at < kBoundMax ? at : kBoundMax;
    a.sum3->patch_n = 0;
  }
  __syncthreads();
  for (uint32_t k = 0; k < g && k < 64; k++)
    for (int e = threadIdx.x; e < s_keep[k]; e += blockDim.x)
      if (s_at[k] + e < kBoundMax) a.bound[s_at[k] + e] = gs[k].open[e];
  __syncthreads();
  if (threadIdx.x == 0) {
    const int n = s_n;
    uint64_t S0 = 0;
    for (int k = 0; k < 64 && k < n; k++) S0 |= (uint64_t)((a.bound[n - 1 - k] >> 56) == '{') << k;
    h->S0 = S0;
    h->open_n = n;
  }
}

// this shard's first error (document token numbering) and root words
__global__ void k_final_shard(Stage2Args a) {
  const Ctrl *c = a.ctrl;
  const View vw = view_of(a);
  Sum3 *r = a.sum3;
  r->err_key = ~0ULL;
  r->offset = -1;
  if (c->utf8_pos != ~0ULL) return;
  if (c->err_key != ~0ULL) {
    const uint64_t i = c->err_key >> 8;
    const int code = (int)(c->err_key & 0xFF);
    r->err_key = c->err_key;
    if (i >= vw.S_total) r->offset = (long long)a.len;
    else if (code == kCapacity) r->offset = -1;  // a number longer than the resident halo
    else if (code == kStringError) r->offset = (long long)c->str_err;
    else r->offset = (long long)a.idx[i - vw.token_base];
  }
  const uint64_t E = a.sh->E_total;
  if (vw.token_base == 0 && vw.tape_base == 0 && a.sh->g == 0) a.tape[0] = tape_word(kTagRoot, E);
  if (vw.is_last) a.tape[E - vw.tape_base] = tape_word(kTagRoot, 0);
}

// document result from all shards' first errors; bracket patches into this
// shard's part of the tape
__global__ void __launch_bounds__(256) k_shard_finish(Stage2Args a, const Sum3 *gs) {
  Ctrl *c = a.ctrl;
  Shard *h = a.sh;
  const uint32_t G = h->G;
  if (threadIdx.x == 0) {
    if (c->utf8_pos != ~0ULL) {
      c->code = kUtf8Error;
      c->offset = (long long)c->utf8_pos;
    } else if (h->S_total == 0) {
      c->code = kEmpty;
      c->offset = -1;
    } else {
      unsigned long long best = ~0ULL;
      long long off = -1;
      for (uint32_t k = 0; k < G; k++)
        if (gs[k].err_key < best) {
          best = gs[k].err_key;
          off = gs[k].offset;
        }
      if (best != ~0ULL) {
        c->code = (int)(best & 0xFF);
        c->offset = off;
      } else {
        c->code = kOk;
        c->offset = -1;
      }
    }
  }
  if (c->utf8_pos != ~0ULL) return;
  const uint64_t lo = h->tape_base, hi = h->tape_base + c->tape_words;  // local words [1, tape_words)
  for (uint32_t k = 0; k < G; k++) {
    const uint32_t n = gs[k].patch_n < (uint32_t)kBoundMax ? gs[k].patch_n : (uint32_t)kBoundMax;
    for (uint32_t e = threadIdx.x; e < n; e += blockDim.x) {
      const uint64_t at = gs[k].patch[2 * e];
      if (at > lo && at < hi && at - lo < a.tape_cap) a.tape[at - lo] = gs[k].patch[2 * e + 1];
    }
  }
}

__global__ void k_stage1_final(Ctrl *c) {
  if (c->utf8_pos != ~0ULL) {
    c->code = kUtf8Error;
    c->offset = (long long)c->utf8_pos;
  } else {
    c->code = kOk;
    c->offset = -1;
  }
}

}  // namespace

Stage2Sizes stage2_sizes(uint64_t cap) {
  Stage2Sizes z;
  z.chunks = (cap + kStructTok - 1) / kStructTok + 1;
  z.tiles = (cap + kTokPerTile - 1) / kTokPerTile + 1;
  // every level padded by one group (vector loads of a whole group)
  z.n1 = (cap + 15) / 16 + 32;
  z.n2 = (cap + 255) / 256 + 32;
  z.n3 = (cap + 4095) / 4096 + 32;
  uint64_t n = (cap + 4095) / 4096, off = 0;
  for (int k = 0; k < 4; k++) {
    n = (n + 15) / 16;
    z.hi_off[k] = off;
    off += (n + 32 + 15) & ~(uint64_t)15;
  }
  z.nhi = off;
  return z;
}

cudaError_t init_launch(Ctrl *ctrl, uint64_t *s1rec, uint64_t s1words, uint64_t *s2rec,
                        uint64_t s2words, cudaStream_t stream) {
  uint64_t m = s1words > s2words ? s1words : s2words;
  unsigned blocks = (unsigned)((m + 255) / 256);
  if (blocks < 1) blocks = 1;
  if (blocks > 1184) blocks = 1184;
  k_init<<<blocks, 256, 0, stream>>>(ctrl, s1rec, s1words, s2rec, s2words);
  return cudaGetLastError();
}

cudaError_t stage1_finalize_launch(Ctrl *ctrl, cudaStream_t stream) {
  k_stage1_final<<<1, 1, 0, stream>>>(ctrl);
  return cudaGetLastError();
}

static unsigned grid_tokens(const Stage2Args &a) {
  const int sms = a.num_sms > 0 ? a.num_sms : 148;
  uint64_t g = (a.cap_tokens + 255) / 256;
  unsigned g2 = (unsigned)(g < (uint64_t)sms * 16 ? g : (uint64_t)sms * 16);
  return g2 < 1 ? 1 : g2;
}

static void launch_stack(const Stage2Args &a, cudaStream_t stream) {
  const int sms = a.num_sms > 0 ? a.num_sms : 148;
  uint64_t nst = (a.cap_tokens + 4095) / 4096;
  unsigned gs = (unsigned)(nst < (uint64_t)sms * 4 ? nst : (uint64_t)sms * 4);
  k_stack<0><<<gs < 1 ? 1 : gs, 256, 0, stream>>>(a);
  k_stack_scan<<<1, kStkScan, 0, stream>>>(a);
  k_stack<1><<<gs < 1 ? 1 : gs, 256, 0, stream>>>(a);
}

static void launch_struct(const Stage2Args &a, cudaStream_t stream) {
  const int sms = a.num_sms > 0 ? a.num_sms : 148;
  uint64_t nt = (a.cap_tokens + kK3Tile - 1) / kK3Tile;
  unsigned g3 = (unsigned)(nt < (uint64_t)sms * 4 ? nt : (uint64_t)sms * 4);
  if (a.records) k_struct<2><<<g3 < 1 ? 1 : g3, 256, 0, stream>>>(a);
  else if (a.sh) k_struct<1><<<g3 < 1 ? 1 : g3, 256, 0, stream>>>(a);
  else k_struct<0><<<g3 < 1 ? 1 : g3, 256, 0, stream>>>(a);
}

cudaError_t stats_launch(const Stage2Args &a, unsigned long long *cnt, cudaStream_t stream) {
  const int sms = a.num_sms > 0 ? a.num_sms : 148;
  k_stats<<<sms * 4, 256, 0, stream>>>(a, cnt);
  return cudaGetLastError();
}

cudaError_t records_init_launch(const Stage2Args &a, cudaStream_t stream) {
  k_records_init<<<1184, 256, 0, stream>>>(a);
  return cudaGetLastError();
}

cudaError_t records_stage2_launch(const Stage2Args &a, cudaStream_t stream, int *launches,
                                  const Stage2Fork *fork) {
  const unsigned g2 = grid_tokens(a);
  if (fork) {
    // side stream: the container kinds next to the scalars / numbers (k_stack
    // reads only stage 1's token records; k_struct needs the fail flags
    // k_scalars and k_numbers leave in them, so it stays behind both)
    cudaEventRecord(fork->fork, stream);
    cudaStreamWaitEvent(fork->side, fork->fork, 0);
    launch_stack(a, fork->side);
    cudaEventRecord(fork->join, fork->side);
  }
  k_scalars<<<g2, 256, 0, stream>>>(a);
  k_numbers<<<g2, 256, 0, stream>>>(a);
  k_slow<<<8, 64, 0, stream>>>(a);
  k_tree<<<1, 1024, 0, stream>>>(a);
  if (fork) cudaStreamWaitEvent(stream, fork->join, 0);
  else launch_stack(a, stream);
  launch_struct(a, stream);
  k_final_records<<<1184, 256, 0, stream>>>(a);
  *launches = 9;
  return cudaGetLastError();
}

// ---- streamed jt_parse: stage 2 in two token ranges ------------------------
__global__ void k_range_a(Stage2Args a, const uint64_t *known, const TokRange *prev, TokRange *r,
                          TokRange *host) {
  const Ctrl *c = a.ctrl;
  const uint64_t n = *known;  // index entries stage 1 has produced so far
  const uint64_t lo = prev ? prev->hi : 0;
  uint64_t hi = n > 0 ? (n - 1) / 4096 * 4096 : 0;  // token hi exists
  if (hi < lo) hi = lo;
  TokRange v{};
  v.lo = lo;
  v.hi = hi;
  v.avail = n;
  v.num_lo = prev ? c->num_count : 0u;
  v.slow_lo = prev ? c->slow_count : 0u;
  v.patch_lim = prev ? prev->tape_end : 0;
  v.tape_end = hi > lo ? a.tape_idx[hi] : (prev ? prev->tape_end : 1);
  *r = v;
  if (host) {  // host-mapped (no copy queued behind the bulk D2H copies); tape_end
    // last: the host polls it (nonzero) to queue the range's tape copy early
    TokRange hv = v;
    hv.tape_end = 0;
    *host = hv;
    __threadfence_system();
    *(volatile uint64_t *)&host->tape_end = v.tape_end;
  }
  if (!prev) a.patch[0] = 0;
}

__global__ void k_range_b(Stage2Args a, const TokRange *ra, TokRange *rb) {
  const Ctrl *c = a.ctrl;
  TokRange v{};
  v.lo = ra->hi;
  v.hi = v.avail = c->S;
  v.num_lo = c->num_count;
  v.slow_lo = c->slow_count;
  v.fin = 1;
  v.patch_lim = ra->tape_end;
  *rb = v;
}

cudaError_t range_a_launch(const Stage2Args &a_in, const uint64_t *known, const TokRange *prev, TokRange *r,
                           TokRange *host, cudaStream_t stream, int *launches, const Stage2Fork *fork) {
  Stage2Args a = a_in;
  a.range = r;
  const unsigned g2 = grid_tokens(a);
  k_range_a<<<1, 1, 0, stream>>>(a, known, prev, r, host);
  if (fork) {  // k_stack next to the scalar / number / tree kernels
    cudaEventRecord(fork->fork, stream);
    cudaStreamWaitEvent(fork->side, fork->fork, 0);
    launch_stack(a, fork->side);
    cudaEventRecord(fork->join, fork->side);
  }
  k_scalars<<<g2, 256, 0, stream>>>(a);
  k_numbers<<<g2, 256, 0, stream>>>(a);
  k_slow<<<8, 64, 0, stream>>>(a);
  k_tree<<<1, 1024, 0, stream>>>(a);
  if (fork) cudaStreamWaitEvent(stream, fork->join, 0);
  else launch_stack(a, stream);
  launch_struct(a, stream);
  *launches = 9;
  return cudaGetLastError();
}

cudaError_t range_b_launch(const Stage2Args &a_in, const TokRange *ra, TokRange *rb, cudaStream_t stream,
                           int *launches, const Stage2Fork *fork) {
  Stage2Args a = a_in;
  a.range = rb;
  const unsigned g2 = grid_tokens(a);
  k_range_b<<<1, 1, 0, stream>>>(a, ra, rb);
  if (fork) {  // k_stack next to the scalar / number / tree kernels (stage2_launch)
    cudaEventRecord(fork->fork, stream);
    cudaStreamWaitEvent(fork->side, fork->fork, 0);
    launch_stack(a, fork->side);
    cudaEventRecord(fork->join, fork->side);
  }
  k_scalars<<<g2, 256, 0, stream>>>(a);
  k_numbers<<<g2, 256, 0, stream>>>(a);
  k_slow<<<8, 64, 0, stream>>>(a);
  k_tree<<<1, 1024, 0, stream>>>(a);
  if (fork) cudaStreamWaitEvent(stream, fork->join, 0);
  else launch_stack(a, stream);
  launch_struct(a, stream);
  k_final<<<1, 1, 0, stream>>>(a);
  *launches = 10;
  return cudaGetLastError();
}

cudaError_t shard_sum1_launch(const Stage2Args &a, Sum1 *out, cudaStream_t stream) {
  k_sum1<<<1, 1, 0, stream>>>(a, out);
  return cudaGetLastError();
}

cudaError_t shard_phase2_launch(const Stage2Args &a, const Sum1 *gathered, Sum2 *out,
                                cudaStream_t stream, int *launches) {
  const unsigned g2 = grid_tokens(a);
  k_apply1<<<1, 1, 0, stream>>>(a, gathered);
  k_scalars<<<g2, 256, 0, stream>>>(a);
  k_numbers<<<g2, 256, 0, stream>>>(a);
  k_slow<<<8, 64, 0, stream>>>(a);
  k_tree<<<1, 1024, 0, stream>>>(a);
  k_bound<<<1, 1024, 0, stream>>>(a, out);
  *launches = 6;
  return cudaGetLastError();
}

cudaError_t shard_phase3_launch(const Stage2Args &a, const Sum2 *gathered, cudaStream_t stream,
                                int *launches) {
  k_apply2<<<1, 1024, 0, stream>>>(a, gathered);
  launch_stack(a, stream);
  launch_struct(a, stream);
  k_final_shard<<<1, 1, 0, stream>>>(a);
  *launches = 6;
  return cudaGetLastError();
}

cudaError_t shard_finish_launch(const Stage2Args &a, const Sum3 *gathered, cudaStream_t stream) {
  k_shard_finish<<<1, 256, 0, stream>>>(a, gathered);
  return cudaGetLastError();
}

// ---- distinct_values over the device-resident parse (§8f rank 4) ----------
// document.cpp:134-192: a scalar is selected when, walking up from it, the
// object keys met (arrays are looked through between keys, not below the
// last one) end with the path's keys; the first key may sit at any depth.
// One thread per token: the innermost step needs ':' + key before the token,
// every further container is found by the previous-smaller-depth query on
// the stage-2 min tree (psv), so the walk is a few loads per level.
__device__ __forceinline__ bool key_is(const Stage2Args &a, const DistinctQuery &q, uint64_t key, int k) {
  if ((a.tok[key] & 0xFF) != '"') return false;
  const uint8_t *s = a.strings + a.aux[key];
  const uint32_t n = (uint32_t)s[0] | ((uint32_t)s[1] << 8) | ((uint32_t)s[2] << 16) | ((uint32_t)s[3] << 24);
  const uint32_t b = q.key_off[k], e = q.key_off[k + 1];
  if (n != e - b) return false;
  for (uint32_t j = 0; j < n; j++)
    if (s[4 + j] != q.key_bytes[b + j]) return false;
  return true;
}

__global__ void __launch_bounds__(256) k_distinct_match(Stage2Args a, DistinctQuery q, uint32_t *match,
                                                        uint32_t *count) {
  const uint64_t S = a.ctrl->S;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < S; i += stride) {
    const uint32_t v = a.tok[i];
    const uint32_t c = v & 0xFF;
    const bool scalar = c == '"' || c == 't' || c == 'f' || c == 'n' || c == '-' || (c - '0') < 10u;
    int d = tok_depth(v);
    if (!scalar || d <= 0 || i < 2 || (a.tok[i - 1] & 0xFF) != ':') continue;
    if (!key_is(a, q, i - 2, q.nkeys - 1)) continue;
    int k = q.nkeys - 2;
    int64_t cur = psv(a, (int64_t)i, d - 1);  // the object holding the last key
    d--;
    bool ok = true;
    while (k >= 0) {
      if (cur < 1 || d <= 0) {  // the root: keys left over
        ok = false;
        break;
      }
      if ((a.tok[cur - 1] & 0xFF) == ':') {  // a member value: its key must be the next one
        if (cur < 2 || !key_is(a, q, (uint64_t)cur - 2, k)) {
          ok = false;
          break;
        }
        k--;
      }  // else an array element: looked through
      if (k < 0) break;
      cur = psv(a, cur, d - 1);
      d--;
    }
    if (ok) match[atomicAdd(count, 1u)] = (uint32_t)i;
  }
}

__global__ void k_distinct_values(Stage2Args a, const uint32_t *match, uint32_t count, DistinctVal *vals,
                                  uint32_t *len) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= count) return;
  const uint32_t t = a.tape_idx[match[k]];
  const uint64_t w = a.tape[t];
  DistinctVal r{};
  r.tag = (uint32_t)(w >> 56);
  if (r.tag == 'l' || r.tag == 'd') {
    r.bits = a.tape[t + 1];
  } else if (r.tag == '"') {
    const uint8_t *s = a.strings + (w & kPayloadMask);
    r.len = (uint32_t)s[0] | ((uint32_t)s[1] << 8) | ((uint32_t)s[2] << 16) | ((uint32_t)s[3] << 24);
    r.bits = w & kPayloadMask;  // source offset until the scan
  }
  vals[k] = r;
  len[k] = r.len;
}

// one warp per string
__global__ void k_distinct_strings(Stage2Args a, const DistinctVal *vals, const uint32_t *off, uint32_t count,
                                   uint8_t *out) {
  const uint32_t k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (k >= count) return;
  const DistinctVal r = vals[k];
  if (r.tag != '"') return;
  const uint8_t *s = a.strings + r.bits + 4;
  for (uint32_t j = lane; j < r.len; j += 32) out[off[k] + j] = s[j];
}

// Exclusive prefix sum of n u32 values (n <= 2^32 - 1; sums wrap mod 2^32,
// the caller bounds them): one CTA, each thread a contiguous chunk summed in
// registers, a CTA scan of the chunk sums, then each chunk rewritten.  The
// distinct_values string offsets (count = selected values) are its only user.
__global__ void __launch_bounds__(1024) k_scan_u32(const uint32_t *in, uint32_t *out, uint32_t n) {
  __shared__ uint32_t s_warp[32];
  const uint32_t per = (n + 1023) / 1024;
  const uint32_t lo = min(n, threadIdx.x * per), hi = min(n, lo + per);
  uint32_t sum = 0;
  for (uint32_t k = lo; k < hi; k++) sum += in[k];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t inc = sum;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) inc += o;
  }
  if (lane == 31) s_warp[warp] = inc;
  __syncthreads();
  uint32_t run = inc - sum;
  for (int k = 0; k < warp; k++) run += s_warp[k];
  for (uint32_t k = lo; k < hi; k++) {
    const uint32_t v = in[k];
    out[k] = run;
    run += v;
  }
}

cudaError_t scan_u32_launch(const uint32_t *in, uint32_t *out, uint32_t n, cudaStream_t stream) {
  if (n) k_scan_u32<<<1, 1024, 0, stream>>>(in, out, n);
  return cudaGetLastError();
}

cudaError_t distinct_match_launch(const Stage2Args &a, const DistinctQuery &q, uint32_t *match,
                                  uint32_t *count, cudaStream_t stream) {
  const int sms = a.num_sms > 0 ? a.num_sms : 148;
  k_distinct_match<<<sms * 8, 256, 0, stream>>>(a, q, match, count);
  return cudaGetLastError();
}

cudaError_t distinct_values_launch(const Stage2Args &a, const uint32_t *match, uint32_t count,
                                   DistinctVal *vals, uint32_t *len, cudaStream_t stream) {
  if (count) k_distinct_values<<<(count + 255) / 256, 256, 0, stream>>>(a, match, count, vals, len);
  return cudaGetLastError();
}

cudaError_t distinct_strings_launch(const Stage2Args &a, const DistinctVal *vals, const uint32_t *off,
                                    uint32_t count, uint8_t *out, cudaStream_t stream) {
  if (count) k_distinct_strings<<<(unsigned)(((uint64_t)count * 32 + 255) / 256), 256, 0, stream>>>(a, vals, off, count, out);
  return cudaGetLastError();
}

cudaError_t stage2_launch(const Stage2Args &a, cudaStream_t stream, int *launches,
                          cudaEvent_t *ev, const Stage2Fork *fork) {
  const Stage2Sizes z = stage2_sizes(a.cap_tokens);
  const int sms = a.num_sms > 0 ? a.num_sms : 148;
  // K2: one thread per token, grid sized for the capacity bound, grid-stride
  uint64_t g = (a.cap_tokens + 255) / 256;
  unsigned g2 = (unsigned)(g < (uint64_t)sms * 16 ? g : (uint64_t)sms * 16);
  if (g2 < 1) g2 = 1;
  const bool forked = fork && !ev;
  if (forked) {  // k_stack reads only stage 1's token records
    cudaEventRecord(fork->fork, stream);
    cudaStreamWaitEvent(fork->side, fork->fork, 0);
    launch_stack(a, fork->side);
  }
  k_scalars<<<g2, 256, 0, stream>>>(a);
  if (forked) {  // the upper tree levels (from k_scalars' level 3) next to the numbers
    cudaEventRecord(fork->fork, stream);
    cudaStreamWaitEvent(fork->side, fork->fork, 0);
    k_tree<<<1, 1024, 0, fork->side>>>(a);
    cudaEventRecord(fork->join, fork->side);
  }
  k_numbers<<<g2, 256, 0, stream>>>(a);
  if (ev) cudaEventRecord(ev[0], stream);
  k_slow<<<8, 64, 0, stream>>>(a);  // rare work; small grid keeps the local-memory reservation small
  if (ev) cudaEventRecord(ev[1], stream);
  if (!forked) k_tree<<<1, 1024, 0, stream>>>(a);
  if (ev) cudaEventRecord(ev[2], stream);
  if (forked) cudaStreamWaitEvent(stream, fork->join, 0);
  else launch_stack(a, stream);  // container kinds (scope bits) for k_struct
  // k_struct reads the fail flags k_scalars / k_numbers leave in the token
  // records (errors are reported in token order): it cannot run next to them
  launch_struct(a, stream);
  if (ev) cudaEventRecord(ev[3], stream);
  k_final<<<1, 1, 0, stream>>>(a);
  if (ev) cudaEventRecord(ev[4], stream);
  *launches = 9;
  return cudaGetLastError();
}

}  // namespace jt
