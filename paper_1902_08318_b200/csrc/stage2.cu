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
#include "stage2.h"
#include "strparse.cuh"

namespace jt {

namespace {

constexpr int kWarps2 = kS2Threads / 32;

struct InAt {
  const uint8_t *in;
  __device__ __forceinline__ uint32_t operator()(uint64_t i) const { return in[i]; }
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

// ---- K2: scalars, one thread per token ---------------------------------

__global__ void __launch_bounds__(256) k_scalars(Stage2Args a) {
  Ctrl *ctrl = a.ctrl;
  if (ctrl->utf8_pos != ~0ULL) return;
  const uint64_t S = ctrl->S;
  const unsigned long long str_err = ctrl->str_err;
  const uint32_t total_sb = (uint32_t)ctrl->string_bytes;
  const InAt at{a.in};
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u); base < S;
       base += stride) {
    const uint64_t i = base + (threadIdx.x & 31);
    const bool live = i < S;
    const uint32_t rec = live ? a.tok[i] : 0u;
    // chunk minimum of depth_before (16 tokens = half a warp)
    int m = live ? (int)(int16_t)(rec >> 16) : 0x7FFF;
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (live && (i & 15) == 0) a.chunk_min[i >> 4] = (int16_t)m;
    if (!live) continue;
    const uint32_t c = rec & 0xFF;
    uint32_t fail = 0;
    if (c == '"') {
      const uint32_t p = a.idx[i];
      const unsigned long long end = i + 1 < S ? a.idx[i + 1] : a.len + 1;
      fail = str_err >= p && str_err < end;  // the failing string holds the minimum
      if (!fail) {
        const uint32_t so = a.aux[i];
        const uint32_t nx = i + 1 < S ? a.aux[i + 1] : total_sb;
        const uint32_t len = nx - so - 4;
        uint8_t *f = a.strings + so;
        f[0] = (uint8_t)len;
        f[1] = (uint8_t)(len >> 8);
        f[2] = (uint8_t)(len >> 16);
        f[3] = (uint8_t)(len >> 24);
        a.tape[a.tape_idx[i]] = tape_word('"', so);
      }
    } else if (c == 't' || c == 'f' || c == 'n') {
      const uint32_t p = a.idx[i];
      fail = !str::atom_ok(at, a.len, p, c);
      if (!fail) a.tape[a.tape_idx[i]] = (uint64_t)c << 56;
    } else if (c == '-' || (c - '0') < 10u) {
      const uint32_t p = a.idx[i];
      num::NumResult r = num::parse_number(at, a.len, p);
      const uint32_t t = a.tape_idx[i];
      if (r.kind == num::kNumFail) {
        fail = 1;
      } else if (r.kind == num::kNumSlow) {
        a.tape[t] = (uint64_t)'d' << 56;
        uint32_t slot = atomicAdd(&ctrl->slow_count, 1u);
        a.slow[2 * slot] = (uint32_t)i;
        a.slow[2 * slot + 1] = t;
      } else {
        a.tape[t] = (uint64_t)(r.kind == num::kNumInt ? 'l' : 'd') << 56;
        a.tape[t + 1] = r.bits;
      }
    }
    if (fail) a.tok[i] = rec | 0x100u;
  }
}

// ---- K2S: exact fallback for hard floats ----------------------------------

__global__ void __launch_bounds__(128) k_slow(Stage2Args a) {
  Ctrl *ctrl = a.ctrl;
  if (ctrl->utf8_pos != ~0ULL) return;
  const uint32_t n = ctrl->slow_count;
  const InAt at{a.in};
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    uint32_t tokn = a.slow[2 * k], slot = a.slow[2 * k + 1];
    num::Decimal dec;
    uint64_t bits;
    if (num::slow_decimal(at, a.len, a.idx[tokn], dec, &bits)) a.tape[slot + 1] = bits;
    else atomicOr(&a.tok[tokn], 1u << 8);  // binary64 overflow -> NUMBER_ERROR
  }
}

// ---- KT: depth min-tree above the chunks --------------------------------

__global__ void __launch_bounds__(256) k_tree(Stage2Args a) {
  __shared__ bool s_last;
  Ctrl *ctrl = a.ctrl;
  if (ctrl->utf8_pos != ~0ULL) return;
  const uint64_t S = ctrl->S;
  const uint64_t nchunks = (S + kTokPerThread - 1) / kTokPerThread;
  const uint64_t ntiles = (S + kTokPerTile - 1) / kTokPerTile;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < ntiles;
       t += (uint64_t)gridDim.x * blockDim.x) {
    int m = 0x7FFF;
    const uint64_t e = min((t + 1) * kS2Threads, nchunks);
    for (uint64_t c = t * kS2Threads; c < e; c++) m = min(m, (int)a.chunk_min[c]);
    a.tile_min[t] = (int16_t)m;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(&ctrl->tree_done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const uint64_t nsup = (ntiles + kTilesPerSuper - 1) / kTilesPerSuper;
  const uint64_t nsup2 = (nsup + kSupersPerSuper2 - 1) / kSupersPerSuper2;
  for (uint64_t s = threadIdx.x; s < nsup; s += blockDim.x) {
    int m = 0x7FFF;
    const uint64_t e = min((s + 1) * kTilesPerSuper, ntiles);
    for (uint64_t t = s * kTilesPerSuper; t < e; t++) m = min(m, (int)((volatile int16_t *)a.tile_min)[t]);
    a.super_min[s] = (int16_t)m;
  }
  __syncthreads();
  for (uint64_t s = threadIdx.x; s < nsup2; s += blockDim.x) {
    int m = 0x7FFF;
    const uint64_t e = min((s + 1) * kSupersPerSuper2, nsup);
    for (uint64_t t = s * kSupersPerSuper2; t < e; t++) m = min(m, (int)a.super_min[t]);
    a.super2_min[s] = (int16_t)m;
  }
}

// ---- K3: structure --------------------------------------------------------

// nearest j < i whose depth_before <= L (the innermost container open at i
// when L = depth_before(i) - 1), or -1
__device__ int64_t psv(const Stage2Args &a, int64_t i, int L) {
  if (i <= 0) return -1;
  int64_t j = i - 1;
  const int64_t lo = (i - 1) & ~(int64_t)(kTokPerThread - 1);
  for (; j >= lo; --j)
    if (tok_depth(a.tok[j]) <= L) return j;
  int64_t c = lo / kTokPerThread - 1;  // chunks of the same tile
  int64_t found_chunk = -1;
  const int64_t clo = (lo / kTokPerThread) & ~(int64_t)(kS2Threads - 1);
  for (; c >= clo; --c)
    if (a.chunk_min[c] <= L) {
      found_chunk = c;
      break;
    }
  if (found_chunk < 0) {
    int64_t tile = clo / kS2Threads;  // tiles of the same super
    int64_t found_tile = -1;
    const int64_t tlo = tile & ~(int64_t)(kTilesPerSuper - 1);
    for (int64_t t = tile - 1; t >= tlo; --t)
      if (a.tile_min[t] <= L) {
        found_tile = t;
        break;
      }
    if (found_tile < 0) {
      int64_t sup = tlo / kTilesPerSuper;
      int64_t found_sup = -1;
      const int64_t slo = sup & ~(int64_t)(kSupersPerSuper2 - 1);
      for (int64_t s = sup - 1; s >= slo; --s)
        if (a.super_min[s] <= L) {
          found_sup = s;
          break;
        }
      if (found_sup < 0) {
        for (int64_t s2 = slo / kSupersPerSuper2 - 1; s2 >= 0; --s2)
          if (a.super2_min[s2] <= L) {
            for (int64_t s = s2 * kSupersPerSuper2 + kSupersPerSuper2 - 1; s >= s2 * kSupersPerSuper2; --s)
              if (a.super_min[s] <= L) {
                found_sup = s;
                break;
              }
            break;
          }
        if (found_sup < 0) return -1;
      }
      for (int64_t t = found_sup * kTilesPerSuper + kTilesPerSuper - 1; t >= found_sup * kTilesPerSuper; --t)
        if (a.tile_min[t] <= L) {
          found_tile = t;
          break;
        }
      if (found_tile < 0) return -1;
    }
    for (int64_t cc = found_tile * kS2Threads + kS2Threads - 1; cc >= found_tile * kS2Threads; --cc)
      if (a.chunk_min[cc] <= L) {
        found_chunk = cc;
        break;
      }
    if (found_chunk < 0) return -1;
  }
  for (j = found_chunk * kTokPerThread + kTokPerThread - 1; j >= found_chunk * kTokPerThread; --j)
    if (tok_depth(a.tok[j]) <= L) return j;
  return -1;
}

// tape index of token j (chunk start + widths of the tokens before it)
__device__ __forceinline__ uint32_t tape_of(const Stage2Args &a, int64_t j) { return a.tape_idx[j]; }

enum : int { M_V = 0, M_OF, M_AF, M_K, M_C, M_A };

__device__ __forceinline__ void report(Ctrl *ctrl, uint64_t tokn, int code) {
  atomicMin(&ctrl->err_key, ((unsigned long long)tokn << 8) | (unsigned)code);
}

__global__ void __launch_bounds__(128) k_struct(Stage2Args a) {
  Ctrl *ctrl = a.ctrl;
  if (ctrl->utf8_pos != ~0ULL) return;
  const uint64_t S = ctrl->S;
  const uint64_t nchunks = (S + kTokPerThread - 1) / kTokPerThread;
  for (uint64_t chunk = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; chunk < nchunks;
       chunk += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i0 = chunk * kTokPerThread;
    const uint64_t i1 = min(i0 + kTokPerThread, S);
    uint32_t t = a.tape_idx[i0];

    // entry state from the two previous tokens (A.5 arrival rules)
    int mode = M_V;
    if (i0 > 0) {
      uint32_t v1 = a.tok[i0 - 1];
      uint32_t c1 = v1 & 0xFF;
      if (c1 == '{') mode = M_OF;
      else if (c1 == '[') mode = M_AF;
      else if (c1 == ':') mode = M_V;
      else if (c1 == ',') {
        int64_t j = psv(a, (int64_t)i0 - 1, tok_depth(v1) - 1);
        mode = (j >= 0 && (a.tok[j] & 0xFF) == '{') ? M_K : M_V;
      } else if (c1 == '"') {
        mode = M_A;
        if (i0 >= 2) {
          uint32_t v2 = a.tok[i0 - 2];
          uint32_t c2 = v2 & 0xFF;
          if (c2 == '{') mode = M_C;
          else if (c2 == ',') {
            int64_t j = psv(a, (int64_t)i0 - 2, tok_depth(v2) - 1);
            if (j >= 0 && (a.tok[j] & 0xFF) == '{') mode = M_C;
          }
        }
      } else {
        mode = M_A;
      }
    }

    uint32_t stk[kTokPerThread];  // local openers: tape index | is_object << 31
    int sp = 0;
    int far_level = -100;  // cache of the last far container lookup
    uint32_t far_tape = 0;
    bool far_obj = false;
    int err = 0;
    uint64_t i = i0;
    int depth_after = 0;
    for (; i < i1; i++) {
      const uint32_t v = a.tok[i];
      const uint32_t c = v & 0xFF;
      const bool fail = (v >> 8) & 1;
      const int D = tok_depth(v);
      depth_after = D + tok_delta(c);
      bool again;
      do {
        again = false;
        bool close = false, have_top = false, top_obj = false;
        uint32_t top_tape = 0;
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
                top_tape = stk[sp - 1] & 0x7FFFFFFFu;
              } else {
                top_tape = t - 1;  // the opener is the previous token
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
              top_tape = stk[sp - 1] & 0x7FFFFFFFu;
              top_obj = stk[sp - 1] >> 31;
            } else {
              if (far_level != D - 1) {
                int64_t j = psv(a, (int64_t)i, D - 1);
                if (j < 0) {
                  err = kTapeError;
                  break;
                }
                far_level = D - 1;
                far_obj = (a.tok[j] & 0xFF) == '{';
                far_tape = tape_of(a, j);
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
          if (top_local) sp--;
          else far_level = -100;
          a.tape[t] = tape_word((uint8_t)c, top_tape);
          a.tape[top_tape] = tape_word(top_obj ? '{' : '[', t + 1);
          mode = M_A;
        }
      } while (again && !err);
      if (err) break;
      t += tok_width(c);
    }
    if (err) {
      report(ctrl, i, err);
      continue;
    }
    if (i1 == S && !(mode == M_A && depth_after == 0)) report(ctrl, S, kTapeError);
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
  z.chunks = (cap + kTokPerThread - 1) / kTokPerThread + 1;
  z.tiles = (cap + kTokPerTile - 1) / kTokPerTile + 1;
  z.supers = (z.tiles + kTilesPerSuper - 1) / kTilesPerSuper + 1;
  z.supers2 = (z.supers + kSupersPerSuper2 - 1) / kSupersPerSuper2 + 1;
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

cudaError_t stage2_launch(const Stage2Args &a, cudaStream_t stream, int *launches,
                          cudaEvent_t *ev) {
  const Stage2Sizes z = stage2_sizes(a.cap_tokens);
  const int sms = a.num_sms > 0 ? a.num_sms : 148;
  // K2: one thread per token, grid sized for the capacity bound, grid-stride
  uint64_t g = (a.cap_tokens + 255) / 256;
  unsigned g2 = (unsigned)(g < (uint64_t)sms * 16 ? g : (uint64_t)sms * 16);
  if (g2 < 1) g2 = 1;
  k_scalars<<<g2, 256, 0, stream>>>(a);
  if (ev) cudaEventRecord(ev[0], stream);
  k_slow<<<sms, 128, 0, stream>>>(a);
  if (ev) cudaEventRecord(ev[1], stream);
  unsigned gt = (unsigned)((z.tiles + 255) / 256);
  if (gt > (unsigned)sms) gt = (unsigned)sms;
  if (gt < 1) gt = 1;
  k_tree<<<gt, 256, 0, stream>>>(a);
  if (ev) cudaEventRecord(ev[2], stream);
  uint64_t nthreads = z.chunks;
  unsigned g3 = (unsigned)((nthreads + 127) / 128);
  if (g3 > (unsigned)sms * 16) g3 = (unsigned)sms * 16;
  if (g3 < 1) g3 = 1;
  k_struct<<<g3, 128, 0, stream>>>(a);
  if (ev) cudaEventRecord(ev[3], stream);
  k_final<<<1, 1, 0, stream>>>(a);
  if (ev) cudaEventRecord(ev[4], stream);
  *launches = 5;
  return cudaGetLastError();
}

}  // namespace jt
