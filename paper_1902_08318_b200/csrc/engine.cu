// engine.cu — host side of the B200 parser: the jsontape C ABI.
//
// Mirrors proj/src/capi.cpp (the reference's C ABI) call for call, but every
// parse runs on the GPU:
//   jt_parser  = one CUDA stream + a grow-only device arena (padded input,
//                two structural-index buffers, look-back records, token
//                records, tape, strings) + pinned control block.
//   jt_parse   = H2D copy into the padded input -> K1 -> K2..K4 -> one D2H of
//                the control block -> D2H of tape and strings on success.
//   jt_stage1 / jt_stage2 keep input and index device-resident in between.
// There is no CPU fallback: without a CUDA device jt_parser_new returns NULL
// and nothing else can be called.
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <charconv>
#include <condition_variable>
#include <functional>
#include <thread>
#include <map>
#include <mutex>
#include <set>
#include <new>
#include <string>
#include <vector>

#include "../../include/jsontape.h"
#include "../../include/jsontape_b200.h"
#include "stage1.h"
#include "jt_common.cuh"
#include "stage2.h"

namespace {

constexpr size_t kPad = 64;  // proj/src/indexer.h:17
constexpr size_t kShardBoundOff = (sizeof(jt::Shard) + 255) & ~(size_t)255;

// JT_CANARY=1 (the test environment's overrun check; compute-sanitizer is
// not available on the GPU pool): every device buffer keeps >= 64 KiB past
// what the current call asked for, filled with 0xA5 when it is sized, and
// canary_check verifies them after the call, aborting with the buffer and
// offset of the first byte a kernel wrote past its capacity.
bool canary_on() {
  static const bool v = [] {
    const char *e = getenv("JT_CANARY");
    return e && e[0] == '1';
  }();
  return v;
}
constexpr uint8_t kCanary = 0xA5;
constexpr size_t kCanaryBytes = 64 << 10;

struct DevBuf {
  void *p = nullptr;
  size_t cap = 0;
  size_t req = 0;  // bytes the last ensure asked for (canary mode: [req, cap) is the canary)
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  bool ensure(size_t bytes) {
    const bool canary = canary_on();
    if (bytes + (canary ? kCanaryBytes : 0) <= cap) {
      if (canary) arm(bytes);
      return true;
    }
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    size_t want = std::max(bytes + (canary ? kCanaryBytes : 0), (size_t)1 << 20);
    want = (want + (1u << 20) - 1) & ~(size_t)((1u << 20) - 1);
    if (cudaMalloc(&p, want) != cudaSuccess) {
      cudaGetLastError();
      p = nullptr;
      return false;
    }
    cap = want;
    if (canary) arm(bytes);
    return true;
  }
  // the canary: [req, req + kCanaryBytes) (a grow-only buffer reused for a
  // smaller call has far more slack than that; overruns land right past req)
  size_t canary_end() const { return std::min(cap, req + kCanaryBytes); }
  void arm(size_t bytes) {
    req = bytes;
    cudaDeviceSynchronize();  // nothing in flight may still write the buffer
    cudaMemset((uint8_t *)p + bytes, kCanary, canary_end() - bytes);
    cudaDeviceSynchronize();
  }
  template <class T>
  T *as() const {
    return (T *)p;
  }
};

}  // namespace

namespace {

// Host storage of documents: page-locked blocks from a process-wide pool, so
// the tape and string buffer come back from HBM at full PCIe/C2C speed and a
// document costs no page faults or zero fill (a std::vector would do both).
// Blocks are size classes (powers of two >= 1 MiB), recycled on
// jt_document_free from any thread, never returned to the OS.
struct PinnedPool {
  std::mutex m;
  std::multimap<size_t, void *> free_blocks;
  static PinnedPool &get() {
    static PinnedPool pool;
    return pool;
  }
  void *take(size_t bytes, size_t *cap, bool *pinned) {
    size_t c = (size_t)1 << 20;
    while (c < bytes) c <<= 1;
    *cap = c;
    {
      std::lock_guard<std::mutex> g(m);
      auto it = free_blocks.find(c);
      if (it != free_blocks.end()) {
        void *b = it->second;
        free_blocks.erase(it);
        *pinned = true;
        return b;
      }
    }
    void *b = nullptr;
    if (cudaMallocHost(&b, c) == cudaSuccess) {
      *pinned = true;
      return b;
    }
    cudaGetLastError();
    *pinned = false;  // pageable fallback, freed with free()
    return malloc(c);
  }
  void give(void *b, size_t cap) {
    std::lock_guard<std::mutex> g(m);
    free_blocks.emplace(cap, b);
  }
};

// vector-like view of part of a document block
template <class T>
struct Span {
  T *p = nullptr;
  size_t n = 0;
  size_t size() const { return n; }
  T *data() const { return p; }
  const T &operator[](size_t i) const { return p[i]; }
  const T *begin() const { return p; }
  const T *end() const { return p + n; }
  bool operator==(const Span &o) const { return n == o.n && (n == 0 || memcmp(p, o.p, n * sizeof(T)) == 0); }
};

// Parallel host memcpy for pageable jt_parse input: a copy engine can only
// read page-locked memory, so a pageable document goes up through a small
// pinned staging ring, and one core's memcpy (~10 GB/s) cannot keep a
// ~55 GB/s PCIe link busy.  `copy` splits the bytes over the helper threads
// and the caller; persistent threads, one pool per parser.
class CopyPool {
 public:
  explicit CopyPool(int helpers) {
    for (int w = 0; w < helpers; w++) th_.emplace_back([this, w] { run(w + 1); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> g(m_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto &t : th_) t.join();
  }
  void copy(void *dst, const void *src, size_t n) {
    const int parts = (int)th_.size() + 1;
    if (n < ((size_t)1 << 20) || parts == 1) {
      memcpy(dst, src, n);
      return;
    }
    {
      std::lock_guard<std::mutex> g(m_);
      dst_ = (uint8_t *)dst;
      src_ = (const uint8_t *)src;
      n_ = n;
      left_.store(parts - 1);
      gen_++;
    }
    cv_.notify_all();
    part(0, parts);
    while (left_.load(std::memory_order_acquire) != 0) std::this_thread::yield();
  }

 private:
  void part(int w, int parts) {
    const size_t step = (n_ / parts + 4095) & ~(size_t)4095;
    const size_t b = std::min(n_, step * (size_t)w), e = std::min(n_, b + step);
    const size_t end = w + 1 == parts ? n_ : e;
    if (end > b) memcpy(dst_ + b, src_ + b, end - b);
  }
  void run(int w) {
    uint64_t seen = 0;
    for (;;) {
      std::unique_lock<std::mutex> g(m_);
      cv_.wait(g, [&] { return stop_ || gen_ != seen; });
      if (stop_) return;
      seen = gen_;
      g.unlock();
      part(w, (int)th_.size() + 1);
      left_.fetch_sub(1, std::memory_order_release);
    }
  }
  std::vector<std::thread> th_;
  std::mutex m_;
  std::condition_variable cv_;
  uint64_t gen_ = 0;
  bool stop_ = false;
  std::atomic<int> left_{0};
  uint8_t *dst_ = nullptr;
  const uint8_t *src_ = nullptr;
  size_t n_ = 0;
};

// host memory the copy engines cannot read directly (not page-locked or
// registered): jt_parse stages it
bool is_pageable(const void *ptr) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return at.type == cudaMemoryTypeUnregistered;
}

}  // namespace

// Layout read by paper_1902_08318_b200/jsontape.py (Document): tape pointer,
// words, strings pointer, bytes.
struct jt_document {
  Span<uint64_t> tape;
  Span<uint8_t> strings;
  void *block = nullptr;
  size_t block_cap = 0;
  bool pinned = false;
  // streamed jt_parse: the string buffer has its own block (sized before
  // the parse knows it), the tape the first one
  void *sblock = nullptr;
  size_t sblock_cap = 0;
  bool spinned = false;
  static void release(void *b, size_t cap, bool pin) {
    if (!b) return;
    if (pin) PinnedPool::get().give(b, cap);
    else free(b);
  }
  ~jt_document() {
    release(block, block_cap, pinned);
    release(sblock, sblock_cap, spinned);
  }
  bool alloc(size_t words, size_t bytes) {
    const size_t tb = (words * 8 + 63) & ~(size_t)63;
    block = PinnedPool::get().take(tb + bytes + 64, &block_cap, &pinned);
    if (!block) return false;
    tape = Span<uint64_t>{(uint64_t *)block, words};
    strings = Span<uint8_t>{(uint8_t *)block + tb, bytes};
    return true;
  }
  // string buffer of up to `cap` bytes (its size is set once known)
  bool alloc_strings(size_t cap) {
    sblock = PinnedPool::get().take(cap + 64, &sblock_cap, &spinned);
    if (!sblock) return false;
    strings = Span<uint8_t>{(uint8_t *)sblock, 0};
    return true;
  }
  bool alloc_tape(size_t words) {
    release(block, block_cap, pinned);  // a block taken before the size was known
    block = nullptr;
    block = PinnedPool::get().take(words * 8 + 64, &block_cap, &pinned);
    if (!block) return false;
    tape = Span<uint64_t>{(uint64_t *)block, words};
    return true;
  }
};

struct jt_parser {
  int device = 0;
  int num_sms = 148;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  DevBuf in;               // padded input
  DevBuf idx[2];           // structural index, double-buffered
  DevBuf aux;              // per index entry: string-buffer prefix (with the last K1 run)
  int cur = 0;             // idx[cur] = index of the last successful stage 1
  DevBuf s1rec, s2rec;     // look-back records
  DevBuf tok, tape_idx, m1, m2, mhi, slow, numlist, scopebits, tile_flags;  // m3 lives in s2rec (zeroed by init)
  DevBuf tape, strings;
  DevBuf ctrl;
  jt::Ctrl *h_ctrl = nullptr;  // pinned
  uint64_t in_len = 0;         // bytes in `in` (retained input)
  size_t in_zeroed_to = 0;     // zero tail maintained up to here
  bool have_index = false;
  uint64_t index_count = 0;
  mutable std::vector<uint32_t> h_index;
  mutable bool h_index_valid = false;
  uint64_t last_tape_len = 0, last_string_bytes = 0;
  bool last_ok = false;
  int launches = 0;
  std::string err;
  uint64_t s1_str_err = ~0ULL, s1_string_bytes = 0, s1_tape_words = 0;  // retained with the index
  bool s1_full = false;  // the retained index came with K1's stage-2 arrays
  uint64_t pending_len = 0;
  int pending_idx = -1;
  bool pending_full = true;
  // captured launch sequences for repeated resident parses (one per index buffer)
  struct Graph {
    cudaGraphExec_t exec = nullptr;
    uint64_t len = ~0ULL;
    cudaStream_t stream = nullptr;
    uint64_t sig = 0;
    int launches = 0;
  } graph[2], graph_s1[2];  // full parse / jt_stage1 (index only), per index buffer
  // byte-range shard of a document (shard.h), between jt_b200_shard_begin
  // and jt_b200_shard_finish
  bool shard_on = false;
  jt::Shard *h_shard = nullptr;  // pinned
  DevBuf shard;                  // Shard + open-container stack
  uint64_t shard_len = 0;        // document length
  uint64_t res_lo = 0, res_hi = 0;  // resident byte range of a shard's document (res_hi 0: all)
  // streamed jt_parse (parse_stream): copy stream, per-chunk events, chunk
  // tile counters and carry states, stage-1 control block snapshot
  cudaStream_t copy_stream = nullptr;
  cudaStream_t d2h_stream = nullptr;  // string pieces back while the input goes up
  cudaStream_t side_stream = nullptr;  // k_stack next to the scalar kernels (stage2_launch)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  jt::Stage2Fork fork{};
  std::vector<cudaEvent_t> chunk_ev, piece_ev;
  cudaEvent_t ev_d2h = nullptr;
  uint64_t *h_piece_sb = nullptr;     // pinned, host-mapped: string bytes up to each piece's end
  uint64_t h_piece_cap = 0;
  cudaEvent_t ev_start = nullptr, ev_s1 = nullptr;
  DevBuf stream_words;
  DevBuf qbuf, qstr;  // distinct_values query: keys, matches, values, lengths, offsets, scan | strings
  jt::Ctrl *h_ctrl_s1 = nullptr;  // pinned
  cudaStream_t s2_stream = nullptr;   // early stage-2 ranges: high priority, ahead of later pieces' stage 1
  // streamed jt_parse, stage 2 in two token ranges (parse_stream)
  DevBuf rngbuf;                      // TokRange A, B | stage-1 token count at piece cA
  DevBuf patchbuf;                    // range B's openers below range A's tape end
  jt::TokRange *h_range = nullptr;    // pinned copies of the early ranges
  unsigned long long *h_patch = nullptr;  // pinned copy of the patch list
  cudaEvent_t ev_rng[5] = {};         // early range k done (its TokRange on the host); [4]: the last range
  cudaStream_t ta_stream = nullptr;   // the early ranges' tape words back to the host
  // NDJSON record mode (jt_b200_parse_records)
  DevBuf recs, nlbuf;
  DevBuf minbuf;  // jt_minify: look-back records, counter, total, output
  // host copy of the per-record results: a page-locked block from the pool
  // (4M records = 188 MB come back at link speed, no zero fill)
  jt::RecordResult *h_records = nullptr;
  size_t h_records_cap = 0;  // block bytes
  bool h_records_pinned = false;
  bool h_records_valid = false;
  const jt::RecordResult *rec_results = nullptr;
  uint64_t rec_n = 0;
  uint8_t rec_last_byte = 0;
  // pageable jt_parse input: pinned staging slots (one upload group each),
  // the event after each slot's H2D copy, and the memcpy pool that fills them
  std::vector<void *> stage_slot;
  std::vector<cudaEvent_t> stage_ev;
  size_t stage_bytes = 0;
  CopyPool *copy_pool = nullptr;
  // optional per-kernel timing: ev[0] before init, then one per launch
  bool prof = false;
  cudaEvent_t ev[8] = {};
  int prof_n = 0;
};

namespace {

// Every call runs on the parser's device (a parser is bound to the device
// current at jt_parser_new), whatever device the calling thread has selected.
struct DevGuard {
  int prev = -1;
  explicit DevGuard(const jt_parser *p) {
    int d = -1;
    if (p && cudaGetDevice(&d) == cudaSuccess && d != p->device && cudaSetDevice(p->device) == cudaSuccess)
      prev = d;
  }
  ~DevGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

__global__ void k_canary(const uint8_t *b, size_t n, unsigned long long *first) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    if (b[i] != kCanary) atomicMin(first, (unsigned long long)i);
}

// canary mode: abort if any kernel of the call `what` wrote past a buffer's
// requested bytes
void canary_check(jt_parser *p, const char *what) {
  if (!canary_on()) return;
  struct Named {
    const char *name;
    const DevBuf *b;
  } bufs[] = {{"in", &p->in}, {"idx0", &p->idx[0]}, {"idx1", &p->idx[1]}, {"aux", &p->aux},
              {"s1rec", &p->s1rec}, {"s2rec", &p->s2rec}, {"tok", &p->tok}, {"tape_idx", &p->tape_idx},
              {"m1", &p->m1}, {"m2", &p->m2}, {"mhi", &p->mhi}, {"slow", &p->slow},
              {"numlist", &p->numlist}, {"scopebits", &p->scopebits}, {"tile_flags", &p->tile_flags},
              {"tape", &p->tape}, {"strings", &p->strings}, {"ctrl", &p->ctrl}, {"shard", &p->shard},
              {"stream_words", &p->stream_words}, {"qbuf", &p->qbuf}, {"qstr", &p->qstr},
              {"rngbuf", &p->rngbuf}, {"patchbuf", &p->patchbuf}, {"recs", &p->recs}, {"nlbuf", &p->nlbuf},
              {"minbuf", &p->minbuf}};
  unsigned long long *d = nullptr, h = ~0ULL;
  cudaDeviceSynchronize();
  if (cudaMalloc(&d, 8) != cudaSuccess) return;
  for (const Named &x : bufs) {
    if (!x.b->p || x.b->canary_end() <= x.b->req) continue;
    cudaMemcpy(d, &h, 8, cudaMemcpyHostToDevice);
    k_canary<<<64, 256>>>((const uint8_t *)x.b->p + x.b->req, x.b->canary_end() - x.b->req, d);
    unsigned long long f = ~0ULL;
    cudaMemcpy(&f, d, 8, cudaMemcpyDeviceToHost);
    if (f != ~0ULL) {
      fprintf(stderr, "JT_CANARY: after %s: buffer %s (%zu bytes requested) written at +%llu past its end\n",
              what, x.name, x.b->req, f);
      abort();
    }
  }
  cudaFree(d);
}

bool cuda_ok(jt_parser *p, cudaError_t e, const char *what) {
  if (e == cudaSuccess) return true;
  p->err = std::string(what) + ": " + cudaGetErrorString(e);
  cudaGetLastError();
  return false;
}

void set_off(long long *o, long long v) {
  if (o) *o = v;
}

size_t round_up(size_t v, size_t m) { return (v + m - 1) / m * m; }

// capacity of the padded input for `len` bytes: stage 1 reads whole 16 KiB
// tiles, stage 2 reads up to 64 bytes past len (escape / atom lookahead)
size_t input_capacity(uint64_t len) { return round_up((size_t)len + kPad, jt::kStage1Tile) + kPad; }

bool ensure_input(jt_parser *p, uint64_t len) {
  size_t need = input_capacity(len);
  size_t old = p->in.cap;
  if (!p->in.ensure(need)) return false;
  if (p->in.cap != old) p->in_zeroed_to = 0;
  return true;
}

// zero [len, tile end + pad) so stage 1 and the lookaheads read zeros
bool zero_tail(jt_parser *p, uint64_t len) {
  size_t end = input_capacity(len);
  return cuda_ok(p, cudaMemsetAsync(p->in.as<uint8_t>() + len, 0, end - len, p->stream),
                 "memset input tail");
}

// Device buffers sized from len before the parse knows S (S <= len: every
// byte can be structural).  The string buffer is at most 2 len + 2 bytes:
// each byte weighs at most 1 except an opening quote (4), and every opening
// quote is followed by content or a closing quote (0).  (The reference
// reserves len + 4 S + 64, tape_builder.cpp:152.)
bool ensure_stage1(jt_parser *p, uint64_t len, int which) {
  size_t cap_tok = (size_t)len + 16;
  if (!p->idx[which].ensure((cap_tok + 16) * sizeof(uint32_t))) return false;
  if (!p->aux.ensure((cap_tok + 16) * sizeof(uint32_t))) return false;
  if (!p->strings.ensure(2 * (size_t)len + 256)) return false;
  if (!p->tok.ensure((cap_tok + 16) * sizeof(uint32_t))) return false;
  if (!p->tape_idx.ensure((cap_tok + 16) * sizeof(uint32_t))) return false;
  if (!p->tile_flags.ensure(jt::stage1_records(len) * sizeof(uint32_t) + 64)) return false;
  if (!p->s1rec.ensure(jt::stage1_records(len) * 9 * sizeof(uint64_t) + 64)) return false;
  if (!p->ctrl.ensure(sizeof(jt::Ctrl))) return false;
  return true;
}

// Number tokens start at least two bytes apart (a number token's first byte
// follows whitespace or a structural character), so the number and slow-float
// lists hold at most len / 2 + 1 entries.  The tape of a document that parses
// has at most len + 3 words (a bracket, string or atom costs at least as many
// bytes as words; a number's second word is paid by the separator or closer
// after it); longer tapes only come from documents that fail, whose tape
// writes past the capacity are dropped (Stage2Args::tape_cap).  The reference
// reserves 2 S + 3 words (tape_builder.cpp:148).  NDJSON records add two root
// words per record (a record can be 2 bytes: "1\n"), so they keep 2 len.
bool ensure_stage2(jt_parser *p, uint64_t len, bool records = false) {
  uint64_t cap = len + 16;
  jt::Stage2Sizes z = jt::stage2_sizes(cap);
  const uint64_t nums = len / 2 + 32;
  bool ok = p->s2rec.ensure(z.n3 * sizeof(int32_t) + 128 + (cap / 4096 + 2) * 32)  /* m3 + 4 words per k_stack tile */ &&
            p->m1.ensure(z.n1 * sizeof(int16_t)) && p->m2.ensure(z.n2 * sizeof(int16_t)) &&
            p->mhi.ensure(z.nhi * sizeof(int16_t) + 64) &&
            p->slow.ensure(nums * sizeof(uint32_t)) &&
            p->numlist.ensure(nums * sizeof(uint32_t)) &&
            p->scopebits.ensure((cap / 32 + 16) * sizeof(uint32_t)) &&
            p->tape.ensure(((records ? 2 * cap : cap) + 16) * sizeof(uint64_t));
  return ok;
}

// layout_tiles: tiles the record arrays are laid out for (the range's own
// count unless a streamed document shares one layout across its pieces)
jt::Stage1Args s1_args(jt_parser *p, uint64_t len, int which, uint64_t begin = 0,
                       uint64_t end = ~0ULL, uint64_t layout_tiles = 0) {
  jt::Stage1Args a{};
  a.begin = begin;
  a.end = end == ~0ULL ? len : end;
  a.last_tile = ~0ULL;
  jt::Ctrl *c = p->ctrl.as<jt::Ctrl>();
  a.in = p->in.as<uint8_t>();
  a.len = len;
  a.idx = p->idx[which].as<uint32_t>();
  a.aux = p->aux.as<uint32_t>();
  a.strings = p->strings.as<uint8_t>();
  a.tokrec = p->tok.as<uint32_t>();
  a.tape_idx = p->tape_idx.as<uint32_t>();
  a.tile_flags = p->tile_flags.as<uint32_t>();
  uint64_t nt = layout_tiles ? layout_tiles : jt::stage1_records(a.end - a.begin);
  a.fn = (uint32_t *)p->s1rec.as<uint64_t>();  // 2 x ntiles u32 in the ntiles-word channel-1 area
  a.carry = a.fn + nt;
  a.rec_count = p->s1rec.as<uint64_t>() + ((nt + 1) & ~1ULL);  // 16-byte aligned: the look-back's vector loads
  a.tile_counter = &c->s1_tile_counter;
  a.utf8_pos = &c->utf8_pos;
  a.str_err = &c->str_err;
  a.total = &c->S;
  a.total_strings = &c->string_bytes;
  a.tape_words = &c->tape_words;
  a.depth_total = &c->depth_total;
  return a;
}

// cap_len: bytes whose tokens this parse handles (the shard's range, or len)
jt::Stage2Args s2_args(jt_parser *p, uint64_t len, int which, uint64_t cap_len = ~0ULL,
                       bool sharded = false) {
  if (cap_len == ~0ULL) cap_len = len;
  jt::Stage2Args a{};
  a.in = p->in.as<uint8_t>();
  a.len = len;
  a.idx = p->idx[which].as<uint32_t>();
  a.aux = p->aux.as<uint32_t>();
  a.ctrl = p->ctrl.as<jt::Ctrl>();
  a.tok = p->tok.as<uint32_t>();
  a.tape_idx = p->tape_idx.as<uint32_t>();
  a.tile_flags = p->tile_flags.as<uint32_t>();
  jt::Stage2Sizes z = jt::stage2_sizes(cap_len + 16);
  a.m1 = p->m1.as<int16_t>();
  a.m2 = p->m2.as<int16_t>();
  a.m3 = p->s2rec.as<int32_t>();
  a.mhi = p->mhi.as<int16_t>();
  for (int k = 0; k < 4; k++) a.hi_off[k] = z.hi_off[k];
  a.slow = p->slow.as<uint32_t>();
  a.numlist = p->numlist.as<uint32_t>();
  a.scopebits = p->scopebits.as<uint32_t>();
  a.stk_rec = (uint64_t *)((uint8_t *)p->s2rec.p + ((z.n3 * sizeof(int32_t) + 64 + 63) & ~(size_t)63));
  a.tape = p->tape.as<uint64_t>();
  a.tape_cap = p->tape.cap / sizeof(uint64_t);
  a.strings = p->strings.as<uint8_t>();
  a.cap_tokens = cap_len + 16;
  a.num_sms = p->num_sms;
  if (sharded) {
    a.sh = p->shard.as<jt::Shard>();
    a.bound = (uint64_t *)(p->shard.as<uint8_t>() + kShardBoundOff);
  }
  return a;
}

// signature of every device pointer baked into a captured graph
uint64_t buffers_sig(jt_parser *p, int which) {
  const void *ptrs[] = {p->in.p, p->idx[which].p, p->aux.p, p->s1rec.p, p->s2rec.p,
                        p->tok.p, p->tape_idx.p, p->m1.p, p->m2.p, p->mhi.p, p->slow.p,
                        p->tape.p, p->strings.p, p->ctrl.p, p->numlist.p, p->scopebits.p,
                        p->tile_flags.p,
                        (const void *)p->h_ctrl};
  uint64_t h = 1469598103934665603ULL;
  for (const void *q : ptrs) h = (h ^ (uint64_t)(uintptr_t)q) * 1099511628211ULL;
  return h;
}

bool enqueue_direct(jt_parser *p, uint64_t len, int which, bool full);

const jt::Stage2Fork *stage2_fork(jt_parser *p) {
  if (!p->side_stream) return nullptr;
  p->fork = jt::Stage2Fork{p->side_stream, p->ev_fork, p->ev_join};
  return &p->fork;
}

// Full parses without profiling replay a CUDA graph of the 9 launches + the
// control-block D2H (captured on first use for this length/stream/buffers).
bool enqueue(jt_parser *p, uint64_t len, int which, bool full) {
  if (p->prof) return enqueue_direct(p, len, which, full);
  auto &g = full ? p->graph[which] : p->graph_s1[which];
  const uint64_t sig = buffers_sig(p, which);
  if (!(g.exec && g.len == len && g.stream == p->stream && g.sig == sig)) {
    if (g.exec) cudaGraphExecDestroy(g.exec);
    g.exec = nullptr;
    cudaGraph_t graph = nullptr;
    if (!cuda_ok(p, cudaStreamBeginCapture(p->stream, cudaStreamCaptureModeThreadLocal), "capture"))
      return enqueue_direct(p, len, which, full);
    bool ok = enqueue_direct(p, len, which, full);
    cudaError_t e = cudaStreamEndCapture(p->stream, &graph);
    if (!ok || e != cudaSuccess || !graph) {
      cudaGetLastError();
      if (graph) cudaGraphDestroy(graph);
      return enqueue_direct(p, len, which, full);
    }
    e = cudaGraphInstantiate(&g.exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) {
      cudaGetLastError();
      g.exec = nullptr;
      return enqueue_direct(p, len, which, full);
    }
    g.len = len;
    g.stream = p->stream;
    g.sig = sig;
    g.launches = p->launches;
  }
  p->launches = g.launches;
  return cuda_ok(p, cudaGraphLaunch(g.exec, p->stream), "graph launch");
}

// Enqueue init + K1 (+ stage 2) for `len` resident bytes; index -> idx[which]
bool enqueue_direct(jt_parser *p, uint64_t len, int which, bool full) {
  p->launches = 0;
  p->prof_n = 0;
  if (p->prof) cudaEventRecord(p->ev[0], p->stream);
  jt::Stage2Sizes z = jt::stage2_sizes(len + 16);
  uint64_t s1w = jt::stage1_records(len) * 9 + 1;  // + the alignment word before the count records (s1_args)
  // m3 (int32, built by atomicMax); the k_stack records behind it are written before they are read
  uint64_t s2w = full ? ((z.n3 * 4 + 64 + 63) / 64) * 8 : 0;
  if (!cuda_ok(p, jt::init_launch(p->ctrl.as<jt::Ctrl>(), p->s1rec.as<uint64_t>(), s1w,
                                  p->s2rec.as<uint64_t>(), s2w, p->stream),
               "init"))
    return false;
  p->launches++;
  if (p->prof) cudaEventRecord(p->ev[1], p->stream);
  if (full) {
    if (!cuda_ok(p, jt::stage1_launch(s1_args(p, len, which), p->stream), "stage1")) return false;
    p->launches += jt::kStage1Launches;
  } else {  // jt_stage1: the index alone (k_index); stage 2 rebuilds the rest
    if (!cuda_ok(p, jt::index_launch(s1_args(p, len, which), p->stream), "index")) return false;
    p->launches += jt::kIndexLaunches;
  }
  if (p->prof) cudaEventRecord(p->ev[2], p->stream);
  if (full) {
    int n = 0;
    if (!cuda_ok(p, jt::stage2_launch(s2_args(p, len, which), p->stream, &n,
                                      p->prof ? p->ev + 3 : nullptr, stage2_fork(p)),
                 "stage2"))
      return false;
    p->launches += n;
    if (p->prof) p->prof_n = 7;
  } else {
    if (!cuda_ok(p, jt::stage1_finalize_launch(p->ctrl.as<jt::Ctrl>(), p->stream), "stage1 final"))
      return false;
    p->launches++;
  }
  return cuda_ok(p, cudaMemcpyAsync(p->h_ctrl, p->ctrl.p, sizeof(jt::Ctrl), cudaMemcpyDeviceToHost,
                                    p->stream),
                 "ctrl D2H");
}

// wait for the enqueued work and publish its results into the parser
jt_error finish(jt_parser *p, int which, bool full, long long *off) {
  if (!cuda_ok(p, cudaStreamSynchronize(p->stream), "sync")) {
    set_off(off, -1);
    return JT_CAPACITY;
  }
  canary_check(p, full ? "parse" : "stage 1");
  const jt::Ctrl &c = *p->h_ctrl;
  p->last_ok = false;
  if (c.code != jt::kUtf8Error) {  // the reference refreshes the index only then
    p->cur = which;
    p->have_index = true;
    p->index_count = c.S;
    p->s1_str_err = c.str_err;
    p->s1_string_bytes = c.string_bytes;
    p->s1_tape_words = c.tape_words;
    p->s1_full = full;  // index-only stage 1: no stage-2 arrays yet
    p->h_index_valid = false;
  }
  set_off(off, c.offset);
  if (full && c.code == jt::kOk && (c.string_bytes >= (1ULL << 32) || c.tape_words >= (1ULL << 32))) {
    // string offsets and tape indices travel as u32 between the kernels: a
    // document whose string buffer or tape reaches 2^32 cannot be represented
    // (only inputs > ~2.4 GiB can get there); fail like an allocation failure
    // (capi.cpp:81-84) instead of returning wrapped offsets
    set_off(off, -1);
    return JT_CAPACITY;
  }
  if (full && c.code == jt::kOk) {
    p->last_ok = true;
    p->last_tape_len = c.tape_len;
    p->last_string_bytes = c.string_bytes;
  }
  return (jt_error)c.code;
}

bool upload(jt_parser *p, const char *data, size_t len) {
  if (!ensure_input(p, len)) return false;
  if (len && !cuda_ok(p, cudaMemcpyAsync(p->in.p, data, len, cudaMemcpyHostToDevice, p->stream),
                      "input H2D"))
    return false;
  if (!zero_tail(p, len)) return false;
  p->in_len = len;
  return true;
}

jt_document *download(jt_parser *p) {
  jt_document *d = new (std::nothrow) jt_document;
  if (!d) return nullptr;
  if (!d->alloc(p->last_tape_len, p->last_string_bytes)) {
    delete d;
    return nullptr;
  }
  if (p->last_tape_len)
    cudaMemcpyAsync(d->tape.data(), p->tape.p, p->last_tape_len * 8, cudaMemcpyDeviceToHost, p->stream);
  if (p->last_string_bytes)
    cudaMemcpyAsync(d->strings.data(), p->strings.p, p->last_string_bytes, cudaMemcpyDeviceToHost,
                    p->stream);
  if (!cuda_ok(p, cudaStreamSynchronize(p->stream), "download")) {
    delete d;
    return nullptr;
  }
  return d;
}

// ---- streamed jt_parse --------------------------------
// The host input goes up in kStreamChunk pieces on a copy stream; stage 1 of
// each piece starts as soon as it has landed (K0b carries the carry state
// from the previous piece, K1's count look-back spans pieces through the
// document's tile numbering), so the upload hides stage 1.  The string
// buffer is complete after stage 1 and comes back while stage 2 runs.
constexpr uint64_t kStreamChunkDefault = 4ULL << 20;  // multiple of kStage1Tile
uint64_t stream_chunk() {  // JT_CHUNK_KB: A/B of the piece size (a multiple of 16 KiB)
  static const uint64_t v = [] {
    const char *e = getenv("JT_CHUNK_KB");
    const long k = e ? atol(e) : 0;
    return k >= 256 ? ((uint64_t)k << 10) / jt::kStage1Tile * jt::kStage1Tile : kStreamChunkDefault;
  }();
  return v;
}
constexpr uint64_t kStreamMin = 8ULL << 20;    // shorter documents: one upload

bool ensure_stream(jt_parser *p, uint64_t nch) {
  if (!p->copy_stream &&
      cudaStreamCreateWithFlags(&p->copy_stream, cudaStreamNonBlocking) != cudaSuccess) {
    cudaGetLastError();
    p->copy_stream = nullptr;
    return false;
  }
  if (!p->h_ctrl_s1 && cudaMallocHost((void **)&p->h_ctrl_s1, sizeof(jt::Ctrl)) != cudaSuccess) {
    cudaGetLastError();
    p->h_ctrl_s1 = nullptr;
    return false;
  }
  auto mk = [](cudaEvent_t *e) {
    return *e || cudaEventCreateWithFlags(e, cudaEventDisableTiming) == cudaSuccess;
  };
  if (!mk(&p->ev_start) || !mk(&p->ev_s1) || !mk(&p->ev_d2h)) return false;
  while (p->chunk_ev.size() < nch) {
    cudaEvent_t e = nullptr;
    if (!mk(&e)) return false;
    p->chunk_ev.push_back(e);
  }
  while (p->piece_ev.size() < nch) {
    cudaEvent_t e = nullptr;
    if (!mk(&e)) return false;
    p->piece_ev.push_back(e);
  }
  if (!p->d2h_stream &&
      cudaStreamCreateWithFlags(&p->d2h_stream, cudaStreamNonBlocking) != cudaSuccess) {
    cudaGetLastError();
    p->d2h_stream = nullptr;
    return false;
  }
  if (p->h_piece_cap < nch) {
    if (p->h_piece_sb) cudaFreeHost(p->h_piece_sb);
    p->h_piece_sb = nullptr;
    p->h_piece_cap = 0;
    if (cudaMallocHost((void **)&p->h_piece_sb, nch * sizeof(uint64_t)) != cudaSuccess) {
      cudaGetLastError();
      p->h_piece_sb = nullptr;
      return false;
    }
    p->h_piece_cap = nch;
  }
  return p->stream_words.ensure(nch * 2 * sizeof(uint32_t) + 64);  // tile counters + carry states
}

constexpr size_t kPatchWords = 2 + 2 * jt::kPatchMax;
constexpr int kMaxRanges = 4;  // early stage-2 ranges of a streamed parse (+ the last one)

bool ensure_ranges(jt_parser *p) {
  if (!p->s2_stream) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    if (cudaStreamCreateWithPriority(&p->s2_stream, cudaStreamNonBlocking, hi) != cudaSuccess) {
      cudaGetLastError();
      p->s2_stream = nullptr;
      return false;
    }
  }
  if (!p->ta_stream && cudaStreamCreateWithFlags(&p->ta_stream, cudaStreamNonBlocking) != cudaSuccess) {
    cudaGetLastError();
    p->ta_stream = nullptr;
    return false;
  }
  for (cudaEvent_t &e : p->ev_rng)
    if (!e && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      e = nullptr;
      return false;
    }
  if (!p->h_range && cudaMallocHost((void **)&p->h_range, kMaxRanges * sizeof(jt::TokRange)) != cudaSuccess) {
    cudaGetLastError();
    p->h_range = nullptr;
    return false;
  }
  if (!p->h_patch && cudaMallocHost((void **)&p->h_patch, kPatchWords * 8) != cudaSuccess) {
    cudaGetLastError();
    p->h_patch = nullptr;
    return false;
  }
  return p->rngbuf.ensure((kMaxRanges + 1) * sizeof(jt::TokRange) + kMaxRanges * 8 + 64) &&
         p->patchbuf.ensure(kPatchWords * 8);
}

// pinned staging ring for pageable input: kStageSlots slots of `bytes`
constexpr int kStageSlots = 4;
bool ensure_stager(jt_parser *p, size_t bytes) {
  if (p->stage_bytes < bytes) {
    jt_document::release(p->h_records, p->h_records_cap, p->h_records_pinned);
  for (void *s : p->stage_slot) cudaFreeHost(s);
    p->stage_slot.clear();
    p->stage_bytes = 0;
    for (int k = 0; k < kStageSlots; k++) {
      void *s = nullptr;
      if (cudaMallocHost(&s, bytes) != cudaSuccess) {
        cudaGetLastError();
        return false;
      }
      p->stage_slot.push_back(s);
    }
    p->stage_bytes = bytes;
  }
  while (p->stage_ev.size() < (size_t)kStageSlots) {
    cudaEvent_t e = nullptr;
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    p->stage_ev.push_back(e);
  }
  if (!p->copy_pool) {
    // JT_COPY_THREADS: threads filling the slots (default: up to 8 of the cores)
    const char *e = getenv("JT_COPY_THREADS");
    long t = e ? atol(e) : 0;
    if (t <= 0) t = std::min<long>(8, std::max<unsigned>(1u, std::thread::hardware_concurrency()));
    p->copy_pool = new (std::nothrow) CopyPool((int)t - 1);
    if (!p->copy_pool) return false;
  }
  return true;
}

jt_error parse_stream(jt_parser *p, const char *data, uint64_t len, jt_document **out, long long *off) {
  static const bool trace = getenv("JT_TRACE") != nullptr;
  auto now_us = []() {
    return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
  };
  const double t0 = trace ? now_us() : 0;
  if (out) *out = nullptr;
  const int which = p->cur ^ 1;
  const uint64_t kStreamChunk = stream_chunk();
  const uint64_t nch = (len + kStreamChunk - 1) / kStreamChunk;
  const uint64_t ntiles = jt::stage1_records(len);
  if (!ensure_input(p, len) || !ensure_stage1(p, len, which) || !ensure_stage2(p, len) ||
      !ensure_stream(p, nch)) {
    set_off(off, -1);
    return JT_CAPACITY;
  }
  // stage 2 in token ranges: early range k covers the tokens of the pieces up
  // to rcut[k] (rounded down to 4096 tokens) and runs on a high-priority
  // stream while the later pieces upload; its tape words go back to the host
  // during the upload; the last range finishes the document after the last
  // piece.  Cuts at JT_RANGE_PCTS % of the pieces (default 30,60,85,96; "0": none:
  // a late fourth cut leaves the last range 4% of the tokens, C4 e2e 41 -> 43 GB/s).
  static const std::vector<uint64_t> pcts = [] {
    std::vector<uint64_t> v;
    const char *e = getenv("JT_RANGE_PCTS");
    std::string str = e ? e : "30,60,85,96";
    size_t at = 0;
    while (at < str.size() && (int)v.size() < kMaxRanges) {
      const long x = atol(str.c_str() + at);
      if (x > 0 && x < 100 && (v.empty() || (uint64_t)x > v.back())) v.push_back((uint64_t)x);
      const size_t c = str.find(',', at);
      if (c == std::string::npos) break;
      at = c + 1;
    }
    return v;
  }();
  std::vector<int64_t> rcut;  // piece after whose stage 1 early range k starts
  if (nch >= 3 && !pcts.empty() && ensure_ranges(p))
    for (uint64_t q : pcts) {
      const int64_t c = std::max<int64_t>(0, (int64_t)(nch * q / 100) - 1);
      if (c + 1 < (int64_t)nch && (rcut.empty() || c > rcut.back())) rcut.push_back(c);
    }
  const int nR = (int)rcut.size();
  const int64_t cA = nR ? rcut[0] : -1;  // >= 0: ranges on
  jt::TokRange *dr = p->rngbuf.as<jt::TokRange>();
  uint64_t *tokA = (uint64_t *)(dr + kMaxRanges + 1);  // token count at each cut
  if (nR) memset((void *)p->h_range, 0, kMaxRanges * sizeof(jt::TokRange));  // nothing in flight writes it
  cudaEvent_t tr_ev[2 * kMaxRanges + 3] = {};  // JT_TRACE: device times of the ranges
  if (trace)
    for (auto &e : tr_ev) cudaEventCreate(&e);
  cudaStream_t cs = p->copy_stream;
  uint32_t *counters = p->stream_words.as<uint32_t>(), *states = counters + nch;
  p->launches = 0;
  jt::Stage2Sizes z = jt::stage2_sizes(len + 16);
  const uint64_t s1w = ntiles * 9 + 1;
  const uint64_t s2w = ((z.n3 * 4 + 64 + 63) / 64) * 8;  // m3 only (enqueue_direct)
  bool ok = cuda_ok(p, jt::init_launch(p->ctrl.as<jt::Ctrl>(), p->s1rec.as<uint64_t>(), s1w,
                                       p->s2rec.as<uint64_t>(), s2w, p->stream),
                    "init") &&
            cuda_ok(p, cudaMemsetAsync(counters, 0, nch * sizeof(uint32_t), p->stream), "counters") &&
            cuda_ok(p, cudaEventRecord(p->ev_start, p->stream), "event") &&
            (!trace || cudaEventRecord(tr_ev[2 * kMaxRanges + 2], p->stream) == cudaSuccess) &&
            cuda_ok(p, cudaStreamWaitEvent(cs, p->ev_start, 0), "wait");
  p->launches = 1;
  // uploads: zero tail first (the last piece's stage 1 reads it), then the pieces
  uint8_t *in = p->in.as<uint8_t>();
  ok = ok && cuda_ok(p, cudaMemsetAsync(in + len, 0, input_capacity(len) - len, cs), "tail");
  // PCIe moves both directions at once far better with large copies (1 MiB:
  // 58 GB/s aggregate, 4 MiB: 83, 16 MiB: 93 measured here), so uploads go in
  // copies of up_pieces pieces (each piece's event after its copy) and the
  // string bytes come back in batches of at least d2h_min (defaults 2 pieces,
  // 4 MiB: C1 e2e 33.1 -> 33.8 GB/s, A/B by JT_UP_PIECES / JT_D2H_MIN_KB)
  // (page-locked documents of 256 MiB and more: 4 pieces = 16 MiB per copy,
  // C4 1 GiB e2e 41 -> 44 GB/s; smaller ones keep 8 MiB so stage 1 starts
  // early; pageable input, filled into the staging ring by host memcpy, keeps
  // 8 MiB groups: C4 36.4 GB/s with 8 MiB, 31.6 with 16 MiB)
  static const uint64_t up_env = [] {
    const char *e = getenv("JT_UP_PIECES");
    const long v = e ? atol(e) : 0;
    return (uint64_t)(v > 0 ? v : 0);
  }();
  const bool pageable = is_pageable(data);
  const uint64_t up_pieces = up_env ? up_env : (!pageable && len >= (256ULL << 20) ? 4 : 2);
  static const uint64_t d2h_min = [] {
    const char *e = getenv("JT_D2H_MIN_KB");
    const long v = e ? atol(e) : -1;
    return v >= 0 ? (uint64_t)v << 10 : (uint64_t)4 << 20;
  }();
  // A pageable document goes up through the pinned staging ring: each
  // upload group is memcpy'd into a free slot by the copy pool, then copied
  // from there; its pieces' stage 1 is enqueued right after it, and the
  // string pieces of finished pieces start back in between.
  const bool staged = pageable && ensure_stager(p, up_pieces * kStreamChunk);
  auto upload_group = [&](uint64_t c0) {
    const uint64_t c1 = std::min(nch, c0 + up_pieces);
    const uint64_t b = c0 * kStreamChunk, e = std::min(len, c1 * kStreamChunk);
    if (staged) {
      const uint64_t grp = c0 / up_pieces;
      const int s = (int)(grp % kStageSlots);
      void *slot = p->stage_slot[s];
      ok = ok && (grp < (uint64_t)kStageSlots || cuda_ok(p, cudaEventSynchronize(p->stage_ev[s]), "slot"));
      if (ok) p->copy_pool->copy(slot, data + b, e - b);
      ok = ok && cuda_ok(p, cudaMemcpyAsync(in + b, slot, e - b, cudaMemcpyHostToDevice, cs), "H2D") &&
           cuda_ok(p, cudaEventRecord(p->stage_ev[s], cs), "event");
    } else {
      ok = ok && cuda_ok(p, cudaMemcpyAsync(in + b, data + b, e - b, cudaMemcpyHostToDevice, cs), "H2D");
    }
    for (uint64_t c = c0; ok && c < c1; c++) ok = cuda_ok(p, cudaEventRecord(p->chunk_ev[c], cs), "event");
  };
  if (!staged)
    for (uint64_t c0 = 0; ok && c0 < nch; c0 += up_pieces) upload_group(c0);
  // the string bytes of each piece go back as soon as its stage 1 is done,
  // while later pieces are still uploading (the copy engines run both
  // directions at once); the string-buffer size is not known yet, so the
  // host block is sized for 5/4 of the input and the rare document with a
  // larger buffer is fetched whole after stage 1
  jt_document *d = nullptr;
  bool early = false;
  uint64_t sb_done = 0;
  // the early ranges' tape words [1, tapeA) go back as each range is done,
  // into a host tape block sized from the input (a larger tape is fetched
  // whole), on their own stream: the string pieces' stream is waited on by
  // k_tile_lengths, these copies must not delay stage 1
  uint64_t tapeA = 0, tape_cap = 0;
  int r_next = 0;
  bool r_stop = false;
  // A range publishes its tape end (host-mapped, written first thing by
  // k_range_a), so its copy is queued behind its completion event while it
  // still runs: no host polling delay between the range and its copy.
  auto published = [&](int k) { return *(volatile uint64_t *)&p->h_range[k].tape_end != 0; };
  auto tape_a = [&](bool block) {
    while (r_next < nR && d && tape_cap) {
      if (!block && !published(r_next) && cudaEventQuery(p->ev_rng[r_next]) != cudaSuccess) return;
      if (!published(r_next) && !cuda_ok(p, cudaEventSynchronize(p->ev_rng[r_next]), "sync")) return;
      const uint64_t lo = r_next ? p->h_range[r_next - 1].tape_end : 1, te = p->h_range[r_next].tape_end;
      if (!r_stop && te >= lo && te <= tape_cap && lo == (tapeA ? tapeA : 1)) {
        if (te > lo &&
            !(cuda_ok(p, cudaStreamWaitEvent(p->ta_stream, p->ev_rng[r_next], 0), "wait") &&
              cuda_ok(p, cudaMemcpyAsync(d->tape.p + lo, p->tape.as<uint64_t>() + lo, (te - lo) * 8,
                                         cudaMemcpyDeviceToHost, p->ta_stream),
                      "tape range D2H")))
          r_stop = true;
        else
          tapeA = te;
      } else {
        r_stop = true;  // the rest comes back with the last range
      }
      if (trace) fprintf(stderr, " range %d done %.0f us: tape words %llu\n", r_next, now_us() - t0,
                         (unsigned long long)te);
      r_next++;
    }
  };
  if (ok && out) {
    d = new (std::nothrow) jt_document;
    // the early path lets kernels (k_tile_lengths) write into the host block:
    // only when it is page-locked (a pageable fallback block is filled by
    // plain copies after stage 1 instead)
    early = d && d->alloc_strings(len + len / 4 + 64) && d->spinned;
    if (early && cA >= 0 && d->alloc_tape(len / 8 + 1024)) tape_cap = d->tape.n;
  }
  // string pieces of the pieces whose stage 1 is enqueued (c < enq) and done
  uint64_t c_next = 0, enq = 0;
  auto drain = [&](bool block) {
    while (early && c_next < enq) {
      const uint64_t c = c_next;
      if (!block && cudaEventQuery(p->piece_ev[c]) != cudaSuccess) {
        cudaGetLastError();
        return;
      }
      if (!cuda_ok(p, cudaEventSynchronize(p->piece_ev[c]), "sync")) {
        early = false;
        return;
      }
      if (trace && (c < 2 || c + 2 >= nch || c % 4 == 0)) fprintf(stderr, " piece %d done %.0f us\n", (int)c, now_us() - t0);
      const uint64_t e = p->h_piece_sb[c];
      if (e > d->sblock_cap - 64 || e < sb_done) {  // too large: fetched whole below
        early = false;
        return;
      }
      c_next++;
      if ((int64_t)c > cA) tape_a(false);
      if (e < sb_done + d2h_min && c + 1 < nch) continue;  // batch small string pieces
      if (e > sb_done &&
          !cuda_ok(p, cudaMemcpyAsync(d->strings.p + sb_done, p->strings.as<uint8_t>() + sb_done, e - sb_done,
                                      cudaMemcpyDeviceToHost, p->d2h_stream),
                   "strings piece D2H")) {
        early = false;
        return;
      }
      sb_done = e;
    }
  };
  // stage 1 piece by piece, each after its upload
  for (uint64_t c = 0; ok && c < nch; c++) {
    if (staged && c % up_pieces == 0) {
      drain(false);
      upload_group(c);
      if (!ok) break;
    }
    const uint64_t b = c * kStreamChunk, e = std::min(len, b + kStreamChunk);
    jt::Stage1Args a = s1_args(p, len, which, b, e, ntiles);
    a.rec_tile0 = b / jt::kStage1Tile;
    a.last_tile = ntiles - 1;
    a.fn += a.rec_tile0;
    a.carry += a.rec_tile0;
    a.tile_counter = counters + c;
    a.init_state = c ? states + c - 1 : nullptr;
    a.out_state = states + c;
    a.sb_out = p->h_piece_sb + c;
    // K1 runs one tile behind the piece boundaries: a tile's last block may
    // read a few bytes past the tile (an escape straddling it), which for a
    // piece's last tile are the next piece's, still uploading
    jt::Stage1Args k1 = a;
    k1.begin = c == 0 ? 0 : b - jt::kStage1Tile;
    k1.end = c + 1 == nch ? len : e - jt::kStage1Tile;
    k1.rec_tile0 = k1.begin / jt::kStage1Tile;
    k1.carry = a.carry - a.rec_tile0 + k1.rec_tile0;
    k1.fn = a.fn - a.rec_tile0 + k1.rec_tile0;
    int rk = -1;  // early range starting after this piece
    for (int q = 0; q < nR; q++)
      if (rcut[q] == (int64_t)c) rk = q;
    if (rk >= 0) k1.tok_out = tokA + rk;
    ok = cuda_ok(p, cudaStreamWaitEvent(p->stream, p->chunk_ev[c], 0), "wait") &&
         cuda_ok(p, jt::stage1_chunk_carry(a, p->stream), "stage1 carry") &&
         cuda_ok(p, jt::stage1_chunk_main(k1, p->stream), "stage1 chunk") &&
         cuda_ok(p, cudaEventRecord(p->piece_ev[c], p->stream), "event");
    p->launches += jt::kStage1Launches;
    if (ok && rk >= 0) {  // early range rk next to the later pieces' stage 1
      jt::Stage2Args s2a = s2_args(p, len, which);
      s2a.patch = p->patchbuf.as<unsigned long long>();
      int nA = 0;
      ok = cuda_ok(p, cudaStreamWaitEvent(p->s2_stream, p->piece_ev[c], 0), "wait") &&
           (!trace || cudaEventRecord(tr_ev[2 * rk], p->s2_stream) == cudaSuccess) &&
           cuda_ok(p, jt::range_a_launch(s2a, tokA + rk, rk ? dr + rk - 1 : nullptr, dr + rk, p->h_range + rk,
                                         p->s2_stream, &nA, stage2_fork(p)),
                   "range") &&
           cuda_ok(p, cudaEventRecord(p->ev_rng[rk], p->s2_stream), "event");
      if (trace) cudaEventRecord(tr_ev[2 * rk + 1], p->s2_stream);
      p->launches += nA;
    }
    enq = c + 1;
  }
  if (trace) fprintf(stderr, " enqueued %.0f us\n", now_us() - t0);
  if (ok && d) {
    drain(true);
    // length fields left to k_tile_lengths are patched into the host copy
    // too, after the last piece is down
    ok = cuda_ok(p, cudaEventRecord(p->ev_d2h, p->d2h_stream), "event") &&
         cuda_ok(p, cudaStreamWaitEvent(p->stream, p->ev_d2h, 0), "wait");
  }
  const double t2 = trace ? now_us() : 0;
  jt::Stage1Args la = s1_args(p, len, which, 0, len, ntiles);
  if (early) la.strings_host = d->strings.p;
  ok = ok && cuda_ok(p, jt::stage1_lengths_launch(la, ntiles, p->stream), "lengths") &&
       cuda_ok(p, cudaMemcpyAsync(p->h_ctrl_s1, p->ctrl.p, sizeof(jt::Ctrl), cudaMemcpyDeviceToHost,
                                  p->stream),
               "ctrl D2H") &&
       cuda_ok(p, cudaEventRecord(p->ev_s1, p->stream), "event");
  p->launches += 1;
  int n2 = 0;
  if (cA >= 0) {
    // the last range: the rest of the document, on the early ranges' stream
    // right after the last piece's stage 1 (it does not need the string
    // pieces' copies k_tile_lengths waits for); openers below the early
    // ranges' tape end as patches.  The parser's stream joins it (finish).
    jt::Stage2Args s2b = s2_args(p, len, which);
    s2b.patch = p->patchbuf.as<unsigned long long>();
    cudaStream_t sb = p->s2_stream;
    ok = ok && cuda_ok(p, cudaStreamWaitEvent(sb, p->piece_ev[nch - 1], 0), "wait") &&
         cuda_ok(p, jt::range_b_launch(s2b, dr + nR - 1, dr + nR, sb, &n2, stage2_fork(p)), "range B") &&
         cuda_ok(p, cudaMemcpyAsync(p->h_patch, p->patchbuf.p, kPatchWords * 8, cudaMemcpyDeviceToHost, sb),
                 "patch D2H") &&
         cuda_ok(p, cudaMemcpyAsync(p->h_ctrl, p->ctrl.p, sizeof(jt::Ctrl), cudaMemcpyDeviceToHost, sb),
                 "ctrl D2H") &&
         cuda_ok(p, cudaEventRecord(p->ev_rng[kMaxRanges], sb), "event") &&
         cuda_ok(p, cudaStreamWaitEvent(p->stream, p->ev_rng[kMaxRanges], 0), "wait");
  } else {
    ok = ok && cuda_ok(p, jt::stage2_launch(s2_args(p, len, which), p->stream, &n2, nullptr, stage2_fork(p)),
                       "stage2") &&
         cuda_ok(p, cudaMemcpyAsync(p->h_ctrl, p->ctrl.p, sizeof(jt::Ctrl), cudaMemcpyDeviceToHost,
                                    p->stream),
                 "ctrl D2H");
  }
  p->launches += n2;
  if (ok) tape_a(true);  // the early ranges' tape words not yet on their way
  if (!ok || !cuda_ok(p, cudaEventSynchronize(p->ev_s1), "sync")) {
    cudaStreamSynchronize(p->stream);
    cudaStreamSynchronize(cs);
    cudaStreamSynchronize(p->d2h_stream);
    if (cA >= 0) {
      cudaStreamSynchronize(p->s2_stream);
      cudaStreamSynchronize(p->ta_stream);
    }
    delete d;
    set_off(off, -1);
    return JT_CAPACITY;
  }
  const double t3 = trace ? now_us() : 0;
  // stage 1 is done: the string buffer is final (and, if it came back piece
  // by piece, already on the host); otherwise fetch it while stage 2 runs
  const jt::Ctrl c1 = *p->h_ctrl_s1;
  if (d && (!early || (c1.utf8_pos == ~0ULL && sb_done != c1.string_bytes))) {
    cudaStreamSynchronize(p->d2h_stream);  // no copy may still target its blocks
    if (cA >= 0) cudaStreamSynchronize(p->ta_stream);
    tapeA = 0;
    delete d;  // not (completely) fetched piece by piece: the whole buffer below
    d = nullptr;
    early = false;
  }
  if (out && c1.utf8_pos == ~0ULL && d && early) {
    d->strings.n = c1.string_bytes;
    if (tapeA && c1.tape_words + 1 <= tape_cap) {
      d->tape.n = c1.tape_words + 1;  // range A's words are in it already
    } else {
      if (tapeA) cudaStreamSynchronize(p->ta_stream);  // before the block is recycled
      tapeA = 0;
      if (!d->alloc_tape(c1.tape_words + 1)) {
        delete d;
        d = nullptr;
      }
    }
  } else if (out && c1.utf8_pos == ~0ULL) {
    d = new (std::nothrow) jt_document;
    if (d && !d->alloc(c1.tape_words + 1, c1.string_bytes)) {
      delete d;
      d = nullptr;
    }
    if (d && c1.string_bytes &&
        !cuda_ok(p, cudaMemcpyAsync(d->strings.data(), p->strings.p, c1.string_bytes,
                                    cudaMemcpyDeviceToHost, cs),
                 "strings D2H")) {
      delete d;
      d = nullptr;
    }
  }
  jt_error e = finish(p, which, true, off);  // waits for stage 2
  cudaStreamSynchronize(cs);
  if (cA >= 0) cudaStreamSynchronize(p->ta_stream);  // the early ranges' tape words
  const double t4 = trace ? now_us() : 0;
  if (e != JT_OK || !out) {
    delete d;
    return e;
  }
  const uint64_t t_lo = tapeA ? tapeA : 0;  // words below came back with range A
  if (!d || d->tape.size() != p->last_tape_len || t_lo > p->last_tape_len ||
      !cuda_ok(p, cudaMemcpyAsync(d->tape.data() + t_lo, p->tape.as<uint64_t>() + t_lo,
                                  (p->last_tape_len - t_lo) * 8, cudaMemcpyDeviceToHost, p->stream),
               "tape D2H") ||
      !cuda_ok(p, cudaStreamSynchronize(p->stream), "sync")) {
    delete d;
    set_off(off, -1);
    return JT_CAPACITY;
  }
  if (tapeA) {  // the root word and range B's openers of containers range A opened
    d->tape.data()[0] = jt::tape_word(jt::kTagRoot, p->last_tape_len - 1);
    const uint64_t n = std::min<uint64_t>(p->h_patch[0], jt::kPatchMax);
    for (uint64_t q = 0; q < n; q++)
      if (p->h_patch[2 + 2 * q] < p->last_tape_len) d->tape.data()[p->h_patch[2 + 2 * q]] = p->h_patch[3 + 2 * q];
  }
  p->in_len = len;
  *out = d;
  if (trace && nR) {
    float t[2 * kMaxRanges];
    for (int q = 0; q < 2 * nR; q++) cudaEventElapsedTime(&t[q], tr_ev[2 * kMaxRanges + 2], tr_ev[q]);
    for (int q = 0; q < nR; q++) fprintf(stderr, " range %d on the device: started %.0f us, done %.0f us\n", q, 1e3 * t[2 * q], 1e3 * t[2 * q + 1]);
  }
  if (trace)
    for (auto &e : tr_ev) cudaEventDestroy(e);
  if (trace)
    fprintf(stderr, "parse_stream: pieces+D2H enqueued %.0f us, stage 1 done %.0f, stage 2 done %.0f, tape down %.0f (early %d)\n",
            t2 - t0, t3 - t0, t4 - t0, now_us() - t0, (int)early);
  return e;
}

jt_error parse_resident(jt_parser *p, uint64_t len, jt_document **out, long long *off) {
  if (out) *out = nullptr;
  if (len >= (1ULL << 32)) {  // indexer.cpp:33-34
    set_off(off, -1);
    return JT_CAPACITY;
  }
  int which = p->cur ^ 1;
  if (!ensure_stage1(p, len, which) || !ensure_stage2(p, len)) {
    set_off(off, -1);
    return JT_CAPACITY;
  }
  if (!enqueue(p, len, which, true)) {
    set_off(off, -1);
    return JT_CAPACITY;
  }
  jt_error e = finish(p, which, true, off);
  if (e == JT_OK && out) {
    *out = download(p);
    if (!*out) {
      set_off(off, -1);
      return JT_CAPACITY;
    }
  }
  return e;
}


// Byte-range shard setup (shard.h) for jt_b200_shard_begin.
int shard_setup(jt_parser *p, size_t len, unsigned g, unsigned G, size_t begin, size_t end) {
  if (G == 0 || g >= G || (uint64_t)len >= (1ULL << 32) || begin % jt::kStage1Tile != 0 ||
      !(begin < end) || end > len || (g + 1 == G) != (end == len) || (g == 0) != (begin == 0)) {
    p->err = "shard_begin: bad shard layout";
    return -1;
  }
  if (!p->h_shard && cudaMallocHost((void **)&p->h_shard, sizeof(jt::Shard)) != cudaSuccess) {
    cudaGetLastError();
    p->h_shard = nullptr;
    p->err = "shard_begin: pinned allocation";
    return -1;
  }
  if (p->res_hi && (p->res_lo > (begin >= 64 ? begin - 64 : 0) ||
                    p->res_hi < (end + 64 < len ? end + 64 : len))) {
    p->err = "shard_begin: the resident range must cover [begin - 64, end + 64)";
    return -1;
  }
  const uint64_t range = end - begin;
  if (!ensure_input(p, len) || !ensure_stage1(p, range, 0) || !ensure_stage2(p, range) ||
      !p->shard.ensure(kShardBoundOff + jt::kBoundMax * sizeof(uint64_t))) {
    p->err = "shard_begin: device allocation";
    return -1;
  }
  jt::Shard h{};
  h.g = g;
  h.G = G;
  h.begin = begin;
  h.end = end;
  h.len = len;
  h.streamed = 0u;
  h.res_hi = p->res_hi && p->res_hi < len ? p->res_hi : 0;
  *p->h_shard = h;
  if (!cuda_ok(p, cudaMemcpyAsync(p->shard.p, p->h_shard, sizeof(jt::Shard), cudaMemcpyHostToDevice,
                                  p->stream),
               "shard upload"))
    return -1;
  p->shard_on = true;
  p->shard_len = len;
  p->in_len = len;
  p->cur = 0;
  p->last_ok = false;
  p->have_index = false;
  p->h_index_valid = false;
  return 0;
}

}  // namespace

extern "C" {

jt_parser *jt_parser_new(void) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  jt_parser *p = new (std::nothrow) jt_parser;
  if (!p) return nullptr;
  p->device = dev;
  cudaDeviceGetAttribute(&p->num_sms, cudaDevAttrMultiProcessorCount, dev);
  if (cudaStreamCreateWithFlags(&p->own_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaMallocHost((void **)&p->h_ctrl, sizeof(jt::Ctrl)) != cudaSuccess ||
      !p->ctrl.ensure(sizeof(jt::Ctrl))) {
    cudaGetLastError();
    if (p->own_stream) cudaStreamDestroy(p->own_stream);
    if (p->h_ctrl) cudaFreeHost(p->h_ctrl);
    delete p;
    return nullptr;
  }
  p->stream = p->own_stream;
  // optional: without the side stream stage 2 runs k_stack in line
  if (cudaStreamCreateWithFlags(&p->side_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&p->ev_join, cudaEventDisableTiming) != cudaSuccess) {
    cudaGetLastError();
    if (p->side_stream) cudaStreamDestroy(p->side_stream);
    p->side_stream = nullptr;
  }
  jt::stage1_configure();  // kernel attributes once, outside any capture
  return p;
}

void jt_parser_free(jt_parser *p) {
  DevGuard dg_(p);
  if (!p) return;
  cudaStreamSynchronize(p->stream);
  for (auto &g : p->graph)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  for (auto &g : p->graph_s1)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  if (p->own_stream) cudaStreamDestroy(p->own_stream);
  if (p->side_stream) {
    cudaStreamSynchronize(p->side_stream);
    cudaStreamDestroy(p->side_stream);
  }
  if (p->ev_fork) cudaEventDestroy(p->ev_fork);
  if (p->ev_join) cudaEventDestroy(p->ev_join);
  if (p->h_ctrl) cudaFreeHost(p->h_ctrl);
  if (p->h_shard) cudaFreeHost(p->h_shard);
  if (p->copy_stream) {
    cudaStreamSynchronize(p->copy_stream);
    cudaStreamDestroy(p->copy_stream);
  }
  if (p->d2h_stream) {
    cudaStreamSynchronize(p->d2h_stream);
    cudaStreamDestroy(p->d2h_stream);
  }
  for (cudaEvent_t e : p->piece_ev) cudaEventDestroy(e);
  if (p->ev_d2h) cudaEventDestroy(p->ev_d2h);
  if (p->h_piece_sb) cudaFreeHost(p->h_piece_sb);
  for (cudaEvent_t e : p->chunk_ev) cudaEventDestroy(e);
  if (p->ev_start) cudaEventDestroy(p->ev_start);
  if (p->ev_s1) cudaEventDestroy(p->ev_s1);
  if (p->h_ctrl_s1) cudaFreeHost(p->h_ctrl_s1);
  if (p->s2_stream) {
    cudaStreamSynchronize(p->s2_stream);
    cudaStreamDestroy(p->s2_stream);
  }
  if (p->h_range) cudaFreeHost(p->h_range);
  if (p->h_patch) cudaFreeHost(p->h_patch);
  for (void *s : p->stage_slot) cudaFreeHost(s);
  for (cudaEvent_t e : p->stage_ev) cudaEventDestroy(e);
  delete p->copy_pool;
  for (cudaEvent_t e : p->ev_rng)
    if (e) cudaEventDestroy(e);
  if (p->ta_stream) {
    cudaStreamSynchronize(p->ta_stream);
    cudaStreamDestroy(p->ta_stream);
  }
  delete p;
}

void jt_parser_set_flags(jt_parser *p, int use_clmul, int fast_extract, int vector_classify) {
  DevGuard dg_(p);
  (void)p;
  (void)use_clmul;
  (void)fast_extract;
  (void)vector_classify;
}

jt_error jt_parse(jt_parser *p, const char *data, size_t len, jt_document **out,
                  long long *error_offset) {
  DevGuard dg_(p);
  if (out) *out = nullptr;
  if ((uint64_t)len >= (1ULL << 32)) {
    set_off(error_offset, -1);
    return JT_CAPACITY;
  }
  if ((uint64_t)len >= kStreamMin) {
    return parse_stream(p, data, len, out, error_offset);
  }
  if (!upload(p, data, len)) {
    set_off(error_offset, -1);
    return JT_CAPACITY;
  }
  return parse_resident(p, len, out, error_offset);
}

jt_error jt_stage1(jt_parser *p, const char *data, size_t len, long long *error_offset) {
  DevGuard dg_(p);
  if ((uint64_t)len >= (1ULL << 32)) {
    set_off(error_offset, -1);
    return JT_CAPACITY;
  }
  if (!upload(p, data, len)) {
    set_off(error_offset, -1);
    return JT_CAPACITY;
  }
  return jt_b200_stage1_resident(p, len, error_offset);
}

size_t jt_index_count(const jt_parser *p) { return p->have_index ? (size_t)p->index_count : 0; }

const uint32_t *jt_index_positions(const jt_parser *p) {
  DevGuard dg_(p);
  if (!p->h_index_valid) {
    p->h_index.assign(p->index_count + 8, 0u);
    if (p->index_count)
      cudaMemcpy(p->h_index.data(), p->idx[p->cur].p, p->index_count * 4, cudaMemcpyDeviceToHost);
    p->h_index_valid = true;
  }
  return p->h_index.data();
}

jt_error jt_stage2(jt_parser *p, jt_document **out, long long *error_offset) {
  DevGuard dg_(p);
  if (out) *out = nullptr;
  uint64_t len = p->in_len;
  if (!ensure_stage2(p, len)) {
    set_off(error_offset, -1);
    return JT_CAPACITY;
  }
  if (p->have_index && !p->s1_full) {
    // the last jt_stage1 built the index alone (k_index): K1 rebuilds the
    // same index with the string payload and token arrays, then stage 2
    // (after a UTF-8-failed jt_stage1 the reference would run on its stale
    // index; this reports the retained input's own verdict)
    if (!ensure_stage1(p, len, p->cur) || !enqueue(p, len, p->cur, true)) {
      set_off(error_offset, -1);
      return JT_CAPACITY;
    }
    jt_error e = finish(p, p->cur, true, error_offset);
    if (e == JT_OK && out) {
      *out = download(p);
      if (!*out) {
        set_off(error_offset, -1);
        return JT_CAPACITY;
      }
    }
    return e;
  }
  // re-run stage 2 over the retained input, index and string payload:
  // reset the records, then restore the stage-1 results into the control block
  jt::Stage2Sizes z = jt::stage2_sizes(len + 16);
  p->launches = 0;
  if (!cuda_ok(p, jt::init_launch(nullptr, p->s1rec.as<uint64_t>(), 0, p->s2rec.as<uint64_t>(),
                                  ((z.n3 * 4 + 64 + 63) / 64) * 8 + ((len + 16) / 256 + 2) * 4,
                                  p->stream),
               "init")) {
    set_off(error_offset, -1);
    return JT_CAPACITY;
  }
  jt::Ctrl c0{};
  c0.utf8_pos = ~0ULL;
  c0.err_key = ~0ULL;
  c0.S = p->have_index ? p->index_count : 0;
  c0.str_err = p->s1_str_err;
  c0.string_bytes = p->s1_string_bytes;
  c0.tape_words = p->s1_tape_words;
  c0.code = -1;
  c0.offset = -1;
  *p->h_ctrl = c0;
  cudaMemcpyAsync(p->ctrl.p, p->h_ctrl, sizeof(jt::Ctrl), cudaMemcpyHostToDevice, p->stream);
  int n = 0;
  if (!cuda_ok(p, jt::stage2_launch(s2_args(p, len, p->cur), p->stream, &n, nullptr, stage2_fork(p)),
               "stage2") ||
      !cuda_ok(p, cudaMemcpyAsync(p->h_ctrl, p->ctrl.p, sizeof(jt::Ctrl), cudaMemcpyDeviceToHost,
                                  p->stream),
               "ctrl")) {
    set_off(error_offset, -1);
    return JT_CAPACITY;
  }
  p->launches = n + 1;
  if (!cuda_ok(p, cudaStreamSynchronize(p->stream), "sync")) {
    set_off(error_offset, -1);
    return JT_CAPACITY;
  }
  canary_check(p, "stage 2");
  const jt::Ctrl &c = *p->h_ctrl;
  set_off(error_offset, c.offset);
  p->last_ok = c.code == jt::kOk;
  if (p->last_ok) {
    p->last_tape_len = c.tape_len;
    p->last_string_bytes = c.string_bytes;
    if (out) {
      *out = download(p);
      if (!*out) {
        set_off(error_offset, -1);
        return JT_CAPACITY;
      }
    }
  }
  return (jt_error)c.code;
}

void jt_document_free(jt_document *doc) { delete doc; }

int jt_document_equal(const jt_document *a, const jt_document *b) {
  return a->tape == b->tape && a->strings == b->strings ? 1 : 0;
}

// text dump, same format as tape_dump (proj/src/tape_builder.cpp:277-350)
char *jt_document_dump(const jt_document *doc) {
  std::string out;
  char buf[64];
  auto num = [&](uint64_t v) {
    auto r = std::to_chars(buf, buf + sizeof(buf), v);
    out.append(buf, r.ptr);
  };
  const auto &t = doc->tape;
  for (size_t i = 0; i < t.size(); i++) {
    uint64_t w = t[i];
    uint8_t tag = (uint8_t)(w >> 56);
    uint64_t pl = w & jt::kPayloadMask;
    num(i);
    out += " : ";
    switch (tag) {
      case 'r':
        out += "r\t// pointing to ";
        num(pl);
        break;
      case '{':
      case '[':
        out += (char)tag;
        out += "\t// pointing to next tape location ";
        num(pl);
        out += " (first node after the scope)";
        break;
      case '}':
      case ']':
        out += (char)tag;
        out += "\t// pointing to previous tape location ";
        num(pl);
        out += " (start of the scope)";
        break;
      case '"': {
        out += "string \"";
        uint32_t n = 0;
        memcpy(&n, doc->strings.data() + pl, 4);
        out.append((const char *)doc->strings.data() + pl + 4, n);
        out += '"';
        break;
      }
      case 'l': {
        out += "integer ";
        auto r = std::to_chars(buf, buf + sizeof(buf), (int64_t)t[i + 1]);
        out.append(buf, r.ptr);
        i++;
        break;
      }
      case 'd': {
        out += "double ";
        double v;
        memcpy(&v, &t[i + 1], 8);
        auto r = std::to_chars(buf, buf + sizeof(buf), v);
        out.append(buf, r.ptr);
        i++;
        break;
      }
      case 't': out += "true"; break;
      case 'f': out += "false"; break;
      case 'n': out += "null"; break;
    }
    out += '\n';
  }
  char *s = (char *)malloc(out.size() + 1);
  if (s) memcpy(s, out.c_str(), out.size() + 1);
  return s;
}

}  // extern "C"

namespace {

// (kind, bits, bytes) ordered as scalar_value (document.h:71-90)
struct DVal {
  int k;
  uint64_t bits;
  std::string bytes;
  bool operator<(const DVal &o) const {
    if (k != o.k) return k < o.k;
    return k == 5 ? bytes < o.bytes : bits < o.bits;
  }
};

// one value per line, as the reference prints scalar_value (document.cpp:108-131)
std::string format_distinct(const std::set<DVal> &vals) {
  std::string out;
  char buf[64];
  for (const DVal &v : vals) {
    switch (v.k) {
      case 0: out += "null"; break;
      case 1: out += "false"; break;
      case 2: out += "true"; break;
      case 3: out.append(buf, std::to_chars(buf, buf + sizeof(buf), (int64_t)v.bits).ptr); break;
      case 4: {
        double d;
        memcpy(&d, &v.bits, 8);
        out.append(buf, std::to_chars(buf, buf + sizeof(buf), d).ptr);
        break;
      }
      default: out += '"' + v.bytes + '"';
    }
    out += '\n';
  }
  return out;
}

char *malloc_string(const std::string &out) {
  char *r = (char *)malloc(out.size() + 1);
  if (!r) return nullptr;
  memcpy(r, out.data(), out.size());
  r[out.size()] = 0;
  return r;
}

std::vector<std::string> split_path(const char *path) {
  std::vector<std::string> keys;
  for (const char *a = path;;) {
    const char *dot = strchr(a, '.');
    keys.emplace_back(a, dot ? (size_t)(dot - a) : strlen(a));
    if (!dot) break;
    a = dot + 1;
  }
  return keys;
}

}  // namespace

extern "C" {

// Sorted distinct scalars at a dotted key path (capi.cpp:143-151,
// document.cpp:134-192): the first key matches at any depth, later keys must
// follow directly, arrays are looked through.  Host-side walk of the
// document's tape (a non-hot export).
char *jt_document_distinct(const jt_document *doc, const char *path) {
  std::string out;
  if (doc && path && *path && doc->tape.size() > 2) {
    const std::vector<std::string> keys = split_path(path);
    const uint64_t *t = doc->tape.data();
    const uint8_t *sb = doc->strings.data();
    auto tag = [&](uint64_t i) { return (uint8_t)(t[i] >> 56); };
    auto pay = [&](uint64_t i) { return t[i] & ((1ULL << 56) - 1); };
    auto next = [&](uint64_t i) -> uint64_t {  // index after the value at i
      const uint8_t g = tag(i);
      return (g == '{' || g == '[') ? pay(i) : (g == 'l' || g == 'd') ? i + 2 : i + 1;
    };
    auto str = [&](uint64_t i) {
      uint32_t n;
      memcpy(&n, sb + pay(i), 4);
      return std::string((const char *)sb + pay(i) + 4, n);
    };
    std::set<DVal> vals;
    auto scalar = [&](uint64_t i) {
      const uint8_t g = tag(i);
      if (g == 'n') vals.insert({0, 0, {}});
      else if (g == 'f') vals.insert({1, 0, {}});
      else if (g == 't') vals.insert({2, 0, {}});
      else if (g == 'l') vals.insert({3, t[i + 1], {}});
      else if (g == 'd') vals.insert({4, t[i + 1], {}});
      else if (g == '"') vals.insert({5, 0, str(i)});
    };
    // children of the container at i: (key index or 0, value index)
    auto each = [&](uint64_t i, auto &&fn) {
      const bool obj = tag(i) == '{';
      for (uint64_t c = i + 1, stop = pay(i) - 1; c < stop;) {
        const uint64_t v = obj ? c + 1 : c;
        fn(obj ? c : 0, v);
        c = next(v);
      }
    };
    std::function<void(uint64_t, size_t)> follow = [&](uint64_t i, size_t k) {
      const uint8_t g = tag(i);
      if (k == keys.size()) {
        if (g != '{' && g != '[') scalar(i);
        return;
      }
      if (g == '{')
        each(i, [&](uint64_t key, uint64_t v) {
          if (str(key) == keys[k]) follow(v, k + 1);
        });
      else if (g == '[')
        each(i, [&](uint64_t, uint64_t v) { follow(v, k); });
    };
    std::function<void(uint64_t)> search = [&](uint64_t i) {
      const uint8_t g = tag(i);
      if (g == '{')
        each(i, [&](uint64_t key, uint64_t v) {
          if (str(key) == keys[0]) follow(v, 1);
          search(v);
        });
      else if (g == '[')
        each(i, [&](uint64_t, uint64_t v) { search(v); });
    };
    search(1);  // document_root (document.cpp:99)
    out = format_distinct(vals);
  }
  return malloc_string(out);
}

// distinct_values of the parser's last successful parse, on the device
// (§8f rank 4, "parse + select"): k_distinct_match selects the scalars, the
// values and their string bytes are gathered into a compact buffer (one D2H
// each), and the host only sorts the selected values; same text as
// jt_document_distinct on the downloaded document.  NULL without such a
// parse or on a device error.
char *jt_b200_distinct(jt_parser *p, const char *path) {
  DevGuard dg_(p);
  if (!p || !p->last_ok || !path) return nullptr;
  std::set<DVal> vals;
  if (!*path) return malloc_string(std::string());
  const std::vector<std::string> keys = split_path(path);
  if (keys.size() > (size_t)jt::kDistinctMaxKeys) {
    p->err = "distinct: too many keys";
    return nullptr;
  }
  const uint64_t S = p->index_count, len = p->in_len;
  jt::DistinctQuery q{};
  std::string kb;
  q.nkeys = (int)keys.size();
  for (size_t k = 0; k < keys.size(); k++) {
    q.key_off[k] = (uint32_t)kb.size();
    kb += keys[k];
  }
  q.key_off[keys.size()] = (uint32_t)kb.size();
  // qbuf: count | keys | match[S] | vals[S] | len[S] | off[S]
  const size_t a_keys = 256, a_match = round_up(a_keys + kb.size() + 1, 256);
  const size_t a_vals = round_up(a_match + 4 * S + 4, 256), a_len = round_up(a_vals + 16 * S, 256);
  const size_t a_off = round_up(a_len + 4 * S + 4, 256), a_tmp = round_up(a_off + 4 * S + 4, 256);
  if (!p->qbuf.ensure(a_tmp + 256)) {
    p->err = "distinct: out of memory";
    return nullptr;
  }
  uint8_t *qb = p->qbuf.as<uint8_t>();
  uint32_t *d_count = (uint32_t *)qb, *d_match = (uint32_t *)(qb + a_match), *d_len = (uint32_t *)(qb + a_len),
           *d_off = (uint32_t *)(qb + a_off);
  jt::DistinctVal *d_vals = (jt::DistinctVal *)(qb + a_vals);
  q.key_bytes = qb + a_keys;
  const jt::Stage2Args a = s2_args(p, len, p->cur);
  uint32_t count = 0;
  if (!cuda_ok(p, cudaMemsetAsync(d_count, 0, 4, p->stream), "memset") ||
      (kb.size() && !cuda_ok(p, cudaMemcpyAsync(qb + a_keys, kb.data(), kb.size(), cudaMemcpyHostToDevice, p->stream),
                             "keys H2D")) ||
      !cuda_ok(p, jt::distinct_match_launch(a, q, d_match, d_count, p->stream), "distinct match") ||
      !cuda_ok(p, cudaMemcpyAsync(&count, d_count, 4, cudaMemcpyDeviceToHost, p->stream), "count D2H") ||
      !cuda_ok(p, cudaStreamSynchronize(p->stream), "sync"))
    return nullptr;
  std::vector<jt::DistinctVal> hv(count);
  std::vector<uint32_t> last(2, 0);
  std::vector<uint8_t> hs;
  if (count) {
    if (!cuda_ok(p, jt::distinct_values_launch(a, d_match, count, d_vals, d_len, p->stream), "distinct values") ||
        !cuda_ok(p, cudaMemsetAsync(d_len + count, 0, 4, p->stream), "memset") ||
        !cuda_ok(p, jt::scan_u32_launch(d_len, d_off, count + 1, p->stream), "scan") ||
        !cuda_ok(p, cudaMemcpyAsync(hv.data(), d_vals, 16 * (size_t)count, cudaMemcpyDeviceToHost, p->stream),
                 "values D2H") ||
        !cuda_ok(p, cudaMemcpyAsync(last.data(), d_off + count, 4, cudaMemcpyDeviceToHost, p->stream), "D2H") ||
        !cuda_ok(p, cudaStreamSynchronize(p->stream), "sync"))
      return nullptr;
    const uint32_t total = last[0];
    if (total) {
      if (!p->qstr.ensure(total) ||
          !cuda_ok(p, jt::distinct_strings_launch(a, d_vals, d_off, count, p->qstr.as<uint8_t>(), p->stream),
                   "distinct strings"))
        return nullptr;
      hs.resize(total);
      std::vector<uint32_t> ho(count);
      if (!cuda_ok(p, cudaMemcpyAsync(hs.data(), p->qstr.p, total, cudaMemcpyDeviceToHost, p->stream), "D2H") ||
          !cuda_ok(p, cudaMemcpyAsync(ho.data(), d_off, 4 * (size_t)count, cudaMemcpyDeviceToHost, p->stream),
                   "D2H") ||
          !cuda_ok(p, cudaStreamSynchronize(p->stream), "sync"))
        return nullptr;
      for (uint32_t k = 0; k < count; k++)
        if (hv[k].tag == '"') hv[k].bits = ho[k];
    }
  }
  canary_check(p, "distinct");
  for (const jt::DistinctVal &r : hv) {
    switch (r.tag) {
      case 'n': vals.insert({0, 0, {}}); break;
      case 'f': vals.insert({1, 0, {}}); break;
      case 't': vals.insert({2, 0, {}}); break;
      case 'l': vals.insert({3, r.bits, {}}); break;
      case 'd': vals.insert({4, r.bits, {}}); break;
      case '"': vals.insert({5, 0, std::string((const char *)hs.data() + r.bits, r.len)}); break;
      default: break;
    }
  }
  return malloc_string(format_distinct(vals));
}

void jt_string_free(char *s) { free(s); }

// capi.cpp:154-167: full parse, then minify_pass (indexer.cpp:58-75) on the
// GPU (k_minify) over the same resident input and its K0 carry-ins
jt_error jt_minify(jt_parser *p, const char *data, size_t len, char *dst, size_t *dst_len,
                   long long *error_offset) {
  DevGuard dg_(p);
  if ((uint64_t)len >= (1ULL << 32)) {
    set_off(error_offset, -1);
    return JT_CAPACITY;
  }
  if (!upload(p, data, len)) {
    set_off(error_offset, -1);
    return JT_CAPACITY;
  }
  jt_error e = parse_resident(p, len, nullptr, error_offset);
  if (e != JT_OK) return e;
  const uint64_t ntiles = jt::stage1_records(len);
  const size_t rec_bytes = round_up(ntiles * 8 + 16, 256);
  if (!p->minbuf.ensure(rec_bytes + len + 256)) {
    set_off(error_offset, -1);
    return JT_CAPACITY;
  }
  jt::MinifyArgs a{};
  a.in = p->in.as<uint8_t>();
  a.len = len;
  a.carry = s1_args(p, len, p->cur).carry;
  a.rec = p->minbuf.as<uint64_t>();
  a.tile_counter = (uint32_t *)(a.rec + ntiles);
  a.total = a.rec + ntiles + 1;
  a.out = p->minbuf.as<uint8_t>() + rec_bytes;
  a.ntiles = ntiles;
  uint64_t total = 0;
  if (!cuda_ok(p, cudaMemsetAsync(p->minbuf.p, 0, (ntiles + 2) * 8, p->stream), "memset") ||
      !cuda_ok(p, jt::minify_launch(a, p->stream), "minify") ||
      !cuda_ok(p, cudaMemcpyAsync(&total, a.total, 8, cudaMemcpyDeviceToHost, p->stream), "D2H") ||
      !cuda_ok(p, cudaStreamSynchronize(p->stream), "sync") ||
      (total && !cuda_ok(p, cudaMemcpy(dst, a.out, total, cudaMemcpyDeviceToHost), "D2H"))) {
    set_off(error_offset, -1);
    return JT_CAPACITY;
  }
  canary_check(p, "minify");
  if (dst_len) *dst_len = total;
  return JT_OK;
}

// capi.cpp:169-191 / stats.cpp:5-47: parse, then the counts as device
// reductions over the token records, tape tags and input (k_stats)
jt_error jt_compute_stats(jt_parser *p, const char *data, size_t len, jt_stats *out,
                          long long *error_offset) {
  DevGuard dg_(p);
  if ((uint64_t)len >= (1ULL << 32)) {
    set_off(error_offset, -1);
    return JT_CAPACITY;
  }
  if (!upload(p, data, len)) {
    set_off(error_offset, -1);
    return JT_CAPACITY;
  }
  jt_error e = parse_resident(p, len, nullptr, error_offset);
  if (e != JT_OK) return e;
  if (!p->minbuf.ensure(256)) {
    set_off(error_offset, -1);
    return JT_CAPACITY;
  }
  unsigned long long *cnt = p->minbuf.as<unsigned long long>();
  unsigned long long h[9] = {0};
  if (!cuda_ok(p, cudaMemsetAsync(cnt, 0, sizeof(h), p->stream), "memset") ||
      !cuda_ok(p, jt::stats_launch(s2_args(p, len, p->cur), cnt, p->stream), "stats") ||
      !cuda_ok(p, cudaMemcpyAsync(h, cnt, sizeof(h), cudaMemcpyDeviceToHost, p->stream), "D2H") ||
      !cuda_ok(p, cudaStreamSynchronize(p->stream), "sync")) {
    set_off(error_offset, -1);
    return JT_CAPACITY;
  }
  canary_check(p, "stats");
  jt_stats s{};
  s.integers = h[0];
  s.floats = h[1];
  s.strings = h[2];
  s.non_ascii_bytes = h[3];
  s.objects = h[4];
  s.arrays = h[5];
  s.nulls = h[6];
  s.trues = h[7];
  s.falses = h[8];
  s.structurals = p->index_count;
  s.bytes = len;
  s.bytes_per_structural = s.structurals ? (double)len / (double)s.structurals : 0.0;
  if (out) *out = s;
  return JT_OK;
}

int jt_oracle_validate(const char *data, size_t len) {
  jt_parser *p = jt_parser_new();
  if (!p) return 0;
  jt_error e = jt_parse(p, data, len, nullptr, nullptr);
  jt_parser_free(p);
  return e == JT_OK ? 1 : 0;
}

char *jt_generate(const char *kind, uint64_t size, uint64_t seed, size_t *len_out) {
  (void)kind;
  (void)size;
  (void)seed;
  if (len_out) *len_out = 0;
  return nullptr;
}

const char *jt_error_name(jt_error code) {
  switch (code) {
    case JT_OK: return "OK";
    case JT_UTF8_ERROR: return "UTF8_ERROR";
    case JT_STRING_ERROR: return "STRING_ERROR";
    case JT_NUMBER_ERROR: return "NUMBER_ERROR";
    case JT_TAPE_ERROR: return "TAPE_ERROR";
    case JT_DEPTH_ERROR: return "DEPTH_ERROR";
    case JT_CAPACITY: return "CAPACITY";
    default: return "EMPTY";
  }
}

// ---- B200 extensions -------------------------------------------------------

void *jt_b200_input_buffer(jt_parser *p, size_t len) {
  DevGuard dg_(p);
  if ((uint64_t)len >= (1ULL << 32)) return nullptr;
  if (!ensure_input(p, len) || !zero_tail(p, len)) return nullptr;
  if (!cuda_ok(p, cudaStreamSynchronize(p->stream), "sync")) return nullptr;
  return p->in.p;
}

int jt_b200_copy_in(jt_parser *p, const void *src, size_t len) {
  DevGuard dg_(p);
  if (!jt_b200_input_buffer(p, len)) return -1;
  if (len && !cuda_ok(p, cudaMemcpyAsync(p->in.p, src, len, cudaMemcpyDefault, p->stream), "copy_in"))
    return -1;
  p->in_len = len;
  return cuda_ok(p, cudaStreamSynchronize(p->stream), "sync") ? 0 : -1;
}

// Enqueue (no wait) a copy of bytes [offset, offset + n) of a host or device
// document `src` into the same positions of the input buffer.
int jt_b200_copy_in_range(jt_parser *p, const void *src, size_t offset, size_t n) {
  DevGuard dg_(p);
  if (offset + n > p->in.cap) return -1;
  if (n && !cuda_ok(p, cudaMemcpyAsync(p->in.as<uint8_t>() + offset, (const uint8_t *)src + offset, n,
                                       cudaMemcpyDefault, p->stream),
                    "copy_in_range"))
    return -1;
  return 0;
}

jt_error jt_b200_stage1_resident(jt_parser *p, size_t len, long long *error_offset) {
  DevGuard dg_(p);
  if ((uint64_t)len >= (1ULL << 32)) {
    set_off(error_offset, -1);
    return JT_CAPACITY;
  }
  p->in_len = len;
  int which = p->cur ^ 1;
  if (!ensure_stage1(p, len, which) || !enqueue(p, len, which, false)) {
    set_off(error_offset, -1);
    return JT_CAPACITY;
  }
  return finish(p, which, false, error_offset);
}

jt_error jt_b200_parse_resident(jt_parser *p, size_t len, long long *error_offset) {
  DevGuard dg_(p);
  p->in_len = len;
  return parse_resident(p, len, nullptr, error_offset);
}

jt_error jt_b200_parse_async(jt_parser *p, size_t len) {
  DevGuard dg_(p);
  if ((uint64_t)len >= (1ULL << 32)) return JT_CAPACITY;
  p->in_len = len;
  int which = p->cur ^ 1;
  if (!ensure_stage1(p, len, which) || !ensure_stage2(p, len) || !enqueue(p, len, which, true))
    return JT_CAPACITY;
  p->pending_len = len;
  p->pending_idx = which;
  p->pending_full = true;
  return JT_OK;
}

jt_error jt_b200_stage1_async(jt_parser *p, size_t len) {
  DevGuard dg_(p);
  if ((uint64_t)len >= (1ULL << 32)) return JT_CAPACITY;
  p->in_len = len;
  int which = p->cur ^ 1;
  if (!ensure_stage1(p, len, which) || !enqueue(p, len, which, false)) return JT_CAPACITY;
  p->pending_len = len;
  p->pending_idx = which;
  p->pending_full = false;
  return JT_OK;
}

jt_error jt_b200_finish(jt_parser *p, long long *error_offset) {
  DevGuard dg_(p);
  if (p->pending_idx < 0) {
    set_off(error_offset, -1);
    return JT_CAPACITY;
  }
  int which = p->pending_idx;
  p->pending_idx = -1;
  return finish(p, which, p->pending_full, error_offset);
}

const uint32_t *jt_b200_device_index(const jt_parser *p, size_t *count) {
  DevGuard dg_(p);
  if (count) *count = jt_index_count(p);
  return p->idx[p->cur].as<uint32_t>();
}

const uint64_t *jt_b200_device_tape(const jt_parser *p, size_t *words) {
  DevGuard dg_(p);
  if (words) *words = p->last_ok ? p->last_tape_len : 0;
  return p->tape.as<uint64_t>();
}

const uint8_t *jt_b200_device_strings(const jt_parser *p, size_t *bytes) {
  DevGuard dg_(p);
  if (bytes) *bytes = p->last_ok ? p->last_string_bytes : 0;
  return p->strings.as<uint8_t>();
}

const uint64_t *jt_b200_document_tape(const jt_document *doc, size_t *words) {
  if (words) *words = doc ? doc->tape.size() : 0;
  return doc ? doc->tape.data() : nullptr;
}

const uint8_t *jt_b200_document_strings(const jt_document *doc, size_t *bytes) {
  if (bytes) *bytes = doc ? doc->strings.size() : 0;
  return doc ? doc->strings.data() : nullptr;
}

jt_document *jt_b200_document_from(const uint64_t *tape, size_t words, const uint8_t *strings, size_t bytes) {
  jt_document *d = new (std::nothrow) jt_document;
  if (!d) return nullptr;
  if (!d->alloc(words, bytes)) {
    delete d;
    return nullptr;
  }
  if (words) memcpy(d->tape.p, tape, words * 8);
  if (bytes) memcpy(d->strings.p, strings, bytes);
  return d;
}

jt_error jt_b200_download(jt_parser *p, jt_document **out) {
  DevGuard dg_(p);
  *out = nullptr;
  if (!p->last_ok) return JT_CAPACITY;
  *out = download(p);
  return *out ? JT_OK : JT_CAPACITY;
}


void jt_b200_set_stream(jt_parser *p, void *cuda_stream) {
  DevGuard dg_(p);
  p->stream = cuda_stream ? (cudaStream_t)cuda_stream : p->own_stream;
}

// ---- NDJSON records (include/jsontape_b200.h) -------------------------------

// Parse the len resident bytes as '\n'-separated records, each as jt_parse of
// the record alone would.  Waits; one host sync after the newline count.
int jt_b200_parse_records(jt_parser *p, size_t len, size_t *n_records) {
  DevGuard dg_(p);
  if (n_records) *n_records = 0;
  if ((uint64_t)len >= (1ULL << 32) || !ensure_input(p, len) || !ensure_stage1(p, len, 0) ||
      !ensure_stage2(p, len, true) ||
      !p->nlbuf.ensure(jt::stage1_records(len) * 2 * sizeof(uint32_t) + 64)) {
    p->err = "parse_records: allocation";
    return -1;
  }
  p->in_len = len;
  p->cur = 0;
  p->have_index = false;
  p->h_index_valid = false;
  p->last_ok = false;
  jt::Stage2Sizes z = jt::stage2_sizes(len + 16);
  const uint64_t s1w = jt::stage1_records(len) * 9 + 1;
  const uint64_t s2w = ((z.n3 * 4 + 64 + 63) / 64) * 8;  // m3 only (enqueue_direct)
  jt::Ctrl *ctrl = p->ctrl.as<jt::Ctrl>();
  jt::Stage1Args a1 = s1_args(p, len, 0);
  a1.records = true;
  a1.nl_count = p->nlbuf.as<uint32_t>();
  a1.nl_base = a1.nl_count + jt::stage1_records(len);
  a1.nl_total = &ctrl->n_newlines;
  if (!cuda_ok(p, jt::init_launch(ctrl, p->s1rec.as<uint64_t>(), s1w, p->s2rec.as<uint64_t>(), s2w,
                                  p->stream),
               "init") ||
      !cuda_ok(p, jt::stage1_records_count(a1, p->stream), "records count") ||
      !cuda_ok(p, cudaMemcpyAsync(p->h_ctrl, p->ctrl.p, sizeof(jt::Ctrl), cudaMemcpyDeviceToHost,
                                  p->stream),
               "ctrl D2H") ||
      (len && !cuda_ok(p, cudaMemcpyAsync(&p->rec_last_byte, p->in.as<uint8_t>() + len - 1, 1,
                                          cudaMemcpyDeviceToHost, p->stream),
                       "last byte")) ||
      !cuda_ok(p, cudaStreamSynchronize(p->stream), "sync"))
    return -1;
  const uint64_t nl = p->h_ctrl->n_newlines, nr = nl + 2;
  const size_t cap_tok = (size_t)len + 16;
  // carve: start (nr+1), kend, tend, send, utf8, serr, end_err (nr each), rec_of (cap_tok),
  // err (nr u64), results (nr)
  const size_t u32s = (nr + 1) + 6 * nr + cap_tok + 64 + 4;
  const size_t bytes = round_up(u32s * 4, 256) + nr * 8 + nr * sizeof(jt::RecordResult) + 512;
  if (!p->recs.ensure(bytes)) {
    p->err = "parse_records: record arrays";
    return -1;
  }
  uint32_t *q = p->recs.as<uint32_t>();
  a1.rec_start = q;
  q += nr + 1;
  a1.rec_kend = q;
  q += nr;
  a1.rec_tend = q;
  q += nr;
  a1.rec_send = q;
  q += nr;
  a1.rec_utf8 = q;
  q += nr;
  a1.rec_serr = q;
  q += nr;
  uint32_t *end_err = q;
  q += nr;
  q = (uint32_t *)(((uintptr_t)q + 15) & ~(uintptr_t)15);  // rec_of is read as uint4 (k_struct)
  a1.rec_of = q;
  unsigned long long *err = (unsigned long long *)(p->recs.as<uint8_t>() + round_up(u32s * 4, 256));
  jt::RecordResult *res = (jt::RecordResult *)(err + nr);
  jt::Stage2Args a2 = s2_args(p, len, 0);
  a2.records = true;
  a2.rec_of = a1.rec_of;
  a2.rec_start = a1.rec_start;
  a2.rec_kend = a1.rec_kend;
  a2.rec_tend = a1.rec_tend;
  a2.rec_send = a1.rec_send;
  a2.rec_utf8 = a1.rec_utf8;
  a2.rec_serr = a1.rec_serr;
  a2.rec_err = err;
  a2.rec_end_err = end_err;
  a2.results = res;
  int n2 = 0;
  if (!cuda_ok(p, jt::records_init_launch(a2, p->stream), "records init") ||
      !cuda_ok(p, jt::stage1_records_main(a1, p->stream), "records stage 1") ||
      !cuda_ok(p, jt::records_stage2_launch(a2, p->stream, &n2, stage2_fork(p)), "records stage 2") ||
      !cuda_ok(p, cudaMemcpyAsync(p->h_ctrl, p->ctrl.p, sizeof(jt::Ctrl), cudaMemcpyDeviceToHost,
                                  p->stream),
               "ctrl D2H") ||
      !cuda_ok(p, cudaStreamSynchronize(p->stream), "sync"))
    return -1;
  p->launches = 1 + 2 + 2 + 1 + n2;
  canary_check(p, "parse_records");
  if (p->h_ctrl->string_bytes >= (1ULL << 32) || p->h_ctrl->tape_words >= (1ULL << 32)) {
    p->err = "parse_records: string buffer or tape reaches 2^32 (u32 offsets)";
    return -1;
  }
  // the input's last byte decides whether a record follows the last '\n'
  // (read from the pinned control copy: no extra sync)
  const uint64_t n = nl + ((len > 0 && p->rec_last_byte != '\n') ? 1 : 0);
  p->rec_results = res;
  p->rec_n = n;
  p->h_records_valid = false;  // results stay on the device until asked for
  // the device tape / string buffer hold all records back to back
  p->last_tape_len = n ? p->h_ctrl->tape_words + 2 * (n - 1) + 1 : 0;
  p->last_string_bytes = p->h_ctrl->string_bytes;
  if (n_records) *n_records = n;
  return 0;
}

// host copy of the last jt_b200_parse_records results (made on first use)
const void *jt_b200_records(jt_parser *p) {
  DevGuard dg_(p);
  if (!p->h_records_valid) {
    const size_t bytes = p->rec_n * sizeof(jt::RecordResult);
    if (bytes > p->h_records_cap) {
      jt_document::release(p->h_records, p->h_records_cap, p->h_records_pinned);
      p->h_records = (jt::RecordResult *)PinnedPool::get().take(bytes, &p->h_records_cap, &p->h_records_pinned);
      if (!p->h_records) {
        p->h_records_cap = 0;
        return nullptr;
      }
    }
    if (bytes && (cudaMemcpyAsync(p->h_records, p->rec_results, bytes, cudaMemcpyDeviceToHost, p->stream) !=
                      cudaSuccess ||
                  cudaStreamSynchronize(p->stream) != cudaSuccess)) {
      cudaGetLastError();
      return nullptr;
    }
    p->h_records_valid = true;
  }
  return p->h_records;
}

// device pointer to the last jt_b200_parse_records results (jt_b200_record[n])
const void *jt_b200_device_records(const jt_parser *p) { return p->rec_results; }

// Copy all records' tape words and string bytes (jt_b200_record ranges) to host.
int jt_b200_records_download(jt_parser *p, uint64_t *tape, uint8_t *strings) {
  DevGuard dg_(p);
  if (p->last_tape_len &&
      !cuda_ok(p, cudaMemcpy(tape, p->tape.p, p->last_tape_len * 8, cudaMemcpyDeviceToHost), "tape D2H"))
    return -1;
  if (p->last_string_bytes &&
      !cuda_ok(p, cudaMemcpy(strings, p->strings.p, p->last_string_bytes, cudaMemcpyDeviceToHost),
               "strings D2H"))
    return -1;
  return 0;
}

// Sizes of the last jt_b200_parse_records output: out[0] tape words, out[1] string bytes.
void jt_b200_records_size(const jt_parser *p, unsigned long long *out) {
  DevGuard dg_(p);
  out[0] = p->last_tape_len;
  out[1] = p->last_string_bytes;
}

// ---- byte-range shards (shard.h, include/jsontape_b200.h) -------------------

size_t jt_b200_shard_summary_bytes(int phase) {
  switch (phase) {
    case 0: return sizeof(jt::Sum0);
    case 1: return sizeof(jt::Sum1);
    case 2: return sizeof(jt::Sum2);
    case 3: return sizeof(jt::Sum3);
    default: return 0;
  }
}

int jt_b200_shard_resident(jt_parser *p, size_t lo, size_t hi) {
  if (hi && lo >= hi) {
    p->err = "shard_resident: empty range";
    return -1;
  }
  p->res_lo = hi ? lo : 0;
  p->res_hi = hi;
  return 0;
}

int jt_b200_shard_begin(jt_parser *p, size_t len, unsigned g, unsigned G, size_t begin, size_t end) {
  DevGuard dg_(p);
  return shard_setup(p, len, g, G, begin, end);
}

// Enqueue phase 0..3 of this shard (shard.h).  `gathered` = device pointer
// to the G summaries of the previous phase (ignored for phase 0); this
// phase's summary goes to the device pointer `summary`.
int jt_b200_shard_phase(jt_parser *p, int phase, const void *gathered, void *summary) {
  DevGuard dg_(p);
  if (!p->shard_on || !summary || (phase > 0 && !gathered)) {
    p->err = "shard_phase: no shard or missing buffers";
    return -1;
  }
  const jt::Shard &h = *p->h_shard;
  const uint64_t len = p->shard_len, range = h.end - h.begin;
  int n = 0;
  bool ok = true;
  switch (phase) {
    case 0: {
      jt::Stage2Sizes z = jt::stage2_sizes(range + 16);
      uint64_t s1w = jt::stage1_records(range) * 9 + 1;
      uint64_t s2w = ((z.n3 * 4 + 64 + 63) / 64) * 8;  // m3 only (enqueue_direct)
      ok = cuda_ok(p, jt::init_launch(p->ctrl.as<jt::Ctrl>(), p->s1rec.as<uint64_t>(), s1w,
                                      p->s2rec.as<uint64_t>(), s2w, p->stream),
                   "init") &&
           cuda_ok(p, jt::stage1_shard_phase0(s1_args(p, len, 0, h.begin, h.end), (jt::Sum0 *)summary,
                                              p->stream),
                   "shard phase 0");
      n = 3;
      break;
    }
    case 1:
      ok = cuda_ok(p, jt::stage1_shard_phase1(s1_args(p, len, 0, h.begin, h.end),
                                              (const jt::Sum0 *)gathered, h.g, p->stream),
                   "shard phase 1") &&
           cuda_ok(p, jt::shard_sum1_launch(s2_args(p, len, 0, range, true), (jt::Sum1 *)summary, p->stream),
                   "shard sum1");
      n = 3;
      break;
    case 2:
      ok = cuda_ok(p, jt::shard_phase2_launch(s2_args(p, len, 0, range, true), (const jt::Sum1 *)gathered,
                                              (jt::Sum2 *)summary, p->stream, &n),
                   "shard phase 2");
      break;
    case 3: {
      jt::Stage2Args a = s2_args(p, len, 0, range, true);
      a.sum3 = (jt::Sum3 *)summary;
      ok = cuda_ok(p, jt::shard_phase3_launch(a, (const jt::Sum2 *)gathered, p->stream, &n),
                   "shard phase 3");
      break;
    }
    default:
      p->err = "shard_phase: phase must be 0..3";
      return -1;
  }
  p->launches = phase == 0 ? n : p->launches + n;
  return ok ? 0 : -1;
}

// Global result from the gathered phase-3 summaries; waits for the shard's
// stream.  On JT_OK this shard's tape words and string bytes stay on the
// device (jt_b200_device_tape / _strings, placed by jt_b200_shard_extent).
jt_error jt_b200_shard_finish(jt_parser *p, const void *gathered, long long *error_offset) {
  DevGuard dg_(p);
  if (!p->shard_on || !gathered) {
    set_off(error_offset, -1);
    return JT_CAPACITY;
  }
  const jt::Shard &h = *p->h_shard;
  const uint64_t range = h.end - h.begin;
  if (!cuda_ok(p, jt::shard_finish_launch(s2_args(p, p->shard_len, 0, range, true),
                                          (const jt::Sum3 *)gathered, p->stream),
               "shard finish") ||
      !cuda_ok(p, cudaMemcpyAsync(p->h_ctrl, p->ctrl.p, sizeof(jt::Ctrl), cudaMemcpyDeviceToHost,
                                  p->stream),
               "ctrl D2H") ||
      !cuda_ok(p, cudaMemcpyAsync(p->h_shard, p->shard.p, sizeof(jt::Shard), cudaMemcpyDeviceToHost,
                                  p->stream),
               "shard D2H") ||
      !cuda_ok(p, cudaStreamSynchronize(p->stream), "sync")) {
    set_off(error_offset, -1);
    return JT_CAPACITY;
  }
  p->launches += 1;
  canary_check(p, "shard_finish");
  const jt::Ctrl &c = *p->h_ctrl;
  set_off(error_offset, c.offset);
  if (c.code != jt::kUtf8Error) {
    p->have_index = true;
    p->index_count = c.S;
    p->h_index_valid = false;
  }
  p->last_ok = c.code == jt::kOk;
  return (jt_error)c.code;
}

// Where this shard's results sit in the document: out[0] = document tape
// index of local tape word out[1], out[2] = local words from there, out[3] =
// document string offset of local string byte 0, out[4] = string bytes,
// out[5] = document index of the shard's first token, out[6] = its tokens.
int jt_b200_shard_extent(const jt_parser *p, unsigned long long *out) {
  DevGuard dg_(p);
  if (!p->shard_on || !p->h_shard) return -1;
  const jt::Shard &h = *p->h_shard;
  const jt::Ctrl &c = *p->h_ctrl;
  const uint64_t lo = h.g == 0 ? 0 : 1;
  const uint64_t hi = c.tape_words + (h.is_last ? 1 : 0);  // local words [lo, hi)
  out[0] = h.tape_base + lo;
  out[1] = lo;
  out[2] = hi - lo;
  out[3] = h.string_base;
  out[4] = c.string_bytes;
  out[5] = h.token_base;
  out[6] = c.S;
  return 0;
}

// Copy this shard's tape words (extent out[2] words) and string bytes
// (out[4]) into host buffers.
int jt_b200_shard_download(jt_parser *p, uint64_t *tape, uint8_t *strings) {
  DevGuard dg_(p);
  unsigned long long e[7];
  if (jt_b200_shard_extent(p, e) != 0) return -1;
  if (e[2] && !cuda_ok(p, cudaMemcpyAsync(tape, p->tape.as<uint64_t>() + e[1], e[2] * 8,
                                          cudaMemcpyDeviceToHost, p->stream),
                       "shard tape D2H"))
    return -1;
  if (e[4] && !cuda_ok(p, cudaMemcpyAsync(strings, p->strings.p, e[4], cudaMemcpyDeviceToHost,
                                          p->stream),
                       "shard strings D2H"))
    return -1;
  return cuda_ok(p, cudaStreamSynchronize(p->stream), "sync") ? 0 : -1;
}

int jt_b200_last_launches(const jt_parser *p) { return p->launches; }

#ifdef JT_TIMELINE
// instrumented builds only: K1 per-tile timeline (16 words per tile)
int jt_b200_timeline(unsigned long long *host, size_t n) {
  return jt::stage1_timeline(host, n) == cudaSuccess ? 0 : -1;
}
#endif

void jt_b200_profile(jt_parser *p, int enable) {
  DevGuard dg_(p);
  if (enable && !p->ev[0])
    for (auto &e : p->ev) cudaEventCreate(&e);
  p->prof = enable != 0;
}

int jt_b200_kernel_times(jt_parser *p, float *ms, int max) {
  DevGuard dg_(p);
  if (!p->prof || p->prof_n == 0) return 0;
  cudaStreamSynchronize(p->stream);
  int n = 0;
  for (int k = 0; k < p->prof_n && n < max; k++, n++)
    if (cudaEventElapsedTime(&ms[n], p->ev[k], p->ev[k + 1]) != cudaSuccess) ms[n] = -1.0f;
  return n;
}

int jt_b200_device(const jt_parser *p) { return p->device; }

size_t jt_b200_device_bytes(const jt_parser *p) {
  const DevBuf *bufs[] = {&p->in, &p->idx[0], &p->idx[1], &p->aux, &p->s1rec, &p->s2rec, &p->tok,
                          &p->tape_idx, &p->m1, &p->m2, &p->mhi, &p->slow, &p->numlist, &p->scopebits,
                          &p->tile_flags, &p->tape, &p->strings, &p->ctrl, &p->shard, &p->stream_words,
                          &p->qbuf, &p->qstr, &p->rngbuf, &p->patchbuf, &p->recs, &p->nlbuf, &p->minbuf};
  size_t t = 0;
  for (const DevBuf *b : bufs) t += b->cap;
  return t;
}

const char *jt_b200_last_error(const jt_parser *p) { return p->err.c_str(); }

}  // extern "C"
