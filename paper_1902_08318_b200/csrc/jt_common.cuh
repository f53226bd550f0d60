// jt_common.cuh — shared device/host helpers for the B200 JSON parse path.
//
// Everything here is __host__ __device__ so the per-block bit algebra can be
// exercised on the CPU (tests/cpu_block_check.cpp) with the exact same code
// the sm_100a kernels run.
#pragma once

#include <stdint.h>

#if defined(__CUDACC__)
#define JT_HD __host__ __device__ __forceinline__
#define JT_D __device__ __forceinline__
#else
#define JT_HD inline
#define JT_D inline
#endif

namespace jt {

// tape tags (proj/src/tape.h:14-26) and word layout (tape.h:28-34)
constexpr uint8_t kTagRoot = 'r';
constexpr uint64_t kPayloadMask = (1ULL << 56) - 1;
constexpr int kMaxDepth = 1024;  // proj/src/tape_builder.cpp:12

JT_HD uint64_t tape_word(uint8_t tag, uint64_t payload) {
  return ((uint64_t)tag << 56) | (payload & kPayloadMask);
}

// error codes, numbering of jt_error (proj/include/jsontape.h:15-24)
enum : int {
  kOk = 0,
  kUtf8Error = 1,
  kStringError = 2,
  kNumberError = 3,
  kTapeError = 4,
  kDepthError = 5,
  kCapacity = 6,
  kEmpty = 7
};

JT_HD int popc64(uint64_t v) {
#if defined(__CUDA_ARCH__)
  return __popcll(v);
#else
  return __builtin_popcountll(v);
#endif
}

JT_HD int popc32(uint32_t v) {
#if defined(__CUDA_ARCH__)
  return __popc(v);
#else
  return __builtin_popcount(v);
#endif
}

// count leading zeros, 64 for 0
JT_HD int clz64(uint64_t v) {
#if defined(__CUDA_ARCH__)
  return __clzll((long long)v);
#else
  return v ? __builtin_clzll(v) : 64;
#endif
}

// count trailing zeros, 64 for 0
JT_HD int ctz64(uint64_t v) {
#if defined(__CUDA_ARCH__)
  return v ? __ffsll((long long)v) - 1 : 64;
#else
  return v ? __builtin_ctzll(v) : 64;
#endif
}

JT_HD int ctz32(uint32_t v) {
#if defined(__CUDA_ARCH__)
  return v ? __ffs((int)v) - 1 : 32;
#else
  return v ? __builtin_ctz(v) : 32;
#endif
}

// PRMT: byte i of the result = byte sel.nibble[i] (0..7) of {lo = a, hi = b}
JT_HD uint32_t byte_perm(uint32_t a, uint32_t b, uint32_t sel) {
#if defined(__CUDA_ARCH__)
  return __byte_perm(a, b, sel);
#else
  uint64_t x = ((uint64_t)b << 32) | a;
  uint32_t r = 0;
  for (int i = 0; i < 4; i++) {
    uint32_t s = (sel >> (4 * i)) & 7;
    r |= (uint32_t)((x >> (8 * s)) & 0xFF) << (8 * i);
  }
  return r;
#endif
}

// bit select: mask bits from a, the others from b (one LOP3, LUT 0xE4; spelled
// in PTX because the compiler otherwise re-associates the shifted operand's
// masks into extra instructions)
JT_HD uint32_t bit_select(uint32_t a, uint32_t b, uint32_t mask) {
#if defined(__CUDA_ARCH__)
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(r) : "r"(a), "r"(b), "r"(mask));
  return r;
#else
  return (a & mask) | (b & ~mask);
#endif
}

}  // namespace jt
