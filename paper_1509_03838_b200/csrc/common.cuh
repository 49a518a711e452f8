// common.cuh -- shared helpers for the sm_100a numerical-entanglement kernels.
//
// Integer semantics follow the reference (two's complement, MSB-truncating
// left shift, arithmetic right shift).  All wrapping arithmetic
// is done on unsigned types so nothing relies on signed-overflow UB.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/nent_b200.h"

#define NENT_MAX_STREAMS 64

namespace nent {

// Row pointer table passed by value (kernel parameter space, constant bank).
struct Rows {
  const void* p[NENT_MAX_STREAMS];
};
struct MutRows {
  void* p[NENT_MAX_STREAMS];
};

void set_error(const char* fmt, ...);

inline Rows to_rows(const void* const* p, int k) {
  Rows r{};
  for (int i = 0; i < k; ++i) r.p[i] = p ? p[i] : nullptr;
  return r;
}
inline MutRows to_mrows(void* const* p, int k) {
  MutRows r{};
  for (int i = 0; i < k; ++i) r.p[i] = p ? p[i] : nullptr;
  return r;
}
int check_launch(const char* what);
// the convolution kernel the calling host thread launched last
// (nent_last_conv_kernel): 1 CUDA-core, 2 mma.sync, 3 tcgen05, 4 tcgen05 fused m = 3
void note_conv_kernel(int k);
// Dynamic shared memory opt-in of `kern` on the current device, done once
// per (device, kernel) and size (thread-safe): NENT_OK or NENT_ERR_CUDA.
int ensure_smem(const void* kern, size_t bytes);
// SM count of the current device when it is an sm_100 part, else -1
// (cached per device ordinal).
int sm100_sms();

__device__ __forceinline__ int64_t wshl(int64_t x, int s) { return (int64_t)((uint64_t)x << s); }
__device__ __forceinline__ int64_t wadd(int64_t a, int64_t b) { return (int64_t)((uint64_t)a + (uint64_t)b); }
__device__ __forceinline__ int64_t wsub(int64_t a, int64_t b) { return (int64_t)((uint64_t)a - (uint64_t)b); }
__device__ __forceinline__ int64_t wmul(int64_t a, int64_t b) { return (int64_t)((uint64_t)a * (uint64_t)b); }
__device__ __forceinline__ int64_t wneg(int64_t a) { return (int64_t)(0 - (uint64_t)a); }

// |x| with numpy's wrap (|INT64_MIN| == INT64_MIN, so it never exceeds hi).
__device__ __forceinline__ int64_t wabs(int64_t x) { return x < 0 ? wneg(x) : x; }
// exact |x| as unsigned (for bounds)
__device__ __forceinline__ uint64_t uabs(int64_t x) { return x < 0 ? 0 - (uint64_t)x : (uint64_t)x; }

template <typename T>
__device__ __forceinline__ int64_t ld(const void* base, int64_t i) {
  return (int64_t)__ldg(reinterpret_cast<const T*>(base) + i);
}
__device__ __forceinline__ int64_t ld_bits(const void* base, int bits, int64_t i) {
  return bits == 32 ? ld<int32_t>(base, i) : ld<int64_t>(base, i);
}
__device__ __forceinline__ void st_bits(void* base, int bits, int64_t i, int64_t v) {
  if (bits == 32)
    reinterpret_cast<int32_t*>(base)[i] = (int32_t)(uint32_t)(uint64_t)v;
  else
    reinterpret_cast<int64_t*>(base)[i] = v;
}

// Warp-aggregated min of a 64-bit index into *dst (used for "first offender").
__device__ __forceinline__ void atomic_min_u64(unsigned long long* dst, unsigned long long v) {
  atomicMin(dst, v);
}

inline int grid_for(int64_t work, int threads, int per_thread, int max_blocks = 148 * 32) {
  int64_t b = (work + (int64_t)threads * per_thread - 1) / ((int64_t)threads * per_thread);
  if (b < 1) b = 1;
  if (b > max_blocks) b = max_blocks;
  return (int)b;
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

}  // namespace nent

#define DISPATCH_IO(ib, ob, ...)                                                           \
  do {                                                                                     \
    if ((ib) == 32 && (ob) == 32) { typedef int32_t TI; typedef int32_t TO; __VA_ARGS__; } \
    else if ((ib) == 32) { typedef int32_t TI; typedef int64_t TO; __VA_ARGS__; }          \
    else if ((ob) == 32) { typedef int64_t TI; typedef int32_t TO; __VA_ARGS__; }          \
    else { typedef int64_t TI; typedef int64_t TO; __VA_ARGS__; }                          \
  } while (0)

#define NENT_CHECK_BITS(b)                                        \
  do {                                                            \
    if ((b) != 32 && (b) != 64) {                                 \
      nent::set_error("element width must be 32 or 64, got %d", (int)(b)); \
      return NENT_ERR_PARAM;                                      \
    }                                                             \
  } while (0)
