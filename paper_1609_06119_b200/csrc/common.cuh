// Shared device/host helpers for the FastBDT B200 hot path.
#pragma once
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <cuda_runtime.h>

namespace bb {

// ---------------------------------------------------------------- errors
void set_error(const std::string& msg);
struct CudaError {
  std::string msg;
};
#define BB_CUDA(call)                                                                   \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess)                                                              \
      throw ::bb::CudaError{std::string(#call) + ": " + cudaGetErrorString(e_) + " (" + \
                            __FILE__ + ":" + std::to_string(__LINE__) + ")"};           \
  } while (0)
#define BB_LAUNCH_CHECK() BB_CUDA(cudaGetLastError())

struct InvalidArg {
  std::string msg;
};

// ---------------------------------------------------------------- keys
// Order-preserving unsigned keys for IEEE floats.  -0.0 is canonicalised to
// +0.0 so equal-comparing values share a key (np.sort/np.searchsorted treat
// them as equal).
__host__ __device__ __forceinline__ uint32_t f32_key(float v) {
  uint32_t b;
#ifdef __CUDA_ARCH__
  b = __float_as_uint(v);
#else
  memcpy(&b, &v, 4);
#endif
  if (b == 0x80000000u) b = 0u;
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__host__ __device__ __forceinline__ uint64_t f64_key(double v) {
  uint64_t b;
#ifdef __CUDA_ARCH__
  b = (uint64_t)__double_as_longlong(v);
#else
  memcpy(&b, &v, 8);
#endif
  if (b == 0x8000000000000000ull) b = 0ull;
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
__host__ __device__ __forceinline__ double key_to_double(uint32_t k) {
  uint32_t b = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
  float f;
#ifdef __CUDA_ARCH__
  f = __uint_as_float(b);
#else
  memcpy(&f, &b, 4);
#endif
  return (double)f;
}
__host__ __device__ __forceinline__ double key_to_double(uint64_t k) {
  uint64_t b = (k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k;
  double f;
#ifdef __CUDA_ARCH__
  f = __longlong_as_double((long long)b);
#else
  memcpy(&f, &b, 8);
#endif
  return f;
}

template <typename T>
struct KeyOf;
template <>
struct KeyOf<float> {
  using K = uint32_t;
  static constexpr int BITS = 32;
  __device__ __forceinline__ static K key(float v) { return f32_key(v); }
  __device__ __forceinline__ static bool finite(float v) {
    return (__float_as_uint(v) & 0x7f800000u) != 0x7f800000u;
  }
  __device__ __forceinline__ static bool isnan_(float v) { return v != v; }
};
template <>
struct KeyOf<double> {
  using K = uint64_t;
  static constexpr int BITS = 64;
  __device__ __forceinline__ static K key(double v) { return f64_key(v); }
  __device__ __forceinline__ static bool finite(double v) {
    return ((uint64_t)__double_as_longlong(v) & 0x7ff0000000000000ull) != 0x7ff0000000000000ull;
  }
  __device__ __forceinline__ static bool isnan_(double v) { return v != v; }
};

// ------------------------------------------------------ fixed-point slots
// An int64 fixed-point accumulator held in shared memory as two u32 limbs
// (lo, hi).  sm_100a has native 32-bit shared atomics only (u64 shared
// atomics are CAS loops, measured 2.6x slower: profiles/r01_microbench_*).
// The lo limb is added with a returning ATOMS.ADD; an unsigned wrap carries
// into hi.  The slot value is (hi:lo) mod 2^64, exact for any sign.
__device__ __forceinline__ void slot_add(uint32_t* slot, long long q) {
  const uint32_t lo = (uint32_t)(unsigned long long)q;
  uint32_t hi = (uint32_t)((unsigned long long)q >> 32);
  const uint32_t old = atomicAdd(slot, lo);
  hi += (old + lo < old) ? 1u : 0u;
  if (hi) atomicAdd(slot + 1, hi);
}
__device__ __forceinline__ long long slot_value(const uint32_t* slot) {
  return (long long)(((unsigned long long)slot[1] << 32) | (unsigned long long)slot[0]);
}

__device__ __forceinline__ unsigned long long as_ull(long long v) { return (unsigned long long)v; }

// --------------------------------------------------------------- misc
__host__ __device__ __forceinline__ int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace bb
