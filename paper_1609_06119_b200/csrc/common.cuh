// Shared device/host helpers for the FastBDT B200 hot path.
#pragma once
#include <cstdlib>
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
// BB_SYNC_DEBUG=1: synchronise after every launch so a faulting kernel is
// reported at its own launch site (debug only)
inline bool sync_debug() {
  static const bool on = getenv("BB_SYNC_DEBUG") != nullptr;
  return on;
}
#define BB_LAUNCH_CHECK()                                   \
  do {                                                      \
    BB_CUDA(cudaGetLastError());                            \
    if (::bb::sync_debug()) BB_CUDA(cudaDeviceSynchronize()); \
  } while (0)

struct InvalidArg {
  std::string msg;
};

// Device-side bounds checks of the check build (make check: -DBB_DEVICE_CHECKS,
// libfastbdt_b200_check.so, loaded with BB_LIB_VARIANT=check); no code in
// the release build.  A failed check prints its location and traps.
#ifdef BB_DEVICE_CHECKS
#define BB_DCHECK(cond)                                                                              \
  do {                                                                                               \
    if (!(cond)) {                                                                                   \
      printf("BB_DCHECK failed: %s at %s:%d block %d thread %d\n", #cond, __FILE__, __LINE__,        \
             (int)blockIdx.x, (int)threadIdx.x);                                                     \
      __trap();                                                                                      \
    }                                                                                                \
  } while (0)
#else
#define BB_DCHECK(cond) \
  do {                  \
  } while (0)
#endif

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

// ------------------------------------------------------ TMA (bulk copy)
// 1-D cp.async.bulk global->shared completing on an mbarrier (sm_90+; SASS
// UBLKCP).  All addresses and sizes must be 16-byte multiples.
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// TMA bulk reduction shared -> global (int64 add at L2; 16-byte aligned, size a multiple of 16)
__device__ __forceinline__ void bulk_reduce_add_u64(void* gdst, const void* ssrc, unsigned bytes) {
  asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.u64 [%0], [%1], %2;" ::"l"(gdst),
               "r"(smem_u32(ssrc)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  const unsigned a = smem_u32(bar);
  unsigned ok = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!ok);
}

// 2-limb slot with the limbs in separate arrays (lo[], hi[]): consecutive
// slots fall in consecutive banks.
__device__ __forceinline__ void slot_add2(uint32_t* lo, uint32_t* hi, int s, long long q) {
  const uint32_t l = (uint32_t)(unsigned long long)q;
  uint32_t h = (uint32_t)((unsigned long long)q >> 32);
  const uint32_t old = atomicAdd(lo + s, l);
  h += (old + l < old) ? 1u : 0u;
  if (h) atomicAdd(hi + s, h);
}

// Rows of every per-row device array are padded to this multiple so that
// whole tiles can be bulk-copied.
constexpr int64_t kRowPad = 1024;

// Bin codes are stored column-major inside 1024-row tiles:
// codes[(tile * d + feature) * kTile + row % kTile].  One tile's feature group
// is one contiguous block (a single bulk copy); one feature of a tile is a
// contiguous 1024-code column (coalesced, vectorisable).
constexpr int kTileLog = 10;
constexpr int kTile = 1 << kTileLog;
__host__ __device__ __forceinline__ int64_t code_index(int64_t row, int f, int d) {
  return ((row >> kTileLog) * d + f) * (int64_t)kTile + (row & (kTile - 1));
}

// ------------------------------------------- programmatic dependent launch
// A kernel launched with cudaLaunchAttributeProgrammaticStreamSerialization
// (bb_capi.cu launch_k) may be scheduled while its predecessor in the stream
// still runs: it must call pdl_wait() before touching anything the
// predecessor wrote (no-op for a plain launch), and pdl_launch() lets its own
// successor be scheduled early in turn.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// --------------------------------------------------------------- misc
__host__ __device__ __forceinline__ int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace bb
