// Weighted ROC AUC on the device (reference pkg/src/binboost/analysis.py:45-70):
// the weighted probability that a signal row outscores a background row,
// ties counting one half.
//
//   1. keys = order-preserving u64 of the f64 scores (common.cuh f64_key;
//      -0.0 == +0.0), payload = row index; LSD radix sort, 4-bit digits
//      (16 stable passes: per-tile digit counts, one digit-major scan over the
//      tiles, stable scatter ranked by a block scan of per-thread counts).
//   2. in sorted order: signal and background weight prefix sums (f64) and
//      the first index of every run of equal keys (max-scan of run starts).
//   3. every run's last row adds S_run * (B_before + B_run / 2); the sum over
//      runs divided by W_sig * W_bkg is the AUC.
// The reference groups by np.unique and sums with bincount / cumsum / np.sum;
// the device sums differ only in rounding order (tests compare at 1e-12).
#pragma once
#include "common.cuh"

namespace bb {

constexpr int kAucTile = 4096;        // elements per radix tile
constexpr int kAucThreads = 256;      // 16 contiguous elements per thread
constexpr int kAucPer = kAucTile / kAucThreads;
constexpr int kAucDigits = 16;        // 4-bit digits

__global__ void k_auc_keys(const double* __restrict__ s, int64_t n, unsigned long long* __restrict__ key,
                           unsigned int* __restrict__ idx) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    key[i] = f64_key(s[i]);
    idx[i] = (unsigned int)i;
  }
}

// per-tile digit counts, digit-major: cnt[digit * tiles + tile]
__global__ void __launch_bounds__(kAucThreads) k_radix_count(const unsigned long long* __restrict__ key, int64_t n,
                                                             int shift, int tiles, unsigned int* __restrict__ cnt) {
  __shared__ unsigned int h[kAucDigits];
  if (threadIdx.x < kAucDigits) h[threadIdx.x] = 0;
  __syncthreads();
  const int64_t t0 = (int64_t)blockIdx.x * kAucTile;
  for (int k = threadIdx.x; k < kAucTile; k += kAucThreads) {
    const int64_t i = t0 + k;
    if (i < n) atomicAdd(&h[(key[i] >> shift) & 15u], 1u);
  }
  __syncthreads();
  if (threadIdx.x < kAucDigits) cnt[(int64_t)threadIdx.x * tiles + blockIdx.x] = h[threadIdx.x];
}

// exclusive scan of m counts in place (one block)
__global__ void __launch_bounds__(1024) k_radix_scan(unsigned int* __restrict__ cnt, int m) {
  __shared__ unsigned int part[1024];
  const int per = (m + 1023) / 1024;
  const int a = threadIdx.x * per, b = min(m, a + per);
  unsigned int s = 0;
  for (int i = a; i < b; ++i) s += cnt[i];
  part[threadIdx.x] = s;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    const unsigned int v = threadIdx.x >= o ? part[threadIdx.x - o] : 0u;
    __syncthreads();
    part[threadIdx.x] += v;
    __syncthreads();
  }
  unsigned int run = part[threadIdx.x] - s;
  for (int i = a; i < b; ++i) {
    const unsigned int c = cnt[i];
    cnt[i] = run;
    run += c;
  }
}

// stable scatter of one tile: thread t owns elements [16t, 16t + 16)
__global__ void __launch_bounds__(kAucThreads) k_radix_scatter(const unsigned long long* __restrict__ kin,
                                                               const unsigned int* __restrict__ vin, int64_t n,
                                                               int shift, int tiles,
                                                               const unsigned int* __restrict__ off,
                                                               unsigned long long* __restrict__ kout,
                                                               unsigned int* __restrict__ vout) {
  __shared__ unsigned int r[kAucDigits * kAucThreads];  // [digit][thread] -> exclusive rank base
  __shared__ unsigned int tot[kAucThreads];
  const int t = threadIdx.x;
  const int64_t e0 = (int64_t)blockIdx.x * kAucTile + (int64_t)t * kAucPer;
  unsigned int c[kAucDigits];
#pragma unroll
  for (int q = 0; q < kAucDigits; ++q) c[q] = 0;
  unsigned long long kk[kAucPer];
#pragma unroll
  for (int j = 0; j < kAucPer; ++j) {
    const int64_t i = e0 + j;
    kk[j] = i < n ? kin[i] : 0ull;
    if (i < n) {
      const int dg = (int)((kk[j] >> shift) & 15u);
#pragma unroll
      for (int q = 0; q < kAucDigits; ++q) c[q] += (dg == q);
    }
  }
#pragma unroll
  for (int q = 0; q < kAucDigits; ++q) r[q * kAucThreads + t] = c[q];
  __syncthreads();
  // block-wide exclusive scan over the digit-major [digit][thread] array:
  // thread t scans 16 consecutive entries, then a scan of the 256 chunk sums
  unsigned int s = 0;
#pragma unroll
  for (int q = 0; q < kAucDigits; ++q) s += r[t * kAucDigits + q];
  tot[t] = s;
  __syncthreads();
  for (int o = 1; o < kAucThreads; o <<= 1) {
    const unsigned int v = t >= o ? tot[t - o] : 0u;
    __syncthreads();
    tot[t] += v;
    __syncthreads();
  }
  unsigned int run = tot[t] - s;
#pragma unroll
  for (int q = 0; q < kAucDigits; ++q) {
    const unsigned int x = r[t * kAucDigits + q];
    r[t * kAucDigits + q] = run;
    run += x;
  }
  __syncthreads();
  // rank of (digit q, thread t) inside the tile = r[q][t] - (elements of smaller digits)
  unsigned int base[kAucDigits];
#pragma unroll
  for (int q = 0; q < kAucDigits; ++q)
    base[q] = off[(int64_t)q * tiles + blockIdx.x] + r[q * kAucThreads + t] - r[q * kAucThreads];
#pragma unroll
  for (int j = 0; j < kAucPer; ++j) {
    const int64_t i = e0 + j;
    if (i >= n) break;
    const int dg = (int)((kk[j] >> shift) & 15u);
    unsigned int pos = 0;
#pragma unroll
    for (int q = 0; q < kAucDigits; ++q)
      if (dg == q) pos = base[q]++;
    BB_DCHECK(pos < (unsigned int)n);
    kout[pos] = kk[j];
    vout[pos] = vin[i];
  }
}

// sorted order: signal / background weights, run-start flags
__global__ void k_auc_prep(const unsigned long long* __restrict__ key, const unsigned int* __restrict__ idx,
                           const signed char* __restrict__ y01, const double* __restrict__ w, int64_t n,
                           double* __restrict__ sw, double* __restrict__ bw, long long* __restrict__ start) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned int r = idx[i];
    const double wi = w ? w[r] : 1.0;
    const bool sig = y01[r] > 0;
    sw[i] = sig ? wi : 0.0;
    bw[i] = sig ? 0.0 : wi;
    start[i] = (i == 0 || key[i] != key[i - 1]) ? (long long)i : -1ll;
  }
}

// block-level inclusive scans (sum for f64, max for int64), three phases
template <typename T, bool MAX>
__device__ __forceinline__ T scan_op(T a, T b) {
  if (MAX) return a > b ? a : b;
  return a + b;
}
template <typename T, bool MAX>
__global__ void __launch_bounds__(1024) k_scan_tiles(T* __restrict__ a, int64_t n, T* __restrict__ sums, T ident) {
  __shared__ T sh[1024];
  const int64_t i = (int64_t)blockIdx.x * 1024 + threadIdx.x;
  T v = i < n ? a[i] : ident;
  sh[threadIdx.x] = v;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    const T u = threadIdx.x >= o ? sh[threadIdx.x - o] : ident;
    __syncthreads();
    sh[threadIdx.x] = scan_op<T, MAX>(sh[threadIdx.x], u);
    __syncthreads();
  }
  if (i < n) a[i] = sh[threadIdx.x];
  if (threadIdx.x == 1023) sums[blockIdx.x] = sh[1023];
}
template <typename T, bool MAX>
__global__ void __launch_bounds__(1024) k_scan_sums_serial(T* __restrict__ sums, int m, T ident) {
  // exclusive scan of the tile totals (one block, sequential chunks)
  __shared__ T part[1024];
  const int per = (m + 1023) / 1024;
  const int a = threadIdx.x * per, b = min(m, a + per);
  T s = ident;
  for (int i = a; i < b; ++i) s = scan_op<T, MAX>(s, sums[i]);
  part[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    T run = ident;
    for (int k = 0; k < 1024; ++k) {
      const T x = part[k];
      part[k] = run;
      run = scan_op<T, MAX>(run, x);
    }
  }
  __syncthreads();
  T run = part[threadIdx.x];
  for (int i = a; i < b; ++i) {
    const T x = sums[i];
    sums[i] = run;
    run = scan_op<T, MAX>(run, x);
  }
}
template <typename T, bool MAX>
__global__ void k_scan_add(T* __restrict__ a, int64_t n, const T* __restrict__ sums) {
  const int64_t i = (int64_t)blockIdx.x * 1024 + threadIdx.x;
  if (i < n && blockIdx.x > 0) a[i] = scan_op<T, MAX>(sums[blockIdx.x], a[i]);
}

// the last row of every run adds S_run * (B_before + B_run / 2); per-block
// partial sums (deterministic tree reduction)
__global__ void __launch_bounds__(256) k_auc_terms(const unsigned long long* __restrict__ key, const double* __restrict__ S,
                                                   const double* __restrict__ Bc, const long long* __restrict__ start,
                                                   int64_t n, double* __restrict__ part) {
  __shared__ double sh[256];
  double acc = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x; i < n; i += (int64_t)gridDim.x * 256) {
    if (i == n - 1 || key[i] != key[i + 1]) {
      const long long s0 = start[i];
      const double s_prev = s0 > 0 ? S[s0 - 1] : 0.0, b_prev = s0 > 0 ? Bc[s0 - 1] : 0.0;
      const double s_run = S[i] - s_prev, b_run = Bc[i] - b_prev;
      acc += s_run * (b_prev + 0.5 * b_run);
    }
  }
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

}  // namespace bb
