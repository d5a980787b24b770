// Exact subsample masks on the GPU (reference sample.py:120-132 driven by
// numpy Generator(PCG64(seed)).permutation, boosting.py:162; numpy's
// algorithm restated in bb_mask.cpp / SURVEY.md Appendix A1).
//
// Per tree, for the signal block then the background block (n rows,
// k = floor(rate*n) active): Fisher-Yates steps i = n-1 .. 1 each draw
// j = random_interval(i) from the u32 stream (rejection on the smallest
// all-ones mask >= i) and swap a[i], a[j].  The active set is
// {a[0..k)} = all values minus the k..n-1 values the steps i >= k move out.
//
//  k_pcg_draws     the u32 draw stream (low, high halves of consecutive
//                  PCG64 XSL-RR outputs), generated in parallel by LCG
//                  jump-ahead.
//  (kernels_seg.cuh assigns the draws to steps: J[i] for steps i >= k.)
//  k_bucket_*      counting sort of the steps by target position.
//  k_resolve       value moved out by step i = follow the chain of later
//                  steps that wrote its target position (see DESIGN.md
//                  §Subsample); marks it removed.
//  k_mask_bits     active bit = not removed, class-block bit order.
#pragma once
#include "common.cuh"

namespace bb {

struct U128 {
  unsigned long long lo, hi;
};

__host__ __device__ __forceinline__ U128 u128_mul(U128 a, U128 b) {
  U128 r;
#ifdef __CUDA_ARCH__
  r.lo = a.lo * b.lo;
  r.hi = __umul64hi(a.lo, b.lo) + a.lo * b.hi + a.hi * b.lo;
#else
  const unsigned __int128 x = ((unsigned __int128)a.hi << 64 | a.lo) * ((unsigned __int128)b.hi << 64 | b.lo);
  r.lo = (unsigned long long)x;
  r.hi = (unsigned long long)(x >> 64);
#endif
  return r;
}
__host__ __device__ __forceinline__ U128 u128_add(U128 a, U128 b) {
  U128 r;
  r.lo = a.lo + b.lo;
  r.hi = a.hi + b.hi + (r.lo < a.lo ? 1ull : 0ull);
  return r;
}
__host__ __device__ __forceinline__ unsigned long long xsl_rr(U128 s) {
  const unsigned long long x = s.hi ^ s.lo;
  const unsigned rot = (unsigned)(s.hi >> 58);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

// (A_m, C_m) with s_m = A_m * s + C_m, for m = 2^j, j = 0..63
struct PcgJump {
  U128 A[64], C[64];
};

// device RNG state between trees (numpy bit_generator.state layout)
struct RngState {
  U128 s, inc;
  int has_uint32;
  unsigned int uinteger;
};

__host__ __device__ __forceinline__ U128 pcg_jump(const PcgJump& J, U128 s, unsigned long long m) {
  for (int j = 0; m; ++j, m >>= 1)
    if (m & 1ull) s = u128_add(u128_mul(J.A[j], s), J.C[j]);
  return s;
}

// u32 draw number `idx` of the stream that starts at state `r`
__device__ __forceinline__ unsigned int draw_at(const PcgJump& J, const RngState& r, long long idx) {
  if (r.has_uint32) {
    if (idx == 0) return r.uinteger;
    idx -= 1;
  }
  const U128 st = pcg_jump(J, r.s, (unsigned long long)(idx >> 1) + 1ull);
  const unsigned long long o = xsl_rr(st);
  return (idx & 1) ? (unsigned int)(o >> 32) : (unsigned int)o;
}

constexpr int kDrawChunk = 64;  // PCG outputs per thread

// draws [j_lo, j_hi) of the buffer (a chunk's draws are generated in two
// parts: the first jobs' range on the critical stream, the rest overlapped).
// A warp owns 32 * kDrawChunk consecutive outputs, lane l the outputs
// l, l + 32, ...: one jump to its first output, then the 32-step LCG map
// (A_32, C_32) per output, so each warp-wide store covers 256 contiguous
// bytes of the buffer.
__global__ void k_pcg_draws(const PcgJump* __restrict__ Jp, const RngState* __restrict__ rs,
                            unsigned int* __restrict__ draws, long long j_lo, long long j_hi) {
  const RngState r = *rs;
  const long long h = r.has_uint32 ? 1 : 0;
  const long long out_lo = j_lo > h ? (j_lo - h) / 2 : 0;   // first output touching [j_lo, j_hi)
  const long long out_hi = (j_hi - h + 1) / 2;              // outputs before this cover j < j_hi
  const long long gt = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const long long wbase = out_lo + (gt >> 5) * 32 * kDrawChunk;
  if (wbase >= out_hi) return;
  if (wbase == 0 && lane == 0 && h && j_lo == 0) draws[0] = r.uinteger;
  const long long q0 = wbase + lane;
  U128 s = pcg_jump(*Jp, r.s, (unsigned long long)q0 + 1ull);  // state after output q0
  const U128 a = Jp->A[5], c = Jp->C[5];                       // 32 steps
  const long long q1 = min(out_hi, wbase + 32 * kDrawChunk);
  for (long long qq = q0; qq < q1; qq += 32) {
    const unsigned long long o = xsl_rr(s);
    const long long j = h + 2 * qq;
    if (j >= j_lo && j + 1 < j_hi && !h) {
      *reinterpret_cast<uint2*>(draws + j) = make_uint2((unsigned int)o, (unsigned int)(o >> 32));
    } else {
      if (j >= j_lo && j < j_hi) draws[j] = (unsigned int)o;
      if (j + 1 >= j_lo && j + 1 < j_hi) draws[j + 1] = (unsigned int)(o >> 32);
    }
    s = u128_add(u128_mul(a, s), c);
  }
}

__device__ __forceinline__ unsigned int smear(unsigned int x) {
  return x ? (0xffffffffu >> __clz((int)x)) : 0u;  // smallest 2^k - 1 >= x
}

// ----------------------------------------------------------- resolution
__global__ void k_bucket_count(const int* __restrict__ J, int k, int n, int* __restrict__ cnt) {
  for (int t = k + blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x)
    atomicAdd(&cnt[J[t]], 1);
}

__global__ void k_bucket_fill(const int* __restrict__ J, int k, int n, const int* __restrict__ off,
                              int* __restrict__ fill, int* __restrict__ bucket) {
  for (int t = k + blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    const int p = J[t];
    const int slot = atomicAdd(&fill[p], 1);
    bucket[off[p] + slot] = t;
  }
}

// steps targeting one position, ascending (buckets are tiny)
__global__ void k_bucket_sort(const int* __restrict__ cnt, const int* __restrict__ off, int n, int* __restrict__ bucket) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
    const int c = cnt[p];
    if (c < 2) continue;
    int* b = bucket + off[p];
    for (int x = 1; x < c; ++x) {
      const int v = b[x];
      int y = x - 1;
      while (y >= 0 && b[y] > v) {
        b[y + 1] = b[y];
        --y;
      }
      b[y + 1] = v;
    }
  }
}

// value removed by step i: V(J[i], i), following the chain of later steps
// (V(p, t) = p if no step t' > t targets p, else V(t*, t*) with
// t* = min{t' > t : J[t'] = p})
__global__ void k_resolve(const int* __restrict__ J, int k, int n, const int* __restrict__ cnt,
                          const int* __restrict__ off, const int* __restrict__ bucket,
                          unsigned char* __restrict__ removed) {
  for (int i = k + blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    int p = J[i], t = i;
    for (;;) {
      const int c = cnt[p];
      const int* b = bucket + off[p];
      int nxt = -1;
      for (int x = 0; x < c; ++x) {
        const int v = b[x];
        if (v > t) {
          nxt = v;
          break;
        }
      }
      if (nxt < 0) break;
      p = nxt;
      t = nxt;
    }
    removed[p] = 1;
  }
}

// Sort-free resolution (replaces the bucket pipeline below on the fit path).
// Follow a value instead of a step: value v starts at position v; while it
// sits at position p it is hit (moved to a final position >= k, i.e.
// removed) iff a step t targets p while it is there, and it leaves p at step
// p (to J[p]) if p >= k.  Steps run downward, so v sits at p from the step
// that brought it there (prev) down to p, and a hit exists iff
// up[p] = min{t > p : J[t] = p} < prev.  J[p] == p keeps v at p until p
// is final: removed.  A value that reaches p < k unhit stays active.
// (Equal to the chain rule of k_resolve on every case of
// tests/test_gpu_parity.py; derivation in DESIGN.md §Kernels.)
constexpr int kUpNone = 0x7f7f7f7f;  // up[] initial value (memset 0x7f): no step targets the position

__global__ void k_up_min(const int* __restrict__ J, int k, int n, int* __restrict__ up) {
  const int t0 = k > 1 ? k : 1;
  for (int t = t0 + blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    const int p = J[t];
    if (p != t) atomicMin(&up[p], t);
  }
}

__global__ void k_resolve_values(const int* __restrict__ J, int k, int n, const int* __restrict__ up,
                                 unsigned char* __restrict__ removed) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    int p = v, prev = kUpNone;  // no step before the first position: up[p] < kUpNone iff some step targets p
    unsigned char rem = 0;
    for (;;) {
      if (__ldg(&up[p]) < prev) { rem = 1; break; }
      if (p < k) break;
      const int j = __ldg(&J[p]);
      if (j == p) { rem = 1; break; }
      prev = p;
      p = j;
    }
    removed[v] = rem;
  }
}

// active bits, class-block order: bit g < n_sig -> signal value g, else
// background value g - n_sig
__global__ void k_mask_bits(const unsigned char* __restrict__ rem_sig, const unsigned char* __restrict__ rem_bkg,
                            long long n_sig, long long n, unsigned int* __restrict__ bits) {
  const long long words = (n + 31) / 32;
  for (long long w = (long long)blockIdx.x * blockDim.x + threadIdx.x; w < words;
       w += (long long)gridDim.x * blockDim.x) {
    unsigned int v = 0;
    for (int b = 0; b < 32; ++b) {
      const long long g = w * 32 + b;
      if (g >= n) break;
      const bool act = g < n_sig ? !rem_sig[g] : !rem_bkg[g - n_sig];
      v |= (act ? 1u : 0u) << b;
    }
    bits[w] = v;
  }
}

// this rank's active bits from the global class-block bits (row-sharded
// fits): local row j < n_sig_l is global signal row s0 + j, otherwise global
// background row b0 + (j - n_sig_l) at bit n_sig_g + ...
__global__ void k_mask_slice(const unsigned int* __restrict__ gbits, long long n_l, long long n_sig_l,
                             long long n_sig_g, long long s0, long long b0, unsigned int* __restrict__ bits) {
  const long long words = (n_l + 31) / 32;
  for (long long w = (long long)blockIdx.x * blockDim.x + threadIdx.x; w < words;
       w += (long long)gridDim.x * blockDim.x) {
    unsigned int v = 0;
    for (int b = 0; b < 32; ++b) {
      const long long j = w * 32 + b;
      if (j >= n_l) break;
      const long long g = j < n_sig_l ? s0 + j : n_sig_g + b0 + (j - n_sig_l);
      v |= ((gbits[g >> 5] >> (g & 31)) & 1u) << b;
    }
    bits[w] = v;
  }
}

// --------------------------------------------------------------- scan
// exclusive scan of n ints: per-block sums, single-CTA scan of the sums,
// per-block exclusive scan with the carried offset
constexpr int kScanBlock = 1024;  // elements per block (256 threads x 4)

__global__ void k_scan_block_sums(const int* __restrict__ in, int n, int* __restrict__ sums) {
  __shared__ int s[8];
  const int base = blockIdx.x * kScanBlock;
  int v = 0;
  for (int j = threadIdx.x; j < kScanBlock; j += blockDim.x)
    if (base + j < n) v += in[base + j];
  v = __reduce_add_sync(0xffffffffu, v);
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s[w];
    sums[blockIdx.x] = t;
  }
}

__global__ void k_scan_sums(int* __restrict__ sums, int nb) {
  // single CTA, sequential chunks of blockDim
  __shared__ int carry;
  __shared__ int ws[32];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < nb; base += blockDim.x) {
    const int i = base + threadIdx.x;
    const int v = i < nb ? sums[i] : 0;
    int incl = v;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if ((threadIdx.x & 31) >= o) incl += y;
    }
    if ((threadIdx.x & 31) == 31) ws[threadIdx.x >> 5] = incl;
    __syncthreads();
    if (threadIdx.x < 32) {
      int w = threadIdx.x < (int)(blockDim.x >> 5) ? ws[threadIdx.x] : 0;
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, w, o);
        if (threadIdx.x >= o) w += y;
      }
      ws[threadIdx.x] = w;
    }
    __syncthreads();
    const int excl = carry + ((threadIdx.x >= 32) ? ws[(threadIdx.x >> 5) - 1] : 0) + incl - v;
    __syncthreads();
    if (i < nb) sums[i] = excl;
    if (threadIdx.x == blockDim.x - 1) carry = excl + v;
    __syncthreads();
  }
}

// also clears the bucket fill cursors and the removed flags of the same
// positions (saves two memsets per class block and tree on the host)
__global__ void k_scan_apply(const int* __restrict__ in, int n, const int* __restrict__ sums, int* __restrict__ out,
                             int* __restrict__ fill_zero, unsigned char* __restrict__ removed_zero) {
  __shared__ int ws[8];
  const int base = blockIdx.x * kScanBlock;
  const int t = threadIdx.x;  // 256 threads, 4 consecutive elements each
  int v[4], loc = 0;
  for (int j = 0; j < 4; ++j) {
    const int i = base + t * 4 + j;
    v[j] = i < n ? in[i] : 0;
    loc += v[j];
  }
  int incl = loc;
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if ((t & 31) >= o) incl += y;
  }
  if ((t & 31) == 31) ws[t >> 5] = incl;
  __syncthreads();
  int woff = 0;
  for (int w = 0; w < (t >> 5); ++w) woff += ws[w];
  int run = sums[blockIdx.x] + woff + incl - loc;
  for (int j = 0; j < 4; ++j) {
    const int i = base + t * 4 + j;
    if (i < n) {
      out[i] = run;
      fill_zero[i] = 0;
      removed_zero[i] = 0;
    }
    run += v[j];
  }
}

}  // namespace bb
