// Equal-frequency binning on the GPU (reference binning.py:52-79,
// sample.py:79-117).
//
//  1. k_transpose_keys  row-major X (f32|f64) -> column-major order-preserving
//                       keys [d][n]; NaN -> key 0; per-feature finite / NaN
//                       counts (M_f for the target ranks).
//  2. k_select_hist /   MSD radix SELECT of the B-1 order statistics
//     k_select_scan     sorted_finite[floor(k*M/B)] per feature: each pass
//                       histograms one digit of the keys that still share a
//                       prefix with some target, then every target picks its
//                       digit.  Exact: the boundary is the key itself.
//  3. k_class_*         stable signal|background partition positions (the
//                       reference's class blocks, sample.py:112-116).
//  4. k_codes           code = 1 + #{boundaries <= v} (searchsorted right),
//                       NaN -> 0, written column-major in class-block order.
#pragma once
#include "common.cuh"

namespace bb {

// ---------------------------------------------------------------- 1
template <typename T>
__global__ void k_transpose_keys(const T* __restrict__ X, int64_t n, int d,
                                 typename KeyOf<T>::K* __restrict__ keys,  // [d][n]
                                 unsigned long long* __restrict__ finite_cnt,
                                 unsigned long long* __restrict__ nan_cnt) {
  using K = typename KeyOf<T>::K;
  // tile: 32 rows x 32 features through shared memory
  __shared__ K tile[32][33];
  __shared__ unsigned int s_fin[32], s_nan[32];
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  const int64_t row0 = (int64_t)blockIdx.x * 32;
  const int f0 = blockIdx.y * 32;
  if (ty == 0) { s_fin[tx] = 0; s_nan[tx] = 0; }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int64_t row = row0 + r;
    const int f = f0 + tx;
    K k = 0;
    if (row < n && f < d) {
      const T v = X[row * d + f];
      if (KeyOf<T>::isnan_(v)) {
        k = 0;
        atomicAdd(&s_nan[tx], 1u);
      } else {
        k = KeyOf<T>::key(v);
        if (KeyOf<T>::finite(v)) atomicAdd(&s_fin[tx], 1u);
      }
    }
    tile[r][tx] = k;
  }
  __syncthreads();
  for (int c = ty; c < 32; c += 8) {
    const int f = f0 + c;
    const int64_t row = row0 + tx;
    if (f < d && row < n) keys[(int64_t)f * n + row] = tile[tx][c];
  }
  if (ty == 0 && f0 + tx < d) {
    if (s_fin[tx]) atomicAdd(&finite_cnt[f0 + tx], (unsigned long long)s_fin[tx]);
    if (s_nan[tx]) atomicAdd(&nan_cnt[f0 + tx], (unsigned long long)s_nan[tx]);
  }
}

// ---------------------------------------------------------------- 2
// Per-feature selection state (targets are the B-1 boundary ranks, sorted,
// so their prefixes are non-decreasing and groups are contiguous runs).
template <typename K>
struct SelectState {
  K* tgt_prefix;          // [d][nt]   resolved high bits of each target key
  unsigned long long* tgt_rank;  // [d][nt] residual rank within its prefix group
  int* tgt_group;         // [d][nt]   group index of the target
  K* grp_prefix;          // [d][nt]   distinct prefixes (sorted)
  int* grp_count;         // [d]       number of groups
  int* grp_first_tgt;     // [d][nt]   first target of each group
  unsigned int* hist;     // [d][hist_cap]
  const unsigned long long* finite_cnt;  // [d]
  int nt;                 // B - 1
  int64_t hist_cap;       // counters per feature
};

template <typename K>
__global__ void k_select_init(SelectState<K> st, int B) {
  const int f = blockIdx.x;
  const unsigned long long M = st.finite_cnt[f];
  for (int t = threadIdx.x; t < st.nt; t += blockDim.x) {
    const int64_t o = (int64_t)f * st.nt + t;
    st.tgt_prefix[o] = 0;
    // rank floor(k*M/B), k = t+1 (binning.py:69-70)
    st.tgt_rank[o] = (unsigned long long)(((unsigned __int128)(t + 1) * M) / (unsigned)B);
    st.tgt_group[o] = 0;
  }
  if (threadIdx.x == 0) {
    st.grp_count[f] = 1;
    st.grp_prefix[(int64_t)f * st.nt] = 0;
    st.grp_first_tgt[(int64_t)f * st.nt] = 0;
  }
}

// 16-bit hash of a group prefix for k_select_hist's membership filter
template <typename K>
__device__ __forceinline__ unsigned int select_filter_hash(K pre) {
  unsigned int x = (unsigned int)pre;
  if (sizeof(K) == 8) x ^= (unsigned int)((unsigned long long)pre >> 32) * 0x85EBCA6Bu;
  return (x * 0x9E3779B1u) >> 16;
}

// Histogram one digit.  resolved = number of high key bits already fixed
// for every group; db = digit bits this pass.
template <typename K>
__global__ void __launch_bounds__(256) k_select_hist(const K* __restrict__ keys, int64_t n, SelectState<K> st,
                                                     int resolved, int db, int smem_bins) {
  extern __shared__ unsigned int s_hist[];
  constexpr int KB = sizeof(K) * 8;
  const int f = blockIdx.y;
  const int ng = st.grp_count[f];
  if (st.finite_cnt[f] == 0) return;
  const K* col = keys + (int64_t)f * n;
  const K* gp = st.grp_prefix + (int64_t)f * st.nt;
  unsigned int* gh = st.hist + (int64_t)f * st.hist_cap;
  const int nbins = ng << db;
  const bool use_smem = nbins <= smem_bins;
  if (use_smem) {
    for (int i = threadIdx.x; i < nbins; i += blockDim.x) s_hist[i] = 0;
    __syncthreads();
  }
  const K kneg = (K)~(K)0 >> 1;  // not used; placeholder for clarity
  (void)kneg;
  // finite keys lie strictly between key(-inf) and key(+inf)
  K key_ninf, key_pinf;
  if (KB == 32) {
    key_ninf = (K)(~0xFF800000u);
    key_pinf = (K)0xFF800000u;
  } else {
    key_ninf = (K)(~0xFFF0000000000000ull);
    key_pinf = (K)0xFFF0000000000000ull;
  }
  const unsigned int dmask = (1u << db) - 1u;
  // Group lookup.  Up to 12 resolved bits: an exact bitmap of the groups'
  // prefixes, the group index is the prefix's rank among the set bits (groups
  // are sorted by prefix).  Beyond: a 64K-bit one-hash filter rejects the keys
  // of no group (from the third pass on > 99 % of a column: only the target
  // order statistics' buckets are refined) before the binary search.
  __shared__ unsigned int s_bm[2048];
  __shared__ int s_pre[128];
  const bool exact = resolved > 0 && resolved <= 12;
  if (resolved > 0) {
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) s_bm[i] = 0u;
    __syncthreads();
    for (int i = threadIdx.x; i < ng; i += blockDim.x) {
      const K pre = __ldg(&gp[i]);
      const unsigned int h = exact ? (unsigned int)pre : select_filter_hash<K>(pre);
      atomicOr(&s_bm[h >> 5], 1u << (h & 31));
    }
    __syncthreads();
    if (exact && threadIdx.x < 128) {
      int c = 0;
      for (int w = 0; w < (int)threadIdx.x; ++w) c += __popc(s_bm[w]);
      s_pre[threadIdx.x] = c;
    }
    __syncthreads();
  }
  // kSelU keys per thread and round, loaded before any is processed: one
  // 4-byte load in flight per thread bounds a full-occupancy SM at ~10 GB/s
  // (measured 0.8 TB/s per pass on the whole GPU before)
  constexpr int kSelU = 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31;
  for (int64_t w0 = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); w0 < n; w0 += kSelU * stride) {
    K kk[kSelU];
#pragma unroll
    for (int u = 0; u < kSelU; ++u) {
      const int64_t i = w0 + u * stride + lane;
      kk[u] = i < n ? col[i] : key_pinf;  // out of range: treated as non-finite (no group)
    }
#pragma unroll
    for (int u = 0; u < kSelU; ++u) {
      if (w0 + u * stride >= n) break;  // warp-uniform
      const K k = kk[u];
      int g = -1;
      if (k > key_ninf && k < key_pinf) {
        if (resolved == 0) {
          g = 0;
        } else if (exact) {
          const unsigned int pre = (unsigned int)(k >> (KB - resolved));
          const unsigned int w = s_bm[pre >> 5], b = pre & 31u;
          if ((w >> b) & 1u) g = s_pre[pre >> 5] + __popc(w & ((1u << b) - 1u));
        } else {
          const K pre = k >> (KB - resolved);
          const unsigned int h = select_filter_hash<K>(pre);
          if ((s_bm[h >> 5] >> (h & 31)) & 1u) {
            int lo = 0, hi = ng - 1;
            while (lo < hi) {
              const int mid = (lo + hi) >> 1;
              if (__ldg(&gp[mid]) < pre) lo = mid + 1; else hi = mid;
            }
            if (__ldg(&gp[lo]) == pre) g = lo;
          }
        }
      }
      const unsigned int digit = (g >= 0) ? (unsigned int)((k >> (KB - resolved - db)) & dmask) : 0u;
      const int bin = (g >= 0) ? (g << db) + (int)digit : -1;
      // warp aggregation of equal bins (heavy ties: discrete features)
      if (__any_sync(0xffffffffu, bin >= 0)) {
        const unsigned int peers = __match_any_sync(0xffffffffu, bin);
        const int leader = __ffs(peers) - 1;
        if (bin >= 0 && lane == leader) {
          const unsigned int c = __popc(peers);
          if (use_smem) atomicAdd(&s_hist[bin], c); else atomicAdd(&gh[bin], c);
        }
      }
    }
  }
  if (use_smem) {
    __syncthreads();
    for (int i = threadIdx.x; i < nbins; i += blockDim.x)
      if (s_hist[i]) atomicAdd(&gh[i], s_hist[i]);
  }
}

// One CTA per feature: every target picks its digit, then groups are rebuilt
// from the distinct new prefixes.  One warp scans one group's histogram.
template <typename K>
__global__ void __launch_bounds__(1024) k_select_scan(SelectState<K> st, int db) {
  const int f = blockIdx.x;
  if (st.finite_cnt[f] == 0) return;
  const int nt = st.nt;
  const int ng = st.grp_count[f];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  unsigned int* gh = st.hist + (int64_t)f * st.hist_cap;
  K* tp = st.tgt_prefix + (int64_t)f * nt;
  unsigned long long* tr = st.tgt_rank + (int64_t)f * nt;
  int* tg = st.tgt_group + (int64_t)f * nt;
  const int* gft = st.grp_first_tgt + (int64_t)f * nt;
  const int nbins = 1 << db;
  const int per_lane = (nbins + 31) / 32;  // <= 128
  // lane owns bins [lane*per_lane, (lane+1)*per_lane), summed in sub-blocks
  // of kSub bins (offsets kept in registers); each lane then resolves its own
  // target per round of 32 (owner lane by a shuffle search over the lanes'
  // inclusive sums, then the sub-block, then <= kSub bins walked in global).
  constexpr int kSub = 16, kMaxSub = 8;  // per_lane <= 128
  const int nsub = (per_lane + kSub - 1) / kSub;
  for (int g = warp; g < ng; g += nwarps) {
    const unsigned int* h = gh + ((int64_t)g << db);
    const int lb = lane * per_lane;
    const int le = min(nbins, lb + per_lane);
    unsigned long long sub_excl[kMaxSub];
    unsigned long long local = 0;
#pragma unroll
    for (int sb = 0; sb < kMaxSub; ++sb) {
      sub_excl[sb] = local;
      if (sb < nsub) {
        unsigned long long ss = 0;
        for (int j = 0; j < kSub; ++j) {
          const int b = lb + sb * kSub + j;
          if (sb * kSub + j < per_lane && b < le) ss += h[b];
        }
        local += ss;
      }
    }
    unsigned long long incl = local;
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const unsigned long long excl = incl - local;
    const int t_begin = gft[g];
    const int t_end = (g + 1 < ng) ? gft[g + 1] : nt;
    for (int tb = t_begin; tb < t_end; tb += 32) {
      const int t = tb + lane;
      const bool act = t < t_end;
      const unsigned long long r = act ? tr[t] : ~0ull;
      // owner = first lane whose inclusive sum exceeds r
      int owner = 0;
      for (int step = 16; step >= 1; step >>= 1) {
        const unsigned long long v = __shfl_sync(0xffffffffu, incl, min(31, owner + step - 1));
        if (owner + step <= 32 && v <= r) owner += step;
      }
      if (__shfl_sync(0xffffffffu, incl, owner) <= r) owner = 32;  // r past every bin: no digit
      const int src = min(owner, 31);
      const unsigned long long oe = __shfl_sync(0xffffffffu, excl, src);
      const unsigned long long rin = r - oe;
      int sidx = 0;
      unsigned long long se_sel = 0;
#pragma unroll
      for (int sb = 0; sb < kMaxSub; ++sb) {
        const unsigned long long se = __shfl_sync(0xffffffffu, sub_excl[sb], src);
        if (sb < nsub && se <= rin) { sidx = sb; se_sel = se; }
      }
      if (act && owner < 32) {
        unsigned long long c = rin - se_sel;
        const int ob = owner * per_lane;
        const int oend = min(nbins, ob + per_lane);
        int b = ob + sidx * kSub;
        for (; b < oend - 1; ++b) {
          const unsigned long long hb = h[b];
          if (c < hb) break;
          c -= hb;
        }
        tr[t] = c;
        tp[t] = (tp[t] << db) | (K)b;
      }
    }
  }
  __syncthreads();
  // rebuild groups: a target starts a group when its prefix differs from the
  // previous one (block-wide ballot scan, blockDim.x targets per round)
  __shared__ int s_wcnt[32];
  __shared__ int s_carry;
  {
    K* gp = st.grp_prefix + (int64_t)f * nt;
    int* gf = st.grp_first_tgt + (int64_t)f * nt;
    int carry = 0;
    for (int base = 0; base < nt; base += blockDim.x) {
      const int t = base + threadIdx.x;
      const bool flag = t < nt && (t == 0 || tp[t] != tp[t - 1]);
      const unsigned int bal = __ballot_sync(0xffffffffu, flag);
      if (lane == 0) s_wcnt[warp] = __popc(bal);
      __syncthreads();
      int before = carry;
      for (int w = 0; w < warp; ++w) before += s_wcnt[w];
      const int idx = before + __popc(bal & ((2u << lane) - 1u));  // inclusive count
      if (t < nt) {
        tg[t] = idx - 1;
        if (flag) {
          gp[idx - 1] = tp[t];
          gf[idx - 1] = t;
        }
      }
      if (threadIdx.x == blockDim.x - 1) s_carry = idx;
      __syncthreads();
      carry = s_carry;
      __syncthreads();
    }
    if (threadIdx.x == 0) st.grp_count[f] = carry;
  }
  // zero the histogram rows this pass used (next pass reuses the buffer)
  const int64_t used = (int64_t)ng << db;
  for (int64_t i = threadIdx.x; i < used; i += blockDim.x) gh[i] = 0;
}

// boundaries (double) and boundary keys from the resolved target keys.
// All-non-finite feature: the zero placeholder (boosting.py:146-155).
template <typename K>
__global__ void k_select_finish(SelectState<K> st, double* __restrict__ bounds, K* __restrict__ bkeys) {
  const int f = blockIdx.x;
  const bool empty = st.finite_cnt[f] == 0;
  for (int t = threadIdx.x; t < st.nt; t += blockDim.x) {
    const int64_t o = (int64_t)f * st.nt + t;
    if (empty) {
      bounds[o] = 0.0;
      bkeys[o] = (sizeof(K) == 4) ? (K)f32_key(0.0f) : (K)f64_key(0.0);
    } else {
      const K k = st.tgt_prefix[o];
      bkeys[o] = k;
      bounds[o] = key_to_double(k);
    }
  }
}

// ---------------------------------------------------------------- 3
// Stable class partition: pos[i] = rank among same-class rows (+ n_sig for
// background), tiles of CLS_TILE rows.
constexpr int CLS_TILE = 2048;

__global__ void k_class_tile_counts(const int8_t* __restrict__ y, int64_t n, int* __restrict__ tile_sig) {
  __shared__ int s;
  if (threadIdx.x == 0) s = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * CLS_TILE;
  int c = 0;
  for (int j = threadIdx.x; j < CLS_TILE; j += blockDim.x) {
    const int64_t i = base + j;
    if (i < n && y[i] > 0) ++c;
  }
  c = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0) atomicAdd(&s, c);
  __syncthreads();
  if (threadIdx.x == 0) tile_sig[blockIdx.x] = s;
}

// single CTA exclusive scan over tiles; tile_sig[n_tiles] = total
__global__ void k_class_scan(int* __restrict__ tile_sig, int n_tiles) {
  __shared__ long long s_carry;
  __shared__ int s_warp[32];
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (int base = 0; base < n_tiles; base += blockDim.x) {
    const int i = base + threadIdx.x;
    const int v = (i < n_tiles) ? tile_sig[i] : 0;
    int incl = v;
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, incl, o);
      if ((threadIdx.x & 31) >= o) incl += u;
    }
    if ((threadIdx.x & 31) == 31) s_warp[threadIdx.x >> 5] = incl;
    __syncthreads();
    if (threadIdx.x < 32) {
      int w = (threadIdx.x < (int)(blockDim.x >> 5)) ? s_warp[threadIdx.x] : 0;
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, w, o);
        if (threadIdx.x >= o) w += u;
      }
      s_warp[threadIdx.x] = w;
    }
    __syncthreads();
    const int warp_off = (threadIdx.x >= 32) ? s_warp[(threadIdx.x >> 5) - 1] : 0;
    const long long excl = s_carry + warp_off + incl - v;
    __syncthreads();
    if (i < n_tiles) tile_sig[i] = (int)excl;
    if (threadIdx.x == blockDim.x - 1) s_carry = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) tile_sig[n_tiles] = (int)s_carry;
}

// pos[i] for every row, plus per-row state in class-block order
__global__ void k_class_positions(const int8_t* __restrict__ y, int64_t n, const int* __restrict__ tile_sig,
                                  int* __restrict__ pos, const double* __restrict__ w_in, double* __restrict__ w_cb) {
  __shared__ int s_warp[32];
  const int64_t base = (int64_t)blockIdx.x * CLS_TILE;
  const int n_sig = tile_sig[gridDim.x];
  int carry = tile_sig[blockIdx.x];
  const int per = CLS_TILE / blockDim.x;  // rows per thread, contiguous
  int flags[8];
  int cnt = 0;
  for (int j = 0; j < per; ++j) {
    const int64_t i = base + (int64_t)threadIdx.x * per + j;
    flags[j] = (i < n && y[i] > 0) ? 1 : 0;
    cnt += flags[j];
  }
  int incl = cnt;
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, incl, o);
    if ((threadIdx.x & 31) >= o) incl += u;
  }
  if ((threadIdx.x & 31) == 31) s_warp[threadIdx.x >> 5] = incl;
  __syncthreads();
  if (threadIdx.x < 32) {
    int w = (threadIdx.x < (int)(blockDim.x >> 5)) ? s_warp[threadIdx.x] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, w, o);
      if (threadIdx.x >= o) w += u;
    }
    s_warp[threadIdx.x] = w;
  }
  __syncthreads();
  int sig_before = carry + ((threadIdx.x >= 32) ? s_warp[(threadIdx.x >> 5) - 1] : 0) + incl - cnt;
  for (int j = 0; j < per; ++j) {
    const int64_t i = base + (int64_t)threadIdx.x * per + j;
    if (i >= n) break;
    int p;
    if (flags[j]) {
      p = sig_before++;
    } else {
      p = n_sig + (int)(i - sig_before);
    }
    pos[i] = p;
    if (w_cb) w_cb[p] = w_in ? w_in[i] : 1.0;
  }
}

// ---------------------------------------------------------------- 4
// codes[code_index(pos[i], f)] = stored code; stored = code - code_off
// (code_off = 1 only for NaN-free data at B = 256 with u8 storage).
// tiled = 0 writes plain column-major [f][code_stride] (bb_bin parity entry).
constexpr int64_t kCodesSmemMax = 200 * 1024;
template <typename K>
__host__ inline size_t codes_smem(int nt) {
  const int64_t b = (int64_t)nt * (int64_t)sizeof(K);
  return b <= kCodesSmemMax ? (size_t)b : 0;
}

template <typename K, typename CodeT>
__global__ void __launch_bounds__(256) k_codes(const K* __restrict__ keys, int64_t n, int nt,
                                               const K* __restrict__ bkeys, const int* __restrict__ pos,
                                               CodeT* __restrict__ codes, int64_t code_stride, int code_off,
                                               int d, int tiled) {
  extern __shared__ unsigned char s_raw[];
  const int f = blockIdx.y;
  const K* bk = bkeys + (int64_t)f * nt;
  // boundary keys in shared memory, or (binning_levels 15 with f64 keys:
  // 256 KB) searched in global memory through the cache
  const bool in_smem = (int64_t)nt * (int64_t)sizeof(K) <= kCodesSmemMax;
  K* sb = in_smem ? reinterpret_cast<K*>(s_raw) : const_cast<K*>(bk);
  if (in_smem) {
    for (int t = threadIdx.x; t < nt; t += blockDim.x) sb[t] = bk[t];
    __syncthreads();
  }
  const K* col = keys + (int64_t)f * n;
  // kCodeU rows per thread and round: their key / position loads are issued
  // together and the upper-bound searches (fixed step count, branch-free) run
  // in lockstep, so several memory and shared-memory latencies overlap
  constexpr int kCodeU = 4;
  int top = 1;
  while (top <= nt) top <<= 1;  // smallest power of two > nt
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += kCodeU * stride) {
    K kk[kCodeU];
    int64_t pp[kCodeU];
    int lo[kCodeU];
#pragma unroll
    for (int u = 0; u < kCodeU; ++u) {
      const int64_t i = i0 + u * stride;
      kk[u] = i < n ? col[i] : (K)0;
      pp[u] = i < n ? (int64_t)pos[i] : -1;
      lo[u] = 0;
    }
    // upper_bound: number of boundary keys <= k
    for (int step = top >> 1; step >= 1; step >>= 1) {
#pragma unroll
      for (int u = 0; u < kCodeU; ++u) {
        const int m = lo[u] + step - 1;
        if (m < nt && sb[m] <= kk[u]) lo[u] += step;
      }
    }
#pragma unroll
    for (int u = 0; u < kCodeU; ++u) {
      if (pp[u] < 0) continue;
      const int code = kk[u] == 0 ? 0 : lo[u] + 1;  // key 0: NaN
      codes[tiled ? code_index(pp[u], f, d) : (int64_t)f * code_stride + pp[u]] = (CodeT)(code - code_off);
    }
  }
}

}  // namespace bb
