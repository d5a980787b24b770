// Forest apply (reference predict_batch / _score_rows / traverse_values /
// _sigmoid2, boosting.py:176-219, trees.py:333-346).
//
// One thread per row.  A CTA stages its rows' raw features in shared memory
// (coalesced tile load; the row-major matrix is read exactly once), then
// every thread walks all trees in tree order: right iff v >= threshold, a
// NaN value or an invalid node stops the walk and emits that node's weight.
// F = f0 + sum(gamma) is accumulated in float64 in tree order, so F is
// bit-identical to the reference given the same node weights.
#pragma once
#include "common.cuh"

namespace bb {

struct ApplyForest {  // device
  int n_trees, depth, n_internal, n_nodes;
  const int* feature;          // [T][I]
  const unsigned char* valid;  // [T][I]
  const double* thr;           // [T][I]
  const double* nw;            // [T][N]
  double f0;
};

constexpr int APPLY_ROWS = 128;

__device__ __forceinline__ double sigmoid2(double f) {
  if (f >= 0.0) return __ddiv_rn(1.0, __dadd_rn(1.0, exp(-2.0 * f)));
  const double e = exp(2.0 * f);
  return __ddiv_rn(e, __dadd_rn(1.0, e));
}

template <typename T>
__global__ void __launch_bounds__(APPLY_ROWS) k_apply(const T* __restrict__ X, int64_t n, int d, ApplyForest fo,
                                                      double* __restrict__ out_p, double* __restrict__ out_F) {
  extern __shared__ unsigned char s_raw[];
  T* tile = reinterpret_cast<T*>(s_raw);  // [APPLY_ROWS][d + 1]
  const int64_t row0 = (int64_t)blockIdx.x * APPLY_ROWS;
  const int rows = (int)min((int64_t)APPLY_ROWS, n - row0);
  const int ld = d + 1;
  const T* src = X + row0 * d;
  for (int e = threadIdx.x; e < rows * d; e += APPLY_ROWS) {
    const int r = e / d, f = e - r * d;
    tile[r * ld + f] = src[e];
  }
  __syncthreads();
  if ((int)threadIdx.x >= rows) return;
  const T* row = tile + threadIdx.x * ld;
  double F = fo.f0;
  for (int t = 0; t < fo.n_trees; ++t) {
    const int* ft = fo.feature + (int64_t)t * fo.n_internal;
    const unsigned char* vt = fo.valid + (int64_t)t * fo.n_internal;
    const double* tt = fo.thr + (int64_t)t * fo.n_internal;
    int nd = 0;
    for (int l = 0; l < fo.depth; ++l) {
      if (!__ldg(&vt[nd])) break;
      const double v = (double)row[__ldg(&ft[nd])];
      if (v != v) break;
      nd = 2 * nd + 1 + (v >= __ldg(&tt[nd]) ? 1 : 0);
    }
    F = __dadd_rn(F, __ldg(&fo.nw[(int64_t)t * fo.n_nodes + nd]));
  }
  const int64_t i = row0 + threadIdx.x;
  if (out_F) out_F[i] = F;
  if (out_p) out_p[i] = sigmoid2(F);
}

// ---------------------------------------------------------------- f32 path
// float32 rows: thresholds pre-rounded to the exact float ceiling (for a
// float v, v >= thr  <=>  v >= ceil_f32(thr)), packed with the feature into
// 8-byte node records (feature < 0: invalid node, stop).  A CTA stages 256
// rows and batches of kApplyTB trees in shared memory; every thread walks
// 4 trees at a time (independent node chains, ILP) and adds the node
// weights to its float64 F in tree order.
constexpr int kApplyRows = 256;
constexpr int kApplyTB = 128;
constexpr int kILP = 4;  // trees walked concurrently per thread (8 measured slower)

struct ApplyF32 {
  int n_trees, depth, n_internal, n_nodes;
  const int2* node;   // [T][I]: x = feature (or -1), y = float bits of ceil_f32(thr)
  const double* nw;   // [T][N]
  double f0;
};

__global__ void __launch_bounds__(kApplyRows) k_apply_f32(const float* __restrict__ X, int64_t n, int d, ApplyF32 fo,
                                                          double* __restrict__ out_p, double* __restrict__ out_F) {
  extern __shared__ __align__(16) unsigned char s_raw[];
  const int ld = d + 1;
  float* tile = reinterpret_cast<float*>(s_raw);  // [kApplyRows][ld]
  unsigned char* after = s_raw + ((size_t)kApplyRows * ld * 4 + 15) / 16 * 16;
  double* s_nw = reinterpret_cast<double*>(after);                                   // [TB][N]
  int2* s_node = reinterpret_cast<int2*>(s_nw + (size_t)kApplyTB * fo.n_nodes);       // [TB][I]
  const int64_t row0 = (int64_t)blockIdx.x * kApplyRows;
  const int rows = (int)min((int64_t)kApplyRows, n - row0);
  const float* src = X + row0 * d;
  for (int e = threadIdx.x; e < rows * d; e += kApplyRows) {
    const int r = e / d, f = e - r * d;
    tile[r * ld + f] = src[e];
  }
  const float* row = tile + threadIdx.x * ld;
  double F = fo.f0;
  const int I = fo.n_internal, N = fo.n_nodes, D = fo.depth;
  for (int tb = 0; tb < fo.n_trees; tb += kApplyTB) {
    const int nt = min(kApplyTB, fo.n_trees - tb);
    __syncthreads();
    for (int e = threadIdx.x; e < nt * I; e += kApplyRows) s_node[e] = fo.node[(int64_t)tb * I + e];
    for (int e = threadIdx.x; e < nt * N; e += kApplyRows) s_nw[e] = fo.nw[(int64_t)tb * N + e];
    __syncthreads();
    if ((int)threadIdx.x < rows) {
      int t = 0;
      for (; t + kILP <= nt; t += kILP) {
        int nd[kILP];
        bool live[kILP];
#pragma unroll
        for (int u = 0; u < kILP; ++u) {
          nd[u] = 0;
          live[u] = true;
        }
        for (int l = 0; l < D; ++l) {
#pragma unroll
          for (int u = 0; u < kILP; ++u) {
            const int2 rec = s_node[(t + u) * I + nd[u]];
            const bool vld = live[u] && rec.x >= 0;
            const float v = vld ? row[rec.x] : 0.0f;
            const bool go = vld && v == v;  // NaN stops at this node
            nd[u] = go ? 2 * nd[u] + 1 + (v >= __int_as_float(rec.y) ? 1 : 0) : nd[u];
            live[u] = go;
          }
        }
#pragma unroll
        for (int u = 0; u < kILP; ++u) F = __dadd_rn(F, s_nw[(t + u) * N + nd[u]]);
      }
      for (; t < nt; ++t) {
        int nd = 0;
        for (int l = 0; l < D; ++l) {
          const int2 rec = s_node[t * I + nd];
          if (rec.x < 0) break;
          const float v = row[rec.x];
          if (v != v) break;
          nd = 2 * nd + 1 + (v >= __int_as_float(rec.y) ? 1 : 0);
        }
        F = __dadd_rn(F, s_nw[t * N + nd]);
      }
    }
  }
  if ((int)threadIdx.x < rows) {
    const int64_t i = row0 + threadIdx.x;
    if (out_F) out_F[i] = F;
    if (out_p) out_p[i] = sigmoid2(F);
  }
}

// ------------------------------------------------------ f32, fixed depth
// Depth-D trees with the invalid-node stops folded into a per-tree leaf
// table: leaf l's weight is that of the first invalid node on its path (the
// walk stops there, trees.py:333-346) or of the leaf node.  The walk is then
// branch-free: D levels of (record, value, compare, child), one leaf-weight
// add per tree in tree order (float64, bit-identical F).  A row with a NaN
// feature stops where that NaN is tested, so it takes the exact per-node
// walk over the original records (global memory; rare).
constexpr int kApplyDRows = 256;
constexpr int kApplyDTB = 64;  // trees per smem batch
#ifndef BB_APPLY_ILP
#define BB_APPLY_ILP 4
#endif
constexpr int kApplyDIlp = BB_APPLY_ILP;  // trees walked together per thread

struct ApplyD {
  int n_trees;
  int t_begin, t_end;  // trees of this launch (a forest may take several launches)
  int first, last;     // first launch: F = f0; last launch: write the probabilities
  const int2* rec;    // [T][2^D - 1]: x = 4 * feature (byte offset; 0 for invalid), y = float bits of ceil_f32(thr)
  const double* leaf; // [T][2^D]
  const int2* node;   // [T][2^D - 1] original records (x = -1: invalid) for NaN rows
  const double* nw;   // [T][2^(D+1) - 1]
  double f0;
};

// root records of up to kApplyRoots trees in the kernel's parameter space:
// the root is the same for every thread of a tree, so its record comes from
// the uniform datapath (constant bank) instead of a shared-memory wavefront
constexpr int kApplyParamRecs = 3900;  // records (8 B) in the parameter space per launch
struct ApplyRoots {
  int2 r[kApplyParamRecs];  // [launch tree][the first PL levels' 2^PL - 1 records]
};

template <int D, int PL>  // PL: levels whose records come from the parameter space (0 .. 3)
__global__ void __launch_bounds__(kApplyDRows) k_apply_d(const float* __restrict__ X, int64_t n, int d, ApplyD fo,
                                                         double* __restrict__ out_p, double* __restrict__ out_F,
                                                         const __grid_constant__ ApplyRoots roots) {
  constexpr int I = (1 << D) - 1, L = 1 << D, N = (1 << (D + 1)) - 1;
  extern __shared__ __align__(16) unsigned char s_raw[];
  const int ld = d + 1;
  float* tile = reinterpret_cast<float*>(s_raw);  // [kApplyDRows][ld]
  unsigned char* after = s_raw + ((size_t)kApplyDRows * ld * 4 + 15) / 16 * 16;
  double* s_leaf = reinterpret_cast<double*>(after);                           // [TB][L]
  int2* s_rec = reinterpret_cast<int2*>(s_leaf + (size_t)kApplyDTB * L);      // [TB][I]
  const int64_t row0 = (int64_t)blockIdx.x * kApplyDRows;
  const int rows = (int)min((int64_t)kApplyDRows, n - row0);
  const float* src = X + row0 * d;
  for (int e = threadIdx.x; e < rows * d; e += kApplyDRows) {
    const int r = e / d, f = e - r * d;
    tile[r * ld + f] = src[e];
  }
  __syncthreads();
  const float* row = tile + threadIdx.x * ld;
  bool has_nan = false;
  if ((int)threadIdx.x < rows)
    for (int f = 0; f < d; ++f) has_nan |= row[f] != row[f];
  double F = fo.f0;
  if (!fo.first && (int)threadIdx.x < rows) F = out_F[row0 + threadIdx.x];  // trees before this launch
  if (has_nan) {
    // exact per-node walk (the generic rule), original records in global memory
    for (int t = fo.t_begin; t < fo.t_end; ++t) {
      int nd = 0;
      for (int l = 0; l < D; ++l) {
        const int2 rc = __ldg(&fo.node[(int64_t)t * I + nd]);
        if (rc.x < 0) break;
        const float v = row[rc.x];
        if (v != v) break;
        nd = 2 * nd + 1 + (v >= __int_as_float(rc.y) ? 1 : 0);
      }
      F = __dadd_rn(F, __ldg(&fo.nw[(int64_t)t * N + nd]));
    }
  }
  constexpr int RP = (1 << PL) - 1;  // parameter records per tree
  for (int tb = fo.t_begin; tb < fo.t_end; tb += kApplyDTB) {
    const int nt = min(kApplyDTB, fo.t_end - tb);
    __syncthreads();
    for (int e = threadIdx.x; e < nt * I; e += kApplyDRows) s_rec[e] = fo.rec[(int64_t)tb * I + e];
    for (int e = threadIdx.x; e < nt * L; e += kApplyDRows) s_leaf[e] = fo.leaf[(int64_t)tb * L + e];
    __syncthreads();
    if (has_nan || (int)threadIdx.x >= rows) continue;
    // byte offsets: records hold the feature's byte offset in the row, the
    // node index walks as off = 8 * node (child: 2 off + 8 + 8 p)
    const unsigned char* rb = reinterpret_cast<const unsigned char*>(row);
    const unsigned char* recb = reinterpret_cast<const unsigned char*>(s_rec);
    const unsigned char* leafb = reinterpret_cast<const unsigned char*>(s_leaf) - 8 * I;
    int t = 0;
    for (; t + kApplyDIlp <= nt; t += kApplyDIlp) {
      int off[kApplyDIlp];
#pragma unroll
      for (int u = 0; u < kApplyDIlp; ++u) off[u] = 0;
#pragma unroll
      for (int l = 0; l < D; ++l) {
#pragma unroll
        for (int u = 0; u < kApplyDIlp; ++u) {
          int2 rc;
          const int2* pr = roots.r + (tb - fo.t_begin + t + u) * RP;  // uniform: the same tree for all threads
          if (l < PL && l == 0) {
            rc = pr[0];
          } else if (l < PL && l == 1) {  // node 1 or 2: off = 8 or 16
            rc = off[u] == 8 ? pr[1] : pr[2];
          } else if (l < PL && l == 2) {  // nodes 3 .. 6: off = 24 .. 48
            const int2 a = off[u] & 8 ? pr[3] : pr[4];  // 24: node 3, 32: node 4
            const int2 b = off[u] & 8 ? pr[5] : pr[6];  // 40: node 5, 48: node 6
            rc = off[u] < 40 ? a : b;
          } else {
            rc = *reinterpret_cast<const int2*>(recb + (t + u) * (8 * I) + off[u]);
          }
          const float v = *reinterpret_cast<const float*>(rb + rc.x);
          off[u] = 2 * off[u] + 8 + (v >= __int_as_float(rc.y) ? 8 : 0);
        }
      }
#pragma unroll
      for (int u = 0; u < kApplyDIlp; ++u)
        F = __dadd_rn(F, *reinterpret_cast<const double*>(leafb + (t + u) * (8 * L) + off[u]));
    }
    for (; t < nt; ++t) {
      int off = 0;
#pragma unroll
      for (int l = 0; l < D; ++l) {
        const int2 rc = *reinterpret_cast<const int2*>(recb + t * (8 * I) + off);
        const float v = *reinterpret_cast<const float*>(rb + rc.x);
        off = 2 * off + 8 + (v >= __int_as_float(rc.y) ? 8 : 0);
      }
      F = __dadd_rn(F, *reinterpret_cast<const double*>(leafb + t * (8 * L) + off));
    }
  }
  if ((int)threadIdx.x < rows) {
    const int64_t i = row0 + threadIdx.x;
    if (out_F) out_F[i] = F;
    if (out_p && fo.last) out_p[i] = sigmoid2(F);
  }
}

}  // namespace bb
