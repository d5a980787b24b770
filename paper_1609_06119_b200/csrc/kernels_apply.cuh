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

}  // namespace bb
