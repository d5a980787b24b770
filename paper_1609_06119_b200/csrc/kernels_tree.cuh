// Per-tree kernels of the boosting loop (reference trees.py:139-315,
// boosting.py:109-114,165-171).  Data layout in HBM:
//   codes  [d][stride]   u8|u16 bin codes, column-major, class-block row order
//   node   [n]           u8|u16 heap node id of every row
//   q      [n]           int64 fixed-point effective weight, 0 when inactive
//   F, w   [n]           float64 score, user weight (w may be absent = 1.0)
//   mask   [n/32]        u32 active bits of the current tree
//   hist   [2][nodes][d][B]  int64 per-layer (class, node, feature, code-1)
#pragma once
#include "common.cuh"

namespace bb {

struct TreeArrays {  // device, all trees
  int* feature;      // [T][I]
  int* cut;          // [T][I]
  unsigned char* valid;
  double* gain;
  double* thr;
  double* nw;        // [T][N] shrunk node weights
  double* pur;       // [T][N]
  const int* forced; // [T][I] -2: free, -1: forced invalid, else f*65536+cut
};

__device__ __forceinline__ int row_label(int64_t i, int64_t n_sig) { return i < n_sig ? 1 : -1; }

// r = 2y*expit(-2yF) = (2y) * (1/(1+exp(2yF)))  (boosting.py:109-114; expit
// is 1/(1+exp(-x)) bit-for-bit).  Explicit _rn intrinsics keep
// the compiler from contracting into FMAs.
__device__ __forceinline__ double residual_of(double F, int lab) {
  const double two_y = 2.0 * (double)lab;
  const double e = exp(__dmul_rn(two_y, F));
  const double s = __ddiv_rn(1.0, __dadd_rn(1.0, e));
  return __dmul_rn(two_y, s);
}
__device__ __forceinline__ double boost_weight_of(double r) {
  const double a = fabs(r);
  return __dmul_rn(a, __dsub_rn(2.0, a));
}

__global__ void k_fill_f64(double* __restrict__ a, int64_t n, double v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) a[i] = v;
}
__global__ void k_iota(int* __restrict__ a, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) a[i] = (int)i;
}

// In-place exclusive scan of 64 counters in shared memory by one warp (two
// per lane); returns the total to every lane.
__device__ __forceinline__ int warp_excl_scan_64(int* a, int lane) {
  const int x0 = a[2 * lane], x1 = a[2 * lane + 1];
  int incl = x0 + x1;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  const int excl = incl - (x0 + x1);
  a[2 * lane] = excl;
  a[2 * lane + 1] = excl + x0;
  return __shfl_sync(0xffffffffu, incl, 31);
}

// ---------------------------------------------------------------- refresh
// F += gamma_prev[node] (score update of the previous tree, all rows), then
// responses, boost weights and the quantised effective weight of tree t.
// Row lists are appended per CTA tile: entries are ranked per key in shared
// memory, one global atomic per (tile, key) reserves their block (a global
// counter per key hit by every warp serialises at L2: 5x slower at cfg3).
constexpr int kListTileRows = 2048;  // rows per CTA tile (512 threads x 4)
constexpr int kListThreads = 512;
static_assert(kListTileRows / kListThreads * (kListThreads / 32) == 64, "warp_excl_scan_64: 64 (row group, warp) counters");
constexpr int kStageNodes = 127;     // staged refresh walk: internal nodes (depth <= 7)

// Leaf of row i in tree `tree` over its bin codes (trees.py:318-330): an
// invalid node or a missing code stops the walk.
template <typename CodeT>
__device__ __forceinline__ int walk_leaf(const CodeT* __restrict__ codes, int d, int code_off, int64_t i,
                                         const TreeArrays& ta, int tree, int n_internal, int depth) {
  int nd = 0;
  for (int l = 0; l < depth; ++l) {
    const int64_t e = (int64_t)tree * n_internal + nd;
    if (!__ldg(&ta.valid[e])) break;
    const int c = (int)codes[code_index(i, __ldg(&ta.feature[e]), d)] + code_off;
    if (c == 0) break;
    nd = 2 * nd + 1 + (c > __ldg(&ta.cut[e]) ? 1 : 0);
  }
  return nd;
}

template <typename CodeT, typename NodeT>
__global__ void k_walk_leaves(const CodeT* __restrict__ codes, int d, int code_off, int64_t n, TreeArrays ta, int tree,
                              int n_internal, int depth, NodeT* __restrict__ node) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    node[i] = (NodeT)walk_leaf(codes, d, code_off, i, ta, tree, n_internal, depth);
}

// walk_tree >= 0 (row-list fits): the previous tree's leaf of every row is
// found by walking that tree over the codes (no per-row node ids are kept);
// otherwise it is node[i].
template <typename NodeT, typename CodeT>
__global__ void __launch_bounds__(kListThreads, 3) k_update_refresh(int64_t n, int64_t n_sig, double* __restrict__ F,
                                                                NodeT* __restrict__ node, const double* __restrict__ w,
                                                                long long* __restrict__ q,
                                                                const unsigned int* __restrict__ mask,
                                                                const double* __restrict__ nw_prev, double two_s,
                                                                int* __restrict__ cnt, int* __restrict__ lrow,
                                                                long long* __restrict__ lq,
                                                                const CodeT* __restrict__ codes, int d, int code_off,
                                                                TreeArrays ta, int walk_tree, int n_internal,
                                                                int depth, int stage_slots) {
  __shared__ int s_base[2];
  constexpr int R = kListTileRows / kListThreads;
  __shared__ int s_wc[2 * R * (kListThreads / 32)];  // per (class, row group, warp): count, then rank base
  // staged walk (stage_slots > 0, n_internal <= kStageNodes): the code columns
  // of the previous tree's distinct cut features are copied into shared
  // memory per tile with coalesced 16-byte loads, and every row walks the tree
  // there.  The gather walk below spends ~58 instructions and one dependent
  // global load per level and row (cfg3: 247 us per tree, issue-bound).
  extern __shared__ __align__(16) unsigned char s_cols[];  // [slot][kListTileRows] codes
  __shared__ int s_rec[kStageNodes];    // node -> (slot << 16) | cut, -1: the walk stops
  __shared__ int s_feat[kStageNodes];   // slot -> feature; scratch: node -> owner node
  __shared__ int s_nslots;
  const bool staged = stage_slots > 0 && nw_prev && walk_tree >= 0;
  pdl_wait();
  pdl_launch();
  if (staged) {
    const int64_t e0 = (int64_t)walk_tree * n_internal;
    const int me = threadIdx.x;
    int f = -1, cut = 0, owner = -1;
    if (me < n_internal && __ldg(&ta.valid[e0 + me])) {
      f = __ldg(&ta.feature[e0 + me]);
      cut = __ldg(&ta.cut[e0 + me]);
      owner = me;  // the first valid node with this feature owns its slot
      for (int j = 0; j < me; ++j)
        if (__ldg(&ta.valid[e0 + j]) && __ldg(&ta.feature[e0 + j]) == f) {
          owner = j;
          break;
        }
    }
    if (me < n_internal) s_feat[me] = owner;
    __syncthreads();
    int slot = 0;
    if (me < n_internal && owner >= 0)
      for (int j = 0; j < owner; ++j) slot += (s_feat[j] == j);
    if (me == 0) {
      int c = 0;
      for (int j = 0; j < n_internal; ++j) c += (s_feat[j] == j);
      s_nslots = c;
    }
    __syncthreads();
    if (me < n_internal) {
      s_rec[me] = owner >= 0 ? ((slot << 16) | cut) : -1;
      if (owner == me) s_feat[slot] = f;
    }
    __syncthreads();
  }
  const bool gather_rec = !staged && nw_prev && walk_tree >= 0 && n_internal <= kStageNodes;
  if (gather_rec) {
    if ((int)threadIdx.x < n_internal) {
      const int64_t e = (int64_t)walk_tree * n_internal + threadIdx.x;
      s_rec[threadIdx.x] = __ldg(&ta.valid[e]) ? ((__ldg(&ta.feature[e]) << 16) | __ldg(&ta.cut[e])) : -1;
    }
    __syncthreads();
  }
  const int64_t code_tiles = (n + kTile - 1) >> kTileLog;
  for (int64_t t0 = (int64_t)blockIdx.x * kListTileRows; t0 < n; t0 += (int64_t)gridDim.x * kListTileRows) {
    int loc[R];
    long long qs[R];
    double fr[R], wr[R];
    unsigned mw[R];
#pragma unroll
    for (int k = 0; k < R; ++k) {  // loads first: their latencies overlap
      const int64_t i = t0 + k * kListThreads + threadIdx.x;
      const bool in = i < n;
      fr[k] = in ? F[i] : 0.0;
      wr[k] = (in && w) ? w[i] : 1.0;
      mw[k] = in ? mask[i >> 5] : 0u;
    }
    if (staged) {
      constexpr int kVecPerCol = kTile * (int)sizeof(CodeT) / 16;               // 16-byte vectors per code-tile column
      constexpr int kColsPerTile = kListTileRows / kTile;                        // code tiles per CTA tile
      const int64_t T0 = t0 >> kTileLog;
      // thread -> (vector v of code-tile column h); the slot advances by a
      // constant per round (kListThreads is a multiple of the vectors per slot)
      constexpr int kVecPerSlot = kVecPerCol * kColsPerTile;
      static_assert(kListThreads % kVecPerSlot == 0 || kVecPerSlot % kListThreads == 0, "staging map");
      if (kListThreads >= kVecPerSlot) {
        constexpr int kSlotStep = kListThreads / kVecPerSlot > 0 ? kListThreads / kVecPerSlot : 1;
        const int v = threadIdx.x % kVecPerCol, h = (threadIdx.x / kVecPerCol) % kColsPerTile;
        if (T0 + h < code_tiles) {
          const uint4* col0 = reinterpret_cast<const uint4*>(codes + (T0 + h) * d * (int64_t)kTile) + v;
          uint4* dst0 = reinterpret_cast<uint4*>(s_cols) + h * kVecPerCol + v;
          const int ns = s_nslots;
          for (int sl = threadIdx.x / kVecPerSlot; sl < ns; sl += kSlotStep)
            dst0[sl * kVecPerSlot] = __ldg(col0 + s_feat[sl] * (kTile * (int)sizeof(CodeT) / 16));
        }
      } else {
        const int nvec = s_nslots * kVecPerSlot;
        for (int idx = threadIdx.x; idx < nvec; idx += kListThreads) {
          const int v = idx % kVecPerCol, h = (idx / kVecPerCol) % kColsPerTile, sl = idx / kVecPerSlot;
          if (T0 + h >= code_tiles) continue;
          const uint4* src = reinterpret_cast<const uint4*>(codes + ((T0 + h) * d + s_feat[sl]) * (int64_t)kTile) + v;
          reinterpret_cast<uint4*>(s_cols)[(sl * kColsPerTile + h) * kVecPerCol + v] = __ldg(src);
        }
      }
      __syncthreads();
      const CodeT* sc = reinterpret_cast<const CodeT*>(s_cols);
      {
        // the R rows' walks in lockstep (branch-free: a stopped row keeps its
        // node), so the shared-memory latencies of a level overlap
        int nd[R];
        bool live[R];
#pragma unroll
        for (int k = 0; k < R; ++k) {
          nd[k] = 0;
          live[k] = true;
        }
        for (int l = 0; l < depth; ++l) {
#pragma unroll
          for (int k = 0; k < R; ++k) {
            const int r = k * kListThreads + threadIdx.x;
            const int rec = s_rec[nd[k]];
            const int c = (int)sc[(max(rec, 0) >> 16) * kListTileRows + r] + code_off;
            live[k] = live[k] && rec >= 0 && c != 0;
            nd[k] = live[k] ? 2 * nd[k] + 1 + (c > (rec & 0xffff) ? 1 : 0) : nd[k];
          }
        }
#pragma unroll
        for (int k = 0; k < R; ++k) {
          const int64_t i = t0 + k * kListThreads + threadIdx.x;
          if (i < n) {
            fr[k] = __dadd_rn(fr[k], nw_prev[nd[k]]);
            F[i] = fr[k];
          }
        }
      }
      // s_cols is rewritten only after the list phase's barriers (or, without
      // lists, after the barrier below)
      if (!lrow) __syncthreads();
    } else if (gather_rec) {
      // gather walk over packed node records in shared memory (feature << 16 |
      // cut): the R rows in lockstep, branch-free, one global code per level
      int nd[R];
      bool live[R];
      int64_t base[R];
#pragma unroll
      for (int k = 0; k < R; ++k) {
        const int64_t i = t0 + k * kListThreads + threadIdx.x;
        nd[k] = 0;
        live[k] = i < n;
        base[k] = (i >> kTileLog) * d * (int64_t)kTile + (i & (kTile - 1));
      }
      for (int l = 0; l < depth; ++l) {
#pragma unroll
        for (int k = 0; k < R; ++k) {
          const int rec = s_rec[nd[k]];
          live[k] = live[k] && rec >= 0;
          const int c = live[k] ? (int)codes[base[k] + (int64_t)(rec >> 16) * kTile] + code_off : 0;
          live[k] = live[k] && c != 0;
          nd[k] = live[k] ? 2 * nd[k] + 1 + (c > (rec & 0xffff) ? 1 : 0) : nd[k];
        }
      }
#pragma unroll
      for (int k = 0; k < R; ++k) {
        const int64_t i = t0 + k * kListThreads + threadIdx.x;
        if (i < n) {
          fr[k] = __dadd_rn(fr[k], nw_prev[nd[k]]);
          F[i] = fr[k];
        }
      }
    } else if (nw_prev && walk_tree >= 0) {
      // the R rows' walks in lockstep: independent gather chains overlap
      int nd[R];
      bool live[R];
#pragma unroll
      for (int k = 0; k < R; ++k) {
        nd[k] = 0;
        live[k] = t0 + k * kListThreads + threadIdx.x < n;
      }
      for (int l = 0; l < depth; ++l) {
#pragma unroll
        for (int k = 0; k < R; ++k) {
          if (!live[k]) continue;
          const int64_t i = t0 + k * kListThreads + threadIdx.x;
          const int64_t e = (int64_t)walk_tree * n_internal + nd[k];
          if (!__ldg(&ta.valid[e])) { live[k] = false; continue; }
          const int c = (int)codes[code_index(i, __ldg(&ta.feature[e]), d)] + code_off;
          if (c == 0) { live[k] = false; continue; }
          nd[k] = 2 * nd[k] + 1 + (c > __ldg(&ta.cut[e]) ? 1 : 0);
        }
      }
#pragma unroll
      for (int k = 0; k < R; ++k) {
        const int64_t i = t0 + k * kListThreads + threadIdx.x;
        if (i < n) {
          fr[k] = __dadd_rn(fr[k], nw_prev[nd[k]]);
          F[i] = fr[k];
        }
      }
    } else if (nw_prev) {
#pragma unroll
      for (int k = 0; k < R; ++k) {
        const int64_t i = t0 + k * kListThreads + threadIdx.x;
        if (i < n) {
          fr[k] = __dadd_rn(fr[k], nw_prev[node[i]]);
          F[i] = fr[k];
        }
      }
    }
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const int64_t i = t0 + k * kListThreads + threadIdx.x;
      loc[k] = -1;
      qs[k] = 0;
      if (i < n) {
        const int lab = row_label(i, n_sig);
        const double r = residual_of(fr[k], lab);
        const double bw = boost_weight_of(r);
        const bool act = (mw[k] >> (i & 31)) & 1u;
        const long long qv = act ? __double2ll_rn(__dmul_rn(__dmul_rn(wr[k], bw), two_s)) : 0ll;
        // row-list fits keep q in the lists; q[] then holds the active rows'
        // fixed-point RESPONSE rint(w r 2^S), read by k_advance_list when a row
        // reaches its final node (trees.py:231-244) instead of a second exp
        q[i] = !lrow ? qv : (act ? __double2ll_rn(__dmul_rn(__dmul_rn(wr[k], r), two_s)) : 0ll);
        if (walk_tree < 0) node[i] = 0;
        qs[k] = qv;
        if (lrow && act) loc[k] = i < n_sig ? 0 : 1;  // class, ranked below
      }
      // layer-1 row lists (kernels_hist_list.cuh): class regions [0, n_sig),
      // [n_sig, n).  Ranks follow the row order inside the tile (per (row
      // group k, warp) counts, scanned in that order), so a list is sorted
      // by row within each tile block and the histogram's row gathers stream
      if (lrow) {
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, cls = loc[k];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const unsigned m = __ballot_sync(0xffffffffu, cls == c);
          if (lane == 0) s_wc[(c * R + k) * (kListThreads / 32) + warp] = __popc(m);
          if (cls == c) loc[k] = (c << 30) | __popc(m & ((1u << lane) - 1u));
        }
      }
    }
    if (!lrow) continue;
    __syncthreads();
    if (threadIdx.x < 64) {  // warp c: exclusive scan of class c's (k, warp) counts in row order
      const int c = threadIdx.x >> 5;
      const int run = warp_excl_scan_64(s_wc + c * R * (kListThreads / 32), threadIdx.x & 31);
      if ((threadIdx.x & 31) == 0) s_base[c] = run ? atomicAdd(cnt + c, run) : 0;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < R; ++k)
      if (loc[k] >= 0) {
        const int c = loc[k] >> 30;
        loc[k] += s_wc[(c * R + k) * (kListThreads / 32) + (threadIdx.x >> 5)];
      }
#pragma unroll
    for (int k = 0; k < R; ++k) {
      if (loc[k] < 0) continue;
      const int64_t i = t0 + k * kListThreads + threadIdx.x;
      const int c = loc[k] >> 30;
      const int64_t pos = (c ? n_sig : 0) + s_base[c] + (loc[k] & 0x3fffffff);
      BB_DCHECK(pos >= 0 && pos < (c ? n : n_sig));
      lrow[pos] = (int)i;
      lq[pos] = qs[k];
    }
    __syncthreads();
  }
}

// final score update only (after the last tree, optional)
template <typename NodeT>
__global__ void k_update_scores(int64_t n, double* __restrict__ F, const NodeT* __restrict__ node,
                                const double* __restrict__ nw) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    F[i] = __dadd_rn(F[i], nw[node[i]]);
}

// ---------------------------------------------------------------- histogram
// One launch per layer builds signal and background histograms for every
// node x feature (trees.py:139-167).  Work item = (class block, feature
// group, node group, contiguous run of row tiles).  Per tile, one thread
// bulk-copies (TMA, cp.async.bulk) the node ids, fixed-point weights and the
// group's code columns into a double-buffered shared-memory stage; the CTA
// compacts the rows that contribute (in class range, at this layer, in the
// node group, q != 0 — inactive rows carry q == 0) and every thread then
// adds its rows' weights into (node, feature, code) slots held in shared
// memory as 2-limb int64 (lo limb: returning 32-bit ATOMS; a wrap carries
// into the hi limb).  Measured better than two non-returning atomics per
// update (16/16 split): fewer shared-atomic wavefronts.
// Missing codes (bin 0) are skipped: the split search never reads slot 0
// (trees.py:181-186).  At the end each CTA merges its slots into the global
// histogram with native 64-bit global reductions.
struct HistPlan {
  int start, nodes;          // layer_start, nodes in layer
  int fg, n_fg;              // features per group, groups
  int ngs, n_ng;             // nodes per node group, node groups
  int tile;                  // rows per tile (= kTile)
  int tiles_sig0, tiles_sig1, tiles_bkg0, tiles_bkg1;  // tile ranges per class
  int split_sig, split_bkg;  // CTAs per group per class
  int smem;                  // dynamic shared memory bytes
  int prof;                  // debug (BB_HIST_PROFILE=1): thread 0's per-phase cycles into g_hist_prof
  int sib;                   // 1: build left children only (right = parent - left in k_split)
  int global_only;           // bins too wide for any shared-memory plan (levels 12..15)
};

__device__ unsigned long long g_hist_prof[8];

constexpr int kHistThreads = 512;
#ifndef BB_HIST_ILP
#define BB_HIST_ILP 8
#endif
constexpr int kHistIlp = BB_HIST_ILP;  // returning low-limb atomics in flight per thread
constexpr int kHistFlushTiles = 1 << 20;  // 2-limb slots are exact int64 sums (no periodic flush needed)

__host__ __device__ __forceinline__ int align16(int x) { return (x + 15) & ~15; }

template <typename CodeT, typename NodeT>
__host__ __device__ __forceinline__ int hist_buf_bytes(int tile, int fcount) {
  return align16(tile * (int)sizeof(NodeT)) + tile * 8 + fcount * tile * (int)sizeof(CodeT);
}

template <typename CodeT, typename NodeT>
__global__ void __launch_bounds__(kHistThreads, 1)
    k_layer_hist(const CodeT* __restrict__ codes, int code_off, const NodeT* __restrict__ node,
                 const long long* __restrict__ q, int64_t n, int64_t n_sig, int d, int B, HistPlan p,
                 unsigned long long* __restrict__ hist) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int groups = p.n_fg * p.n_ng;
  const int group = blockIdx.x % groups;
  const int part = blockIdx.x / groups;
  const int fgi = group % p.n_fg, ngi = group / p.n_fg;
  int cls, ta, tb;
  int64_t clo, chi;
  if (part < p.split_sig) {
    cls = 0;
    clo = 0;
    chi = n_sig;
    const int nt = p.tiles_sig1 - p.tiles_sig0;
    ta = p.tiles_sig0 + (int)((int64_t)nt * part / p.split_sig);
    tb = p.tiles_sig0 + (int)((int64_t)nt * (part + 1) / p.split_sig);
  } else {
    cls = 1;
    clo = n_sig;
    chi = n;
    const int k = part - p.split_sig;
    const int nt = p.tiles_bkg1 - p.tiles_bkg0;
    ta = p.tiles_bkg0 + (int)((int64_t)nt * k / p.split_bkg);
    tb = p.tiles_bkg0 + (int)((int64_t)nt * (k + 1) / p.split_bkg);
  }
  const int f0 = fgi * p.fg;
  const int fcount = min(p.fg, d - f0);
  const int n0 = ngi * p.ngs;
  const int built = p.sib ? p.nodes >> 1 : p.nodes;  // histogram nodes built by this launch
  const int ncount = min(p.ngs, built - n0);
  const int nslots = ncount * fcount * B;
  const int tile = p.tile;
  uint32_t* lo = reinterpret_cast<uint32_t*>(smem);
  uint32_t* hi = lo + nslots + 32;  // slots nslots .. nslots+31: per-lane dummies
  unsigned char* stage = smem + align16((nslots + 32) * 8);
  const int bufb = hist_buf_bytes<CodeT, NodeT>(tile, fcount);
  uint32_t* list = reinterpret_cast<uint32_t*>(stage + 2 * bufb);
  uint64_t* bar = reinterpret_cast<uint64_t*>(list + tile);
  int* counter = reinterpret_cast<int*>(bar + 2);

  for (int i = threadIdx.x; i < 2 * (nslots + 32); i += kHistThreads) lo[i] = 0u;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
    counter[0] = 0;
    counter[1] = 0;
  }
  __syncthreads();

  auto issue = [&](int k, int buf) {
    unsigned char* b = stage + buf * bufb;
    const int64_t row0 = (int64_t)k * tile;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(&bar[buf], (unsigned)(tile * (int)sizeof(NodeT) + tile * 8 + fcount * tile * (int)sizeof(CodeT)));
    tma_load_1d(b, node + row0, tile * sizeof(NodeT), &bar[buf]);
    tma_load_1d(b + align16(tile * (int)sizeof(NodeT)), q + row0, tile * 8, &bar[buf]);
    unsigned char* cb = b + align16(tile * (int)sizeof(NodeT)) + tile * 8;
    tma_load_1d(cb, codes + ((int64_t)k * d + f0) * kTile, fcount * kTile * sizeof(CodeT), &bar[buf]);
  };

  // smem slots -> global int64 histogram (value = l sum + h sum * 2^16)
  auto flush = [&](bool zero) {
    for (int s = threadIdx.x; s < nslots; s += kHistThreads) {
      const long long v = (long long)(((unsigned long long)hi[s] << 32) | (unsigned long long)lo[s]);
      if (zero) {
        lo[s] = 0u;
        hi[s] = 0u;
      }
      if (v != 0) {
        const int bb = s % B;
        const int j = (s / B) % fcount;
        const int nd = s / (B * fcount);
        const int ln = p.sib ? 2 * (n0 + nd) : (n0 + nd);
        const int64_t g = (((int64_t)cls * p.nodes + ln) * d + (f0 + j)) * B + bb;
        atomicAdd(&hist[g], as_ull(v));
      }
    }
  };
  if (threadIdx.x == 0 && ta < tb) issue(ta, 0);
  for (int k = ta; k < tb; ++k) {
    const int it = k - ta, buf = it & 1;
    if (threadIdx.x == 0) {
      if (k + 1 < tb) issue(k + 1, buf ^ 1);
      counter[(it + 1) & 1] = 0;
    }
    const bool pf = (p.prof & 1) && threadIdx.x == 0;
    const long long t0 = pf ? clock64() : 0;
    mbar_wait(&bar[buf], (it >> 1) & 1);
    const long long t1 = pf ? clock64() : 0;
    const unsigned char* b = stage + buf * bufb;
    const NodeT* nt = reinterpret_cast<const NodeT*>(b);
    const long long* qt = reinterpret_cast<const long long*>(b + align16(tile * (int)sizeof(NodeT)));
    const CodeT* ct = reinterpret_cast<const CodeT*>(b + align16(tile * (int)sizeof(NodeT)) + tile * 8);
    const int64_t row0 = (int64_t)k * tile;
    // compaction of contributing rows (order irrelevant: integer sums)
    for (int rl = threadIdx.x; rl < tile; rl += kHistThreads) {
      const int64_t r = row0 + rl;
      const int ln = (int)nt[rl] - p.start;  // node within the layer
      const int nd = (p.sib ? (ln >> 1) : ln) - n0;
      const bool ok = r >= clo && r < chi && ln >= 0 && ln < p.nodes && !(p.sib && (ln & 1)) && nd >= 0 &&
                      nd < ncount && qt[rl] != 0;
      const unsigned m = __ballot_sync(0xffffffffu, ok);
      int base = 0;
      if ((threadIdx.x & 31) == 0 && m) base = atomicAdd(&counter[it & 1], __popc(m));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (ok) list[base + __popc(m & ((1u << (threadIdx.x & 31)) - 1u))] = (uint32_t)rl | ((uint32_t)nd << 16);
    }
    const long long t2 = pf ? clock64() : 0;
    __syncthreads();
    const long long t3 = pf ? clock64() : 0;
    const int n_act = counter[it & 1];
    // one thread per compacted row, looping over the group's features: the
    // row's node and q are read once and every code load is independent.
    // Each update is one returning u32 add on the low limb (8 in flight)
    // plus an add of the high word and carry on the high limb when nonzero:
    // the fewest shared-memory wavefronts per update (bank conflicts make
    // each warp-wide atomic ~3.5 wavefronts).  A missing code (NaN bin) goes
    // to this lane's dummy slot (nslots + lane), never read.
    const int dummy = nslots + (threadIdx.x & 31);
    for (int ai = threadIdx.x; ai < n_act; ai += kHistThreads) {
      const uint32_t e = list[ai];
      const int rl = (int)(e & 0xffffu);
      const int nd = (int)(e >> 16);
      const long long qq = qt[rl];
      const uint32_t l = (uint32_t)(unsigned long long)qq;
      const uint32_t h = (uint32_t)((unsigned long long)qq >> 32);
      const int sb = nd * fcount * B - 1 + code_off;
      const CodeT* cp = ct + rl;
      int j = 0;
      for (; j + kHistIlp <= fcount; j += kHistIlp) {
        int sl[kHistIlp];
        uint32_t old[kHistIlp];
#pragma unroll
        for (int u = 0; u < kHistIlp; ++u) {
          const int c = (int)cp[(j + u) * kTile];
          sl[u] = (c + code_off != 0) ? sb + (j + u) * B + c : dummy;
        }
#pragma unroll
        for (int u = 0; u < kHistIlp; ++u) old[u] = atomicAdd(lo + sl[u], l);
#pragma unroll
        for (int u = 0; u < kHistIlp; ++u) {
          const uint32_t hh = h + ((old[u] + l < old[u]) ? 1u : 0u);
          if (hh) atomicAdd(hi + sl[u], hh);
        }
      }
      for (; j < fcount; ++j) {
        const int c = (int)cp[j * kTile];
        const int sl = (c + code_off != 0) ? sb + j * B + c : dummy;
        const uint32_t o = atomicAdd(lo + sl, l);
        const uint32_t hh = h + ((o + l < o) ? 1u : 0u);
        if (hh) atomicAdd(hi + sl, hh);
      }
    }
    const long long t4 = pf ? clock64() : 0;
    __syncthreads();
    if (pf) {
      const long long t5 = clock64();
      atomicAdd(&g_hist_prof[0], (unsigned long long)(t1 - t0));  // TMA wait
      atomicAdd(&g_hist_prof[1], (unsigned long long)(t2 - t1));  // compaction
      atomicAdd(&g_hist_prof[2], (unsigned long long)(t3 - t2));  // barrier 1
      atomicAdd(&g_hist_prof[3], (unsigned long long)(t4 - t3));  // atomics
      atomicAdd(&g_hist_prof[4], (unsigned long long)(t5 - t4));  // barrier 2
      atomicAdd(&g_hist_prof[5], 1ull);
    }
    if ((it & (kHistFlushTiles - 1)) == kHistFlushTiles - 1 && k + 1 < tb) {
      flush(true);
      __syncthreads();
    }
  }
  flush(false);
}

// Warp-independent variant of k_layer_hist (same plan, slots and sums): warp
// 16 is a producer issuing the tiles' bulk copies behind full/empty
// mbarriers; compute warp w compacts and accumulates its own 64 rows of
// each tile with no CTA-wide barrier, so warps drift up to a tile apart and
// the shared atomic pipe stays busy across tile boundaries.
#ifndef BB_HIST_WARPS
#define BB_HIST_WARPS 16
#endif
constexpr int kHistWarps = BB_HIST_WARPS;  // compute warps; each owns 1024 / kHistWarps rows of a tile
constexpr int kHistWRows = 1024 / kHistWarps;
constexpr int kHistWThreads = 32 * (kHistWarps + 1);

template <typename CodeT, typename NodeT>
__global__ void __launch_bounds__(kHistWThreads, 1)
    k_layer_hist_w(const CodeT* __restrict__ codes, int code_off, const NodeT* __restrict__ node,
                   const long long* __restrict__ q, int64_t n, int64_t n_sig, int d, int B, HistPlan p,
                   unsigned long long* __restrict__ hist) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int groups = p.n_fg * p.n_ng;
  const int group = blockIdx.x % groups;
  const int part = blockIdx.x / groups;
  const int fgi = group % p.n_fg, ngi = group / p.n_fg;
  int cls, ta, tb;
  int64_t clo, chi;
  if (part < p.split_sig) {
    cls = 0;
    clo = 0;
    chi = n_sig;
    const int nt = p.tiles_sig1 - p.tiles_sig0;
    ta = p.tiles_sig0 + (int)((int64_t)nt * part / p.split_sig);
    tb = p.tiles_sig0 + (int)((int64_t)nt * (part + 1) / p.split_sig);
  } else {
    cls = 1;
    clo = n_sig;
    chi = n;
    const int k = part - p.split_sig;
    const int nt = p.tiles_bkg1 - p.tiles_bkg0;
    ta = p.tiles_bkg0 + (int)((int64_t)nt * k / p.split_bkg);
    tb = p.tiles_bkg0 + (int)((int64_t)nt * (k + 1) / p.split_bkg);
  }
  const int f0 = fgi * p.fg;
  const int fcount = min(p.fg, d - f0);
  const int n0 = ngi * p.ngs;
  const int built = p.sib ? p.nodes >> 1 : p.nodes;
  const int ncount = min(p.ngs, built - n0);
  const int nslots = ncount * fcount * B;
  const int tile = p.tile;
  uint32_t* lo = reinterpret_cast<uint32_t*>(smem);
  uint32_t* hi = lo + nslots + 32;
  unsigned char* stage = smem + align16((nslots + 32) * 8);
  const int bufb = hist_buf_bytes<CodeT, NodeT>(tile, fcount);
  uint32_t* list = reinterpret_cast<uint32_t*>(stage + 2 * bufb);  // [warp][kHistWRows]
  uint64_t* full = reinterpret_cast<uint64_t*>(list + tile);
  uint64_t* empty = full + 2;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

  for (int i = threadIdx.x; i < 2 * (nslots + 32); i += kHistWThreads) lo[i] = 0u;
  if (threadIdx.x == 0) {
    for (int b = 0; b < 2; ++b) {
      mbar_init(&full[b], 1);
      mbar_init(&empty[b], kHistWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == kHistWarps) {
    // ---- producer
    if (lane == 0) {
      for (int k = ta; k < tb; ++k) {
        const int it = k - ta, buf = it & 1;
        if (it >= 2) mbar_wait(&empty[buf], (unsigned)(((it >> 1) - 1) & 1));
        unsigned char* b = stage + buf * bufb;
        const int64_t row0 = (int64_t)k * tile;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&full[buf], (unsigned)(tile * (int)sizeof(NodeT) + tile * 8 + fcount * tile * (int)sizeof(CodeT)));
        tma_load_1d(b, node + row0, tile * sizeof(NodeT), &full[buf]);
        tma_load_1d(b + align16(tile * (int)sizeof(NodeT)), q + row0, tile * 8, &full[buf]);
        tma_load_1d(b + align16(tile * (int)sizeof(NodeT)) + tile * 8, codes + ((int64_t)k * d + f0) * kTile,
                    fcount * kTile * sizeof(CodeT), &full[buf]);
      }
    }
  } else {
    // ---- compute warps
    uint32_t* wl = list + warp * kHistWRows;
    const int dummy = nslots + lane;
    const unsigned lt = (1u << lane) - 1u;
    for (int k = ta; k < tb; ++k) {
      const int it = k - ta, buf = it & 1;
      mbar_wait(&full[buf], (unsigned)((it >> 1) & 1));
      const unsigned char* b = stage + buf * bufb;
      const NodeT* nt = reinterpret_cast<const NodeT*>(b);
      const long long* qt = reinterpret_cast<const long long*>(b + align16(tile * (int)sizeof(NodeT)));
      const CodeT* ct = reinterpret_cast<const CodeT*>(b + align16(tile * (int)sizeof(NodeT)) + tile * 8);
      const int64_t row0 = (int64_t)k * tile;
      int cnt = 0;
#pragma unroll
      for (int h = 0; h < kHistWRows / 32; ++h) {
        const int rl = warp * kHistWRows + h * 32 + lane;
        const int64_t r = row0 + rl;
        const int ln = (int)nt[rl] - p.start;
        const int nd = (p.sib ? (ln >> 1) : ln) - n0;
        const bool ok = r >= clo && r < chi && ln >= 0 && ln < p.nodes && !(p.sib && (ln & 1)) && nd >= 0 &&
                        nd < ncount && qt[rl] != 0;
        const unsigned m = __ballot_sync(0xffffffffu, ok);
        if (ok) wl[cnt + __popc(m & lt)] = (uint32_t)rl | ((uint32_t)nd << 16);
        cnt += __popc(m);
      }
      __syncwarp();
      for (int ai = lane; ai < cnt; ai += 32) {
        const uint32_t e = wl[ai];
        const int rl = (int)(e & 0xffffu);
        const int nd = (int)(e >> 16);
        const long long qq = qt[rl];
        const uint32_t l = (uint32_t)(unsigned long long)qq;
        const uint32_t h = (uint32_t)((unsigned long long)qq >> 32);
        const int sb = nd * fcount * B - 1 + code_off;
        const CodeT* cp = ct + rl;
        int j = 0;
        for (; j + kHistIlp <= fcount; j += kHistIlp) {
          int sl[kHistIlp];
          uint32_t old[kHistIlp];
#pragma unroll
          for (int u = 0; u < kHistIlp; ++u) {
            const int c = (int)cp[(j + u) * kTile];
            sl[u] = (c + code_off != 0) ? sb + (j + u) * B + c : dummy;
          }
#pragma unroll
          for (int u = 0; u < kHistIlp; ++u) old[u] = atomicAdd(lo + sl[u], l);
#pragma unroll
          for (int u = 0; u < kHistIlp; ++u) {
            const uint32_t hh = h + ((old[u] + l < old[u]) ? 1u : 0u);
            if (hh) atomicAdd(hi + sl[u], hh);
          }
        }
        for (; j < fcount; ++j) {
          const int c = (int)cp[j * kTile];
          const int sl = (c + code_off != 0) ? sb + j * B + c : dummy;
          const uint32_t o = atomicAdd(lo + sl, l);
          const uint32_t hh = h + ((o + l < o) ? 1u : 0u);
          if (hh) atomicAdd(hi + sl, hh);
        }
      }
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[buf])) : "memory");
    }
  }
  __syncthreads();
  // flush: int64 rows [node][feature][bin] staged in the drained ring, one TMA
  // bulk reduction per row (scattered 64-bit global atomics cost ~1 LSU
  // cycle per lane: ~10 us per CTA for cfg2's 20k slots)
  const int cap_rows = (2 * bufb) / (B * 8);
  if (cap_rows >= 1 && (B & 1) == 0) {
    long long* st = reinterpret_cast<long long*>(stage);
    const int rows = ncount * fcount;
    for (int r0 = 0; r0 < rows; r0 += cap_rows) {
      const int rn = min(cap_rows, rows - r0);
      for (int e = threadIdx.x; e < rn * B; e += kHistWThreads) {
        const int s = r0 * B + e;  // slot = (nd * fcount + j) * B + bin = row * B + bin
        st[e] = (long long)(((unsigned long long)hi[s] << 32) | (unsigned long long)lo[s]);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      for (int rl = threadIdx.x; rl < rn; rl += kHistWThreads) {
        const int row = r0 + rl, nd = row / fcount, j = row - nd * fcount;
        const int ln = p.sib ? 2 * (n0 + nd) : (n0 + nd);
        bulk_reduce_add_u64(hist + (((int64_t)cls * p.nodes + ln) * d + (f0 + j)) * B, st + (size_t)rl * B,
                            (unsigned)B * 8u);
      }
      asm volatile("cp.async.bulk.commit_group;\ncp.async.bulk.wait_group 0;" ::: "memory");
      __syncthreads();
    }
    return;
  }
  for (int s = threadIdx.x; s < nslots; s += kHistWThreads) {
    const long long v = (long long)(((unsigned long long)hi[s] << 32) | (unsigned long long)lo[s]);
    if (v != 0) {
      const int bb = s % B;
      const int j = (s / B) % fcount;
      const int nd = s / (B * fcount);
      const int ln = p.sib ? 2 * (n0 + nd) : (n0 + nd);
      const int64_t g = (((int64_t)cls * p.nodes + ln) * d + (f0 + j)) * B + bb;
      atomicAdd(&hist[g], as_ull(v));
    }
  }
}

// Layer histogram straight into global memory (int64 RED.ADD, L2-resident
// layer histogram) for layers whose shared-memory plan would need many
// (node, feature) groups, each re-reading every row: one pass over the rows,
// one thread per (row, 8-feature block).  Same slots, same exact sums.
template <typename CodeT, typename NodeT>
__global__ void __launch_bounds__(256)
    k_layer_hist_g(const CodeT* __restrict__ codes, int code_off, const NodeT* __restrict__ node,
                   const long long* __restrict__ q, int64_t n, int64_t n_sig, int d, int B, HistPlan p,
                   unsigned long long* __restrict__ hist) {
  const int nfb = (d + 7) >> 3;
  const int per_tile = kTile * nfb;  // (feature block, row) items of a tile
  const int64_t tiles = (n + kTile - 1) / kTile;
  // grid-stride over tiles, 32-bit item math inside a tile (the 64-bit
  // divisions of a flat item index cost more than the loads they address)
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const CodeT* ct = codes + tile * (int64_t)d * kTile;
    for (int e = threadIdx.x; e < per_tile; e += blockDim.x) {
      // consecutive threads take consecutive rows of one feature block (coalesced codes)
      const int fb = e >> kTileLog, rl = e & (kTile - 1);
      const int64_t r = tile * kTile + rl;
      if (r >= n) continue;
      const int ln = (int)node[r] - p.start;
      if (ln < 0 || ln >= p.nodes || (p.sib && (ln & 1))) continue;
      const long long qq = q[r];
      if (qq == 0) continue;
      const int cls = r >= n_sig ? 1 : 0;
      unsigned long long* hb = hist + ((int64_t)cls * p.nodes + ln) * d * B - 1 + code_off;
      const int f0 = fb * 8, f1 = min(d, f0 + 8);
#pragma unroll 8
      for (int f = f0; f < f1; ++f) {
        const int c = (int)ct[f * kTile + rl];
        if (c + code_off != 0) atomicAdd(hb + (int64_t)f * B + c, as_ull(qq));
      }
    }
  }
}

// ---------------------------------------------------------------- split
// CPH prefix scan + separation gain + argmax (trees.py:117-136,170-204),
// fixed-point definition shared with oracle/binboost_np.py:_gains_fixed.
// Grid (nodes, feature chunks); each CTA scans its features' signal and
// background histograms, keeps the first maximum over flat (f, c-1), and the
// last CTA of a node reduces the chunks and writes the cut.
struct SplitScratch {
  double* best_gain;       // [nodes][n_fc]
  int* best_flat;          // [nodes][n_fc]
  double* forced_gain;     // [nodes]
  unsigned int* done;      // [nodes]
};

__device__ __forceinline__ double g_term(long long s_q, long long b_q, double scale) {
  const long long den_q = s_q + b_q;
  if (den_q <= 0) return 0.0;
  const double s = __dmul_rn((double)s_q, scale);
  const double den = __dmul_rn((double)den_q, scale);
  return __ddiv_rn(__dmul_rn(s, s), den);
}

__device__ __forceinline__ bool better(double g, int flat, double bg, int bflat) {
  return (g > bg) || (g == bg && flat < bflat);
}

template <int THREADS>
__global__ void __launch_bounds__(THREADS) k_split(unsigned long long* __restrict__ hist_u, int d, int B, int start,
                                                   int nodes, int fc_size, int final_layer, double scale, int tree,
                                                   int n_internal, TreeArrays ta, const double* __restrict__ bounds,
                                                   SplitScratch sc, unsigned long long* __restrict__ par_u, int sib,
                                                   int keep, const int* __restrict__ cnt) {
  pdl_wait();
  pdl_launch();
  long long* hist = reinterpret_cast<long long*>(hist_u);
  long long* par = reinterpret_cast<long long*>(par_u);  // previous layer [2][nodes/2][d][B] (sib)
  const int node = blockIdx.x;
  const int fci = blockIdx.y;
  const int n_fc = gridDim.y;
  const int heap = start + node;
  const int fc = ta.forced ? ta.forced[(int64_t)tree * n_internal + heap] : -2;
  const int per = (B + THREADS - 1) / THREADS;  // consecutive codes per thread (<= 8)
  __shared__ long long s_ws[THREADS / 32], s_wb[THREADS / 32];
  __shared__ double s_bg[THREADS / 32];
  __shared__ int s_bf[THREADS / 32];
  double best_g = -INFINITY;
  int best_flat = 0x7fffffff;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int fbeg = fci * fc_size, fend = min(d, fbeg + fc_size);
  // sibling subtraction (sib): the histogram launch built the left children
  // only; a right child is its parent minus its left sibling (integer sums:
  // exact), or empty if the parent was not split.  A right child's CTA
  // zeroes the parent it consumed; a non-final layer keeps its histograms as
  // the next layer's parents, a final one is cleared by the host (memset).
  // sib == 2 (row-list fits): the child with fewer active rows was built
  // (kernels_hist_list.cuh lh_build_right); `right` = this node is the derived one
  bool built_right = false;
  if (sib == 2) {
    const int lc = start + (node & ~1);
    built_right = (__ldcg(cnt + 2 * lc + 2) + __ldcg(cnt + 2 * lc + 3)) < (__ldcg(cnt + 2 * lc) + __ldcg(cnt + 2 * lc + 1));
  }
  const bool right = sib && (((node & 1) != 0) != built_right);
  const int sibn = node ^ 1;  // the built sibling of a derived node
  const int pnode = node >> 1, pnodes = nodes >> 1;
  const bool pvalid = right && ta.valid[(int64_t)tree * n_internal + ((start - 1) >> 1) + pnode] != 0;
  if (per > 8) {
    // wide bins (B > 8 * THREADS, binning_levels 12..15): two passes per
    // feature, node totals first, then chunks of 8 * THREADS codes with the
    // CPH prefix carried across chunks (same gains, same first-max order)
    constexpr int CH = 8 * THREADS;
    __shared__ long long s_red[2][THREADS / 32];
    for (int f = fbeg; f < fend; ++f) {
      long long* hs = hist + ((int64_t)node * d + f) * B;
      long long* hb = hist + (((int64_t)nodes + node) * d + f) * B;
      long long* ls = right ? hist + ((int64_t)sibn * d + f) * B : nullptr;
      long long* lb = right ? hist + (((int64_t)nodes + sibn) * d + f) * B : nullptr;
      long long* ps = right ? par + ((int64_t)pnode * d + f) * B : nullptr;
      long long* pb = right ? par + (((int64_t)pnodes + pnode) * d + f) * B : nullptr;
      auto val = [&](int c, long long& a, long long& b) {
        if (right) {
          a = pvalid ? ps[c] - ls[c] : 0;
          b = pvalid ? pb[c] - lb[c] : 0;
        } else {
          a = hs[c];
          b = hb[c];
        }
      };
      long long ts = 0, tb = 0;
      for (int c = threadIdx.x; c < B; c += THREADS) {
        long long a, b;
        val(c, a, b);
        ts += a;
        tb += b;
      }
      for (int o = 16; o > 0; o >>= 1) {
        ts += __shfl_xor_sync(0xffffffffu, ts, o);
        tb += __shfl_xor_sync(0xffffffffu, tb, o);
      }
      if (lane == 0) { s_red[0][warp] = ts; s_red[1][warp] = tb; }
      __syncthreads();
      long long tot_s = 0, tot_b = 0;
      for (int w = 0; w < THREADS / 32; ++w) { tot_s += s_red[0][w]; tot_b += s_red[1][w]; }
      __syncthreads();
      long long carry_s = 0, carry_b = 0;
      for (int ch0 = 0; ch0 < B; ch0 += CH) {
        long long vs[8], vb[8];
        long long qs = 0, qb = 0;
        const int c0 = ch0 + threadIdx.x * 8;
        for (int j = 0; j < 8; ++j) {
          const int c = c0 + j;
          vs[j] = 0;
          vb[j] = 0;
          if (c < B) {
            val(c, vs[j], vb[j]);
            if (right) {
              if (!final_layer) { hs[c] = vs[j]; hb[c] = vb[j]; }
              ps[c] = 0;
              pb[c] = 0;
            }
          }
          qs += vs[j];
          qb += vb[j];
        }
        long long is = qs, ib = qb;
        for (int o = 1; o < 32; o <<= 1) {
          const long long us = __shfl_up_sync(0xffffffffu, is, o);
          const long long ub = __shfl_up_sync(0xffffffffu, ib, o);
          if (lane >= o) { is += us; ib += ub; }
        }
        if (lane == 31) { s_ws[warp] = is; s_wb[warp] = ib; }
        __syncthreads();
        long long off_s = 0, off_b = 0, ch_s = 0, ch_b = 0;
        for (int w = 0; w < THREADS / 32; ++w) {
          if (w < warp) { off_s += s_ws[w]; off_b += s_wb[w]; }
          ch_s += s_ws[w];
          ch_b += s_wb[w];
        }
        __syncthreads();
        long long cs = carry_s + off_s + is - qs, cb = carry_b + off_b + ib - qb;
        for (int j = 0; j < 8; ++j) {
          const int c = c0 + j;
          cs += vs[j];
          cb += vb[j];
          if (c >= B - 1) break;
          const long long rs = tot_s - cs, rb = tot_b - cb;
          double g = -INFINITY;
          if (cs + cb > 0 && rs + rb > 0)
            g = __dsub_rn(__dadd_rn(g_term(cs, cb, scale), g_term(rs, rb, scale)), g_term(tot_s, tot_b, scale));
          const int flat = f * (B - 1) + c;
          if (better(g, flat, best_g, best_flat)) { best_g = g; best_flat = flat; }
          if (fc >= 0 && (fc >> 16) == f && (fc & 0xffff) == c + 1) sc.forced_gain[node] = g;
        }
        if (!sib && !keep) {
          for (int j = 0; j < 8; ++j) {
            const int c = c0 + j;
            if (c < B) { hs[c] = 0; hb[c] = 0; }
          }
        }
        carry_s += ch_s;
        carry_b += ch_b;
      }
    }
  }
  for (int f = fbeg; f < fend && per <= 8; ++f) {
    long long* hs = hist + ((int64_t)node * d + f) * B;
    long long* hb = hist + (((int64_t)nodes + node) * d + f) * B;
    long long vs[8], vb[8];
    long long ts = 0, tb = 0;
    const int c0 = threadIdx.x * per;
    if (right) {
      long long* ls = hist + ((int64_t)sibn * d + f) * B;
      long long* lb = hist + (((int64_t)nodes + sibn) * d + f) * B;
      long long* ps = par + ((int64_t)pnode * d + f) * B;
      long long* pb = par + (((int64_t)pnodes + pnode) * d + f) * B;
      for (int j = 0; j < per; ++j) {
        const int c = c0 + j;
        vs[j] = 0;
        vb[j] = 0;
        if (c < B) {
          if (pvalid) {
            vs[j] = ps[c] - ls[c];
            vb[j] = pb[c] - lb[c];
          }
          if (!final_layer) {  // the next layer's parent
            hs[c] = vs[j];
            hb[c] = vb[j];
          }
          ps[c] = 0;  // only this CTA reads the parent
          pb[c] = 0;
        }
        ts += vs[j];
        tb += vb[j];
      }
    } else {
      for (int j = 0; j < per; ++j) {
        const int c = c0 + j;
        vs[j] = (c < B) ? hs[c] : 0;
        vb[j] = (c < B) ? hb[c] : 0;
        ts += vs[j];
        tb += vb[j];
      }
    }
    // block-wide exclusive scan of (ts, tb)
    long long is = ts, ib = tb;
    for (int o = 1; o < 32; o <<= 1) {
      const long long us = __shfl_up_sync(0xffffffffu, is, o);
      const long long ub = __shfl_up_sync(0xffffffffu, ib, o);
      if (lane >= o) { is += us; ib += ub; }
    }
    if (lane == 31) { s_ws[warp] = is; s_wb[warp] = ib; }
    __syncthreads();
    long long off_s = 0, off_b = 0, tot_s = 0, tot_b = 0;
    for (int w = 0; w < THREADS / 32; ++w) {
      if (w < warp) { off_s += s_ws[w]; off_b += s_wb[w]; }
      tot_s += s_ws[w];
      tot_b += s_wb[w];
    }
    __syncthreads();
    long long cs = off_s + is - ts, cb = off_b + ib - tb;
    for (int j = 0; j < per; ++j) {
      const int c = c0 + j;  // 0-based code index: cut bin c+1 keeps codes 1..c+1 left
      cs += vs[j];
      cb += vb[j];
      if (c >= B - 1) break;
      const long long rs = tot_s - cs, rb = tot_b - cb;
      double g = -INFINITY;
      if (cs + cb > 0 && rs + rb > 0)
        g = __dsub_rn(__dadd_rn(g_term(cs, cb, scale), g_term(rs, rb, scale)), g_term(tot_s, tot_b, scale));
      const int flat = f * (B - 1) + c;
      if (better(g, flat, best_g, best_flat)) { best_g = g; best_flat = flat; }
      if (fc >= 0 && (fc >> 16) == f && (fc & 0xffff) == c + 1) sc.forced_gain[node] = g;
    }
    // without sibling subtraction a layer zeroes what it consumed, unless the
    // next layer subtracts from it (keep)
    if (!sib && !keep) {
      for (int j = 0; j < per; ++j) {
        const int c = c0 + j;
        if (c < B) { hs[c] = 0; hb[c] = 0; }
      }
    }
  }
  // block argmax
  for (int o = 16; o > 0; o >>= 1) {
    const double og = __shfl_down_sync(0xffffffffu, best_g, o);
    const int of = __shfl_down_sync(0xffffffffu, best_flat, o);
    if (better(og, of, best_g, best_flat)) { best_g = og; best_flat = of; }
  }
  if (lane == 0) { s_bg[warp] = best_g; s_bf[warp] = best_flat; }
  __syncthreads();
  __shared__ bool s_last;
  if (threadIdx.x == 0) {
    for (int w = 1; w < THREADS / 32; ++w)
      if (better(s_bg[w], s_bf[w], best_g, best_flat)) { best_g = s_bg[w]; best_flat = s_bf[w]; }
    sc.best_gain[node * n_fc + fci] = best_g;
    sc.best_flat[node * n_fc + fci] = best_flat;
    __threadfence();
    const unsigned prev = atomicAdd(&sc.done[node], 1u);
    s_last = (prev == (unsigned)n_fc - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // the last CTA of the node reduces the chunks' bests in parallel (a serial
  // loop of dependent L2 reads cost ~10 us with 40 chunks)
  double g = -INFINITY;
  int flat = 0x7fffffff;
  for (int k = threadIdx.x; k < n_fc; k += THREADS) {
    const double kg = __ldcg(sc.best_gain + node * n_fc + k);
    const int kf = __ldcg(sc.best_flat + node * n_fc + k);
    if (better(kg, kf, g, flat)) { g = kg; flat = kf; }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double og = __shfl_down_sync(0xffffffffu, g, o);
    const int of = __shfl_down_sync(0xffffffffu, flat, o);
    if (better(og, of, g, flat)) { g = og; flat = of; }
  }
  if (lane == 0) { s_bg[warp] = g; s_bf[warp] = flat; }
  __syncthreads();
  if (threadIdx.x != 0) return;
  for (int w = 1; w < THREADS / 32; ++w)
    if (better(s_bg[w], s_bf[w], g, flat)) { g = s_bg[w]; flat = s_bf[w]; }
  sc.done[node] = 0u;
  const int64_t o = (int64_t)tree * n_internal + heap;
  bool ok;
  int f = -1, cut = 0;
  if (fc == -1) {
    ok = false;
  } else if (fc >= 0) {
    ok = true;
    f = fc >> 16;
    cut = fc & 0xffff;
    g = ((volatile double*)sc.forced_gain)[node];
  } else {
    ok = isfinite(g) && (g > 0.0 || (g == 0.0 && !final_layer));
    if (ok) { f = flat / (B - 1); cut = flat % (B - 1) + 1; }
  }
  ta.valid[o] = ok ? 1 : 0;
  ta.feature[o] = ok ? f : -1;
  ta.cut[o] = ok ? cut : 0;
  ta.gain[o] = ok ? g : 0.0;
  ta.thr[o] = ok ? bounds[(int64_t)f * (B - 1) + cut - 1] : __longlong_as_double(0x7ff8000000000000ll);
}

// ---------------------------------------------------------------- advance
constexpr int kAdvMaxNodes = 128;  // layer nodes with row lists (depth <= 8)
// Move every row at the layer to its child (trees.py:207-228 for active rows,
// which traverse_bins, trees.py:318-330, repeats for all rows): left iff
// code <= cut; invalid cut or missing code parks the row.  Advancing ALL rows
// makes the final node the leaf traverse_bins would find.  On the last layer
// the active rows' (eff, resp) fixed-point sums are accumulated per final
// node, from which k_node_weights derives every node's sums (trees.py:231-244).
template <typename CodeT, typename NodeT>
__global__ void __launch_bounds__(kListThreads, 4) k_advance(const CodeT* __restrict__ codes, int d, int code_off,
                                                         NodeT* __restrict__ node, int64_t n, int64_t n_sig, int start,
                                                         int tree, int n_internal, TreeArrays ta, int last_layer,
                                                         int n_nodes, const long long* __restrict__ q,
                                                         const unsigned int* __restrict__ mask,
                                                         const double* __restrict__ F, const double* __restrict__ w,
                                                         double two_s, unsigned long long* __restrict__ sums,
                                                         int* __restrict__ cnt, int* __restrict__ lrow,
                                                         long long* __restrict__ lq, int sib) {
  extern __shared__ uint32_t s_sums[];  // [2 cls][n_nodes][2 kinds] 2-limb
  __shared__ int s_reg[2 * kAdvMaxNodes];  // list region of (class, node of this layer)
  __shared__ int s_cnt[4 * kAdvMaxNodes], s_base[4 * kAdvMaxNodes];  // per (child, class) of the tile
  constexpr int R = kListTileRows / kListThreads;
  const int* feat = ta.feature + (int64_t)tree * n_internal;
  const int* cutp = ta.cut + (int64_t)tree * n_internal;
  const unsigned char* vld = ta.valid + (int64_t)tree * n_internal;
  const bool lists = lrow != nullptr && !last_layer;
  const int nodes = start + 1;           // nodes of this layer: heap [start, 2 start]
  const int c0 = 2 * start + 1, nkeys = 4 * nodes;  // children heap [c0, c0 + 2 nodes), key = 2 (child - c0) + class
  if (last_layer) {
    for (int i = threadIdx.x; i < 2 * n_nodes * 2 * 2; i += blockDim.x) s_sums[i] = 0u;
  }
  if (lists && threadIdx.x == 0) {
    // class-major prefix of this layer's active counts (kernels_hist_list.cuh lh_segments)
    int off = 0;
    for (int k = 0; k < 2; ++k)
      for (int p = 0; p < nodes; ++p) {
        s_reg[k * nodes + p] = off;
        off += cnt[2 * (start + p) + k];
      }
  }
  for (int64_t t0 = (int64_t)blockIdx.x * kListTileRows; t0 < n; t0 += (int64_t)gridDim.x * kListTileRows) {
    if (lists) {
      for (int k = threadIdx.x; k < nkeys; k += blockDim.x) s_cnt[k] = 0;
    }
    __syncthreads();
    // loads batched across the tile's R rows per thread (node ids, then the
    // cut tables, then the code gathers) so their latencies overlap
    int key[R], loc[R], ndv[R], fv[R];
    bool act[R];
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const int64_t i = t0 + k * kListThreads + threadIdx.x;
      ndv[k] = i < n ? (int)node[i] : -1;
      act[k] = i < n && ((mask[i >> 5] >> (i & 31)) & 1u);
    }
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const bool go = ndv[k] >= start && vld[ndv[k]];
      fv[k] = go ? feat[ndv[k]] : -1;
    }
    int cv[R];
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const int64_t i = t0 + k * kListThreads + threadIdx.x;
      cv[k] = fv[k] >= 0 ? (int)codes[code_index(i, fv[k], d)] + code_off : 0;
    }
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const int64_t i = t0 + k * kListThreads + threadIdx.x;
      key[k] = -1;
      loc[k] = 0;
      int nd = ndv[k];
      if (fv[k] >= 0 && cv[k] != 0) {
        nd = 2 * nd + 1 + (cv[k] > cutp[nd] ? 1 : 0);
        node[i] = (NodeT)nd;
        if (lists && act[k]) key[k] = 2 * (nd - c0) + (i < n_sig ? 0 : 1);
      }
      if (last_layer && act[k]) {
        const int lab = row_label(i, n_sig);
        const int cls = lab > 0 ? 0 : 1;
        const double r = residual_of(F[i], lab);
        const double wi = w ? w[i] : 1.0;
        const long long qr = __double2ll_rn(__dmul_rn(__dmul_rn(wi, r), two_s));
        uint32_t* sp = s_sums + 4 * (cls * n_nodes + nd);
        slot_add(sp, q[i]);
        slot_add(sp + 2, qr);
      }
    }
    if (!lists) continue;
    {  // rank within the tile: one shared atomic per warp and key
      const int lane = threadIdx.x & 31;
#pragma unroll
      for (int k = 0; k < R; ++k) {
        const unsigned grp = __match_any_sync(0xffffffffu, key[k]);
        const int leader = __ffs(grp) - 1;
        int b0 = 0;
        if (key[k] >= 0 && lane == leader) b0 = atomicAdd(&s_cnt[key[k]], __popc(grp));
        b0 = __shfl_sync(0xffffffffu, b0, leader);
        loc[k] = b0 + __popc(grp & ((1u << lane) - 1u));
      }
    }
    __syncthreads();
    // active rows entering a child: counted per (child, class); the rows of
    // the children a histogram builds are listed in the parent's region (left
    // child from its start, right child from its end)
    for (int k = threadIdx.x; k < nkeys; k += blockDim.x)
      s_base[k] = s_cnt[k] ? atomicAdd(cnt + 2 * c0 + k, s_cnt[k]) : 0;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < R; ++k) {
      if (key[k] < 0) continue;
      const int child = c0 + (key[k] >> 1), cls = key[k] & 1;
      const bool left = child & 1;
      if (!left && sib) continue;
      const int par = (child - 1) >> 1;
      const int old = s_base[key[k]] + loc[k];
      const int reg = s_reg[cls * nodes + (par - start)];
      const int pos = left ? reg + old : reg + cnt[2 * par + cls] - 1 - old;
      const int64_t i = t0 + k * kListThreads + threadIdx.x;
      BB_DCHECK(pos >= 0 && pos < n && old < cnt[2 * par + cls]);
      lrow[pos] = (int)i;
      lq[pos] = q[i];
    }
    __syncthreads();
  }
  if (last_layer) {
    __syncthreads();
    for (int k = threadIdx.x; k < 2 * n_nodes * 2; k += blockDim.x) {
      const long long v = slot_value(s_sums + 2 * k);
      if (v != 0) atomicAdd(&sums[k], as_ull(v));
    }
  }
}

// ---------------------------------------------------------------- weights
// Node sums of every node from the final-node sums (subtree totals, exact
// integers), node weight sum(w r)/sum(w bw) with the 1e-12 guard, purity,
// shrinkage (trees.py:297-304, boosting.py:168).  One CTA; zeroes sums.
__global__ void k_node_weights(unsigned long long* __restrict__ sums_u, int n_nodes, int depth, double scale,
                               double shrinkage, int tree, TreeArrays ta) {
  extern __shared__ long long s_tot[];  // [2 cls][n_nodes][2]
  pdl_wait();
  pdl_launch();
  long long* sums = reinterpret_cast<long long*>(sums_u);
  const int m = 2 * n_nodes * 2;
  for (int k = threadIdx.x; k < m; k += blockDim.x) {
    s_tot[k] = sums[k];
    sums[k] = 0;
  }
  __syncthreads();
  // bottom-up: internal node p (layers depth .. 1) adds its children
  for (int layer = depth; layer >= 1; --layer) {
    const int first = (1 << (layer - 1)) - 1, cnt = 1 << (layer - 1);
    for (int k = threadIdx.x; k < cnt * 4; k += blockDim.x) {
      const int p = first + (k >> 2), cls = (k >> 1) & 1, kind = k & 1;
      const int a = 2 * p + 1, b = 2 * p + 2;
      s_tot[(cls * n_nodes + p) * 2 + kind] += s_tot[(cls * n_nodes + a) * 2 + kind] + s_tot[(cls * n_nodes + b) * 2 + kind];
    }
    __syncthreads();
  }
  for (int p = threadIdx.x; p < n_nodes; p += blockDim.x) {
    const long long es = s_tot[(0 * n_nodes + p) * 2 + 0], eb = s_tot[(1 * n_nodes + p) * 2 + 0];
    const long long rs = s_tot[(0 * n_nodes + p) * 2 + 1], rb = s_tot[(1 * n_nodes + p) * 2 + 1];
    const double den = __dmul_rn((double)(es + eb), scale);
    const double num = __dmul_rn((double)(rs + rb), scale);
    const double esd = __dmul_rn((double)es, scale);
    const double gam = (fabs(den) >= 1e-12) ? __ddiv_rn(num, den) : 0.0;
    const double pur = (den >= 1e-12) ? __ddiv_rn(esd, den) : 0.0;
    ta.nw[(int64_t)tree * n_nodes + p] = __dmul_rn(gam, shrinkage);
    ta.pur[(int64_t)tree * n_nodes + p] = pur;
  }
}

}  // namespace bb
