// C-ABI and host driver of the FastBDT B200 hot path (include/fastbdt_b200.h).
//
// bb_fit is the B200 restatement of fit_forest (reference
// pkg/src/binboost/boosting.py:117-173): GPU binning, class-block layout,
// then per tree one refresh kernel and per layer histogram -> split ->
// advance kernels, all stream-ordered with no host synchronisation inside
// the tree loop.  The host only generates the next tree's subsample bits
// (exact numpy PCG64 restatement, bb_mask.cpp) while the GPU works.
#include <algorithm>
#include <cstdlib>
#include <chrono>
#include <cmath>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include <cudaTypedefs.h>
#include <nvtx3/nvToolsExt.h>

#include "../../include/fastbdt_b200.h"
#include "bb_mask.h"
#include "bb_nccl.h"
#include "bb_stage.h"
#include "common.cuh"
#include "kernels_apply.cuh"
#include "kernels_binning.cuh"
#include "kernels_mask.cuh"
#include "kernels_seg.cuh"
#include "kernels_tree.cuh"
#include "kernels_hist_fl.cuh"
#include "kernels_hist_list.cuh"
#include "kernels_auc.cuh"

namespace bb {

static thread_local std::string g_err;

// NVTX ranges (header-only nvtx3: free unless a profiler attaches) around
// the fit's phases, every tree and every layer
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
void set_error(const std::string& msg) { g_err = msg; }

// numpy's pairwise float64 summation (numpy/_core/src/umath/loops_utils.h
// pairwise_sum, PW_BLOCKSIZE 128, 8-way unroll); used by prior()
// (boosting.py:79-80 calls np.sum).
static double pairwise(const double* a, int64_t n) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; ++i) res += a[i];
    return res;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int64_t i;
    for (i = 8; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i];
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return pairwise(a, n2) + pairwise(a + n2, n - n2);
}

// S = 32 - ceil(log2(max|w|)) so |w*bw| * 2^S <= 2^32 (bw <= 1):
// one returning 32-bit shared atomic per update for non-negative weights.
static int fixed_shift_for(double max_abs_w) {
  if (!(max_abs_w > 0.0)) return 32;
  int e;
  const double m = std::frexp(max_abs_w, &e);
  const int ceil_log2 = (m == 0.5) ? e - 1 : e;
  return 32 - ceil_log2;
}

struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int sm_count = 148;
  std::mutex mu;
  NcclComm comm;  // world > 1: row-sharded fits
  HostStager stage;  // pinned staging of pageable host buffers (bb_stage.h)
};

// class-block layout of this rank's rows inside the global blocks
struct Shard {
  int64_t n_sig_g = 0, n_bkg_g = 0;  // global block sizes
  int64_t s0 = 0, b0 = 0;            // this rank's offsets in each block
  int64_t n_sig_l = 0;               // this rank's signal rows
  bool dist = false;
};

// numpy's pairwise summation (pairwise() above) on the device: the host
// enumerates the recursion's leaves (<= 128 elements), a kernel sums each
// leaf with numpy's rule, the host combines the leaf sums in recursion order
static void pw_leaves(int64_t off, int64_t n, std::vector<long long>& lo, std::vector<int>& ln) {
  if (n <= 128) {
    lo.push_back(off);
    ln.push_back((int)n);
    return;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  pw_leaves(off, n2, lo, ln);
  pw_leaves(off + n2, n - n2, lo, ln);
}

static double pw_combine(int64_t n, const double* leaf, size_t& k) {
  if (n <= 128) return leaf[k++];
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  const double a = pw_combine(n2, leaf, k);
  const double b = pw_combine(n - n2, leaf, k);
  return a + b;
}

__global__ void k_pairwise_leaves(const double* __restrict__ a, const long long* __restrict__ off,
                                  const int* __restrict__ len, int L, double* __restrict__ out) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < L; e += gridDim.x * blockDim.x) {
    const double* x = a + off[e];
    const int n = len[e];
    double res;
    if (n < 8) {
      res = 0.0;
      for (int i = 0; i < n; ++i) res = __dadd_rn(res, x[i]);
    } else {
      double r[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = x[j];
      int i;
      for (i = 8; i < n - (n % 8); i += 8)
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], x[i + j]);
      res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                      __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
      for (; i < n; ++i) res = __dadd_rn(res, x[i]);
    }
    out[e] = res;
  }
}

// max |w| (as ordered bits) and a non-finite flag
__global__ void k_weight_stats(const double* __restrict__ w, int64_t n, unsigned long long* __restrict__ maxbits,
                               unsigned int* __restrict__ bad) {
  double m = 0.0;
  bool b = false;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double v = w[i];
    b |= !isfinite(v);
    m = fmax(m, fabs(v));
  }
  for (int o = 16; o > 0; o >>= 1) {
    m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    b |= __shfl_xor_sync(0xffffffffu, (int)b, o) != 0;
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(maxbits, (unsigned long long)__double_as_longlong(m));
    if (b) atomicOr(bad, 1u);
  }
}

// stream-ordered arena: every allocation of one call, freed at the end
struct Arena {
  cudaStream_t s;
  std::vector<void*> ptrs;
  explicit Arena(cudaStream_t st) : s(st) {}
  template <typename T>
  T* alloc(size_t count) {
    void* p = nullptr;
    if (count == 0) count = 1;
    BB_CUDA(cudaMallocAsync(&p, count * sizeof(T), s));
    ptrs.push_back(p);
    return reinterpret_cast<T*>(p);
  }
  void release(void* p) {
    for (auto& q : ptrs)
      if (q == p) {
        cudaFreeAsync(q, s);
        q = nullptr;
      }
  }
  ~Arena() {
    for (void* p : ptrs)
      if (p) cudaFreeAsync(p, s);
  }
};

// Kernel launch with programmatic stream serialization (common.cuh pdl_wait):
// the kernel may be scheduled while the previous kernel of the stream drains.
template <typename... KArgs, typename... Args>
static void launch_k(bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                     Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  BB_CUDA(cudaLaunchKernelEx(&cfg, kern, KArgs(std::forward<Args>(args))...));
}

static int grid_for(int64_t n, int threads, int sm, int per_sm = 8) {
  const int64_t want = ceil_div(n, threads);
  return (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sm * per_sm));
}

static double elapsed_ms(std::chrono::steady_clock::time_point a) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - a).count();
}

// ------------------------------------------------------------- binning
template <typename T>
struct BinResult {
  double* bounds;                       // device [d][B-1]
  typename KeyOf<T>::K* bkeys;          // device [d][B-1]
  std::vector<unsigned long long> finite, nans;
};

constexpr int kSmemHistBins = 8192;  // k_select_hist shared counters

template <typename T>
static void run_select(Ctx& c, Arena& A, const typename KeyOf<T>::K* keys, int64_t n, int d, int levels,
                       const unsigned long long* finite_dev, double* bounds, typename KeyOf<T>::K* bkeys,
                       bool dist = false) {
  using K = typename KeyOf<T>::K;
  constexpr int KB = sizeof(K) * 8;
  const int B = 1 << levels, nt = B - 1;
  SelectState<K> st;
  st.nt = nt;
  st.hist_cap = std::max<int64_t>(4096, (int64_t)nt * 256);
  st.tgt_prefix = A.alloc<K>((size_t)d * nt);
  st.tgt_rank = A.alloc<unsigned long long>((size_t)d * nt);
  st.tgt_group = A.alloc<int>((size_t)d * nt);
  st.grp_prefix = A.alloc<K>((size_t)d * nt);
  st.grp_first_tgt = A.alloc<int>((size_t)d * nt);
  st.grp_count = A.alloc<int>(d);
  st.hist = A.alloc<unsigned int>((size_t)d * st.hist_cap);
  st.finite_cnt = finite_dev;
  BB_CUDA(cudaMemsetAsync(st.hist, 0, (size_t)d * st.hist_cap * 4, c.stream));
  k_select_init<K><<<d, 256, 0, c.stream>>>(st, B);
  BB_LAUNCH_CHECK();
  int resolved = 0;
  const int gx = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256 * 8), std::max(1, 2 * c.sm_count * 8 / d + 1)));
  while (resolved < KB) {
    int db = (resolved == 0) ? 12 : 8;
    db = std::min(db, KB - resolved);
    if (n > 0) {
      k_select_hist<K><<<dim3(gx, d), 256, kSmemHistBins * 4, c.stream>>>(keys, n, st, resolved, db, kSmemHistBins);
      BB_LAUNCH_CHECK();
    }
    if (dist) c.comm.all_reduce(st.hist, (size_t)d * st.hist_cap, kNcclU32, kNcclSum, c.stream);
    k_select_scan<K><<<d, 1024, 0, c.stream>>>(st, db);
    BB_LAUNCH_CHECK();
    resolved += db;
  }
  k_select_finish<K><<<d, 256, 0, c.stream>>>(st, bounds, bkeys);
  BB_LAUNCH_CHECK();
}

template <typename T>
static typename KeyOf<T>::K* make_keys(Ctx& c, Arena& A, const T* Xd, int64_t n, int d,
                                       std::vector<unsigned long long>& finite, std::vector<unsigned long long>& nans,
                                       unsigned long long** finite_dev_out, bool dist = false) {
  using K = typename KeyOf<T>::K;
  K* keys = A.alloc<K>((size_t)n * d);
  unsigned long long* cnt = A.alloc<unsigned long long>(2 * (size_t)d);
  BB_CUDA(cudaMemsetAsync(cnt, 0, 2 * (size_t)d * 8, c.stream));
  if (n > 0) {
    k_transpose_keys<T><<<dim3((unsigned)ceil_div(n, 32), (unsigned)ceil_div(d, 32)), dim3(32, 8), 0, c.stream>>>(
        Xd, n, d, keys, cnt, cnt + d);
    BB_LAUNCH_CHECK();
  }
  if (dist) c.comm.all_reduce(cnt, 2 * (size_t)d, kNcclU64, kNcclSum, c.stream);
  finite.assign(d, 0);
  nans.assign(d, 0);
  BB_CUDA(cudaMemcpyAsync(finite.data(), cnt, (size_t)d * 8, cudaMemcpyDeviceToHost, c.stream));
  BB_CUDA(cudaMemcpyAsync(nans.data(), cnt + d, (size_t)d * 8, cudaMemcpyDeviceToHost, c.stream));
  BB_CUDA(cudaStreamSynchronize(c.stream));
  *finite_dev_out = cnt;
  return keys;
}

// ------------------------------------------------------------- tree loop
struct FitStats {
  double mask_ms = 0.0, hist_ms = 0.0;
  int64_t launches = 0, hist_launches = 0;
};

struct FitShape {
  int64_t n, n_sig;
  int d, levels, B, depth, n_internal, n_nodes, T;
};

template <typename CodeT, typename NodeT>
static HistPlan plan_layer(int layer, const FitShape& s, int sm_count, bool sib_ok = true) {
  HistPlan p{};
  p.prof = getenv("BB_HIST_PROFILE") ? atoi(getenv("BB_HIST_PROFILE")) : 0;
  p.nodes = 1 << (layer - 1);
  p.start = p.nodes - 1;
  p.sib = (sib_ok && layer >= 2) ? 1 : 0;  // left children only; right = parent - left (k_split)
  const int built = p.sib ? p.nodes / 2 : p.nodes;
  constexpr int64_t kSmemMax = 227 * 1024 - 1024;
  static const int64_t hist_budget = (getenv("BB_HIST_BUDGET_KB") ? atoi(getenv("BB_HIST_BUDGET_KB")) : 160) * 1024;
  const int64_t fn_budget = std::max<int64_t>(1, hist_budget / ((int64_t)s.B * 8));
  if (built <= fn_budget) {
    p.ngs = built;
    p.n_ng = 1;
    const int fg = (int)std::min<int64_t>(s.d, fn_budget / built);
    p.n_fg = (int)ceil_div(s.d, fg);
    p.fg = (int)ceil_div(s.d, p.n_fg);
  } else {
    p.fg = 1;
    p.n_fg = s.d;
    p.ngs = (int)fn_budget;
    p.n_ng = (int)ceil_div(built, p.ngs);
  }
  const int tile = kTile;
  auto need = [&](int fg) {
    return (int64_t)align16((p.ngs * fg * s.B + 32) * 8) + 2 * (int64_t)hist_buf_bytes<CodeT, NodeT>(tile, fg) + 4 * tile + 64;
  };
  while (p.fg > 1 && need(p.fg) > kSmemMax) {
    p.n_fg += 1;
    p.fg = (int)ceil_div(s.d, p.n_fg);
    p.n_fg = (int)ceil_div(s.d, p.fg);
  }
  while (p.ngs > 1 && need(p.fg) > kSmemMax) {  // a budget above what the stage leaves: fewer nodes per group
    p.ngs -= 1;
    p.n_ng = (int)ceil_div(built, p.ngs);
  }
  if (need(p.fg) > kSmemMax) {
    if (s.B <= 2048) throw InvalidArg{"histogram stage does not fit in shared memory"};
    p.global_only = 1;  // binning_levels 12..15: the global-atomic kernel
  }
  p.tile = tile;
  p.smem = (int)need(p.fg);
  p.tiles_sig0 = 0;
  p.tiles_sig1 = (int)ceil_div(s.n_sig, tile);
  p.tiles_bkg0 = (int)(s.n_sig / tile);
  p.tiles_bkg1 = (int)ceil_div(s.n, tile);
  // one CTA per SM, leaving 9 SMs to the concurrent mask streams (their
  // chain / tail / pass CTAs need room while a histogram launch runs)
  const int groups = p.n_fg * p.n_ng;
  static const int reserve = getenv("BB_HIST_RESERVE") ? atoi(getenv("BB_HIST_RESERVE")) : 9;  // SMs left to the mask streams
  const int per_sm = std::max(1, std::min(2, (int)((228 * 1024) / (p.smem + 2048))));  // resident CTAs per SM
  const int total = std::max(2, (int)(per_sm * (sm_count - reserve) / groups));
  const int ts = p.tiles_sig1 - p.tiles_sig0, tb = p.tiles_bkg1 - p.tiles_bkg0;
  p.split_sig = std::max(1, std::min(ts, (int)std::llround((double)total * ts / (ts + tb))));
  p.split_bkg = std::max(1, std::min(tb, total - p.split_sig));
  return p;
}

// shared-memory plans needing more (node, feature) groups than this (each
// re-reads every row) use the global-atomic histogram instead
static int hist_global_groups() {
  const char* e = getenv("BB_HIST_GLOBAL_GROUPS");  // read per call: tests force either path
  return e ? atoi(e) : 40;  // cfg5 (B = 1024): the warp kernel wins up to ~34 groups (profiles)
}

static bool hist_warp_mode() {  // the warp-independent histogram kernel (BB_HIST_WARP=0: the CTA-barrier one)
  const char* e = getenv("BB_HIST_WARP");
  return !e || atoi(e) != 0;
}

static int hist_reserve() {  // SMs left to the concurrent mask streams during a histogram launch
  static const int r = getenv("BB_HIST_RESERVE") ? atoi(getenv("BB_HIST_RESERVE")) : 9;
  return r;
}

static inline int hist_grid(const HistPlan& p) { return p.n_fg * p.n_ng * (p.split_sig + p.split_bkg); }

// Histogram path: BB_HIST_PATH = fl | w | cta | g (read per call: tests force
// each path); default: feature-lane kernel where its plan fits, else the
// warp-independent one (or global atomics for many-group plans).
static int hist_path_env() {
  const char* e = getenv("BB_HIST_PATH");
  if (!e) return 0;
  if (!strcmp(e, "fl")) return 1;
  if (!strcmp(e, "w")) return 2;
  if (!strcmp(e, "cta")) return 3;
  if (!strcmp(e, "g")) return 4;
  if (!strcmp(e, "list")) return 5;
  return 0;
}

// Tensor maps (driver entry point; no libcuda link) for the feature-lane
// histogram's 2-D code boxes.
static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult qr;
    BB_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &qr));
    if (!f || qr != cudaDriverEntryPointSuccess) throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

// codes viewed as 2-D [tiles * d feature columns][kTile codes], boxes of
// [fpad columns][128 bytes], 128-byte swizzle
template <typename CodeT>
static void make_code_map(CUtensorMap* tm, const CodeT* codes, int64_t tiles, int d, int fpad) {
  const cuuint64_t dims[2] = {(cuuint64_t)kTile, (cuuint64_t)(tiles * d)};
  const cuuint64_t strides[1] = {(cuuint64_t)kTile * sizeof(CodeT)};
  const cuuint32_t box[2] = {(cuuint32_t)(128 / sizeof(CodeT)), (cuuint32_t)fpad};
  const cuuint32_t es[2] = {1, 1};
  const CUresult r = tensor_map_encoder()(
      tm, sizeof(CodeT) == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_UINT16, 2,
      const_cast<CodeT*>(codes), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
}

// Plan of k_layer_hist_fl (kernels_hist_fl.cuh): work types = class x
// feature group (up to 64 features: 32 lanes x 1 row, plus a remainder sub
// with 1, 2 or 4 row copies) x node group (nodes whose lane-interleaved
// 2-limb slots fit next to the ring); one CTA per SM, split across types in
// proportion to their estimated work.  n_types == 0: no feasible plan (wide
// bins).
template <typename CodeT, typename NodeT>
static FlPlan plan_fl(int layer, const FitShape& s, int sm_count, bool sib_ok, const CodeT* codes) {
  FlPlan p{};
  p.nodes = 1 << (layer - 1);
  p.start = p.nodes - 1;
  p.sib = (sib_ok && layer >= 2) ? 1 : 0;
  p.log2b = s.levels;
  const int built = p.sib ? p.nodes / 2 : p.nodes;
  if (s.B > 256) return FlPlan{};
  auto rl = [](int r) { return r > 16 ? 0 : (r > 8 ? 1 : 2); };
  struct FG { int f0, fc0, r0log, fc1, r1log, fpad; };
  constexpr int kSmemMax = 227 * 1024;
  const int subb = (s.B + 1) * 256;
  const int fixed0 = 1024 + kFlMetaBytes + 2 * kFlMaxStages * 8;
  std::vector<FG> fgs;
  int nsub = 1;
  bool ok = false;
  for (int width : {64, 32}) {  // features per type: merged remainder first
    fgs.clear();
    nsub = 1;
    for (int f0 = 0; f0 < s.d; f0 += width) {
      const int r = std::min(width, s.d - f0);
      FG g{};
      g.f0 = f0;
      if (r > 32) {
        g.fc0 = 32; g.r0log = 0; g.fc1 = r - 32; g.r1log = rl(r - 32);
        nsub = 2;
      } else {
        g.fc0 = r; g.r0log = rl(r); g.fc1 = 0; g.r1log = 0;
      }
      g.fpad = (g.fc0 + g.fc1 + 7) & ~7;
      fgs.push_back(g);
    }
    p.stage_bytes = fl_stage_bytes<CodeT, NodeT>(fgs[0].fpad);
    for (int ns : {3, 2}) {
      if (fixed0 + ns * p.stage_bytes + nsub * subb <= kSmemMax) {
        p.stages = ns;
        ok = true;
        break;
      }
    }
    if (ok) break;
  }
  if (!ok) return FlPlan{};
  const int nc_fit = (kSmemMax - fixed0 - p.stages * p.stage_bytes) / (nsub * subb);
  const int n_ng = (int)ceil_div(built, std::min(built, nc_fit));
  // one node group only: every further group re-reads all rows for a
  // shrinking share of contributing ones (measured: cfg3 layers 3-5 at 2, 4,
  // 8 groups run 1.5-2.7x slower than the warp-independent kernel, which
  // holds all of a layer's nodes); BB_HIST_PATH=fl forces it
  const char* pe = getenv("BB_HIST_PATH");
  if (n_ng > 1 && !(pe && !strcmp(pe, "fl"))) return FlPlan{};
  p.ngs = (int)ceil_div(built, n_ng);
  p.hist_bytes = p.ngs * nsub * subb;
  p.smem = fixed0 + p.stages * p.stage_bytes + p.hist_bytes;
  const int64_t tiles = ceil_div(s.n, kTile);
  make_code_map(&p.tm[0], codes, tiles, s.d, fgs[0].fpad);
  if (fgs.back().fpad != fgs[0].fpad) make_code_map(&p.tm[1], codes, tiles, s.d, fgs.back().fpad);
  static const int reserve = getenv("BB_HIST_RESERVE") ? atoi(getenv("BB_HIST_RESERVE")) : 9;
  const int total = std::max(1, sm_count - reserve);
  const int64_t st_sig0 = 0, st_sig1 = ceil_div(s.n_sig, kFlRows);
  const int64_t st_bkg0 = s.n_sig / kFlRows, st_bkg1 = ceil_div(s.n, kFlRows);
  std::vector<FlType> ts;
  std::vector<double> w;
  const double frac0 = 0.5 * (p.sib ? 0.5 : 1.0) / n_ng;  // contributing share of a class's rows (alpha ~ 0.5)
  auto steps = [&](int r_log) {                            // warp steps per row of a sub
    const int R = 1 << r_log;
    return (1.0 - std::pow(1.0 - frac0, R)) / R;
  };
  for (int cls = 0; cls < 2; ++cls) {
    const int64_t a = cls ? st_bkg0 : st_sig0, b = cls ? st_bkg1 : st_sig1;
    if (b <= a) continue;
    for (size_t gi = 0; gi < fgs.size(); ++gi) {
      const FG& g = fgs[gi];
      for (int ng = 0; ng < n_ng; ++ng) {
        FlType t{};
        t.t0 = (int)a;
        t.t1 = (int)b;
        t.cls = (short)cls;
        t.f0 = (short)g.f0;
        t.fc0 = (short)g.fc0;
        t.r0log = (short)g.r0log;
        t.fc1 = (short)g.fc1;
        t.r1log = (short)g.r1log;
        t.fpad = (short)g.fpad;
        t.map = (short)(g.fpad == fgs[0].fpad ? 0 : 1);
        t.n0 = (short)(ng * p.ngs);
        t.ncount = (short)std::min(p.ngs, built - ng * p.ngs);
        w.push_back((double)(b - a) * (0.6 + 3.0 * (steps(g.r0log) + (g.fc1 ? steps(g.r1log) : 0.0))));
        ts.push_back(t);
      }
    }
  }
  if (ts.empty() || (int)ts.size() > kFlMaxTypes || (int)ts.size() > total) return FlPlan{};
  double wsum = 0;
  for (double x : w) wsum += x;
  int used = 0;
  for (size_t i = 0; i < ts.size(); ++i) {
    int k = (int)std::floor(total * w[i] / wsum);
    k = (int)std::max<int64_t>(1, std::min<int64_t>(k, ts[i].t1 - ts[i].t0));
    ts[i].nctas = k;
    used += k;
  }
  // hand the rounding remainder to the heaviest types (per CTA)
  while (used < total) {
    int best = -1;
    double bw = 0;
    for (size_t i = 0; i < ts.size(); ++i) {
      if (ts[i].nctas >= ts[i].t1 - ts[i].t0) continue;
      const double x = w[i] / ts[i].nctas;
      if (x > bw) { bw = x; best = (int)i; }
    }
    if (best < 0) break;
    ts[best].nctas += 1;
    used += 1;
  }
  int cta = 0;
  for (size_t i = 0; i < ts.size(); ++i) {
    ts[i].cta0 = cta;
    for (int k = 0; k < ts[i].nctas && cta + k < 256; ++k) p.cta_type[cta + k] = (unsigned char)i;
    cta += ts[i].nctas;
    p.t[i] = ts[i];
  }
  if (cta > 256) return FlPlan{};
  p.n_types = (int)ts.size();
  p.noflush = getenv("BB_FL_NOFLUSH") ? atoi(getenv("BB_FL_NOFLUSH")) : 0;
  return p;
}

// partial rows per CTA (elements) and the scratch a plan needs
static inline int64_t fl_cta_stride(const FlPlan& p, int B) {
  int rows = 0;
  for (int i = 0; i < p.n_types; ++i) rows = std::max(rows, p.t[i].ncount * (p.t[i].fc0 + p.t[i].fc1));
  return (int64_t)rows * B;
}

static inline int fl_grid(const FlPlan& p) { return p.n_types ? p.t[p.n_types - 1].cta0 + p.t[p.n_types - 1].nctas : 0; }

// one layer histogram launch on the chosen path (same slots, same exact sums)
template <typename CodeT, typename NodeT>
static void launch_layer_hist(const HistPlan& p, const FlPlan& fl, int sm_count, const CodeT* codes, int code_off,
                              const NodeT* node, const long long* q, int64_t n, int64_t n_sig, int d, int B,
                              unsigned long long* hist, cudaStream_t st, long long* partials) {
  const int path = hist_path_env();
  if ((path == 0 || path == 1) && fl.n_types > 0 && !getenv("BB_HIST_WARP") && !getenv("BB_HIST_GLOBAL_GROUPS")) {
    const bool use_partials = getenv("BB_FL_PARTIALS") && atoi(getenv("BB_FL_PARTIALS")) != 0;  // per call: tests
    if (partials && use_partials) {
      FlPlan f2 = fl;
      f2.partials = partials;
      f2.cta_stride = fl_cta_stride(fl, B);
      k_layer_hist_fl<CodeT, NodeT><<<fl_grid(f2), kFlThreads, f2.smem, st>>>(code_off, node, q, n, n_sig, d, B, f2,
                                                                             hist);
      BB_LAUNCH_CHECK();
      int rows = 0;
      for (int i = 0; i < f2.n_types; ++i) rows = std::max(rows, f2.t[i].ncount * (f2.t[i].fc0 + f2.t[i].fc1));
      k_fl_reduce<<<dim3(rows, f2.n_types), kFlRedThreads, 0, st>>>(d, B, f2, hist);
    } else {
      k_layer_hist_fl<CodeT, NodeT><<<fl_grid(fl), kFlThreads, fl.smem, st>>>(code_off, node, q, n, n_sig, d, B, fl,
                                                                             hist);
    }
  } else if (path == 4 || p.global_only || (path == 0 && p.n_fg * p.n_ng > hist_global_groups())) {
    k_layer_hist_g<CodeT, NodeT><<<8 * sm_count, 256, 0, st>>>(codes, code_off, node, q, n, n_sig, d, B, p, hist);
  } else if (path == 2 || (path != 3 && hist_warp_mode())) {
    k_layer_hist_w<CodeT, NodeT><<<hist_grid(p), kHistWThreads, p.smem, st>>>(codes, code_off, node, q, n, n_sig, d, B,
                                                                             p, hist);
  } else {
    k_layer_hist<CodeT, NodeT><<<hist_grid(p), kHistThreads, p.smem, st>>>(codes, code_off, node, q, n, n_sig, d, B, p,
                                                                           hist);
  }
  BB_LAUNCH_CHECK();
}

template <typename CodeT, typename NodeT>
static void set_hist_smem_attrs() {
  BB_CUDA(cudaFuncSetAttribute(k_layer_hist<CodeT, NodeT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
  BB_CUDA(cudaFuncSetAttribute(k_layer_hist_w<CodeT, NodeT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
  BB_CUDA(cudaFuncSetAttribute(k_layer_hist_fl<CodeT, NodeT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
}

// GPU subsample-mask generator on its own stream (kernels_mask.cuh).  One
// cluster launch parses a chunk of up to kChunk trees back to back (the u32
// draw stream is continuous across trees), so the 8-SM cluster is placed
// once per chunk; the per-tree resolution kernels follow.
constexpr int kChunk = 8;

// segment table of a block of n rows (kernels_seg.cuh seg_geom)
struct SegPlan {
  std::vector<SegTab> tab;
  std::vector<int2> tasks;
  int n_rec = 0;
};

// standard deviation of a job's draw count: sum over steps of (1-q)/q^2,
// q = (i+1)/(mask+1), integrated per band: (M+1)(1/qa - 1/qb + ln(qa/qb))
static double seg_draws_sd(int n) {
  double var = 0.0;
  double x = (double)n;  // i + 1 at the job's first step
  while (x > 1.0 + 1e-9) {
    const unsigned M = smear_host((unsigned)std::max(1.0, std::floor(x - 1.0)));
    const double mp1 = (double)M + 1.0, lowx = mp1 / 2.0;
    const double qa = lowx / mp1, qb = x / mp1;  // q at the band's last and first steps
    var += mp1 * (1.0 / qa - 1.0 / qb + std::log(qa / qb));
    x = lowx;
  }
  return std::sqrt(std::max(0.0, var));
}

// anchor slack of a job: 2 sd of the previous job's draw count
// (its first draw is predicted before that job is parsed), clamped
static long long seg_slack(int n_prev) {
  static const double k = getenv("BB_ANCHOR_SD") ? atof(getenv("BB_ANCHOR_SD")) : 2.0;
  return std::min<long long>(kAnchorSlackMax,
                             std::max<long long>(kAnchorSlackMin, (long long)std::ceil(k * seg_draws_sd(n_prev))));
}

static SegPlan build_seg_plan(int n, long long slack, bool throughput_plan) {
  SegPlan P;
  if (n - 1 < kSegTail) return P;
  long long off = 0;
  SegTab t{};
  // Plan shape.  Large fits (>= 4M rows) are bound by the tree kernels, which
  // share the SMs with phase 1: shorter segments and 3-sd windows cut the
  // phase-1 work (cfg3: 720 -> 663 ms per fit; a start outside its window only
  // costs an exact walk of that segment).  Small fits are bound by the mask
  // pipeline's latency: 5-sd windows (no exact walks on the critical
  // path; cfg2 at 3 sd: 101 -> 112 ms) of 8192 draws (cfg2: 60 ms per fit; 67 ms
  // at 16384 and 101 ms at 32768 draws, whose phase-1 warps the chain then
  // waits for).  BB_SEG_LEN / BB_SEG_SD override.
  const int max_len = getenv("BB_SEG_LEN") ? std::max(256, std::min(kSegMaxLen, atoi(getenv("BB_SEG_LEN"))))
                                           : (throughput_plan ? 16384 : 8192);
  const double window_sd = getenv("BB_SEG_SD") ? atof(getenv("BB_SEG_SD")) : (throughput_plan ? 3.0 : (double)BB_SEG_WINDOW_SD);
  while (seg_geom(n - 1, off, kSegTail, &t, 2 * slack, max_len, window_sd)) {
    t.rec_off = P.n_rec;
    const int ns = t.nA + t.nB;
    // phase-1 tasks (kernels_seg.cuh): one warp per piece whose window is a
    // small share of its band (few ambiguous draws), else one warp per
    // 512-state sub-window
    auto piece = [&](int pl, int ph, int np, int code, int j0) {
      if (np <= 0) return;
      const double band = (double)smear_host((unsigned)ph) + 1.0;
      static const double ratio = getenv("BB_PIECE_RATIO") ? atof(getenv("BB_PIECE_RATIO")) : 64.0;
      if ((double)(ph - pl + 1 + kSub) * ratio <= band) {
        P.tasks.push_back(int2{(int)P.tab.size(), code});
      } else {
        for (int j = 0; j < np; ++j) P.tasks.push_back(int2{(int)P.tab.size(), j0 + j});
      }
    };
    piece(t.loA, t.hiA, t.nA, -1, 0);
    piece(t.loB, t.hiB, t.nB, -2, t.nA);
    P.n_rec += ns;
    P.tab.push_back(t);
    off += t.len;
    // safety net: ~4x the expected draws of the job in 256-draw segments
    if (P.tab.size() > 64 + (size_t)(4.0 * seg_expected_draws(n - 1) / 256.0)) break;
  }
  return P;
}

struct MaskGen {
  PcgJump* jump = nullptr;
  RngState* rng = nullptr;
  unsigned int* draws = nullptr;
  long long n_draws = 0;
  int* J[2] = {nullptr, nullptr};
  int *cnt = nullptr, *off = nullptr, *fill = nullptr, *bucket = nullptr, *sums = nullptr;
  long long* prof = nullptr;  // BB_PARSE_PROFILE: phase cycles, printed at the end
  unsigned char* removed[2] = {nullptr, nullptr};
  int n[2] = {0, 0}, k[2] = {0, 0};
  int sm = 148;
  Shard sh;                       // sh.dist: slice the global bits to this rank
  long long sh_n_local = 0;       // this rank's rows
  unsigned int* gbits = nullptr;  // global bits scratch (sharded fits)
  // segment-parallel parse (kernels_seg.cuh)
  SegTab* tab[2] = {nullptr, nullptr};
  int2* tasks[2] = {nullptr, nullptr};
  int S[2] = {0, 0}, n_tasks[2] = {0, 0};
  SegRec* rec[2] = {nullptr, nullptr};          // by job parity
  int *seg_start[2] = {nullptr, nullptr}, *n_seg[2] = {nullptr, nullptr};
  long long slack[2] = {0, 0};                    // anchor slack per class
  long long exp_draws[2] = {0, 0};                // expected draws of a job per class
  cudaEvent_t evF[2] = {}, evC = nullptr, evTl = nullptr;
  long long* spos = nullptr;     // true first draw of each job of a chunk
  long long* sanchor = nullptr;  // anchor (predicted first draw + slack) of each job
  long long* stail = nullptr;    // chain -> tail hand-off: draw
  int* stail_i = nullptr;        //                         state
  cudaStream_t sb = nullptr;     // phase 1 stream (overlaps the tails)
  cudaStream_t se = nullptr;     // phase 3 (emit) stream: phase 1 of job j+2 does not queue behind emit(j)
  cudaEvent_t evE[2] = {}, evEnd = nullptr;
  cudaStream_t sg = nullptr;     // the chunk's draws beyond the first two jobs
  cudaEvent_t evPre = nullptr, evG2 = nullptr;
  cudaStream_t sc = nullptr;     // value resolution + mask bits (overlaps the next chunk's parse)
  cudaEvent_t evA = nullptr, evB = nullptr;
  cudaEvent_t evT[kChunk] = {};  // tree t of the chunk emitted (sb -> sc)
  cudaEvent_t evR[2] = {};       // resolution of the chunk that used J half p done (sc -> st)
  int parity = 0;                // J buffer half of the current chunk
  RngState* rng0 = nullptr;

  void init(Arena& A, cudaStream_t st, int64_t n_sig, int64_t n_bkg, double rate, const bb_fit_config& cfg,
            int sm_count) {
    sm = sm_count;
    n[0] = (int)n_sig;
    n[1] = (int)n_bkg;
    k[0] = (int)subsample_count(n_sig, rate);
    k[1] = (int)subsample_count(n_bkg, rate);
    PcgJump hj;
    U128 a{0x4385DF649FCCF645ull, 0x2360ED051FC65DA4ull};
    U128 c{cfg.pcg_inc_lo, cfg.pcg_inc_hi};
    for (int j = 0; j < 64; ++j) {
      hj.A[j] = a;
      hj.C[j] = c;
      c = u128_add(u128_mul(a, c), c);
      a = u128_mul(a, a);
    }
    RngState hr;
    hr.s = U128{cfg.pcg_state_lo, cfg.pcg_state_hi};
    hr.inc = U128{cfg.pcg_inc_lo, cfg.pcg_inc_hi};
    hr.has_uint32 = cfg.pcg_has_uint32;
    hr.uinteger = cfg.pcg_uinteger;
    jump = A.alloc<PcgJump>(1);
    rng = A.alloc<RngState>(1);
    BB_CUDA(cudaMemcpyAsync(jump, &hj, sizeof(hj), cudaMemcpyHostToDevice, st));
    BB_CUDA(cudaMemcpyAsync(rng, &hr, sizeof(hr), cudaMemcpyHostToDevice, st));
    BB_CUDA(cudaStreamSynchronize(st));  // host staging structs go out of scope
    const int64_t steps = n_sig + n_bkg;
    const int chunk = kChunk;
    // E[draws/step] = mean of (mask+1)/(i+1) <= ~1.45 (2 ln 2 asymptotically) and < 2
    // always; beyond the buffer the parse falls back to per-draw jump-ahead
    n_draws = (long long)(2.0 * (double)steps * chunk) + 65536;
    draws = A.alloc<unsigned int>((size_t)n_draws);
    const int nmax = std::max(n[0], n[1]);
    for (int cc = 0; cc < 2; ++cc) {
      J[cc] = A.alloc<int>((size_t)std::max(1, std::max(n[0], n[1])) * chunk * 2);  // stride = larger class; 2 chunks
      removed[cc] = A.alloc<unsigned char>(std::max(1, n[cc]));
    }
    cnt = A.alloc<int>(nmax + 1);
    off = A.alloc<int>(nmax + 1);
    fill = A.alloc<int>(nmax + 1);
    bucket = A.alloc<int>(nmax + 1);
    sums = A.alloc<int>(ceil_div(nmax, kScanBlock) + 1);
    if (getenv("BB_PARSE_PROFILE")) {
      prof = A.alloc<long long>(32);
      BB_CUDA(cudaMemsetAsync(prof, 0, 256, st));
    }
    gbits = A.alloc<unsigned int>((size_t)ceil_div(steps, 32) + 1);
    int smax = 1, rmax = 1;
    for (int cc = 0; cc < 2; ++cc) {
      // class cc's jobs follow jobs of the other class (sig, bkg alternate)
      slack[cc] = seg_slack(n[1 - cc]);
      exp_draws[cc] = n[cc] > 1 ? (long long)std::llround(seg_expected_draws(n[cc] - 1)) : 0;
      const SegPlan P = build_seg_plan(n[cc], slack[cc], (long long)n[0] + n[1] >= 4000000);
      S[cc] = (int)P.tab.size();
      n_tasks[cc] = (int)P.tasks.size();
      tab[cc] = A.alloc<SegTab>(std::max<size_t>(1, P.tab.size()));
      tasks[cc] = A.alloc<int2>(std::max<size_t>(1, P.tasks.size()));
      if (S[cc]) BB_CUDA(cudaMemcpyAsync(tab[cc], P.tab.data(), P.tab.size() * sizeof(SegTab), cudaMemcpyHostToDevice, st));
      if (n_tasks[cc])
        BB_CUDA(cudaMemcpyAsync(tasks[cc], P.tasks.data(), P.tasks.size() * sizeof(int2), cudaMemcpyHostToDevice, st));
      BB_CUDA(cudaStreamSynchronize(st));
      smax = std::max(smax, S[cc]);
      rmax = std::max(rmax, P.n_rec);
      if (getenv("BB_PARSE_PROFILE"))
        fprintf(stderr, "seg plan n=%d: %d segments, %d phase-1 pieces, %d records\n", n[cc], S[cc], n_tasks[cc], P.n_rec);
    }
    for (int q = 0; q < 2; ++q) {
      rec[q] = A.alloc<SegRec>((size_t)rmax);
      seg_start[q] = A.alloc<int>(smax);
      n_seg[q] = A.alloc<int>(1);
    }
    spos = A.alloc<long long>(2 * (size_t)chunk + 2);
    sanchor = A.alloc<long long>(2 * (size_t)chunk + 2);
    stail = A.alloc<long long>(1);
    stail_i = A.alloc<int>(1);
    int lo_prio = 0, hi_prio = 0;
    BB_CUDA(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
    // BB_MASK_PRIO: 0 all mask streams high priority; 1 phase 1 high, emits /
    // resolution / draws normal; 2 all normal (the chain stream stays high)
    static const int prio_mode = getenv("BB_MASK_PRIO") ? atoi(getenv("BB_MASK_PRIO")) : 2;
    const int p_sb = prio_mode >= 2 ? lo_prio : hi_prio, p_rest = prio_mode >= 1 ? lo_prio : hi_prio;
    BB_CUDA(cudaStreamCreateWithPriority(&sb, cudaStreamNonBlocking, p_sb));
    BB_CUDA(cudaEventCreateWithFlags(&evA, cudaEventDisableTiming));
    BB_CUDA(cudaEventCreateWithFlags(&evB, cudaEventDisableTiming));
    BB_CUDA(cudaEventCreateWithFlags(&evC, cudaEventDisableTiming));
    BB_CUDA(cudaEventCreateWithFlags(&evTl, cudaEventDisableTiming));
    for (int q = 0; q < 2; ++q) BB_CUDA(cudaEventCreateWithFlags(&evF[q], cudaEventDisableTiming));
    BB_CUDA(cudaStreamCreateWithPriority(&sc, cudaStreamNonBlocking, p_rest));
    BB_CUDA(cudaStreamCreateWithPriority(&se, cudaStreamNonBlocking, p_rest));
    for (int q = 0; q < 2; ++q) BB_CUDA(cudaEventCreateWithFlags(&evE[q], cudaEventDisableTiming));
    BB_CUDA(cudaEventCreateWithFlags(&evEnd, cudaEventDisableTiming));
    BB_CUDA(cudaStreamCreateWithPriority(&sg, cudaStreamNonBlocking, p_rest));
    BB_CUDA(cudaEventCreateWithFlags(&evPre, cudaEventDisableTiming));
    BB_CUDA(cudaEventCreateWithFlags(&evG2, cudaEventDisableTiming));
    for (int q = 0; q < kChunk; ++q) BB_CUDA(cudaEventCreateWithFlags(&evT[q], cudaEventDisableTiming));
    for (int q = 0; q < 2; ++q) BB_CUDA(cudaEventCreateWithFlags(&evR[q], cudaEventDisableTiming));
    rng0 = A.alloc<RngState>(1);
    BB_CUDA(cudaFuncSetAttribute(k_seg_pass, cudaFuncAttributeMaxDynamicSharedMemorySize, kSegPassSmem));
    BB_CUDA(cudaFuncSetAttribute(k_seg_tail, cudaFuncAttributeMaxDynamicSharedMemorySize, kSegTailSmem));
    BB_CUDA(cudaFuncSetAttribute(k_seg_chain, cudaFuncAttributeMaxDynamicSharedMemorySize, kSegComposeSmem));
  }
  void sync() {
    if (sg) cudaStreamSynchronize(sg);
    if (sb) cudaStreamSynchronize(sb);
    if (se) cudaStreamSynchronize(se);
    if (sc) cudaStreamSynchronize(sc);
  }
  ~MaskGen() {
    if (sg) {
      cudaStreamSynchronize(sg);
      cudaStreamDestroy(sg);
    }
    if (evPre) cudaEventDestroy(evPre);
    if (evG2) cudaEventDestroy(evG2);
    if (se) {
      cudaStreamSynchronize(se);
      cudaStreamDestroy(se);
    }
    for (int q = 0; q < 2; ++q)
      if (evE[q]) cudaEventDestroy(evE[q]);
    if (evEnd) cudaEventDestroy(evEnd);
    if (sb) {
      cudaStreamSynchronize(sb);
      cudaStreamDestroy(sb);
    }
    if (sc) {
      cudaStreamSynchronize(sc);
      cudaStreamDestroy(sc);
    }
    if (evA) cudaEventDestroy(evA);
    if (evB) cudaEventDestroy(evB);
    if (evC) cudaEventDestroy(evC);
    if (evTl) cudaEventDestroy(evTl);
    for (int q = 0; q < 2; ++q)
      if (evF[q]) cudaEventDestroy(evF[q]);
    for (int q = 0; q < kChunk; ++q)
      if (evT[q]) cudaEventDestroy(evT[q]);
    for (int q = 0; q < 2; ++q)
      if (evR[q]) cudaEventDestroy(evR[q]);
  }
  void report(cudaStream_t st) {
    if (!prof) return;
    long long h[32];
    cudaStreamSynchronize(st);
    cudaMemcpy(h, prof, 256, cudaMemcpyDeviceToHost);
    fprintf(stderr, "parse prof:");
    for (int q = 0; q < 32; ++q) fprintf(stderr, " %lld", h[q]);
    fprintf(stderr, "\n");
  }

  // segment-parallel parse of `count` trees (2 * count block jobs)
  int64_t enqueue_seg(cudaStream_t st, int count) {
    int64_t launches = 0;
    const int jobs = 2 * count;
    BB_CUDA(cudaMemcpyAsync(rng0, rng, sizeof(RngState), cudaMemcpyDeviceToDevice, st));
    // job 0 starts at draw 0; job 1's first draw is predicted from job 0's length
    k_seg_init<<<1, 1, 0, st>>>(spos, sanchor, slack[0], exp_draws[0] + slack[1]);
    BB_LAUNCH_CHECK();
    const long long stride = std::max(n[0], n[1]);
    SegArgs base{};
    base.draws = draws;
    base.n_draws = n_draws;
    base.jump = jump;
    base.rng0 = rng0;
    base.rng = rng;
    base.tail_p = stail;
    base.tail_i = stail_i;
    base.prof = prof;
    auto args = [&](int jj) {  // the job-parity buffers of job jj
      SegArgs a = base;
      a.rec = rec[jj & 1];
      a.seg_start = seg_start[jj & 1];
      a.n_seg = n_seg[jj & 1];
      return a;
    };
    auto make_job = [&](int jj) {
      SegJob job{};
      if (jj < jobs) {
        const int t = jj >> 1, cc = jj & 1;
        job.n = n[cc];
        job.k = k[cc];
        job.S = S[cc];
        job.tab = tab[cc];
        job.tasks = tasks[cc];
        job.n_tasks = n_tasks[cc];
        job.J = J[cc] + (size_t)(parity * kChunk + t) * stride;
        job.pos_in = spos + jj;
        job.pos_out = spos + jj + 1;
        job.anchor_in = sanchor + jj;
        job.anchor2_out = jj + 2 < jobs ? sanchor + jj + 2 : nullptr;
        job.next_draws = exp_draws[1 - cc];
        job.slack2 = slack[cc];  // job jj+2 is of this job's class
        job.write_rng = jj == jobs - 1;
      }
      return job;
    };
    auto func = [&](int jj) {  // phase 1 of job jj (stream sb)
      if (jj == 2) BB_CUDA(cudaStreamWaitEvent(sb, evG2, 0));  // draws beyond the first two jobs
      const SegJob job = make_job(jj);
      if (job.n_tasks > 0) {
        SegArgs a = args(jj);
        a.func = job;
        a.emit = SegJob{};
        const int nbf = (int)ceil_div(job.n_tasks, kSubPerCta);
        k_seg_pass<<<nbf, kSegThreads, kSegPassSmem, sb>>>(a, nbf);
        BB_LAUNCH_CHECK();
        launches += 1;
      }
      BB_CUDA(cudaEventRecord(evF[jj & 1], sb));
    };
    auto emit = [&](int jj) {  // phase 3 of job jj (stream se)
      const SegJob job = make_job(jj);
      const int nb = (int)ceil_div(job.S, kSubPerCta);
      if (nb > 0) {
        SegArgs a = args(jj);
        a.func = SegJob{};
        a.emit = job;
        k_seg_pass<<<nb, kSegThreads, kSegPassSmem, se>>>(a, 0);
        BB_LAUNCH_CHECK();
        launches += 1;
      }
    };
    // stream st: chain(j) -> tail(j) -> chain(j+1) ...  Stream sb: phase 1 of
    // job j+2 right after tail(j) (its anchor is then known), overlapping
    // chain(j+1) + tail(j+1).  Stream se: phase 3 of job j after chain(j).
    // Records and segment starts alternate between two buffers by job parity
    // (chain(j+2) waits for emit(j), which reads the same seg_start).
    // BB_MASK_TIMELINE=1 (debug): per-job waits / chain / tail on the critical stream, printed at the end
    static const bool mtl_on = getenv("BB_MASK_TIMELINE") != nullptr;
    std::vector<cudaEvent_t> mtl;
    if (mtl_on) { mtl.emplace_back(); BB_CUDA(cudaEventCreate(&mtl.back())); BB_CUDA(cudaEventRecord(mtl.back(), st)); }
    BB_CUDA(cudaEventRecord(evA, st));
    BB_CUDA(cudaStreamWaitEvent(sb, evA, 0));
    func(0);
    if (jobs > 1) func(1);
    for (int jj = 0; jj < jobs; ++jj) {
      const SegJob job = make_job(jj);
      SegArgs a = args(jj);
      a.func = job;
      a.emit = SegJob{};
      BB_CUDA(cudaStreamWaitEvent(st, evF[jj & 1], 0));  // phase 1 of job jj done
      if (jj == 1) BB_CUDA(cudaStreamWaitEvent(st, evG2, 0));  // job 1 may read past the first part
      if (jj >= 2) BB_CUDA(cudaStreamWaitEvent(st, evE[jj & 1], 0));  // emit of jj-2 read this parity's seg_start
      if (mtl_on) { mtl.emplace_back(); BB_CUDA(cudaEventCreate(&mtl.back())); BB_CUDA(cudaEventRecord(mtl.back(), st)); }
      k_seg_chain<<<1, 64, kSegComposeSmem, st>>>(a);
      BB_LAUNCH_CHECK();
      BB_CUDA(cudaEventRecord(evC, st));
      if (mtl_on) { mtl.emplace_back(); BB_CUDA(cudaEventCreate(&mtl.back())); BB_CUDA(cudaEventRecord(mtl.back(), st)); }
      if (!kFuseTail) {
        k_seg_tail<<<1, 32, kSegTailSmem, st>>>(a);
        BB_LAUNCH_CHECK();
      }
      BB_CUDA(cudaEventRecord(evTl, st));
      if (mtl_on) { mtl.emplace_back(); BB_CUDA(cudaEventCreate(&mtl.back())); BB_CUDA(cudaEventRecord(mtl.back(), st)); }
      launches += 2;
      BB_CUDA(cudaStreamWaitEvent(se, evC, 0));
      emit(jj);
      BB_CUDA(cudaEventRecord(evE[jj & 1], se));
      if (jj & 1) BB_CUDA(cudaEventRecord(evT[jj >> 1], se));  // both jobs of tree jj/2 emitted
      if (jj + 2 < jobs) {
        BB_CUDA(cudaStreamWaitEvent(sb, evTl, 0));
        func(jj + 2);
      }
    }
    BB_CUDA(cudaEventRecord(evB, sb));
    BB_CUDA(cudaStreamWaitEvent(st, evB, 0));
    BB_CUDA(cudaEventRecord(evEnd, se));
    BB_CUDA(cudaStreamWaitEvent(st, evEnd, 0));  // the next chunk's draws overwrite what the emits read
    if (mtl_on) {
      mtl.emplace_back();
      BB_CUDA(cudaEventCreate(&mtl.back()));
      BB_CUDA(cudaEventRecord(mtl.back(), st));
      BB_CUDA(cudaEventSynchronize(mtl.back()));
      // events: start, then per job (before chain, before tail, after tail), then end
      double wait = 0, chain = 0, tail = 0;
      float x;
      for (int jj = 0; jj < jobs; ++jj) {
        cudaEvent_t prev = mtl[3 * jj], c0 = mtl[3 * jj + 1], t0 = mtl[3 * jj + 2], t1 = mtl[3 * jj + 3];
        BB_CUDA(cudaEventElapsedTime(&x, prev, c0)); wait += x;
        BB_CUDA(cudaEventElapsedTime(&x, c0, t0)); chain += x;
        BB_CUDA(cudaEventElapsedTime(&x, t0, t1)); tail += x;
      }
      BB_CUDA(cudaEventElapsedTime(&x, mtl[3 * jobs], mtl.back()));
      BB_CUDA(cudaEventElapsedTime(&x, mtl[0], mtl.back()));
      fprintf(stderr, "mask chunk: %d jobs, total %.3f ms: waits %.3f, chains %.3f, tails %.3f\n", jobs, x, wait, chain, tail);
      for (auto e : mtl) cudaEventDestroy(e);
    }
    return launches;
  }

  // masks of `count` consecutive trees; bits[j] = output words of tree j,
  // ready[j] (optional) recorded when tree j's bits are written
  void enqueue_chunk(cudaStream_t st, unsigned int* const* bits, int count, const cudaEvent_t* ready,
                     int64_t& launches) {
    // the first two jobs' draws on the critical stream, the rest on sg
    // (waited by chain(1) and by phase 1 of jobs >= 2)
    const long long n1 = std::min(n_draws, (long long)(1.25 * (double)(exp_draws[0] + exp_draws[1])) + 65536);
    auto draws_part = [&](long long lo, long long hi, cudaStream_t s2) {
      if (hi <= lo) return;
      const long long outs = (hi - lo) / 2 + 2;
      k_pcg_draws<<<(unsigned)ceil_div(ceil_div(outs, kDrawChunk), 256), 256, 0, s2>>>(jump, rng, draws, lo, hi);
      BB_LAUNCH_CHECK();
    };
    BB_CUDA(cudaEventRecord(evPre, st));
    draws_part(0, n1, st);
    BB_CUDA(cudaStreamWaitEvent(sg, evPre, 0));
    draws_part(n1, n_draws, sg);
    BB_CUDA(cudaEventRecord(evG2, sg));
    BB_CUDA(cudaStreamWaitEvent(st, evR[parity], 0));  // J half free (no-op before its first use)
    launches += enqueue_seg(st, count) + 1;
    const long long stride = std::max(n[0], n[1]);
    const int half = parity * kChunk;
    parity ^= 1;
    st = sc;  // value resolution and mask bits on their own stream
    for (int t = 0; t < count; ++t) {
      BB_CUDA(cudaStreamWaitEvent(sc, evT[t], 0));  // after this tree's jobs' J are emitted
      for (int cc = 0; cc < 2; ++cc) {
        const int nn = n[cc], kk = k[cc];
        int* Jt = J[cc] + (size_t)(half + t) * stride;
        // k == 0: nothing is active (position 0 is never a step target)
        if (kk == 0 || nn <= 1 || kk >= nn) {
          BB_CUDA(cudaMemsetAsync(removed[cc], kk == 0 ? 1 : 0, (size_t)std::max(1, nn), st));
          continue;
        }
        const bool buckets = getenv("BB_MASK_BUCKETS") && atoi(getenv("BB_MASK_BUCKETS")) != 0;  // per call: tests
        if (!buckets) {
          // sort-free resolution (kernels_mask.cuh k_up_min / k_resolve_values)
          BB_CUDA(cudaMemsetAsync(cnt, 0x7f, (size_t)nn * 4, st));  // up[] = 0x7f7f7f7f (no step)
          k_up_min<<<grid_for(nn - kk, 256, sm), 256, 0, st>>>(Jt, kk, nn, cnt);
          k_resolve_values<<<grid_for(nn, 256, sm), 256, 0, st>>>(Jt, kk, nn, cnt, removed[cc]);
          BB_LAUNCH_CHECK();
          launches += 2;
          continue;
        }
        BB_CUDA(cudaMemsetAsync(cnt, 0, (size_t)nn * 4, st));  // fill and removed: cleared by k_scan_apply
        const int g = grid_for(nn - kk, 256, sm);
        k_bucket_count<<<g, 256, 0, st>>>(Jt, kk, nn, cnt);
        const int nb = (int)ceil_div(nn, kScanBlock);
        k_scan_block_sums<<<nb, 256, 0, st>>>(cnt, nn, sums);
        k_scan_sums<<<1, 1024, 0, st>>>(sums, nb);
        k_scan_apply<<<nb, 256, 0, st>>>(cnt, nn, sums, off, fill, removed[cc]);
        k_bucket_fill<<<g, 256, 0, st>>>(Jt, kk, nn, off, fill, bucket);
        k_bucket_sort<<<grid_for(nn, 256, sm), 256, 0, st>>>(cnt, off, nn, bucket);
        k_resolve<<<g, 256, 0, st>>>(Jt, kk, nn, cnt, off, bucket, removed[cc]);
        BB_LAUNCH_CHECK();
        launches += 7;
      }
      const int64_t nt = (int64_t)n[0] + n[1];
      unsigned int* dst = sh.dist ? gbits : bits[t];
      k_mask_bits<<<grid_for(ceil_div(nt, 32), 256, sm), 256, 0, st>>>(removed[0], removed[1], n[0], nt, dst);
      BB_LAUNCH_CHECK();
      launches += 1;
      if (sh.dist) {
        k_mask_slice<<<grid_for(ceil_div(sh_n_local, 32), 256, sm), 256, 0, st>>>(gbits, sh_n_local, sh.n_sig_l,
                                                                                   sh.n_sig_g, sh.s0, sh.b0, bits[t]);
        BB_LAUNCH_CHECK();
        launches += 1;
      }
      if (ready) BB_CUDA(cudaEventRecord(ready[t], st));
    }
    BB_CUDA(cudaEventRecord(evR[half / kChunk], sc));
  }
  // make `st` wait for everything the mask streams have enqueued
  void join(cudaStream_t st) {
    if (!sc) return;
    cudaEvent_t e;
    BB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    BB_CUDA(cudaEventRecord(e, sc));
    BB_CUDA(cudaStreamWaitEvent(st, e, 0));
    BB_CUDA(cudaEventDestroy(e));
  }
};

// Subsample bits of every tree, produced ahead of the fit into a ring of
// kSlots mask buffers: the GPU generator on its own streams (default) or the
// host restatement (flags bit 1).  Created before binning, so the first
// chunk's parse overlaps it (the masks only need the class sizes).
constexpr int kSlots = 2 * kChunk;

struct MaskFeed {
  cudaStream_t st = nullptr;  // the fit's stream
  int64_t n = 0, n_sig = 0;
  int T = 0;
  bool host_masks = false;
  int64_t words = 0;
  double rate = 1.0;
  unsigned int* slots = nullptr;  // [kSlots][words]
  MaskGen mgen;
  cudaStream_t ms = nullptr;
  cudaEvent_t ready[kSlots] = {}, freed[kSlots] = {};
  unsigned int* pinned[kSlots] = {};
  Pcg64 g;
  std::vector<uint32_t> perm;
  int next = 0;
  FitStats* stats = nullptr;

  void init(Ctx& c, Arena& A, int64_t n_, int64_t n_sig_, const bb_fit_config& cfg, const Shard& shard,
            FitStats* stats_) {
    st = c.stream;
    n = n_;
    n_sig = n_sig_;
    T = cfg.n_trees;
    rate = cfg.subsample;
    stats = stats_;
    host_masks = (cfg.flags & 2) != 0 && !shard.dist;
    words = ceil_div(n, 32);
    slots = A.alloc<unsigned int>((size_t)words * kSlots);
    g.state = ((unsigned __int128)cfg.pcg_state_hi << 64) | cfg.pcg_state_lo;
    g.inc = ((unsigned __int128)cfg.pcg_inc_hi << 64) | cfg.pcg_inc_lo;
    g.has_uint32 = cfg.pcg_has_uint32;
    g.uinteger = cfg.pcg_uinteger;
    for (int k = 0; k < kSlots; ++k) {
      BB_CUDA(cudaEventCreateWithFlags(&ready[k], cudaEventDisableTiming));
      BB_CUDA(cudaEventCreateWithFlags(&freed[k], cudaEventDisableTiming));
    }
    if (host_masks) {
      for (int k = 0; k < kSlots; ++k) BB_CUDA(cudaMallocHost(&pinned[k], (size_t)words * 4));
      return;
    }
    // the mask chain is the fit's critical path: highest stream priority
    int prio_lo = 0, prio_hi = 0;
    BB_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    BB_CUDA(cudaStreamCreateWithPriority(&ms, cudaStreamNonBlocking, prio_hi));
    if (shard.dist) {
      mgen.init(A, st, shard.n_sig_g, shard.n_bkg_g, cfg.subsample, cfg, c.sm_count);
      mgen.sh = shard;
      mgen.sh_n_local = n;
    } else {
      mgen.init(A, st, n_sig, n - n_sig, cfg.subsample, cfg, c.sm_count);
    }
  }
  // host path: one tree; GPU path: the chunk starting at t
  int produce(int t) {
    if (host_masks) {
      const int slot = t % kSlots;
      unsigned int* bits = slots + (size_t)slot * words;
      if (t >= kSlots) BB_CUDA(cudaEventSynchronize(freed[slot]));
      const auto tm = std::chrono::steady_clock::now();
      subsample_tree(g, n_sig, n - n_sig, rate, pinned[slot], perm);
      stats->mask_ms += elapsed_ms(tm);
      BB_CUDA(cudaMemcpyAsync(bits, pinned[slot], (size_t)words * 4, cudaMemcpyHostToDevice, st));
      BB_CUDA(cudaEventRecord(ready[slot], st));
      return 1;
    }
    const int cnt = std::min(kChunk, T - t);
    unsigned int* bits[kChunk];
    cudaEvent_t evs[kChunk];
    for (int j = 0; j < cnt; ++j) {
      const int slot = (t + j) % kSlots;
      if (t + j >= kSlots) {
        BB_CUDA(cudaStreamWaitEvent(ms, freed[slot], 0));
        BB_CUDA(cudaStreamWaitEvent(mgen.sc, freed[slot], 0));
      }
      bits[j] = slots + (size_t)slot * words;
      evs[j] = ready[slot];
    }
    mgen.enqueue_chunk(ms, bits, cnt, evs, stats->launches);
    return cnt;
  }
  // masks enqueued up to tree t (+ one chunk of lookahead on the GPU path)
  void ahead(int t) {
    while (next < T && next < t + (host_masks ? 1 : kChunk + 1)) next += produce(next);
  }
  unsigned int* bits(int t) const { return slots + (size_t)(t % kSlots) * words; }
  ~MaskFeed() {
    if (ms) {
      mgen.report(ms);
      cudaStreamSynchronize(ms);
    }
    mgen.sync();  // its streams still wait on ready / freed
    if (ms) cudaStreamDestroy(ms);
    for (int k = 0; k < kSlots; ++k) {
      if (ready[k]) cudaEventDestroy(ready[k]);
      if (freed[k]) cudaEventDestroy(freed[k]);
      if (pinned[k]) cudaFreeHost(pinned[k]);
    }
  }
};

template <typename CodeT, typename NodeT>
static void run_trees(Ctx& c, Arena& A, const FitShape& s, const CodeT* codes, int code_off,
                      const double* w_cb, double f0, int shift, const bb_fit_config& cfg,
                      const bb_forced_cut* forced, int n_forced, const double* bounds_dev, bb_fit_out* out,
                      double* t_trees_ms, FitStats& stats, const Shard& shard, bool any_nan, MaskFeed& feed) {
  const int64_t n = s.n;
  cudaStream_t st = c.stream;
  const double two_s = std::ldexp(1.0, shift), scale = std::ldexp(1.0, -shift);
  const int64_t npad = ceil_div(n, kRowPad) * kRowPad;
  double* F = A.alloc<double>(n);
  NodeT* node = A.alloc<NodeT>(npad);
  long long* q = A.alloc<long long>(npad);
  BB_CUDA(cudaMemsetAsync(node, 0, (size_t)npad * sizeof(NodeT), st));
  BB_CUDA(cudaMemsetAsync(q, 0, (size_t)npad * 8, st));
  const int max_nodes = 1 << (s.depth - 1);
  // two layer histograms: the current layer's and its parent layer's (sibling
  // subtraction); both all-zero between trees
  unsigned long long* hist2 = A.alloc<unsigned long long>((size_t)4 * max_nodes * s.d * s.B);
  BB_CUDA(cudaMemsetAsync(hist2, 0, (size_t)4 * max_nodes * s.d * s.B * 8, st));
  unsigned long long* hbuf[2] = {hist2, hist2 + (size_t)2 * max_nodes * s.d * s.B};
  unsigned long long* sums = A.alloc<unsigned long long>((size_t)2 * s.n_nodes * 2);
  BB_CUDA(cudaMemsetAsync(sums, 0, (size_t)2 * s.n_nodes * 2 * 8, st));
  TreeArrays ta;
  const size_t TI = (size_t)s.T * s.n_internal, TN = (size_t)s.T * s.n_nodes;
  ta.feature = A.alloc<int>(TI);
  ta.cut = A.alloc<int>(TI);
  ta.valid = A.alloc<unsigned char>(TI);
  ta.gain = A.alloc<double>(TI);
  ta.thr = A.alloc<double>(TI);
  ta.nw = A.alloc<double>(TN);
  ta.pur = A.alloc<double>(TN);
  ta.forced = nullptr;
  if (n_forced > 0) {
    std::vector<int> fh(TI, -2);
    for (int k = 0; k < n_forced; ++k) {
      const bb_forced_cut& fc = forced[k];
      if (fc.tree < 0 || fc.tree >= s.T || fc.node < 0 || fc.node >= s.n_internal)
        throw InvalidArg{"forced cut out of range"};
      if (fc.valid && (fc.feature < 0 || fc.feature >= s.d || fc.cut_bin < 1 || fc.cut_bin > s.B - 1))
        throw InvalidArg{"forced cut feature/cut_bin out of range"};
      fh[(size_t)fc.tree * s.n_internal + fc.node] = fc.valid ? (fc.feature << 16) + fc.cut_bin : -1;
    }
    int* fd = A.alloc<int>(TI);
    BB_CUDA(cudaMemcpyAsync(fd, fh.data(), TI * 4, cudaMemcpyHostToDevice, st));
    ta.forced = fd;
  }
  SplitScratch sc;
  sc.best_gain = A.alloc<double>((size_t)max_nodes * s.d);
  sc.best_flat = A.alloc<int>((size_t)max_nodes * s.d);
  sc.forced_gain = A.alloc<double>(max_nodes);
  sc.done = A.alloc<unsigned int>(max_nodes);
  BB_CUDA(cudaMemsetAsync(sc.done, 0, (size_t)max_nodes * 4, st));

  // F = f0 (boosting.py:158-160)
  k_fill_f64<<<grid_for(n, 256, c.sm_count), 256, 0, st>>>(F, n, f0);
  BB_LAUNCH_CHECK();

  std::vector<HistPlan> plans(s.depth + 1);
  // sibling subtraction needs parent = left + right: a row with a missing
  // value at its node's cut feature stops at the node (trees.py:207-228), so
  // it is used only for NaN-free data
  std::vector<FlPlan> fl_plans(s.depth + 1);
  int64_t part_elems = 0;
  for (int l = 1; l <= s.depth; ++l) {
    plans[l] = plan_layer<CodeT, NodeT>(l, s, c.sm_count, !any_nan);
    fl_plans[l] = plan_fl<CodeT, NodeT>(l, s, c.sm_count, !any_nan, codes);
    part_elems = std::max(part_elems, (int64_t)fl_grid(fl_plans[l]) * fl_cta_stride(fl_plans[l], s.B));
  }
  long long* fl_partials = part_elems ? A.alloc<long long>((size_t)part_elems) : nullptr;
  set_hist_smem_attrs<CodeT, NodeT>();

  // node-partitioned row lists + row-major codes (kernels_hist_list.cuh):
  // u8 codes, d <= 64, every built (node, class) list gets a CTA
  // rows of 33..64 features: one 64-feature CTA per SM; BB_LH_GROUPS=1 runs
  // two 32-feature groups of the NW = 8 kernel (two CTAs per SM) instead,
  // measured slower at cfg3 (240 vs 180 us at layer 1: a group's 32-byte
  // half-row reads cost a 64-byte DRAM access each)
  static const bool lh_nw16 = !(getenv("BB_LH_GROUPS") && atoi(getenv("BB_LH_GROUPS")) != 0);
  const int lh_nw = (s.d <= 32 || !lh_nw16) ? 8 : 16;
  const int lh_pitch = s.d <= 32 ? 8 : 16;  // words per row of rc
  const int lh_groups = lh_nw == 8 && s.d > 32 ? 2 : 1;
  // BB_LH_WAVES > 1: that many CTAs per SM slot, scheduled as SMs come free
  // (SMs held by mask CTAs take fewer histogram CTAs) at one more flush each
  static const int lh_waves = getenv("BB_LH_WAVES") ? std::max(1, atoi(getenv("BB_LH_WAVES"))) : 1;
  const int lh_grid = lh_waves * (lh_nw == 8 ? 2 * (c.sm_count - hist_reserve()) : c.sm_count - hist_reserve());
  const int hp_env = hist_path_env();
  const bool lists8 = sizeof(CodeT) == 1 && s.d <= 64 && s.depth <= 8 && (hp_env == 0 || hp_env == 5) &&
                      2 * (1 << (s.depth - 1)) <= lh_grid && !getenv("BB_HIST_WARP") && !getenv("BB_HIST_GLOBAL_GROUPS");
  // u16 codes (more than 256 bins, or 256 bins with missing values) and u8
  // codes of more than 64 features: the 16-feature-group list kernel
  // (k_hist_list16), up to 1024 bins
  const int l16_groups = (int)ceil_div(s.d, kL16Feat);
  const bool lists16 = ((sizeof(CodeT) == 2 && s.B <= kL16Bins) || (sizeof(CodeT) == 1 && s.d > 64)) && s.depth <= 8 &&
                       (hp_env == 0 || hp_env == 5) &&
                       2 * (1 << (s.depth - 1)) * l16_groups <= kLhMaxSegs && !getenv("BB_HIST_WARP") &&
                       !getenv("BB_HIST_GLOBAL_GROUPS") && !(getenv("BB_LIST16") && atoi(getenv("BB_LIST16")) == 0);
  const bool lists = lists8 || lists16;
  uint16_t* rc16 = nullptr;
  uint32_t* rc = nullptr;
  int* lrow[2] = {nullptr, nullptr};
  long long* lq[2] = {nullptr, nullptr};
  int* cnt = nullptr;
  if (lists) {
    for (int b = 0; b < 2; ++b) {
      lrow[b] = A.alloc<int>(npad);
      lq[b] = A.alloc<long long>(npad);
    }
    cnt = A.alloc<int>((size_t)2 * s.n_nodes);
  }
  if (lists16) {
    rc16 = A.alloc<uint16_t>((size_t)npad * kL16Feat * l16_groups);
    BB_CUDA(cudaFuncSetAttribute(k_hist_list16, cudaFuncAttributeMaxDynamicSharedMemorySize, kL16SmemBytes));
    k_rowcodes16<CodeT><<<dim3((unsigned)ceil_div(n, kTile), l16_groups), 256, 0, st>>>(codes, n, s.d, l16_groups,
                                                                                       code_off, rc16);
    BB_LAUNCH_CHECK();
  }
  if (lists8) {
    rc = A.alloc<uint32_t>((size_t)npad * lh_pitch);
    const int tiles = (int)ceil_div(n, kTile);
    const uint8_t* c8 = reinterpret_cast<const uint8_t*>(codes);
    BB_CUDA(cudaFuncSetAttribute(k_hist_list<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, lh_smem_bytes<8>()));
    BB_CUDA(cudaFuncSetAttribute(k_hist_list<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, lh_smem_bytes<16>()));
    BB_CUDA(cudaFuncSetAttribute(k_rowcodes<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * kTile));
    BB_CUDA(cudaFuncSetAttribute(k_rowcodes<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * kTile));
    if (lh_pitch == 8) k_rowcodes<8><<<tiles, 256, (size_t)s.d * kTile, st>>>(c8, n, s.d, rc);
    else k_rowcodes<16><<<tiles, 256, (size_t)s.d * kTile, st>>>(c8, n, s.d, rc);
    BB_LAUNCH_CHECK();
  }

  std::vector<NodeT> leaf_tmp;
  const bool prof = (cfg.flags & 1) != 0;
  std::vector<cudaEvent_t> hev;
  auto hist_event = [&]() {
    cudaEvent_t e;
    BB_CUDA(cudaEventCreate(&e));
    BB_CUDA(cudaEventRecord(e, st));
    hev.push_back(e);
  };
  auto cleanup = [&]() {
    if (getenv("BB_HIST_PROFILE")) {
      unsigned long long h[8];
      cudaStreamSynchronize(st);
      cudaMemcpyFromSymbol(h, g_hist_prof, sizeof(h));
      fprintf(stderr, "hist prof (thread-cycles: wait compact bar1 atomics bar2 n):");
      for (int q = 0; q < 6; ++q) fprintf(stderr, " %llu", h[q]);
      fprintf(stderr, "\n");
    }
    for (auto e : hev) cudaEventDestroy(e);
  };
  const int gridN = grid_for(n, 256, c.sm_count);
  // refresh / advance: 2048-row tiles, grid-stride over exactly the resident
  // CTAs (a grid larger than one wave leaves its tail CTAs for a second pass)
  auto resident = [&](auto kern, size_t smem) {
    int per = 1;
    BB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, kListThreads, smem));
    return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, kListTileRows), (int64_t)std::max(1, per) * c.sm_count));
  };
  // staged refresh walk (kernels_tree.cuh): the previous tree's distinct cut
  // features' code columns in shared memory, 2048 rows per tile
  static const bool stage_off = getenv("BB_REFRESH_STAGE") && atoi(getenv("BB_REFRESH_STAGE")) == 0;
  int stage_slots = std::min(s.n_internal, s.d);
  size_t stage_smem = (size_t)stage_slots * kListTileRows * sizeof(CodeT);
  if (!lists || stage_off || s.n_internal > kStageNodes || stage_smem > 64 * 1024) {
    stage_slots = 0;
    stage_smem = 0;
  }
  if (stage_smem > 0)
    BB_CUDA(cudaFuncSetAttribute(k_update_refresh<NodeT, CodeT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)stage_smem));
  const int gridR = resident(k_update_refresh<NodeT, CodeT>, stage_smem);
  const int gridL = resident(k_advance<CodeT, NodeT>, 0);
  const int gridLL = resident(k_advance<CodeT, NodeT>, (size_t)32 * s.n_nodes);
  const int gridAL = std::max(2 * (1 << std::max(0, s.depth - 1)), resident(k_advance_list<CodeT>, 0));
  const auto t0 = std::chrono::steady_clock::now();
  try {
    // programmatic dependent launch on the tree loop's kernels (BB_PDL=0: plain launches)
    // sibling subtraction mode: 2 = the smaller child is built (row-list fits on
    // one device; a sharded fit builds the left child on every rank, the local
    // counts would disagree), 1 = the left child (BB_SIB_SMALL=0)
    const int sib_mode = lists && !c.comm.active() && !(getenv("BB_SIB_SMALL") && atoi(getenv("BB_SIB_SMALL")) == 0) ? 2 : 1;
    // BB_PDL bits: 1 refresh, 2 histogram, 4 split, 8 advance, 16 node weights
    const int pdl_mask = !lists ? 0 : (getenv("BB_PDL") ? atoi(getenv("BB_PDL")) : 0);
    const bool pdl_r = pdl_mask & 1, pdl_h = pdl_mask & 2, pdl_s = pdl_mask & 4, pdl_a = pdl_mask & 8, pdl_n = pdl_mask & 16;
    const bool tl_on = getenv("BB_TIMELINE") != nullptr;  // debug: main-stream waits for masks
    std::vector<cudaEvent_t> tl;
    if (getenv("BB_MASKS_FIRST") && s.T <= kSlots) {  // debug: every mask before the first tree (tree loop timed alone)
      feed.ahead(s.T);
      BB_CUDA(cudaDeviceSynchronize());
    }
    for (int t = 0; t < s.T; ++t) {
      NvtxRange tree_range("tree");
      feed.ahead(t);
      const int slot = t % kSlots;
      unsigned int* mask = feed.bits(t);
      if (tl_on) {
        tl.emplace_back();
        BB_CUDA(cudaEventCreate(&tl.back()));
        BB_CUDA(cudaEventRecord(tl.back(), st));  // main stream done with tree t-1
      }
      BB_CUDA(cudaStreamWaitEvent(st, feed.ready[slot], 0));
      if (tl_on) {
        tl.emplace_back();
        BB_CUDA(cudaEventCreate(&tl.back()));
        BB_CUDA(cudaEventRecord(tl.back(), st));  // ... and tree t's mask ready
      }
      if (lists) BB_CUDA(cudaMemsetAsync(cnt, 0, (size_t)2 * s.n_nodes * 4, st));
      launch_k(pdl_r, k_update_refresh<NodeT, CodeT>, gridR, kListThreads, stage_smem, st, n, s.n_sig, F, node, w_cb, q,
               mask, t > 0 ? ta.nw + (size_t)(t - 1) * s.n_nodes : nullptr, two_s, cnt, lrow[0], lq[0], codes, s.d,
               code_off, ta, (lists && t > 0) ? t - 1 : -1, s.n_internal, s.depth, stage_slots);
      BB_LAUNCH_CHECK();
      stats.launches += 1;
      for (int layer = 1; layer <= s.depth; ++layer) {
        static const char* kLayerNames[] = {"layer 0", "layer 1", "layer 2", "layer 3", "layer 4", "layer 5", "layer 6",
                                            "layer 7", "layer 8", "layer 9", "layer 10", "layer 11", "layer 12",
                                            "layer 13", "layer 14", "layer 15"};
        NvtxRange layer_range(kLayerNames[layer]);
        const HistPlan& p = plans[layer];
        unsigned long long* hist = hbuf[layer & 1];
        unsigned long long* par = hbuf[(layer - 1) & 1];
        if (prof) hist_event();
        if (lists) {
          const int lb = (layer - 1) & 1;
          if (lists16) {
            const int g16 = c.sm_count - hist_reserve();  // more (segment, group) items than CTAs: row-balanced parts
            launch_k(pdl_h, k_hist_list16, g16, kLhThreads, kL16SmemBytes, st, reinterpret_cast<const uint4*>(rc16),
                     2 * l16_groups, lrow[lb], lq[lb], cnt, layer, p.sib ? sib_mode : 0, s.n_sig, s.d, s.B, p.nodes, hist,
                     l16_groups);
          } else if (lh_nw == 8)
            launch_k(pdl_h, k_hist_list<8>, lh_grid, kLhThreads, lh_smem_bytes<8>(), st, rc, lrow[lb], lq[lb], cnt, layer,
                     p.sib ? sib_mode : 0, s.n_sig, s.d, s.B, code_off, p.nodes, hist, lh_pitch, lh_groups);
          else
            launch_k(pdl_h, k_hist_list<16>, lh_grid, kLhThreads, lh_smem_bytes<16>(), st, rc, lrow[lb], lq[lb], cnt, layer,
                     p.sib ? sib_mode : 0, s.n_sig, s.d, s.B, code_off, p.nodes, hist, 16, 1);
          BB_LAUNCH_CHECK();
        } else {
          launch_layer_hist<CodeT, NodeT>(p, fl_plans[layer], c.sm_count, codes, code_off, node, q, n, s.n_sig, s.d,
                                          s.B, hist, st, fl_partials);
        }
        if (prof) hist_event();
        c.comm.all_reduce(hist, (size_t)2 * p.nodes * s.d * s.B, kNcclI64, kNcclSum, st);  // sharded fits
        stats.launches += 3;
        stats.hist_launches += 1;
        const int nodes = p.nodes;
        const int n_fc_want = std::max(1, std::min(s.d, (2 * c.sm_count + nodes - 1) / nodes));
        const int fc_size = (int)ceil_div(s.d, n_fc_want);
        const int n_fc = (int)ceil_div(s.d, fc_size);
        launch_k(pdl_s && !c.comm.active(), k_split<256>, dim3(nodes, n_fc), 256, 0, st, hist, s.d, s.B, p.start, nodes,
                 fc_size, layer == s.depth ? 1 : 0, scale, t, s.n_internal, ta, bounds_dev, sc, par,
                 p.sib ? sib_mode : 0, (layer < s.depth && plans[layer + 1].sib) ? 1 : 0, cnt);
        BB_LAUNCH_CHECK();
        const bool last = layer == s.depth;
        if (last && p.sib) BB_CUDA(cudaMemsetAsync(hist, 0, (size_t)2 * nodes * s.d * s.B * 8, st));
        if (lists) {
          // the layer's listed active rows only (kernels_hist_list.cuh)
          launch_k(pdl_a, k_advance_list<CodeT>, gridAL, kListThreads, 0, st, codes, s.d, code_off, lrow[(layer - 1) & 1],
                   lq[(layer - 1) & 1], cnt, lrow[layer & 1], lq[layer & 1], layer, t, s.n_internal, ta, last ? 1 : 0,
                   s.n_sig, sums, s.n_nodes, q);
        } else {
          k_advance<CodeT, NodeT><<<last ? gridLL : gridL, kListThreads, last ? (size_t)32 * s.n_nodes : 0, st>>>(
              codes, s.d, code_off, node, n, s.n_sig, p.start, t, s.n_internal, ta, last ? 1 : 0, s.n_nodes, q, mask,
              F, w_cb, two_s, sums, nullptr, nullptr, nullptr, 0);
        }
        BB_LAUNCH_CHECK();
      }
      BB_CUDA(cudaEventRecord(feed.freed[slot], st));
      c.comm.all_reduce(sums, (size_t)2 * s.n_nodes * 2, kNcclI64, kNcclSum, st);  // sharded fits
      launch_k(pdl_n && !c.comm.active(), k_node_weights, 1, 256, (size_t)2 * s.n_nodes * 2 * 8, st, sums, s.n_nodes,
               s.depth, scale, cfg.shrinkage, t, ta);
      BB_LAUNCH_CHECK();
      stats.launches += 1;
      if (out->leaves) {
        if (lists) {  // no per-row node ids in row-list fits: walk the tree
          k_walk_leaves<CodeT, NodeT><<<gridN, 256, 0, st>>>(codes, s.d, code_off, n, ta, t, s.n_internal, s.depth,
                                                              node);
          BB_LAUNCH_CHECK();
        }
        leaf_tmp.resize(n);
        BB_CUDA(cudaMemcpyAsync(leaf_tmp.data(), node, (size_t)n * sizeof(NodeT), cudaMemcpyDeviceToHost, st));
        BB_CUDA(cudaStreamSynchronize(st));
        uint16_t* dst = out->leaves + (size_t)t * n;
        for (int64_t i = 0; i < n; ++i) dst[i] = (uint16_t)leaf_tmp[i];
      }
    }
    if (out->scores) {
      if (lists)
        k_walk_leaves<CodeT, NodeT><<<gridN, 256, 0, st>>>(codes, s.d, code_off, n, ta, s.T - 1, s.n_internal, s.depth,
                                                            node);
      k_update_scores<NodeT><<<gridN, 256, 0, st>>>(n, F, node, ta.nw + (size_t)(s.T - 1) * s.n_nodes);
      BB_LAUNCH_CHECK();
      BB_CUDA(cudaMemcpyAsync(out->scores, F, (size_t)n * 8, cudaMemcpyDeviceToHost, st));
    }
    const double enq_ms = elapsed_ms(t0);  // host time to enqueue every tree (launch-bound if ~ the fit)
    BB_CUDA(cudaStreamSynchronize(st));
    if (tl_on) fprintf(stderr, "timeline: host enqueue %.2f ms, enqueue+sync %.2f ms\n", enq_ms, elapsed_ms(t0));
    if (tl_on && tl.size() >= 2) {
      double wait = 0.0, busy = 0.0;
      int waits = 0;
      for (size_t k = 0; k + 1 < tl.size(); k += 2) {
        float w = 0.f;
        BB_CUDA(cudaEventElapsedTime(&w, tl[k], tl[k + 1]));
        wait += w;
        waits += w > 0.01f;
        if (k + 2 < tl.size()) {
          float b = 0.f;
          BB_CUDA(cudaEventElapsedTime(&b, tl[k + 1], tl[k + 2]));
          busy += b;
        }
      }
      fprintf(stderr, "timeline: main stream waited %.2f ms for masks (%d trees), busy %.2f ms\n", wait, waits, busy);
      for (auto e : tl) cudaEventDestroy(e);
    }
    for (size_t k = 0; k + 1 < hev.size(); k += 2) {
      float msf = 0.f;
      BB_CUDA(cudaEventElapsedTime(&msf, hev[k], hev[k + 1]));
      stats.hist_ms += msf;
    }
  } catch (...) {
    cudaStreamSynchronize(st);
    cleanup();
    throw;
  }
  *t_trees_ms = elapsed_ms(t0);
  cleanup();

  // outputs
  std::vector<unsigned char> vtmp(TI);
  BB_CUDA(cudaMemcpyAsync(out->feature, ta.feature, TI * 4, cudaMemcpyDeviceToHost, st));
  BB_CUDA(cudaMemcpyAsync(out->cut_bin, ta.cut, TI * 4, cudaMemcpyDeviceToHost, st));
  BB_CUDA(cudaMemcpyAsync(out->valid, ta.valid, TI, cudaMemcpyDeviceToHost, st));
  BB_CUDA(cudaMemcpyAsync(out->gain, ta.gain, TI * 8, cudaMemcpyDeviceToHost, st));
  BB_CUDA(cudaMemcpyAsync(out->threshold, ta.thr, TI * 8, cudaMemcpyDeviceToHost, st));
  BB_CUDA(cudaMemcpyAsync(out->node_weight, ta.nw, TN * 8, cudaMemcpyDeviceToHost, st));
  BB_CUDA(cudaMemcpyAsync(out->node_purity, ta.pur, TN * 8, cudaMemcpyDeviceToHost, st));
  BB_CUDA(cudaStreamSynchronize(st));
}

template <typename T>
static void fit_impl(Ctx& c, const void* Xv, bool x_dev, int64_t n, int d, const int8_t* y, bool y_dev,
                     const double* w, bool w_dev, const bb_fit_config& cfg, const bb_forced_cut* forced,
                     int n_forced, bb_fit_out* out) {
  using K = typename KeyOf<T>::K;
  const auto t_all = std::chrono::steady_clock::now();
  cudaStream_t st = c.stream;
  cudaEvent_t ev0, ev1;
  BB_CUDA(cudaEventCreate(&ev0));
  BB_CUDA(cudaEventCreate(&ev1));
  BB_CUDA(cudaEventRecord(ev0, st));
  FitStats stats;
  struct EvGuard {
    cudaEvent_t a, b;
    ~EvGuard() { cudaEventDestroy(a); cudaEventDestroy(b); }
  } evg{ev0, ev1};
  Arena A(st);
  const int levels = cfg.binning_levels, B = 1 << levels, nt = B - 1;
  NvtxRange fit_range("bb_fit");
  // ---- upload: labels and weights first (the class-block kernels and the
  // subsample masks need only these), the rows after the first mask chunk
  // has been queued, so its parse overlaps the row upload as well
  auto t_up = std::chrono::steady_clock::now();
  const T* Xd = reinterpret_cast<const T*>(Xv);
  const int8_t* yd = y;
  if (!y_dev) {
    int8_t* p = A.alloc<int8_t>(n);
    c.stage.h2d(p, y, (size_t)n, st);
    yd = p;
  }
  const double* wd = w;
  if (w && !w_dev) {
    double* p = A.alloc<double>(n);
    c.stage.h2d(p, w, (size_t)n * 8, st);
    wd = p;
  }
  double ms_up = elapsed_ms(t_up);
  // ---- class blocks (sample.py:112-116)
  auto t_bin = std::chrono::steady_clock::now();
  const bool dist = c.comm.active();  // row-sharded fit: every rank holds a slice of the rows
  const int n_tiles = (int)ceil_div(n, CLS_TILE);
  int* tile_sig = A.alloc<int>(n_tiles + 1);
  int* pos = A.alloc<int>(n);
  double* w_cb = w ? A.alloc<double>(n) : nullptr;
  k_class_tile_counts<<<n_tiles, 256, 0, st>>>(yd, n, tile_sig);
  BB_LAUNCH_CHECK();
  k_class_scan<<<1, 1024, 0, st>>>(tile_sig, n_tiles);
  BB_LAUNCH_CHECK();
  k_class_positions<<<n_tiles, 256, 0, st>>>(yd, n, tile_sig, pos, wd, w_cb);
  BB_LAUNCH_CHECK();
  int n_sig_i = 0;
  BB_CUDA(cudaMemcpyAsync(&n_sig_i, tile_sig + n_tiles, 4, cudaMemcpyDeviceToHost, st));
  BB_CUDA(cudaStreamSynchronize(st));
  const int64_t n_sig = n_sig_i;
  Shard shard;
  if (dist) {
    // per-rank class counts -> this rank's offsets in the global class blocks
    // (ranks concatenate in rank order: the global row order of the fit)
    const int W = c.comm.world, R = c.comm.rank;
    unsigned long long* cnt = A.alloc<unsigned long long>(2 * (size_t)W);
    std::vector<unsigned long long> h(2 * (size_t)W, 0);
    h[2 * R] = (unsigned long long)n_sig;
    h[2 * R + 1] = (unsigned long long)(n - n_sig);
    BB_CUDA(cudaMemcpyAsync(cnt, h.data(), h.size() * 8, cudaMemcpyHostToDevice, st));
    c.comm.all_reduce(cnt, h.size(), kNcclU64, kNcclSum, st);
    BB_CUDA(cudaMemcpyAsync(h.data(), cnt, h.size() * 8, cudaMemcpyDeviceToHost, st));
    BB_CUDA(cudaStreamSynchronize(st));
    shard.dist = true;
    shard.n_sig_l = n_sig;
    for (int r = 0; r < W; ++r) {
      if (r < R) {
        shard.s0 += (int64_t)h[2 * r];
        shard.b0 += (int64_t)h[2 * r + 1];
      }
      shard.n_sig_g += (int64_t)h[2 * r];
      shard.n_bkg_g += (int64_t)h[2 * r + 1];
    }
    if (shard.n_sig_g + shard.n_bkg_g >= ((int64_t)1 << 31)) throw InvalidArg{"at most 2^31-1 rows per fit"};
    if (shard.n_sig_g == 0 || shard.n_bkg_g == 0) throw InvalidArg{"training data must contain both classes"};
  } else if (n_sig == 0 || n_sig == n) {
    throw InvalidArg{"training data must contain both classes"};
  }
  // ---- subsample masks: they need only the class sizes, so the first
  // chunk's parse starts now and overlaps the binning below
  MaskFeed feed;
  feed.init(c, A, n, n_sig, cfg, shard, &stats);
  feed.ahead(0);
  if (!x_dev) {
    t_up = std::chrono::steady_clock::now();
    T* p = A.alloc<T>((size_t)n * d);
    c.stage.h2d(p, Xv, (size_t)n * d * sizeof(T), st);
    Xd = p;
    ms_up += elapsed_ms(t_up);
  }
  // user weights: per-class pairwise-sum leaves and max |w| on the device
  // (read back after the binning kernels are queued)
  std::vector<long long> pw_off;
  std::vector<int> pw_len;
  double* pw_out = nullptr;
  unsigned long long* wstat = nullptr;
  size_t L_sig = 0;
  if (w) {
    pw_leaves(0, n_sig, pw_off, pw_len);
    L_sig = pw_off.size();
    pw_leaves(n_sig, n - n_sig, pw_off, pw_len);
    const int L = (int)pw_off.size();
    long long* d_off = A.alloc<long long>(L);
    int* d_len = A.alloc<int>(L);
    pw_out = A.alloc<double>(L);
    wstat = A.alloc<unsigned long long>(2);
    BB_CUDA(cudaMemcpyAsync(d_off, pw_off.data(), (size_t)L * 8, cudaMemcpyHostToDevice, st));
    BB_CUDA(cudaMemcpyAsync(d_len, pw_len.data(), (size_t)L * 4, cudaMemcpyHostToDevice, st));
    BB_CUDA(cudaMemsetAsync(wstat, 0, 16, st));
    k_pairwise_leaves<<<grid_for(L, 128, c.sm_count), 128, 0, st>>>(w_cb, d_off, d_len, L, pw_out);
    BB_LAUNCH_CHECK();
    k_weight_stats<<<grid_for(n, 256, c.sm_count), 256, 0, st>>>(w_cb, n, wstat,
                                                               reinterpret_cast<unsigned int*>(wstat + 1));
    BB_LAUNCH_CHECK();
    BB_CUDA(cudaStreamSynchronize(st));  // host vectors pw_off / pw_len go out of use
  }
  // ---- binning
  NvtxRange bin_range("binning");
  std::vector<unsigned long long> finite, nans;
  unsigned long long* finite_dev = nullptr;
  K* keys = make_keys<T>(c, A, Xd, n, d, finite, nans, &finite_dev, dist);
  if (!x_dev) A.release(const_cast<T*>(Xd));
  double* bounds = A.alloc<double>((size_t)d * nt);
  K* bkeys = A.alloc<K>((size_t)d * nt);
  run_select<T>(c, A, keys, n, d, levels, finite_dev, bounds, bkeys, dist);
  bool any_nan = false;
  for (int f = 0; f < d; ++f) any_nan |= nans[f] > 0;
  const int64_t stride = ceil_div(n, kTile) * kTile;  // rows incl. tile padding
  FitShape s{n, n_sig, d, levels, B, cfg.depth, (1 << cfg.depth) - 1, (1 << (cfg.depth + 1)) - 1, cfg.n_trees};
  // prior (boosting.py:76-83) and the fixed-point shift from the user weights
  double w_sig, w_bkg, max_abs = 1.0;
  if (w) {
    std::vector<double> leaf(pw_off.size());
    unsigned long long hs[2];
    BB_CUDA(cudaMemcpyAsync(leaf.data(), pw_out, leaf.size() * 8, cudaMemcpyDeviceToHost, st));
    BB_CUDA(cudaMemcpyAsync(hs, wstat, 16, cudaMemcpyDeviceToHost, st));
    BB_CUDA(cudaStreamSynchronize(st));
    if ((unsigned int)hs[1] != 0u) throw InvalidArg{"user weights must be finite"};
    size_t k0 = 0, k1 = L_sig;
    w_sig = pw_combine(n_sig, leaf.data(), k0);
    w_bkg = pw_combine(n - n_sig, leaf.data(), k1);
    std::memcpy(&max_abs, &hs[0], 8);
  } else {
    w_sig = (double)n_sig;
    w_bkg = (double)(n - n_sig);
  }
  if (dist) {
    // global class weights (exact for unit weights; for user weights the
    // caller passes the reference's pairwise f0 in f0_override) and the
    // global weight magnitude for the common fixed-point shift
    double* red = A.alloc<double>(3);
    double hv[3] = {w_sig, w_bkg, max_abs};
    BB_CUDA(cudaMemcpyAsync(red, hv, 24, cudaMemcpyHostToDevice, st));
    c.comm.all_reduce(red, 2, kNcclF64, kNcclSum, st);
    c.comm.all_reduce(red + 2, 1, kNcclF64, kNcclMax, st);
    BB_CUDA(cudaMemcpyAsync(hv, red, 24, cudaMemcpyDeviceToHost, st));
    BB_CUDA(cudaStreamSynchronize(st));
    w_sig = hv[0];
    w_bkg = hv[1];
    max_abs = hv[2];
  }
  double f0 = (w_sig <= 0.0 || w_bkg <= 0.0) ? 0.0 : 0.5 * std::log(w_sig / w_bkg);
  if (!std::isnan(cfg.f0_override)) f0 = cfg.f0_override;
  const int shift = fixed_shift_for(max_abs);
  double ms_trees = 0.0;
  auto launch_codes = [&](auto* codes, int off) {
    using CodeT = std::remove_pointer_t<decltype(codes)>;
    // padding rows of the last tile hold code 0: the feature-lane histogram
    // adds zeros for rows that do not contribute, at their (in-range) codes
    if (n % kTile)
      BB_CUDA(cudaMemsetAsync(codes + (size_t)(ceil_div(n, kTile) - 1) * d * kTile, 0, (size_t)d * kTile * sizeof(CodeT),
                              st));
    BB_CUDA(cudaFuncSetAttribute(k_codes<K, CodeT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    k_codes<K, CodeT><<<dim3((unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256 * 4), 4 * c.sm_count / d + 1)), d),
                        256, codes_smem<K>(nt), st>>>(keys, n, nt, bkeys, pos, codes, stride, off, d, 1);
    BB_LAUNCH_CHECK();
  };
  auto after_codes = [&]() {
    A.release(keys);
  };
  double ms_bin = 0.0;
  auto go = [&](auto* codes, int off) {
    using CodeT = std::remove_pointer_t<decltype(codes)>;
    launch_codes(codes, off);
    after_codes();
    BB_CUDA(cudaStreamSynchronize(st));
    ms_bin = elapsed_ms(t_bin);
    if (s.depth <= 7)
      run_trees<CodeT, uint8_t>(c, A, s, codes, off, w_cb, f0, shift, cfg, forced, n_forced, bounds, out, &ms_trees,
                                stats, shard, any_nan, feed);
    else
      run_trees<CodeT, uint16_t>(c, A, s, codes, off, w_cb, f0, shift, cfg, forced, n_forced, bounds, out, &ms_trees,
                                 stats, shard, any_nan, feed);
  };
  if (B <= 255) {
    go(A.alloc<uint8_t>((size_t)d * stride), 0);
  } else if (B == 256 && !any_nan) {
    go(A.alloc<uint8_t>((size_t)d * stride), 1);
  } else {
    go(A.alloc<uint16_t>((size_t)d * stride), 0);
  }
  auto t_dn = std::chrono::steady_clock::now();
  BB_CUDA(cudaMemcpyAsync(out->boundaries, bounds, (size_t)d * nt * 8, cudaMemcpyDeviceToHost, st));
  BB_CUDA(cudaEventRecord(ev1, st));
  BB_CUDA(cudaStreamSynchronize(st));
  float dev_ms = 0.f;
  BB_CUDA(cudaEventElapsedTime(&dev_ms, ev0, ev1));
  *out->f0 = f0;
  *out->fixed_shift = shift;
  if (out->n_sig) *out->n_sig = n_sig;
  if (out->timing_ms) {
    out->timing_ms[0] = ms_up;
    out->timing_ms[1] = ms_bin;
    out->timing_ms[2] = ms_trees;
    out->timing_ms[3] = elapsed_ms(t_dn);
    out->timing_ms[4] = elapsed_ms(t_all);
    out->timing_ms[5] = dev_ms;
    out->timing_ms[6] = stats.hist_ms;
    out->timing_ms[7] = (double)stats.hist_launches;
    out->timing_ms[8] = (double)(stats.launches + 9 + 2 * (KeyOf<T>::BITS == 32 ? 4 : 8));
    out->timing_ms[9] = stats.mask_ms;
  }
}

// ------------------------------------------------------------- ROC AUC
// analysis.py:45-70 on the device (kernels_auc.cuh).  p, y01, w (w may be
// null) are device arrays of n rows; returns the AUC and the class totals.
static double auc_device(Ctx& c, Arena& A, const double* p, const int8_t* y01, const double* w, int64_t n,
                         double* w_sig_out, double* w_bkg_out) {
  cudaStream_t st = c.stream;
  unsigned long long* k[2] = {A.alloc<unsigned long long>(n), A.alloc<unsigned long long>(n)};
  unsigned int* v[2] = {A.alloc<unsigned int>(n), A.alloc<unsigned int>(n)};
  const int tiles = (int)ceil_div(n, kAucTile);
  unsigned int* cnt = A.alloc<unsigned int>((size_t)kAucDigits * tiles);
  k_auc_keys<<<grid_for(n, 256, c.sm_count), 256, 0, st>>>(p, n, k[0], v[0]);
  BB_LAUNCH_CHECK();
  int cur = 0;
  for (int shift = 0; shift < 64; shift += 4) {
    k_radix_count<<<tiles, kAucThreads, 0, st>>>(k[cur], n, shift, tiles, cnt);
    k_radix_scan<<<1, 1024, 0, st>>>(cnt, kAucDigits * tiles);
    k_radix_scatter<<<tiles, kAucThreads, 0, st>>>(k[cur], v[cur], n, shift, tiles, cnt, k[cur ^ 1], v[cur ^ 1]);
    BB_LAUNCH_CHECK();
    cur ^= 1;
  }
  double* S = A.alloc<double>(n);
  double* Bc = A.alloc<double>(n);
  long long* start = A.alloc<long long>(n);
  k_auc_prep<<<grid_for(n, 256, c.sm_count), 256, 0, st>>>(k[cur], v[cur], reinterpret_cast<const signed char*>(y01),
                                                           w, n, S, Bc, start);
  BB_LAUNCH_CHECK();
  const int nb = (int)ceil_div(n, 1024);
  double* sums_d = A.alloc<double>(nb);
  long long* sums_l = A.alloc<long long>(nb);
  for (double* a : {S, Bc}) {
    k_scan_tiles<double, false><<<nb, 1024, 0, st>>>(a, n, sums_d, 0.0);
    k_scan_sums_serial<double, false><<<1, 1024, 0, st>>>(sums_d, nb, 0.0);
    k_scan_add<double, false><<<nb, 1024, 0, st>>>(a, n, sums_d);
    BB_LAUNCH_CHECK();
  }
  k_scan_tiles<long long, true><<<nb, 1024, 0, st>>>(start, n, sums_l, -1ll);
  k_scan_sums_serial<long long, true><<<1, 1024, 0, st>>>(sums_l, nb, -1ll);
  k_scan_add<long long, true><<<nb, 1024, 0, st>>>(start, n, sums_l);
  BB_LAUNCH_CHECK();
  const int tb = (int)std::min<int64_t>(1024, ceil_div(n, 256));
  double* part = A.alloc<double>(tb);
  k_auc_terms<<<tb, 256, 0, st>>>(k[cur], S, Bc, start, n, part);
  BB_LAUNCH_CHECK();
  std::vector<double> hp(tb);
  double tot[2];
  BB_CUDA(cudaMemcpyAsync(hp.data(), part, (size_t)tb * 8, cudaMemcpyDeviceToHost, st));
  BB_CUDA(cudaMemcpyAsync(&tot[0], S + n - 1, 8, cudaMemcpyDeviceToHost, st));
  BB_CUDA(cudaMemcpyAsync(&tot[1], Bc + n - 1, 8, cudaMemcpyDeviceToHost, st));
  BB_CUDA(cudaStreamSynchronize(st));
  double won = 0.0;
  for (double x : hp) won += x;
  *w_sig_out = tot[0];
  *w_bkg_out = tot[1];
  if (!(tot[0] > 0.0) || !(tot[1] > 0.0)) throw InvalidArg{"roc_auc needs both classes with positive total weight"};
  return won / (tot[0] * tot[1]);
}

// ------------------------------------------------------------- elimination
// Batched refits for elimination_importance (analysis.py:104-173): the
// training rows are uploaded, class-blocked and binned ONCE (boundaries of a
// feature do not depend on the other features), and the validation rows are
// binned with the training boundaries once.  Each refit gathers the code
// columns of its feature subset, runs the tree loop, applies the forest to
// the validation codes (traverse over codes == traverse over values,
// SURVEY.md A5) and computes the validation AUC on the device.  Refits of one
// round run concurrently from several contexts (one stream each).
struct ElimSession {
  int device = 0;
  int64_t n = 0, n_sig = 0, nv = 0;
  int d = 0, levels = 0, B = 0, code_bytes = 1, code_off = 0;
  void* codes = nullptr;     // training codes, tiled, class-block order
  double* bounds = nullptr;  // [d][B-1]
  double* w_cb = nullptr;    // class-block training weights (null: unit)
  std::vector<unsigned long long> nans;
  double f0 = 0.0;
  int shift = 32;
  void* vcodes = nullptr;    // validation codes, tiled, input row order
  int8_t* vy = nullptr;
  double* vw = nullptr;
  std::vector<void*> owned;
  template <typename T>
  T* alloc(size_t count) {
    void* p = nullptr;
    BB_CUDA(cudaMalloc(&p, std::max<size_t>(1, count) * sizeof(T)));
    owned.push_back(p);
    return reinterpret_cast<T*>(p);
  }
  ~ElimSession() {
    cudaSetDevice(device);
    for (void* p : owned) cudaFree(p);
  }
};

template <typename CodeT>
__global__ void k_gather_cols(const CodeT* __restrict__ src, int d, const int* __restrict__ cols, int nc,
                              CodeT* __restrict__ dst) {
  const int64_t tile = blockIdx.x;
  const int j = blockIdx.y;
  const CodeT* a = src + (tile * d + cols[j]) * (int64_t)kTile;
  CodeT* b = dst + (tile * nc + j) * (int64_t)kTile;
  for (int r = threadIdx.x; r < kTile; r += blockDim.x) b[r] = a[r];
}

// F and p over tiled validation codes: right iff code > cut_bin (code
// 0 = missing stops), features mapped to the session's columns
template <typename CodeT>
__global__ void k_apply_codes(const CodeT* __restrict__ codes, int64_t n, int d, int code_off,
                              const int* __restrict__ colmap, int T, int depth, const int* __restrict__ feat,
                              const int* __restrict__ cut, const unsigned char* __restrict__ vld,
                              const double* __restrict__ nw, double f0, double* __restrict__ p) {
  const int I = (1 << depth) - 1, N = (1 << (depth + 1)) - 1;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double F = f0;
    for (int t = 0; t < T; ++t) {
      int nd = 0;
      for (int l = 0; l < depth; ++l) {
        const int e = t * I + nd;
        if (!__ldg(&vld[e])) break;
        const int c = (int)codes[code_index(i, __ldg(&colmap[__ldg(&feat[e])]), d)] + code_off;
        if (c == 0) break;
        nd = 2 * nd + 1 + (c > __ldg(&cut[e]) ? 1 : 0);
      }
      F = __dadd_rn(F, __ldg(&nw[(int64_t)t * N + nd]));
    }
    p[i] = sigmoid2(F);
  }
}

template <typename T>
static ElimSession* elim_prepare(Ctx& c, const T* X, int64_t n, int d, const int8_t* y, const double* w, int levels,
                                 const T* Xv, int64_t nv, const int8_t* yv, const double* wv) {
  using K = typename KeyOf<T>::K;
  cudaStream_t st = c.stream;
  auto S = std::make_unique<ElimSession>();
  ElimSession& s = *S;
  s.device = c.device;
  s.n = n;
  s.nv = nv;
  s.d = d;
  s.levels = levels;
  s.B = 1 << levels;
  const int nt = s.B - 1;
  Arena A(st);
  T* Xd = A.alloc<T>((size_t)n * d);
  int8_t* yd = A.alloc<int8_t>(n);
  c.stage.h2d(Xd, X, (size_t)n * d * sizeof(T), st);
  c.stage.h2d(yd, y, (size_t)n, st);
  double* wd = nullptr;
  if (w) {
    wd = A.alloc<double>(n);
    c.stage.h2d(wd, w, (size_t)n * 8, st);
  }
  // class blocks (sample.py:112-116)
  const int n_tiles = (int)ceil_div(n, CLS_TILE);
  int* tile_sig = A.alloc<int>(n_tiles + 1);
  int* pos = A.alloc<int>(n);
  if (w) s.w_cb = s.alloc<double>(n);
  k_class_tile_counts<<<n_tiles, 256, 0, st>>>(yd, n, tile_sig);
  k_class_scan<<<1, 1024, 0, st>>>(tile_sig, n_tiles);
  k_class_positions<<<n_tiles, 256, 0, st>>>(yd, n, tile_sig, pos, wd, s.w_cb);
  BB_LAUNCH_CHECK();
  int n_sig_i = 0;
  BB_CUDA(cudaMemcpyAsync(&n_sig_i, tile_sig + n_tiles, 4, cudaMemcpyDeviceToHost, st));
  BB_CUDA(cudaStreamSynchronize(st));
  s.n_sig = n_sig_i;
  if (s.n_sig == 0 || s.n_sig == n) throw InvalidArg{"training data must contain both classes"};
  // prior (boosting.py:76-83) and the fixed-point shift, as fit_impl
  double w_sig = (double)s.n_sig, w_bkg = (double)(n - s.n_sig), max_abs = 1.0;
  if (w) {
    std::vector<double> hw(s.w_cb ? (size_t)n : 0);
    BB_CUDA(cudaMemcpyAsync(hw.data(), s.w_cb, (size_t)n * 8, cudaMemcpyDeviceToHost, st));
    BB_CUDA(cudaStreamSynchronize(st));
    w_sig = pairwise(hw.data(), s.n_sig);
    w_bkg = pairwise(hw.data() + s.n_sig, n - s.n_sig);
    max_abs = 0.0;
    for (double x : hw) {
      if (!std::isfinite(x)) throw InvalidArg{"user weights must be finite"};
      max_abs = std::max(max_abs, std::fabs(x));
    }
  }
  s.f0 = (w_sig <= 0.0 || w_bkg <= 0.0) ? 0.0 : 0.5 * std::log(w_sig / w_bkg);
  s.shift = fixed_shift_for(max_abs);
  // binning of every feature over the training rows
  std::vector<unsigned long long> finite;
  unsigned long long* finite_dev = nullptr;
  K* keys = make_keys<T>(c, A, Xd, n, d, finite, s.nans, &finite_dev);
  s.bounds = s.alloc<double>((size_t)d * nt);
  K* bkeys = A.alloc<K>((size_t)d * nt);
  run_select<T>(c, A, keys, n, d, levels, finite_dev, s.bounds, bkeys);
  bool any_nan = false;
  for (int f = 0; f < d; ++f) any_nan |= s.nans[f] > 0;
  s.code_bytes = (s.B <= 256) && (s.B <= 255 || !any_nan) ? 1 : 2;
  s.code_off = (s.B == 256 && s.code_bytes == 1) ? 1 : 0;
  const int64_t stride = ceil_div(n, kTile) * kTile;
  auto emit = [&](const K* kk, int64_t rows, const int* pp, void* out) {
    const dim3 g((unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(rows, 256 * 4), 4 * c.sm_count / d + 1)), d);
    const int64_t str = ceil_div(rows, kTile) * kTile;
    if (s.code_bytes == 1) {
      if (rows % kTile)
        BB_CUDA(cudaMemsetAsync((uint8_t*)out + (size_t)(ceil_div(rows, kTile) - 1) * d * kTile, 0, (size_t)d * kTile, st));
      BB_CUDA(cudaFuncSetAttribute(k_codes<K, uint8_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
      k_codes<K, uint8_t><<<g, 256, codes_smem<K>(nt), st>>>(kk, rows, nt, bkeys, pp, (uint8_t*)out, str,
                                                                  s.code_off, d, 1);
    } else {
      if (rows % kTile)
        BB_CUDA(cudaMemsetAsync((uint16_t*)out + (size_t)(ceil_div(rows, kTile) - 1) * d * kTile, 0,
                                (size_t)d * kTile * 2, st));
      BB_CUDA(cudaFuncSetAttribute(k_codes<K, uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
      k_codes<K, uint16_t><<<g, 256, codes_smem<K>(nt), st>>>(kk, rows, nt, bkeys, pp, (uint16_t*)out, str,
                                                                   s.code_off, d, 1);
    }
    BB_LAUNCH_CHECK();
  };
  s.codes = s.code_bytes == 1 ? (void*)s.alloc<uint8_t>((size_t)d * stride) : (void*)s.alloc<uint16_t>((size_t)d * stride);
  emit(keys, n, pos, s.codes);
  // validation rows: keys, codes with the training boundaries, input order
  if (nv > 0) {
    T* Xvd = A.alloc<T>((size_t)nv * d);
    c.stage.h2d(Xvd, Xv, (size_t)nv * d * sizeof(T), st);
    std::vector<unsigned long long> f2, n2;
    unsigned long long* fd2 = nullptr;
    K* vkeys = make_keys<T>(c, A, Xvd, nv, d, f2, n2, &fd2);
    int* vpos = A.alloc<int>(nv);
    k_iota<<<grid_for(nv, 256, c.sm_count), 256, 0, st>>>(vpos, nv);
    const int64_t vstride = ceil_div(nv, kTile) * kTile;
    s.vcodes = s.code_bytes == 1 ? (void*)s.alloc<uint8_t>((size_t)d * vstride)
                                 : (void*)s.alloc<uint16_t>((size_t)d * vstride);
    emit(vkeys, nv, vpos, s.vcodes);
    s.vy = s.alloc<int8_t>(nv);
    BB_CUDA(cudaMemcpyAsync(s.vy, yv, (size_t)nv, cudaMemcpyHostToDevice, st));
    if (wv) {
      s.vw = s.alloc<double>(nv);
      BB_CUDA(cudaMemcpyAsync(s.vw, wv, (size_t)nv * 8, cudaMemcpyHostToDevice, st));
    }
  }
  BB_CUDA(cudaStreamSynchronize(st));
  return S.release();
}

static void elim_fit(Ctx& c, const ElimSession& s, const int* cols, int nc, const bb_fit_config& cfg, double* auc,
                     bb_fit_out* fo) {
  if (nc < 1 || nc > s.d) throw InvalidArg{"need 1..d feature columns"};
  for (int j = 0; j < nc; ++j)
    if (cols[j] < 0 || cols[j] >= s.d) throw InvalidArg{"feature column out of range"};
  if (cfg.binning_levels != s.levels) throw InvalidArg{"binning_levels differs from the prepared session"};
  cudaStream_t st = c.stream;
  Arena A(st);
  const int64_t tiles = ceil_div(s.n, kTile);
  int* cd = A.alloc<int>(nc);
  BB_CUDA(cudaMemcpyAsync(cd, cols, (size_t)nc * 4, cudaMemcpyHostToDevice, st));
  const int nt = s.B - 1;
  double* bsub = A.alloc<double>((size_t)nc * nt);
  for (int j = 0; j < nc; ++j)
    BB_CUDA(cudaMemcpyAsync(bsub + (size_t)j * nt, s.bounds + (size_t)cols[j] * nt, (size_t)nt * 8,
                            cudaMemcpyDeviceToDevice, st));
  bool any_nan = false;
  for (int j = 0; j < nc; ++j) any_nan |= s.nans[cols[j]] > 0;
  const int D = cfg.depth, T = cfg.n_trees, I = (1 << D) - 1, N = (1 << (D + 1)) - 1;
  FitShape fs{s.n, s.n_sig, nc, s.levels, s.B, D, I, N, T};
  std::vector<int> feat((size_t)T * I), cut((size_t)T * I);
  std::vector<unsigned char> vld((size_t)T * I);
  std::vector<double> gain((size_t)T * I), thr((size_t)T * I), nw((size_t)T * N), pur((size_t)T * N);
  bb_fit_out o{};
  if (fo) o = *fo;
  if (!o.feature) o.feature = feat.data();
  if (!o.cut_bin) o.cut_bin = cut.data();
  if (!o.valid) o.valid = vld.data();
  if (!o.gain) o.gain = gain.data();
  if (!o.threshold) o.threshold = thr.data();
  if (!o.node_weight) o.node_weight = nw.data();
  if (!o.node_purity) o.node_purity = pur.data();
  o.leaves = nullptr;
  o.scores = nullptr;
  FitStats stats;
  Shard shard;
  MaskFeed feed;
  feed.init(c, A, s.n, s.n_sig, cfg, shard, &stats);
  feed.ahead(0);
  double ms = 0.0;
  auto go = [&](auto* codes) {
    using CodeT = std::remove_pointer_t<decltype(codes)>;
    CodeT* sub = A.alloc<CodeT>((size_t)tiles * nc * kTile);
    k_gather_cols<CodeT><<<dim3((unsigned)tiles, nc), 256, 0, st>>>(codes, s.d, cd, nc, sub);
    BB_LAUNCH_CHECK();
    if (D <= 7)
      run_trees<CodeT, uint8_t>(c, A, fs, sub, s.code_off, s.w_cb, s.f0, s.shift, cfg, nullptr, 0, bsub, &o, &ms,
                                stats, shard, any_nan, feed);
    else
      run_trees<CodeT, uint16_t>(c, A, fs, sub, s.code_off, s.w_cb, s.f0, s.shift, cfg, nullptr, 0, bsub, &o, &ms,
                                 stats, shard, any_nan, feed);
  };
  if (s.code_bytes == 1) go(static_cast<uint8_t*>(s.codes));
  else go(static_cast<uint16_t*>(s.codes));
  if (fo) {
    if (fo->f0) *fo->f0 = s.f0;
    if (fo->fixed_shift) *fo->fixed_shift = s.shift;
  }
  if (!auc || s.nv == 0) return;
  // validation AUC of the refit
  int* fd = A.alloc<int>((size_t)T * I);
  int* cutd = A.alloc<int>((size_t)T * I);
  unsigned char* vd = A.alloc<unsigned char>((size_t)T * I);
  double* nwd = A.alloc<double>((size_t)T * N);
  std::vector<int> fz((size_t)T * I);
  for (size_t e = 0; e < fz.size(); ++e) fz[e] = o.valid[e] ? o.feature[e] : 0;
  BB_CUDA(cudaMemcpyAsync(fd, fz.data(), fz.size() * 4, cudaMemcpyHostToDevice, st));
  BB_CUDA(cudaMemcpyAsync(cutd, o.cut_bin, (size_t)T * I * 4, cudaMemcpyHostToDevice, st));
  BB_CUDA(cudaMemcpyAsync(vd, o.valid, (size_t)T * I, cudaMemcpyHostToDevice, st));
  BB_CUDA(cudaMemcpyAsync(nwd, o.node_weight, (size_t)T * N * 8, cudaMemcpyHostToDevice, st));
  double* p = A.alloc<double>(s.nv);
  const int g = grid_for(s.nv, 256, c.sm_count);
  if (s.code_bytes == 1)
    k_apply_codes<uint8_t><<<g, 256, 0, st>>>(static_cast<const uint8_t*>(s.vcodes), s.nv, s.d, s.code_off, cd, T, D,
                                              fd, cutd, vd, nwd, s.f0, p);
  else
    k_apply_codes<uint16_t><<<g, 256, 0, st>>>(static_cast<const uint16_t*>(s.vcodes), s.nv, s.d, s.code_off, cd, T,
                                               D, fd, cutd, vd, nwd, s.f0, p);
  BB_LAUNCH_CHECK();
  double ws, wb;
  *auc = auc_device(c, A, p, s.vy, s.vw, s.nv, &ws, &wb);
}

}  // namespace bb

using namespace bb;

// two copy streams and K + 1 events of a row pipeline (bb_predict)
struct PipeStreams {
  cudaStream_t s_in = nullptr, s_out = nullptr;
  cudaEvent_t ev[PinnedRing::kBufs + 1] = {};
  explicit PipeStreams(int) {
    BB_CUDA(cudaStreamCreateWithFlags(&s_in, cudaStreamNonBlocking));
    BB_CUDA(cudaStreamCreateWithFlags(&s_out, cudaStreamNonBlocking));
    for (auto& e : ev) BB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  ~PipeStreams() {
    if (s_in) {
      cudaStreamSynchronize(s_in);
      cudaStreamDestroy(s_in);
    }
    if (s_out) {
      cudaStreamSynchronize(s_out);
      cudaStreamDestroy(s_out);
    }
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
  }
};

struct bb_ctx {
  Ctx c;
};
struct bb_elim {
  ElimSession* s;
};

template <typename Fn>
static int guarded(Fn&& fn) {
  try {
    fn();
    return BB_OK;
  } catch (const InvalidArg& e) {
    set_error(e.msg);
    return BB_EINVAL;
  } catch (const CudaError& e) {
    set_error(e.msg);
    return BB_ECUDA;
  } catch (const std::exception& e) {
    set_error(e.what());
    return BB_ESTATE;
  }
}

extern "C" {

const char* bb_last_error(void) { return g_err.c_str(); }
int bb_abi_version(void) { return BB_ABI_VERSION; }

int bb_device_count(int32_t* out) {
  return guarded([&] {
    int n = 0;
    BB_CUDA(cudaGetDeviceCount(&n));
    *out = n;
  });
}

int bb_ctx_create(int32_t device, bb_ctx** out) {
  return guarded([&] {
    auto* h = new bb_ctx();
    h->c.device = device;
    try {
      BB_CUDA(cudaSetDevice(device));
      // the fit's main stream runs above the mask streams (BB_MASK_PRIO=2
      // default): the mask kernels backfill what the tree kernels leave, and a
      // pending histogram CTA is not starved by queued phase-1 CTAs.
      // cfg3: 728 -> 712 ms per fit; cfg2 unchanged (BB_MAIN_PRIO=0 BB_MASK_PRIO=0: the old order)
      {
        int lo_prio = 0, hi_prio = 0;
        BB_CUDA(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
        const bool main_hi = !(getenv("BB_MAIN_PRIO") && atoi(getenv("BB_MAIN_PRIO")) == 0);
        BB_CUDA(cudaStreamCreateWithPriority(&h->c.stream, cudaStreamNonBlocking, main_hi ? hi_prio : lo_prio));
      }
      BB_CUDA(cudaDeviceGetAttribute(&h->c.sm_count, cudaDevAttrMultiProcessorCount, device));
      // keep freed stream-ordered allocations cached in the device pool: the
      // default threshold (0) returns them to the OS at every synchronisation,
      // so each call would re-map its buffers inside the work it times
      cudaMemPool_t pool;
      BB_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
      uint64_t keep = UINT64_MAX;
      BB_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int bb_ctx_destroy(bb_ctx* ctx) {
  return guarded([&] {
    if (!ctx) return;
    cudaSetDevice(ctx->c.device);
    if (ctx->c.stream) {
      cudaStreamSynchronize(ctx->c.stream);
      cudaStreamDestroy(ctx->c.stream);
    }
    ctx->c.comm.destroy();
    delete ctx;
  });
}

int bb_ctx_init_comm(bb_ctx* ctx, int32_t rank, int32_t world, const uint8_t* unique_id) {
  return guarded([&] {
    if (!ctx || !unique_id) throw InvalidArg{"null argument"};
    if (world < 1 || rank < 0 || rank >= world) throw InvalidArg{"rank must be in [0, world)"};
    std::lock_guard<std::mutex> lock(ctx->c.mu);
    BB_CUDA(cudaSetDevice(ctx->c.device));
    ctx->c.comm.init(rank, world, unique_id);
  });
}

int bb_vgroup_create(int32_t world, bb_vgroup** out) {
  return guarded([&] {
    if (!out || world < 1) throw InvalidArg{"world must be >= 1"};
    auto* g = new VirtualGroup();
    g->world = world;
    *out = reinterpret_cast<bb_vgroup*>(g);
  });
}

int bb_vgroup_destroy(bb_vgroup* g) {
  return guarded([&] { delete reinterpret_cast<VirtualGroup*>(g); });
}

int bb_ctx_init_virtual(bb_ctx* ctx, int32_t rank, bb_vgroup* g) {
  return guarded([&] {
    if (!ctx || !g) throw InvalidArg{"null argument"};
    auto* vg = reinterpret_cast<VirtualGroup*>(g);
    if (rank < 0 || rank >= vg->world) throw InvalidArg{"rank must be in [0, world)"};
    std::lock_guard<std::mutex> lock(ctx->c.mu);
    ctx->c.comm.init_virtual(rank, vg);
  });
}

int bb_fit(bb_ctx* ctx, const void* X, int32_t x_dtype, int32_t x_on_device, int64_t n, int32_t d,
           const int8_t* y01, int32_t y_on_device, const double* w, int32_t w_on_device,
           const bb_fit_config* cfg, const bb_forced_cut* forced, int32_t n_forced, bb_fit_out* out) {
  return guarded([&] {
    if (!ctx || !cfg || !out) throw InvalidArg{"null argument"};
    // a shard of a row-sharded fit may hold a single row (the class check
    // runs on the global counts)
    if (n < (ctx->c.comm.active() ? 1 : 2) || d < 1) throw InvalidArg{"need at least 2 rows and 1 feature"};
    if (n >= (int64_t)1 << 31) throw InvalidArg{"at most 2^31-1 rows per device"};
    if (cfg->n_trees < 1) throw InvalidArg{"n_trees must be >= 1"};
    if (cfg->depth < 1 || cfg->depth > 15) throw InvalidArg{"depth must be in [1, 15]"};
    if (cfg->binning_levels < 1 || cfg->binning_levels > 15)
      throw InvalidArg{"binning_levels must be in [1, 15] on the GPU path (uint16 codes)"};
    if (!(cfg->shrinkage > 0.0 && cfg->shrinkage <= 1.0)) throw InvalidArg{"shrinkage must be in (0, 1]"};
    if (!(cfg->subsample > 0.0 && cfg->subsample <= 1.0)) throw InvalidArg{"subsample must be in (0, 1]"};
    const int64_t hist_bytes = (int64_t)2 * (1 << (cfg->depth - 1)) * d * (1 << cfg->binning_levels) * 8;
    if (hist_bytes > ((int64_t)16 << 30)) throw InvalidArg{"layer histogram exceeds 16 GiB (depth/features/levels)"};
    std::lock_guard<std::mutex> lock(ctx->c.mu);
    BB_CUDA(cudaSetDevice(ctx->c.device));
    if (x_dtype == BB_F32)
      fit_impl<float>(ctx->c, X, x_on_device, n, d, y01, y_on_device, w, w_on_device, *cfg, forced, n_forced, out);
    else if (x_dtype == BB_F64)
      fit_impl<double>(ctx->c, X, x_on_device, n, d, y01, y_on_device, w, w_on_device, *cfg, forced, n_forced, out);
    else
      throw InvalidArg{"x_dtype must be BB_F32 or BB_F64"};
  });
}

int bb_predict(bb_ctx* ctx, const bb_forest* fo, const void* X, int32_t x_dtype, int32_t x_on_device, int64_t n,
               int32_t d, double* out_prob, double* out_score, int32_t out_on_device) {
  return guarded([&] {
    if (!ctx || !fo) throw InvalidArg{"null argument"};
    if (d != fo->n_features)
      throw InvalidArg{"model expects " + std::to_string(fo->n_features) + " features, rows have " + std::to_string(d)};
    if (fo->n_trees < 0 || fo->depth < 1 || fo->depth > 20) throw InvalidArg{"invalid forest shape"};
    // cut features index the row in shared memory: reject out-of-range ones
    for (size_t e = 0, te = (size_t)fo->n_trees * ((1 << fo->depth) - 1); e < te; ++e)
      if (fo->valid[e] && (fo->feature[e] < 0 || fo->feature[e] >= d))
        throw InvalidArg{"cut feature " + std::to_string(fo->feature[e]) + " out of range for " + std::to_string(d) +
                         " features"};
    if (n == 0) return;
    std::lock_guard<std::mutex> lock(ctx->c.mu);
    Ctx& c = ctx->c;
    BB_CUDA(cudaSetDevice(c.device));
    cudaStream_t st = c.stream;
    Arena A(st);
    const int I = (1 << fo->depth) - 1, N = (1 << (fo->depth + 1)) - 1;
    const size_t TI = (size_t)fo->n_trees * I, TN = (size_t)fo->n_trees * N;
    int* feat = A.alloc<int>(TI);
    unsigned char* vld = A.alloc<unsigned char>(TI);
    double* thr = A.alloc<double>(TI);
    double* nw = A.alloc<double>(TN);
    if (TI) {
      BB_CUDA(cudaMemcpyAsync(feat, fo->feature, TI * 4, cudaMemcpyHostToDevice, st));
      BB_CUDA(cudaMemcpyAsync(vld, fo->valid, TI, cudaMemcpyHostToDevice, st));
      BB_CUDA(cudaMemcpyAsync(thr, fo->threshold, TI * 8, cudaMemcpyHostToDevice, st));
      BB_CUDA(cudaMemcpyAsync(nw, fo->node_weight, TN * 8, cudaMemcpyHostToDevice, st));
    }
    ApplyForest af{fo->n_trees, fo->depth, I, N, feat, vld, thr, nw, fo->f0};
    const size_t es = x_dtype == BB_F32 ? 4 : 8;
    const size_t row_bytes = (size_t)d * es;
    // host rows: uploaded and scored in row chunks through pinned staging
    // (bb_stage.h), the chunk's DMA, kernels and result read-back overlapping
    const bool pipe = !x_on_device && !out_on_device && (size_t)n * row_bytes >= HostStager::kMinStaged &&
                      !host_pointer_is_pinned(X) && !getenv("BB_NO_STAGING");
    const void* Xd = X;
    if (!x_on_device) {
      void* p = A.alloc<unsigned char>((size_t)n * row_bytes);
      if (!pipe) c.stage.h2d(p, X, (size_t)n * row_bytes, st);
      Xd = p;
    }
    double* pd = out_prob;
    double* fd = out_score;
    if (!out_on_device) {
      pd = out_prob ? A.alloc<double>(n) : nullptr;
      fd = out_score ? A.alloc<double>(n) : nullptr;
    }
    const size_t smem = (size_t)APPLY_ROWS * (d + 1) * es;
    const size_t smem32 = ((size_t)kApplyRows * (d + 1) * 4 + 15) / 16 * 16 + (size_t)kApplyTB * (N * 8 + I * 8);
    const int D = fo->depth;
    const size_t smemD = ((size_t)kApplyDRows * (d + 1) * 4 + 15) / 16 * 16 +
                         (size_t)kApplyDTB * (((size_t)1 << D) * 8 + (size_t)I * 8);
    // launch_rows(r0, nr): score rows [r0, r0 + nr) on st.  The host staging
    // vectors of the chosen kernel live until the final synchronisation.
    std::function<void(int64_t, int64_t)> launch_rows;
    std::vector<int2> hr, hn;
    std::vector<double> hl;
    std::unique_ptr<ApplyRoots> roots;
    auto rows_at = [&](int64_t r0) { return (const void*)((const char*)Xd + (size_t)r0 * row_bytes); };
    auto at = [](double* p, int64_t r0) { return p ? p + r0 : nullptr; };
    if (x_dtype == BB_F32 && D >= 1 && D <= 6 && smemD <= 200 * 1024) {
      // fixed-depth walk over leaf tables with the invalid-node stops folded in
      hr.resize(TI);
      hn.resize(TI);
      hl.resize((size_t)fo->n_trees << D);
      for (int t = 0; t < fo->n_trees; ++t) {
        for (int k = 0; k < I; ++k) {
          const size_t e = (size_t)t * I + k;
          const double th = fo->threshold[e];
          float tf = (float)th;  // round-to-nearest, then step up if below th
          if ((double)tf < th) tf = std::nextafter(tf, INFINITY);
          int bits;
          std::memcpy(&bits, &tf, 4);
          hr[e] = make_int2(fo->valid[e] ? 4 * fo->feature[e] : 0, bits);
          hn[e] = make_int2(fo->valid[e] ? fo->feature[e] : -1, bits);
        }
        for (int l = 0; l < (1 << D); ++l) {
          int nd = 0, stop = -1;
          for (int lv = 0; lv < D; ++lv) {
            if (!fo->valid[(size_t)t * I + nd]) {
              stop = nd;
              break;
            }
            nd = 2 * nd + 1 + ((l >> (D - 1 - lv)) & 1);
          }
          hl[((size_t)t << D) + l] = fo->node_weight[(size_t)t * N + (stop >= 0 ? stop : nd)];
        }
      }
      int2* rd = A.alloc<int2>(std::max<size_t>(1, TI));
      int2* nd2 = A.alloc<int2>(std::max<size_t>(1, TI));
      double* ld = A.alloc<double>(std::max<size_t>(1, hl.size()));
      if (TI) {
        BB_CUDA(cudaMemcpyAsync(rd, hr.data(), TI * sizeof(int2), cudaMemcpyHostToDevice, st));
        BB_CUDA(cudaMemcpyAsync(nd2, hn.data(), TI * sizeof(int2), cudaMemcpyHostToDevice, st));
      }
      if (!hl.empty()) BB_CUDA(cudaMemcpyAsync(ld, hl.data(), hl.size() * 8, cudaMemcpyHostToDevice, st));
      // the first PL levels' records of each tree come from the kernel's
      // parameter space (uniform loads instead of shared-memory wavefronts);
      // a forest larger than the parameter space takes several launches,
      // each continuing F in tree order
      // (2 levels measured best: cfg4 889 M rows/s; 3 levels need two launches
      // for 1000 trees and a 4-way select: 583 M)
      const int PL = getenv("BB_APPLY_PARAM_LEVELS") ? std::max(0, std::min(std::min(3, D), atoi(getenv("BB_APPLY_PARAM_LEVELS"))))
                                                     : std::min(D, 2);
      const int RP = (1 << PL) - 1;
      const int per_launch = RP ? kApplyParamRecs / RP : fo->n_trees;
      const int n_launch = fo->n_trees > 0 ? (int)ceil_div(fo->n_trees, per_launch) : 1;
      double* fa = fd;
      if (n_launch > 1 && !fa) fa = A.alloc<double>(n);  // F between launches
      roots = std::make_unique<ApplyRoots>();  // host staging; each launch copies its parameters
      launch_rows = [=, &roots, &hr](int64_t r0, int64_t nr) {
        const unsigned gd = (unsigned)ceil_div(nr, kApplyDRows);
        for (int li = 0; li < n_launch; ++li) {
          const int t0 = li * per_launch, t1 = std::min(fo->n_trees, t0 + per_launch);
          for (int t = t0; t < t1; ++t)
            for (int k = 0; k < RP; ++k) roots->r[(t - t0) * RP + k] = hr[(size_t)t * I + k];
          ApplyD ad{fo->n_trees, t0, t1, li == 0 ? 1 : 0, li == n_launch - 1 ? 1 : 0, rd, ld, nd2, nw, fo->f0};
          auto launch = [&](auto kern) {
            BB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
            kern<<<gd, kApplyDRows, smemD, st>>>((const float*)rows_at(r0), nr, d, ad, at(pd, r0), at(fa, r0), *roots);
            BB_LAUNCH_CHECK();
          };
#define BB_APPLY_D(DD)                                      \
  do {                                                      \
    if (PL >= 3 && DD >= 3) launch(k_apply_d<DD, 3>);       \
    else if (PL >= 2 && DD >= 2) launch(k_apply_d<DD, 2>);  \
    else if (PL >= 1) launch(k_apply_d<DD, 1>);             \
    else launch(k_apply_d<DD, 0>);                          \
  } while (0)
          switch (D) {
            case 1: BB_APPLY_D(1); break;
            case 2: BB_APPLY_D(2); break;
            case 3: BB_APPLY_D(3); break;
            case 4: BB_APPLY_D(4); break;
            case 5: BB_APPLY_D(5); break;
            default: BB_APPLY_D(6); break;
          }
#undef BB_APPLY_D
        }
      };
    } else if (x_dtype == BB_F32 && smem32 <= 200 * 1024) {
      // packed node records with float-ceiling thresholds (exact for float rows)
      hn.resize(TI);
      for (size_t e = 0; e < TI; ++e) {
        const double t = fo->threshold[e];
        float tf = (float)t;  // round-to-nearest, then step up if below t
        if ((double)tf < t) tf = std::nextafter(tf, INFINITY);
        int bits;
        std::memcpy(&bits, &tf, 4);
        hn[e] = make_int2(fo->valid[e] ? fo->feature[e] : -1, bits);
      }
      int2* nd = A.alloc<int2>(TI);
      if (TI) BB_CUDA(cudaMemcpyAsync(nd, hn.data(), TI * sizeof(int2), cudaMemcpyHostToDevice, st));
      ApplyF32 a32{fo->n_trees, fo->depth, I, N, nd, nw, fo->f0};
      BB_CUDA(cudaFuncSetAttribute(k_apply_f32, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
      launch_rows = [=](int64_t r0, int64_t nr) {
        k_apply_f32<<<(unsigned)ceil_div(nr, kApplyRows), kApplyRows, smem32, st>>>((const float*)rows_at(r0), nr, d, a32,
                                                                                  at(pd, r0), at(fd, r0));
        BB_LAUNCH_CHECK();
      };
    } else if (x_dtype == BB_F32) {
      BB_CUDA(cudaFuncSetAttribute(k_apply<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
      launch_rows = [=](int64_t r0, int64_t nr) {
        k_apply<float><<<(unsigned)ceil_div(nr, APPLY_ROWS), APPLY_ROWS, smem, st>>>((const float*)rows_at(r0), nr, d, af,
                                                                                   at(pd, r0), at(fd, r0));
        BB_LAUNCH_CHECK();
      };
    } else {
      BB_CUDA(cudaFuncSetAttribute(k_apply<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
      launch_rows = [=](int64_t r0, int64_t nr) {
        k_apply<double><<<(unsigned)ceil_div(nr, APPLY_ROWS), APPLY_ROWS, smem, st>>>((const double*)rows_at(r0), nr, d,
                                                                                    af, at(pd, r0), at(fd, r0));
        BB_LAUNCH_CHECK();
      };
    }
    if (!pipe) {
      launch_rows(0, n);
      if (!out_on_device) {
        if (out_prob) c.stage.d2h(out_prob, pd, (size_t)n * 8, st);
        if (out_score) c.stage.d2h(out_score, fd, (size_t)n * 8, st);
      }
      BB_CUDA(cudaStreamSynchronize(st));
      return;
    }
    // ---- pipelined host rows: chunk i's upload (copy stream), kernels (st)
    // and read-back (second copy stream) overlap chunks i+1 / i-1
    constexpr int K = PinnedRing::kBufs;
    const size_t out_chunk = HostStager::chunk() / 4;
    int64_t rows_c = (int64_t)std::min(HostStager::chunk() / row_bytes, out_chunk / 8);
    rows_c = std::max<int64_t>(1024, rows_c / 1024 * 1024);
    HostStager& hs = c.stage;
    hs.in.ensure(std::max(HostStager::chunk(), (size_t)rows_c * row_bytes));
    if (out_prob) hs.out.ensure(std::max(HostStager::chunk(), (size_t)rows_c * 8));
    if (out_score) hs.out2.ensure(std::max(HostStager::chunk(), (size_t)rows_c * 8));
    PipeStreams ps(c.device);
    const int64_t chunks = ceil_div(n, rows_c);
    cudaEvent_t ev_k[K];
    for (int b = 0; b < K; ++b) ev_k[b] = ps.ev[b];
    auto drain = [&](int64_t j) {
      const int b = (int)(j % K);
      const int64_t r0 = j * rows_c, nr = std::min(rows_c, n - r0);
      if (out_prob) {
        BB_CUDA(cudaEventSynchronize(hs.out.ev(b)));
        parallel_memcpy(out_prob + r0, hs.out.buf(b), (size_t)nr * 8);
      }
      if (out_score) {
        BB_CUDA(cudaEventSynchronize(hs.out2.ev(b)));
        parallel_memcpy(out_score + r0, hs.out2.buf(b), (size_t)nr * 8);
      }
    };
    cudaEvent_t ev_setup = ps.ev[K];
    BB_CUDA(cudaEventRecord(ev_setup, st));  // forest tables uploaded; Xd / pd allocated in stream order
    BB_CUDA(cudaStreamWaitEvent(ps.s_in, ev_setup, 0));
    BB_CUDA(cudaStreamWaitEvent(ps.s_out, ev_setup, 0));
    for (int64_t i = 0; i < chunks; ++i) {
      const int b = (int)(i % K);
      const int64_t r0 = i * rows_c, nr = std::min(rows_c, n - r0);
      if (i >= K) drain(i - K);  // frees out buffer b; in buffer b is guarded by its own event
      BB_CUDA(cudaEventSynchronize(hs.in.ev(b)));
      parallel_memcpy(hs.in.buf(b), (const char*)X + (size_t)r0 * row_bytes, (size_t)nr * row_bytes);
      BB_CUDA(cudaMemcpyAsync((char*)Xd + (size_t)r0 * row_bytes, hs.in.buf(b), (size_t)nr * row_bytes,
                              cudaMemcpyHostToDevice, ps.s_in));
      BB_CUDA(cudaEventRecord(hs.in.ev(b), ps.s_in));
      BB_CUDA(cudaStreamWaitEvent(st, hs.in.ev(b), 0));
      launch_rows(r0, nr);
      BB_CUDA(cudaEventRecord(ev_k[b], st));
      BB_CUDA(cudaStreamWaitEvent(ps.s_out, ev_k[b], 0));
      if (out_prob) {
        BB_CUDA(cudaMemcpyAsync(hs.out.buf(b), pd + r0, (size_t)nr * 8, cudaMemcpyDeviceToHost, ps.s_out));
        BB_CUDA(cudaEventRecord(hs.out.ev(b), ps.s_out));
      }
      if (out_score) {
        BB_CUDA(cudaMemcpyAsync(hs.out2.buf(b), fd + r0, (size_t)nr * 8, cudaMemcpyDeviceToHost, ps.s_out));
        BB_CUDA(cudaEventRecord(hs.out2.ev(b), ps.s_out));
      }
    }
    for (int64_t j = std::max<int64_t>(0, chunks - K); j < chunks; ++j) drain(j);
    BB_CUDA(cudaStreamSynchronize(ps.s_in));
    BB_CUDA(cudaStreamSynchronize(ps.s_out));
    BB_CUDA(cudaStreamSynchronize(st));
  });
}

int bb_bin(bb_ctx* ctx, const void* X, int32_t x_dtype, int64_t n, int32_t d, int32_t levels, double* out_boundaries,
           int16_t* out_codes) {
  return guarded([&] {
    if (!ctx) throw InvalidArg{"null argument"};
    if (levels < 1 || levels > 15) throw InvalidArg{"levels must be in [1, 15]"};
    std::lock_guard<std::mutex> lock(ctx->c.mu);
    Ctx& c = ctx->c;
    BB_CUDA(cudaSetDevice(c.device));
    cudaStream_t st = c.stream;
    Arena A(st);
    const int nt = (1 << levels) - 1;
    auto body = [&](auto tag) {
      using T = decltype(tag);
      using K = typename KeyOf<T>::K;
      T* Xd = A.alloc<T>((size_t)n * d);
      c.stage.h2d(Xd, X, (size_t)n * d * sizeof(T), st);
      std::vector<unsigned long long> fin, nan_;
      unsigned long long* fdev = nullptr;
      K* keys = make_keys<T>(c, A, Xd, n, d, fin, nan_, &fdev);
      double* bounds = A.alloc<double>((size_t)d * nt);
      K* bkeys = A.alloc<K>((size_t)d * nt);
      run_select<T>(c, A, keys, n, d, levels, fdev, bounds, bkeys);
      BB_CUDA(cudaMemcpyAsync(out_boundaries, bounds, (size_t)d * nt * 8, cudaMemcpyDeviceToHost, st));
      if (out_codes) {  // null: boundaries only
        int* pos = A.alloc<int>(n);
        k_iota<<<grid_for(n, 256, c.sm_count), 256, 0, st>>>(pos, n);
        BB_LAUNCH_CHECK();
        uint16_t* codes = A.alloc<uint16_t>((size_t)d * n);
        BB_CUDA(cudaFuncSetAttribute(k_codes<K, uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        k_codes<K, uint16_t><<<dim3((unsigned)std::max<int64_t>(1, ceil_div(n, 1024)), d), 256, codes_smem<K>(nt),
                               st>>>(keys, n, nt, bkeys, pos, codes, n, 0, d, 0);
        BB_LAUNCH_CHECK();
        BB_CUDA(cudaMemcpyAsync(out_codes, codes, (size_t)d * n * 2, cudaMemcpyDeviceToHost, st));
      }
      BB_CUDA(cudaStreamSynchronize(st));
    };
    if (x_dtype == BB_F32) body(float{});
    else if (x_dtype == BB_F64) body(double{});
    else throw InvalidArg{"x_dtype must be BB_F32 or BB_F64"};
  });
}

int bb_layer_hist(bb_ctx* ctx, const uint16_t* codes, const uint16_t* node, const int64_t* q, int64_t n, int64_t n_sig,
                  int32_t d, int32_t levels, int32_t layer, int64_t* out_hist) {
  return guarded([&] {
    if (!ctx) throw InvalidArg{"null argument"};
    if (layer < 1 || layer > 15 || levels < 1 || levels > 15) throw InvalidArg{"bad layer/levels"};
    std::lock_guard<std::mutex> lock(ctx->c.mu);
    Ctx& c = ctx->c;
    BB_CUDA(cudaSetDevice(c.device));
    cudaStream_t st = c.stream;
    Arena A(st);
    const int B = 1 << levels;
    const int64_t npad = ceil_div(n, kRowPad) * kRowPad;
    if (hist_path_env() == 5) {
      // node-partitioned row lists (kernels_hist_list.cuh), built on the host
      // with the fit's region rule (full layer: both children listed)
      if (B > 256 || d > 64) throw InvalidArg{"list histogram: needs B <= 256 and d <= 64"};
      const int code_off = B == 256 ? 1 : 0;
      const int NW = d <= 32 ? 8 : 16;  // row words
      const bool nw16 = !(getenv("BB_LH_GROUPS") && atoi(getenv("BB_LH_GROUPS")) != 0);
      const int groups = (NW == 16 && !nw16) ? 2 : 1;
      std::vector<uint32_t> rch((size_t)npad * NW, 0u);
      for (int f = 0; f < d; ++f)
        for (int64_t i = 0; i < n; ++i) {
          const int v = (int)codes[(size_t)f * n + i] - code_off;
          if (v < 0) throw InvalidArg{"list histogram: B = 256 needs NaN-free codes"};
          rch[(size_t)i * NW + f / 4] |= (uint32_t)v << (8 * (f & 3));
        }
      const int nodes = 1 << (layer - 1), start = nodes - 1;
      const int nn = 2 * nodes + 1;  // heap ids < 2^layer + ...
      std::vector<int> cnth((size_t)2 * (2 * nodes + nodes), 0);
      auto cls_of = [&](int64_t i) { return i < n_sig ? 0 : 1; };
      std::vector<int> lr(std::max<int64_t>(1, n), 0);
      std::vector<long long> lqv(std::max<int64_t>(1, n), 0);
      if (layer == 1) {
        int fill[2] = {0, 0};
        for (int64_t i = 0; i < n; ++i) {
          if (node[i] != 0) continue;
          const int k = cls_of(i);
          const int64_t pos = (k ? n_sig : 0) + fill[k]++;
          lr[pos] = (int)i;
          lqv[pos] = q[i];
        }
        cnth[0] = fill[0];
        cnth[1] = fill[1];
      } else {
        const int ps = (1 << (layer - 2)) - 1, np = 1 << (layer - 2);
        for (int64_t i = 0; i < n; ++i) {
          const int nd = node[i];
          if (nd < start || nd >= start + nodes) continue;
          const int k = cls_of(i), par = (nd - 1) / 2;
          cnth[2 * nd + k] += 1;
          cnth[2 * par + k] += 1;
        }
        std::vector<int> reg(2 * np), fl(2 * np, 0), fr(2 * np, 0);
        int off = 0;
        for (int k = 0; k < 2; ++k)
          for (int pp = 0; pp < np; ++pp) {
            reg[k * np + pp] = off;
            off += cnth[2 * (ps + pp) + k];
          }
        for (int64_t i = 0; i < n; ++i) {
          const int nd = node[i];
          if (nd < start || nd >= start + nodes) continue;
          const int k = cls_of(i), par = (nd - 1) / 2, pl = par - ps;
          int pos;
          if (nd & 1) pos = reg[k * np + pl] + fl[k * np + pl]++;
          else pos = reg[k * np + pl] + cnth[2 * par + k] - 1 - fr[k * np + pl]++;
          lr[pos] = (int)i;
          lqv[pos] = q[i];
        }
      }
      (void)nn;
      uint32_t* rcd = A.alloc<uint32_t>(rch.size());
      int* lrd = A.alloc<int>(lr.size());
      long long* lqd = A.alloc<long long>(lqv.size());
      int* cd = A.alloc<int>(cnth.size());
      BB_CUDA(cudaMemcpyAsync(rcd, rch.data(), rch.size() * 4, cudaMemcpyHostToDevice, st));
      BB_CUDA(cudaMemcpyAsync(lrd, lr.data(), lr.size() * 4, cudaMemcpyHostToDevice, st));
      BB_CUDA(cudaMemcpyAsync(lqd, lqv.data(), lqv.size() * 8, cudaMemcpyHostToDevice, st));
      BB_CUDA(cudaMemcpyAsync(cd, cnth.data(), cnth.size() * 4, cudaMemcpyHostToDevice, st));
      const size_t hsz = (size_t)2 * nodes * d * B;
      unsigned long long* hist = A.alloc<unsigned long long>(hsz);
      BB_CUDA(cudaMemsetAsync(hist, 0, hsz * 8, st));
      const bool k8 = NW == 8 || groups == 2;
      const int grid = k8 ? 2 * c.sm_count : c.sm_count;
      if (k8) {
        BB_CUDA(cudaFuncSetAttribute(k_hist_list<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, lh_smem_bytes<8>()));
        k_hist_list<8><<<grid, kLhThreads, lh_smem_bytes<8>(), st>>>(rcd, lrd, lqd, cd, layer, 0, n_sig, d, B, code_off,
                                                                     nodes, hist, NW, groups);
      } else {
        BB_CUDA(cudaFuncSetAttribute(k_hist_list<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, lh_smem_bytes<16>()));
        k_hist_list<16><<<grid, kLhThreads, lh_smem_bytes<16>(), st>>>(rcd, lrd, lqd, cd, layer, 0, n_sig, d, B,
                                                                       code_off, nodes, hist, 16, 1);
      }
      BB_LAUNCH_CHECK();
      BB_CUDA(cudaStreamSynchronize(st));
      BB_CUDA(cudaMemcpyAsync(out_hist, hist, hsz * 8, cudaMemcpyDeviceToHost, st));
      BB_CUDA(cudaStreamSynchronize(st));
      return;
    }
    std::vector<uint16_t> tiled((size_t)d * npad, 0);
    for (int f = 0; f < d; ++f)
      for (int64_t i = 0; i < n; ++i) tiled[(size_t)code_index(i, f, d)] = codes[(size_t)f * n + i];
    uint16_t* cd = A.alloc<uint16_t>((size_t)d * npad);
    uint16_t* nd = A.alloc<uint16_t>(npad);
    long long* qd = A.alloc<long long>(npad);
    BB_CUDA(cudaMemsetAsync(nd, 0, (size_t)npad * 2, st));
    BB_CUDA(cudaMemsetAsync(qd, 0, (size_t)npad * 8, st));
    BB_CUDA(cudaMemcpyAsync(cd, tiled.data(), (size_t)d * npad * 2, cudaMemcpyHostToDevice, st));
    BB_CUDA(cudaMemcpyAsync(nd, node, (size_t)n * 2, cudaMemcpyHostToDevice, st));
    BB_CUDA(cudaMemcpyAsync(qd, q, (size_t)n * 8, cudaMemcpyHostToDevice, st));
    FitShape s{n, n_sig, d, levels, B, layer, 0, 0, 1};
    const HistPlan p = plan_layer<uint16_t, uint16_t>(layer, s, c.sm_count, false);  // full layer
    const size_t hsz = (size_t)2 * p.nodes * d * B;
    unsigned long long* hist = A.alloc<unsigned long long>(hsz);
    BB_CUDA(cudaMemsetAsync(hist, 0, hsz * 8, st));
    const FlPlan fl = plan_fl<uint16_t, uint16_t>(layer, s, c.sm_count, false, cd);
    set_hist_smem_attrs<uint16_t, uint16_t>();
    const int64_t pe = (int64_t)fl_grid(fl) * fl_cta_stride(fl, B);
    long long* partials = pe ? A.alloc<long long>((size_t)pe) : nullptr;
    launch_layer_hist<uint16_t, uint16_t>(p, fl, c.sm_count, cd, 0, nd, qd, n, n_sig, d, B, hist, st, partials);
    BB_CUDA(cudaStreamSynchronize(st));  // host staging vector lives until here
    BB_CUDA(cudaMemcpyAsync(out_hist, hist, hsz * 8, cudaMemcpyDeviceToHost, st));
    BB_CUDA(cudaStreamSynchronize(st));
  });
}

int bb_split(bb_ctx* ctx, const int64_t* hist, int32_t d, int32_t levels, int32_t layer, int32_t final_layer,
             int32_t shift, const double* boundaries, uint8_t* out_valid, int32_t* out_feature, int32_t* out_cut,
             double* out_gain, double* out_threshold) {
  return guarded([&] {
    if (!ctx) throw InvalidArg{"null argument"};
    if (layer < 1 || layer > 15 || levels < 1 || levels > 15) throw InvalidArg{"bad layer/levels"};
    std::lock_guard<std::mutex> lock(ctx->c.mu);
    Ctx& c = ctx->c;
    BB_CUDA(cudaSetDevice(c.device));
    cudaStream_t st = c.stream;
    Arena A(st);
    const int B = 1 << levels, nodes = 1 << (layer - 1), start = nodes - 1;
    const int n_internal = 2 * nodes - 1;  // heap ids 0 .. start+nodes-1
    const size_t hsz = (size_t)2 * nodes * d * B;
    unsigned long long* hd = A.alloc<unsigned long long>(hsz);
    BB_CUDA(cudaMemcpyAsync(hd, hist, hsz * 8, cudaMemcpyHostToDevice, st));
    double* bd = A.alloc<double>((size_t)d * (B - 1));
    BB_CUDA(cudaMemcpyAsync(bd, boundaries, (size_t)d * (B - 1) * 8, cudaMemcpyHostToDevice, st));
    TreeArrays ta;
    ta.feature = A.alloc<int>(n_internal);
    ta.cut = A.alloc<int>(n_internal);
    ta.valid = A.alloc<unsigned char>(n_internal);
    ta.gain = A.alloc<double>(n_internal);
    ta.thr = A.alloc<double>(n_internal);
    ta.nw = nullptr;
    ta.pur = nullptr;
    ta.forced = nullptr;
    SplitScratch sc;
    sc.best_gain = A.alloc<double>((size_t)nodes * d);
    sc.best_flat = A.alloc<int>((size_t)nodes * d);
    sc.forced_gain = A.alloc<double>(nodes);
    sc.done = A.alloc<unsigned int>(nodes);
    BB_CUDA(cudaMemsetAsync(sc.done, 0, (size_t)nodes * 4, st));
    const int n_fc_want = std::max(1, std::min<int>(d, (2 * c.sm_count + nodes - 1) / nodes));
    const int fc_size = (int)ceil_div(d, n_fc_want);
    const int n_fc = (int)ceil_div(d, fc_size);
    k_split<256><<<dim3(nodes, n_fc), 256, 0, st>>>(hd, d, B, start, nodes, fc_size, final_layer, std::ldexp(1.0, -shift),
                                                   0, n_internal, ta, bd, sc, nullptr, 0, 0, nullptr);
    BB_LAUNCH_CHECK();
    BB_CUDA(cudaMemcpyAsync(out_valid, ta.valid + start, nodes, cudaMemcpyDeviceToHost, st));
    BB_CUDA(cudaMemcpyAsync(out_feature, ta.feature + start, (size_t)nodes * 4, cudaMemcpyDeviceToHost, st));
    BB_CUDA(cudaMemcpyAsync(out_cut, ta.cut + start, (size_t)nodes * 4, cudaMemcpyDeviceToHost, st));
    BB_CUDA(cudaMemcpyAsync(out_gain, ta.gain + start, (size_t)nodes * 8, cudaMemcpyDeviceToHost, st));
    BB_CUDA(cudaMemcpyAsync(out_threshold, ta.thr + start, (size_t)nodes * 8, cudaMemcpyDeviceToHost, st));
    BB_CUDA(cudaStreamSynchronize(st));
  });
}

int bb_subsample_masks(int64_t n_sig, int64_t n_bkg, double rate, int32_t n_trees, const bb_fit_config* rng,
                       uint32_t* out_bits) {
  return guarded([&] {
    if (!rng || !out_bits) throw InvalidArg{"null argument"};
    if (!(rate > 0.0 && rate <= 1.0)) throw InvalidArg{"subsample rate must be in (0, 1]"};
    Pcg64 g;
    g.state = ((unsigned __int128)rng->pcg_state_hi << 64) | rng->pcg_state_lo;
    g.inc = ((unsigned __int128)rng->pcg_inc_hi << 64) | rng->pcg_inc_lo;
    g.has_uint32 = rng->pcg_has_uint32;
    g.uinteger = rng->pcg_uinteger;
    const int64_t words = ceil_div(n_sig + n_bkg, 32);
    std::vector<uint32_t> perm;
    for (int t = 0; t < n_trees; ++t) subsample_tree(g, n_sig, n_bkg, rate, out_bits + (size_t)t * words, perm);
  });
}

int bb_subsample_masks_gpu(bb_ctx* ctx, int64_t n_sig, int64_t n_bkg, double rate, int32_t n_trees,
                           const bb_fit_config* rng, uint32_t* out_bits) {
  return guarded([&] {
    if (!ctx || !rng || !out_bits) throw InvalidArg{"null argument"};
    if (!(rate > 0.0 && rate <= 1.0)) throw InvalidArg{"subsample rate must be in (0, 1]"};
    if (n_sig < 0 || n_bkg < 0 || n_sig + n_bkg >= ((int64_t)1 << 31)) throw InvalidArg{"bad block sizes"};
    std::lock_guard<std::mutex> lock(ctx->c.mu);
    Ctx& c = ctx->c;
    BB_CUDA(cudaSetDevice(c.device));
    cudaStream_t st = c.stream;
    Arena A(st);
    MaskGen mg;
    mg.init(A, st, n_sig, n_bkg, rate, *rng, c.sm_count);
    const int64_t words = ceil_div(n_sig + n_bkg, 32);
    unsigned int* bits = A.alloc<unsigned int>((size_t)std::max<int64_t>(1, words) * n_trees);
    int64_t launches = 0;
    for (int t = 0; t < n_trees; t += kChunk) {
      const int cnt = std::min(kChunk, n_trees - t);
      unsigned int* bp[kChunk];
      for (int j = 0; j < cnt; ++j) bp[j] = bits + (size_t)(t + j) * words;
      mg.enqueue_chunk(st, bp, cnt, nullptr, launches);
    }
    mg.join(st);
    if (words) BB_CUDA(cudaMemcpyAsync(out_bits, bits, (size_t)words * n_trees * 4, cudaMemcpyDeviceToHost, st));
    BB_CUDA(cudaStreamSynchronize(st));
    mg.report(st);
  });
}

double bb_pairwise_sum(const double* a, int64_t n) { return pairwise(a, n); }

}  // extern "C"

int bb_roc_auc(bb_ctx* ctx, const double* scores, const int8_t* y01, const double* w, int64_t n, double* out_auc) {
  return guarded([&] {
    if (!ctx || !scores || !y01 || !out_auc) throw InvalidArg{"null argument"};
    if (n < 1) throw InvalidArg{"roc_auc needs both classes with positive total weight"};
    std::lock_guard<std::mutex> lock(ctx->c.mu);
    Ctx& c = ctx->c;
    BB_CUDA(cudaSetDevice(c.device));
    Arena A(c.stream);
    double* p = A.alloc<double>(n);
    int8_t* y = A.alloc<int8_t>(n);
    double* wd = w ? A.alloc<double>(n) : nullptr;
    c.stage.h2d(p, scores, (size_t)n * 8, c.stream);
    BB_CUDA(cudaMemcpyAsync(y, y01, (size_t)n, cudaMemcpyHostToDevice, c.stream));
    if (w) c.stage.h2d(wd, w, (size_t)n * 8, c.stream);
    double ws, wb;
    *out_auc = auc_device(c, A, p, y, wd, n, &ws, &wb);
  });
}

int bb_elim_create(bb_ctx* ctx, const void* X, int32_t x_dtype, int64_t n, int32_t d, const int8_t* y01,
                   const double* w, int32_t levels, const void* Xv, int64_t n_val, const int8_t* y01_val,
                   const double* w_val, bb_elim** out) {
  return guarded([&] {
    if (!ctx || !X || !y01 || !out) throw InvalidArg{"null argument"};
    if (n < 2 || d < 1) throw InvalidArg{"need at least 2 rows and 1 feature"};
    if (n >= (int64_t)1 << 31 || n_val >= (int64_t)1 << 31) throw InvalidArg{"at most 2^31-1 rows per device"};
    if (levels < 1 || levels > 15) throw InvalidArg{"binning_levels must be in [1, 15] on the GPU path (uint16 codes)"};
    if (n_val > 0 && (!Xv || !y01_val)) throw InvalidArg{"null validation argument"};
    std::lock_guard<std::mutex> lock(ctx->c.mu);
    BB_CUDA(cudaSetDevice(ctx->c.device));
    ElimSession* s;
    if (x_dtype == BB_F32)
      s = elim_prepare<float>(ctx->c, (const float*)X, n, d, y01, w, levels, (const float*)Xv, n_val, y01_val, w_val);
    else if (x_dtype == BB_F64)
      s = elim_prepare<double>(ctx->c, (const double*)X, n, d, y01, w, levels, (const double*)Xv, n_val, y01_val,
                               w_val);
    else
      throw InvalidArg{"x_dtype must be BB_F32 or BB_F64"};
    *out = new bb_elim{s};
  });
}

int bb_elim_fit(bb_ctx* ctx, const bb_elim* e, const int32_t* cols, int32_t n_cols, const bb_fit_config* cfg,
                double* out_auc, bb_fit_out* out) {
  return guarded([&] {
    if (!ctx || !e || !cols || !cfg) throw InvalidArg{"null argument"};
    if (cfg->n_trees < 1) throw InvalidArg{"n_trees must be >= 1"};
    if (cfg->depth < 1 || cfg->depth > 15) throw InvalidArg{"depth must be in [1, 15]"};
    if (!(cfg->shrinkage > 0.0 && cfg->shrinkage <= 1.0)) throw InvalidArg{"shrinkage must be in (0, 1]"};
    if (!(cfg->subsample > 0.0 && cfg->subsample <= 1.0)) throw InvalidArg{"subsample must be in (0, 1]"};
    std::lock_guard<std::mutex> lock(ctx->c.mu);
    BB_CUDA(cudaSetDevice(ctx->c.device));
    if (e->s->device != ctx->c.device) throw InvalidArg{"session and context are on different devices"};
    elim_fit(ctx->c, *e->s, cols, n_cols, *cfg, out_auc, out);
  });
}

int bb_elim_destroy(bb_elim* e) {
  return guarded([&] {
    if (!e) return;
    delete e->s;
    delete e;
  });
}
