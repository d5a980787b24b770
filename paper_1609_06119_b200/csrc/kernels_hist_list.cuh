// Node-partitioned ("list") layer histogram (trees.py:139-167) for u8 codes
// (B <= 256) and d <= 64 features.
//
// Row lists.  The active rows of a tree are kept in per-(node, class) lists
// of (row id, fixed-point weight q): the refresh kernel lists every active
// row for layer 1 (class regions [0, n_sig) and [n_sig, n)), and each
// advance appends the rows entering the next layer's children into the
// parent's region (left child from the region start, right child from its
// end; the region of parent p and class k starts at the class-major prefix
// of the parents' active counts).  A layer's histogram therefore reads only
// the rows of the nodes it builds (with sibling subtraction: the left
// children, ~half the active rows), each once, in one launch for every node.
//
// Row codes.  Codes are gathered from a row-major copy (NW u32 words per
// row, NW = 8 for d <= 32, 16 for d <= 64; zero-padded) with cp.async into a
// per-warp double buffer.
//
// Lane owns a row.  Lane l adds its own row's weight at every feature: at
// step (w, b) it takes byte c of word g of its row (NW = 16: g = (w + l/2)
// mod 16, c = (b + 2 (l&1)) mod 4; NW = 8: g = (w + l/4) mod 8, c = (b + l)
// mod 4).  The 32 lanes then touch 32 distinct features, and the slot word of
// feature 4g + c inside a bin row (NW = 16: 32 (c&1) + 16 (c>>1) + g; NW = 8:
// 4g + c) puts them in 32 distinct banks: every warp-wide atomic is one
// shared-memory wavefront for any codes, with no lane-private copies.  The
// row reads (word g of row l, row pitch NW words) are conflict-free as well
// (checked exhaustively for both NW).  The per-row weight stays in the
// lane's registers (no broadcast meta loads).
//
// Limbs as in the feature-lane kernel: q is added as lo16 = q & 0xffff and
// hi = q >> 16 (signed) with non-returning 32-bit atomics; a slot is exact
// while it takes < 2^15 adds, so a CTA flushes at least every kLhFlushRows
// rows.  Flush: int64 rows [feature][bin] staged in the drained buffers and
// added to the global layer histogram by TMA bulk reductions.
#pragma once
#include "common.cuh"
#include "kernels_tree.cuh"

namespace bb {

constexpr int kLhWarps = 16;
constexpr int kLhThreads = 32 * kLhWarps;
constexpr int kLhFlushRows = 32767;
constexpr int kLhMaxSegs = 512;
#ifndef BB_LH_PF
#define BB_LH_PF 4
#endif
constexpr int kLhPf = BB_LH_PF;  // slices of row codes in flight per warp (registers)

// byte offset of the (lo) slot of feature f in a bin row
template <int NW>
__host__ __device__ __forceinline__ int lh_slot_word(int f) {
  const int g = f >> 2, c = f & 3;
  return NW == 16 ? 32 * (c & 1) + 16 * ((c >> 1) & 1) + g : 4 * g + c;
}
// shared memory: NW = 16: lo limbs [256][64] words, then hi limbs (128 KB);
// NW = 8: bin rows of [32 lo | 32 hi] words (64 KB).  Then the warp buffers.
template <int NW>
__host__ __device__ constexpr int lh_hist_bytes() { return NW == 16 ? 2 * 256 * 64 * 4 : 256 * 64 * 4; }
template <int NW>
__host__ __device__ constexpr int lh_buf_bytes() {  // per-warp slice buffers; also the flush staging (rows of pitch 258 int64)
  return kLhWarps * 32 * NW * 4 > (NW == 16 ? 32 : 16) * 258 * 8 ? kLhWarps * 32 * NW * 4 : (NW == 16 ? 32 : 16) * 258 * 8;
}
template <int NW>
__host__ __device__ constexpr int lh_smem_bytes() { return lh_hist_bytes<NW>() + lh_buf_bytes<NW>() + 16 * kLhMaxSegs + 64; }

// Segments (list ranges) of the histogram launch of `layer`: every built
// node's (class, node) list.  cnt is heap-indexed [node][class].  Layer 1:
// the refresh's class regions [0, n_sig), [n_sig, n).  Layer >= 2: parent p
// (layer-1 node) and class k own the region at the class-major prefix of
// the parents' counts; the left child fills it from the start, the right
// child (built only without sibling subtraction) from the end.
// seg = {list offset, rows, layer-local node index, class}
// Sibling subtraction over the SMALLER child: of the children (c, c + 1) of a
// split node the histogram launch builds the one with fewer active rows
// (right only if strictly fewer; counts are heap-indexed [node][class]).
// Integer sums are exact, so parent - built is the sibling bit for bit.
__device__ __forceinline__ bool lh_build_right(const int* __restrict__ cnt, int left_child) {
  const int l = __ldcg(cnt + 2 * left_child) + __ldcg(cnt + 2 * left_child + 1);
  const int r = __ldcg(cnt + 2 * left_child + 2) + __ldcg(cnt + 2 * left_child + 3);
  return r < l;
}

__device__ __forceinline__ int lh_segments(const int* __restrict__ cnt, int layer, int sib, long long n_sig,
                                           int4* segs) {
  int ns = 0;
  if (layer == 1) {
    segs[ns++] = make_int4(0, __ldcg(cnt + 0), 0, 0);
    segs[ns++] = make_int4((int)n_sig, __ldcg(cnt + 1), 0, 1);
    return ns;
  }
  const int ps = (1 << (layer - 2)) - 1, np = 1 << (layer - 2), st = (1 << (layer - 1)) - 1;
  int off = 0;
  for (int k = 0; k < 2; ++k) {
    for (int p = ps; p < ps + np; ++p) {
      const int cp = __ldcg(cnt + 2 * p + k);
      const int c = 2 * p + 1;
      const int cr = __ldcg(cnt + 2 * (c + 1) + k);
      // sib == 2: the child with fewer active rows (both classes) is built, its
      // sibling is parent - built in k_split (same rule there: lh_build_right)
      const bool build_right = sib == 2 && lh_build_right(cnt, c);
      if (!build_right) segs[ns++] = make_int4(off, __ldcg(cnt + 2 * c + k), c - st, k);
      if (!sib || build_right) segs[ns++] = make_int4(off + cp - cr, cr, c + 1 - st, k);
      off += cp;
    }
  }
  return ns;
}

// CTA -> (segment, row range).  The G CTAs of a launch are split over the
// non-empty segments so that the LARGEST per-CTA row count is minimal: k_s =
// ceil(rows_s / T) CTAs for the smallest T with sum_s k_s <= G (binary search;
// needs G >= the number of non-empty segments, which the host guarantees).
// The first version gave 1 + floor((G - E) rows_s / R) CTAs: up to one CTA per
// segment stayed idle and mid-sized segments ran up to ~30 % over the mean.
// Called by all 32 lanes of warp 0; out = {segment or -1, r0, r1}.
__device__ __forceinline__ void lh_assign(const int4* __restrict__ segs, int ns, int G, int cta, int lane, int* out) {
  constexpr int Q = kLhMaxSegs / 32;
  const unsigned FULL = 0xffffffffu;
  int rows[Q];
  int mx = 0, ne = 0;
  long long tot = 0;
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int s = lane + 32 * q;
    rows[q] = s < ns ? segs[s].y : 0;
    mx = max(mx, rows[q]);
    tot += rows[q];
    ne += rows[q] > 0;
  }
  for (int o = 16; o > 0; o >>= 1) {
    mx = max(mx, __shfl_xor_sync(FULL, mx, o));
    tot += __shfl_xor_sync(FULL, tot, o);
    ne += __shfl_xor_sync(FULL, ne, o);
  }
  if (lane == 0) out[0] = -1;
  if (ne == 0) return;
  const int nq = (ns + 31) >> 5;
  int lo = (int)max(1ll, (tot + G - 1) / G), hi = mx;
  while (lo < hi) {
    const int mid = (int)(((long long)lo + hi) >> 1);
    int c = 0;
    for (int q = 0; q < nq; ++q) c += (rows[q] + mid - 1) / mid;
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(FULL, c, o);
    if (c <= G) hi = mid; else lo = mid + 1;
  }
  const int T = lo;
  int base = 0;
  for (int q = 0; q < nq; ++q) {
    const int k = (rows[q] + T - 1) / T;
    int incl = k;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += y;
    }
    const int first = base + incl - k;
    if (k > 0 && cta >= first && cta < first + k) {
      const int j = cta - first;
      out[0] = lane + 32 * q;
      out[1] = (int)((long long)rows[q] * j / k);
      out[2] = (int)((long long)rows[q] * (j + 1) / k);
    }
    base += __shfl_sync(FULL, incl, 31);
  }
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int NW>
__global__ void __launch_bounds__(kLhThreads, NW == 8 ? 2 : 1)
    k_hist_list(const uint32_t* __restrict__ rc, const int* __restrict__ lrow, const long long* __restrict__ lq,
                const int* __restrict__ cnt, int layer, int sib, long long n_sig, int d, int B, int code_off,
                int nodes, unsigned long long* __restrict__ hist, int pitch, int ngroups) {
  // pitch: row words of rc; ngroups > 1 (NW = 8 over 16-word rows): CTA
  // b takes feature group b % ngroups (features 32 g ..) of the rows it
  // gathers, so two 64 KB-histogram CTAs fit per SM and twice the warps
  // keep gathers in flight (same bytes: each group reads its 32-byte half)
  const int fgrp = (int)blockIdx.x % ngroups, cta = (int)blockIdx.x / ngroups, nctas = (int)gridDim.x / ngroups;
  const int fbase = 32 * fgrp * (NW == 8 ? 1 : 0);
  const uint32_t* rcg = rc + (NW == 8 ? 8 * fgrp : 0);
  const int dtot = d;
  d = min(d - fbase, NW * 4);  // features of this group
  extern __shared__ __align__(16) unsigned char lh_sm[];
  unsigned char* hb = lh_sm;                                             // histogram limbs
  uint32_t* bufs = reinterpret_cast<uint32_t*>(lh_sm + lh_hist_bytes<NW>());  // [warp][2][32 rows][NW]
  int4* segs = reinterpret_cast<int4*>(lh_sm + lh_hist_bytes<NW>() + lh_buf_bytes<NW>());
  __shared__ int s_ns;
  __shared__ int s_asg[3];  // segment, first row, end row of this CTA
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // zero the histogram limbs (before the dependency wait: overlaps the
  // previous kernel's tail under programmatic dependent launch)
  for (int i = threadIdx.x; i < lh_hist_bytes<NW>() / 16; i += kLhThreads)
    reinterpret_cast<uint4*>(hb)[i] = make_uint4(0u, 0u, 0u, 0u);
  pdl_wait();
  pdl_launch();
  if (threadIdx.x == 0) s_ns = lh_segments(cnt, layer, sib, n_sig, segs);
  __syncthreads();
  if (warp == 0) lh_assign(segs, s_ns, nctas, cta, lane, s_asg);
  __syncthreads();
  if (s_asg[0] < 0) return;
  const int4 sg = segs[s_asg[0]];
  BB_DCHECK(sg.x >= 0 && sg.y >= 0 && sg.z >= 0 && sg.z < nodes && (sg.w == 0 || sg.w == 1));
  const int r_begin = s_asg[1], r_end = s_asg[2];
  const int* lr = lrow + sg.x;
  const long long* lqs = lq + sg.x;
  uint32_t* wbuf = bufs + warp * 32 * NW;
  constexpr int CPR = NW / 4;  // 16-byte chunks per row

  // per-lane constants of the rotated schedule
  const uint32_t sel = NW == 16 ? ((lane & 1) ? 0x1032u : 0x3210u)
                                : ((lane & 3) == 0 ? 0x3210u : (lane & 3) == 1 ? 0x0321u : (lane & 3) == 2 ? 0x1032u : 0x2103u);
  const int gsh = NW == 16 ? (lane >> 1) : (lane >> 2);
  uint32_t cb[4];
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    if (NW == 16) {
      const int c = (b + 2 * (lane & 1)) & 3;
      cb[b] = 4u * (uint32_t)(32 * (c & 1) + 16 * ((c >> 1) & 1));
    } else {
      const int c = (b + lane) & 3;
      cb[b] = 4u * (uint32_t)c;
    }
  }

  for (int p0 = r_begin; p0 < r_end; p0 += kLhFlushRows) {
    const int p1 = min(r_end, p0 + kLhFlushRows);
    const int nsl = (p1 - p0 + 31) >> 5;  // 32-row slices of the piece; warp w takes w, w + 16, ...
    // Pipeline per warp: the row codes of the next two slices are in flight
    // in registers (4 lanes per row, 16-byte coalesced loads) while the
    // current slice, stored to the warp's shared buffer, is accumulated.
    uint32_t* sbuf = wbuf;  // [32 rows][NW]
    auto entry = [&](int j, int& row, long long& qq) {  // the lane's own list entry of slice j
      const int sl = warp + kLhWarps * j;
      const int e = p0 + 32 * sl + lane;
      row = -1;
      qq = 0;
      if (sl < nsl && e < p1) {
        row = __ldg(lr + e);
        qq = __ldg(lqs + e);
        BB_DCHECK(row >= 0);
      }
    };
    auto fetch = [&](int row_of_lane, uint4 (&x)[CPR]) {  // lane loads chunk (lane % CPR) of rows lane / CPR + (32 / CPR) t
#pragma unroll
      for (int t = 0; t < CPR; ++t) {
        const int rr = lane / CPR + (32 / CPR) * t;
        const int srow = __shfl_sync(0xffffffffu, row_of_lane, rr);
        x[t] = srow >= 0 ? __ldg(reinterpret_cast<const uint4*>(rcg + (size_t)srow * pitch) + (lane % CPR))
                         : make_uint4(0u, 0u, 0u, 0u);
      }
    };
    auto store = [&](const uint4 (&x)[CPR]) {
#pragma unroll
      for (int t = 0; t < CPR; ++t) {
        const int rr = lane / CPR + (32 / CPR) * t;
        reinterpret_cast<uint4*>(sbuf + rr * NW)[lane % CPR] = x[t];
      }
    };
    auto accumulate = [&](long long qq) {
      const uint32_t qlo = (uint32_t)((unsigned long long)qq & 0xffffull);
      const uint32_t qhi = (uint32_t)(int)(qq >> 16);
      const uint32_t* rowp = sbuf + lane * NW;
      // rows past the piece end carry q = 0 (zero codes): branch-free
#pragma unroll 4
      for (int w = 0; w < NW; ++w) {
        const int g = (w + gsh) & (NW - 1);
        const uint32_t word = __byte_perm(rowp[g], 0u, sel);
        const uint32_t g4 = (uint32_t)(NW == 16 ? 4 * g : 16 * g);
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const uint32_t off = __byte_perm(word, g4 + cb[b], 0x5504u | ((uint32_t)b << 4));
          BB_DCHECK(off + (NW == 16 ? 65536u : 128u) + 4u <= (uint32_t)lh_hist_bytes<NW>());
          atomicAdd(reinterpret_cast<uint32_t*>(hb + off), qlo);
          atomicAdd(reinterpret_cast<uint32_t*>(hb + off + (NW == 16 ? 65536u : 128u)), qhi);
        }
      }
    };
    const int nj = nsl > warp ? (nsl - warp + kLhWarps - 1) / kLhWarps : 0;  // this warp's slices
    // kLhPf slices in flight in registers (register-file capacity, not shared
    // memory, bounds the bytes in flight: 16 warps x kLhPf x 32 rows x NW words)
    // row ids (and q) are loaded one round before the gathers that need them
    constexpr int PF = NW == 8 ? 3 : kLhPf;  // NW = 8 runs 2 CTAs / SM: 64 registers
    long long qv[PF], qn[PF];
    int rn[PF];
    uint4 xv[PF][CPR];
#pragma unroll
    for (int u = 0; u < PF; ++u) {
      int r0;
      entry(u, r0, qv[u]);
      fetch(r0, xv[u]);
      entry(u + PF, rn[u], qn[u]);
    }
    for (int j = 0; j < nj; j += PF) {
#pragma unroll
      for (int u = 0; u < PF; ++u) {
        if (j + u < nj) {
          store(xv[u]);
          __syncwarp();
          fetch(rn[u], xv[u]);  // slice j + u + PF (ids from the previous round)
          const long long qq = qv[u];
          qv[u] = qn[u];
          entry(j + u + 2 * PF, rn[u], qn[u]);
          accumulate(qq);
          __syncwarp();
        }
      }
    }
    __syncthreads();
    // ---- flush: lanes take 32 features whose slots sit in distinct banks (a
    // bin's slot row read is one wavefront; reading one feature's bins would
    // hit one bank 32 times), warps take bins; int64 rows [feature][bin]
    // (pitch B + 2) are staged in the drained buffers and added to the global
    // layer histogram with one bulk reduction per row
    const uint32_t* lo = reinterpret_cast<const uint32_t*>(hb);
    long long* stg = reinterpret_cast<long long*>(bufs);
    const int spitch = B + 2;
    // NW = 16: 2 rounds of 32 feature rows, warps take bins; NW = 8 (2 CTAs
    // per SM, half the staging): 2 rounds of 16 rows, half-warps take bins
    constexpr int RPR = NW == 16 ? 32 : 16;  // staged rows per round
#pragma unroll 1
    for (int round = 0; round < 2; ++round) {
      const int f = NW == 16 ? 4 * (lane & 15) + 2 * (lane >> 4) + round : (lane & 15) + 16 * round;
      const int srow = NW == 16 ? lane : (lane & 15);
      if (f < d) {
        const int wa = lh_slot_word<NW>(f);
        const int b0 = NW == 16 ? warp : 2 * warp + (lane >> 4), bstep = NW == 16 ? kLhWarps : 2 * kLhWarps;
        for (int bin = b0; bin < B; bin += bstep) {
          const int v = bin + 1 - code_off;  // stored code of this bin
          long long val = 0;
          if (v >= 0 && v < 256) {
            if (NW == 16) val = (long long)(int)lo[16384 + v * 64 + wa] * 65536ll + (long long)lo[v * 64 + wa];
            else val = (long long)(int)lo[v * 64 + 32 + wa] * 65536ll + (long long)lo[v * 64 + wa];
          }
          stg[(size_t)srow * spitch + bin] = val;
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (threadIdx.x < RPR) {
        const int ff = NW == 16 ? 4 * (threadIdx.x & 15) + 2 * (threadIdx.x >> 4) + round : threadIdx.x + 16 * round;
        if (ff < d)
          bulk_reduce_add_u64(hist + (((size_t)sg.w * nodes + sg.z) * dtot + fbase + ff) * B,
                              stg + (size_t)threadIdx.x * spitch, (unsigned)B * 8u);
      }
      // the staging rows may be rewritten once the reductions have READ them;
      // only the last round waits for the reductions themselves
      if (round == 0) asm volatile("cp.async.bulk.commit_group;\ncp.async.bulk.wait_group.read 0;" ::: "memory");
      else asm volatile("cp.async.bulk.commit_group;\ncp.async.bulk.wait_group 0;" ::: "memory");
      __syncthreads();
    }
    if (p1 < r_end) {
      for (int i = threadIdx.x; i < lh_hist_bytes<NW>() / 16; i += kLhThreads)
        reinterpret_cast<uint4*>(hb)[i] = make_uint4(0u, 0u, 0u, 0u);
      __syncthreads();
    }
  }
}

// Advance over the row lists (row-list fits; replaces the all-rows k_advance):
// every listed active row of the layer moves to its child (code of the
// node's cut feature > cut bin -> right; trees.py:207-228).  CTAs take
// contiguous pieces of the (node, class) segments, so a CTA's rows share one
// node: its cut is uniform, children are two keys.  Both children are listed
// for the next layer in the node's region (left from its start, right from
// its end; ranks in list order within a tile, one global atomic per tile and
// child).  A row that parks (invalid cut, missing code) leaves the lists and
// adds its (eff, resp) fixed-point sums to its node; on the last layer every
// row adds them to its leaf (trees.py:231-244).  Per-row node ids are not
// kept: the next tree's refresh walks this tree for every row.
template <typename CodeT>
__global__ void __launch_bounds__(kListThreads) k_advance_list(
    const CodeT* __restrict__ codes, int d, int code_off, const int* __restrict__ lrow_in,
    const long long* __restrict__ lq_in, int* __restrict__ cnt, int* __restrict__ lrow_out,
    long long* __restrict__ lq_out, int layer, int tree, int n_internal, TreeArrays ta, int last_layer,
    long long n_sig, unsigned long long* __restrict__ sums, int n_nodes, const long long* __restrict__ q_resp) {
  constexpr int R = kListTileRows / kListThreads;
  constexpr int NWARP = kListThreads / 32;
  __shared__ int4 segs[kLhMaxSegs];
  __shared__ int s_ns, s_asg[3];
  __shared__ int s_reg[2 * kAdvMaxNodes];
  __shared__ int s_wc[2 * R * NWARP];  // per (child side, row group, warp): count, then rank base
  __shared__ int s_base[2];
  __shared__ unsigned long long s_sum[3][2];  // (node, left, right) x (eff, resp), two's complement sums
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int start = (1 << (layer - 1)) - 1, nodes = start + 1;
  pdl_wait();
  pdl_launch();
  if (threadIdx.x == 0) {
    s_ns = lh_segments(cnt, layer, 0, n_sig, segs);
    if (!last_layer) {  // regions of the next layer's lists: class-major prefix of this layer's counts
      int off = 0;
      for (int k = 0; k < 2; ++k)
        for (int p = 0; p < nodes; ++p) {
          s_reg[k * nodes + p] = off;
          off += __ldcg(cnt + 2 * (start + p) + k);
        }
    }
  }
  if (threadIdx.x < 6) s_sum[threadIdx.x >> 1][threadIdx.x & 1] = 0ull;
  __syncthreads();
  if (warp == 0) lh_assign(segs, s_ns, (int)gridDim.x, (int)blockIdx.x, lane, s_asg);
  __syncthreads();
  if (s_asg[0] < 0) return;
  const int s_r0 = s_asg[1], s_r1 = s_asg[2];
  const int4 sg = segs[s_asg[0]];
  const int c = start + sg.z, cls = sg.w;
  const int64_t e_tc = (int64_t)tree * n_internal + c;
  const bool vld = ta.valid[e_tc] != 0;
  const int f = vld ? ta.feature[e_tc] : 0;
  const int cut = vld ? ta.cut[e_tc] : 0;
  const int* lr = lrow_in + sg.x;
  const long long* lqs = lq_in + sg.x;
  const int cnt_c = __ldcg(cnt + 2 * c + cls);
  const int reg = last_layer ? 0 : s_reg[cls * nodes + sg.z];
  long long acc_e[3] = {0, 0, 0}, acc_r[3] = {0, 0, 0};  // per thread: (node, left, right)
  for (int t0 = s_r0; t0 < s_r1; t0 += kListTileRows) {
    int rowv[R], side[R];  // side: 0 left, 1 right, 2 parked, -1 none
    long long qv[R];
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const int e = t0 + k * kListThreads + threadIdx.x;
      rowv[k] = e < s_r1 ? __ldg(lr + e) : -1;
      qv[k] = e < s_r1 ? __ldg(lqs + e) : 0;
    }
    int cv[R];
#pragma unroll
    for (int k = 0; k < R; ++k)
      cv[k] = (rowv[k] >= 0 && vld) ? (int)codes[code_index(rowv[k], f, d)] + code_off : 0;
#pragma unroll
    for (int k = 0; k < R; ++k) {
      side[k] = rowv[k] < 0 ? -1 : (cv[k] == 0 ? 2 : (cv[k] > cut ? 1 : 0));
      if (side[k] == 2 || (last_layer && side[k] >= 0)) {
        // fixed-point (eff, resp) of the row at its final node (k_advance's last-layer rule)
        const long long qr = __ldg(q_resp + rowv[k]);  // rint(w r 2^S), written by the refresh
        const int slot = side[k] == 2 ? 0 : 1 + side[k];
        acc_e[slot] += qv[k];
        acc_r[slot] += qr;
      }
    }
    if (!last_layer) {
#pragma unroll
      for (int k = 0; k < R; ++k)
#pragma unroll
        for (int sd = 0; sd < 2; ++sd) {
          const unsigned m = __ballot_sync(0xffffffffu, side[k] == sd);
          if (lane == 0) s_wc[(sd * R + k) * NWARP + warp] = __popc(m);
          if (side[k] == sd) rowv[k] = (rowv[k] & 0x7fffffff), side[k] = sd + 4 * __popc(m & ((1u << lane) - 1u));
        }
      __syncthreads();
      if (threadIdx.x < 64) {  // warp sd: exclusive scan of side sd's (row group, warp) counts
        const int sd = threadIdx.x >> 5;
        const int run = warp_excl_scan_64(s_wc + sd * R * NWARP, lane);
        if (lane == 0) s_base[sd] = run ? atomicAdd(cnt + 2 * (2 * c + 1 + sd) + cls, run) : 0;
      }
      __syncthreads();
#pragma unroll
      for (int k = 0; k < R; ++k) {
        if (rowv[k] < 0 || (side[k] & 3) > 1) continue;
        const int sd = side[k] & 3;
        const int old = s_base[sd] + s_wc[(sd * R + k) * NWARP + warp] + (side[k] >> 2);
        const int pos = sd == 0 ? reg + old : reg + cnt_c - 1 - old;
        BB_DCHECK(old < cnt_c && pos >= 0);
        lrow_out[pos] = rowv[k];
        lq_out[pos] = qv[k];
      }
      __syncthreads();
    }
  }
  // node sums of this CTA's rows: (parked at c, left child, right child)
#pragma unroll
  for (int s3 = 0; s3 < 3; ++s3) {
    long long e = acc_e[s3], r = acc_r[s3];
    for (int o = 16; o > 0; o >>= 1) {
      e += __shfl_xor_sync(0xffffffffu, e, o);
      r += __shfl_xor_sync(0xffffffffu, r, o);
    }
    if (lane == 0 && (e != 0 || r != 0)) {
      atomicAdd(&s_sum[s3][0], as_ull(e));
      atomicAdd(&s_sum[s3][1], as_ull(r));
    }
  }
  __syncthreads();
  if (threadIdx.x < 6) {
    const int s3 = threadIdx.x >> 1, kind = threadIdx.x & 1;
    const unsigned long long v = s_sum[s3][kind];
    const int nd = s3 == 0 ? c : 2 * c + s3;
    if (v != 0ull && nd < n_nodes) atomicAdd(&sums[((int64_t)cls * n_nodes + nd) * 2 + kind], v);
  }
}

// Row-major copy of the tiled column-major codes (u8): rc[row][NW words],
// bytes of features >= d zero.  One CTA per 1024-row tile.
template <int NW>
__global__ void __launch_bounds__(256) k_rowcodes(const uint8_t* __restrict__ codes, int64_t n, int d,
                                                  uint32_t* __restrict__ rc) {
  extern __shared__ __align__(16) unsigned char rk_sm[];
  const int64_t tile = blockIdx.x;
  const uint8_t* src = codes + tile * (int64_t)d * kTile;
  const int bytes = d * kTile;
  for (int i = threadIdx.x; i < bytes / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(rk_sm)[i] = __ldg(reinterpret_cast<const uint4*>(src) + i);
  __syncthreads();
  for (int r = threadIdx.x; r < kTile; r += blockDim.x) {
    const int64_t row = tile * kTile + r;
    if (row >= n) break;
    uint32_t wv[NW];
#pragma unroll
    for (int j = 0; j < NW; ++j) {
      uint32_t x = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int f = 4 * j + b;
        if (f < d) x |= (uint32_t)rk_sm[f * kTile + r] << (8 * b);
      }
      wv[j] = x;
    }
    uint4* dst = reinterpret_cast<uint4*>(rc + row * NW);
#pragma unroll
    for (int j = 0; j < NW / 4; ++j) dst[j] = make_uint4(wv[4 * j], wv[4 * j + 1], wv[4 * j + 2], wv[4 * j + 3]);
  }
}

// ------------------------------------------------ u16 codes (B <= 1024)
// The same row-list histogram for 2-byte codes (more than 256 bins, or 256
// bins with missing values): features in GROUPS of 16.  A CTA takes one
// (segment, feature group) item (or a row range of one), keeps the group's
// limbs [bin][16 features][lo, hi] (1024 x 32 words = 128 KB) in shared memory
// and reads 32 bytes per listed row: the group's codes from a row-major copy
// (rc16, row pitch 32 B x groups).  Lane owns a row.  Step (a, b), a < 8,
// b < 4: lane l takes word w = (l/4 + a) mod 8 of its row (features 2w, 2w+1)
// and (half h, limb) = ((l mod 4) + b) mod 4: the 32 lanes cover every (w, h,
// limb) once, so the row reads (bank 8 (l mod 4) + w, row pitch 8 words) and
// the atomics (bank 4w + 2h + limb, 32 words per bin) are conflict-free for any
// codes.  rc16 holds SLOTS: code - 1, and kL16Bins (a dummy bin row that is
// never flushed) for a missing value (code 0: its slot is never read,
// trees.py:181-186) and for the padding features of the last group, so the
// accumulation is branch-free.
constexpr int kL16Feat = 16;
constexpr int kL16Bins = 1024;
constexpr int kL16HistBytes = (kL16Bins + 1) * 2 * kL16Feat * 4;                // 128 KB + the dummy bin row
constexpr uint32_t kL16Dummy2 = (uint32_t)kL16Bins * 0x00010001u;               // two dummy slots
constexpr int kL16ChunkBins = 256;                                              // bins per flush round
constexpr int kL16StagePitch = kL16ChunkBins + 2;                               // int64 per staged feature row
constexpr int kL16BufBytes = kL16Feat * kL16StagePitch * 8 > kLhWarps * 32 * 8 * 4 ? kL16Feat * kL16StagePitch * 8
                                                                                 : kLhWarps * 32 * 8 * 4;
constexpr int kL16SmemBytes = kL16HistBytes + kL16BufBytes + 16 * kLhMaxSegs + 64;

__device__ __forceinline__ void red_shared_add_u32(uint32_t saddr, uint32_t v) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(saddr), "r"(v) : "memory");
}

__global__ void __launch_bounds__(kLhThreads, 1)
    k_hist_list16(const uint4* __restrict__ rc16, int pitch16, const int* __restrict__ lrow,
                  const long long* __restrict__ lq, const int* __restrict__ cnt, int layer, int sib, long long n_sig,
                  int d, int B, int nodes, unsigned long long* __restrict__ hist, int ngroups) {
  // rc16: row-major codes, pitch16 uint4 (16 bytes) per row = 2 per feature group
  extern __shared__ __align__(16) unsigned char lh_sm[];
  unsigned char* hb = lh_sm;
  uint32_t* bufs = reinterpret_cast<uint32_t*>(lh_sm + kL16HistBytes);  // [warp][32 rows][8 words]
  int4* segs = reinterpret_cast<int4*>(lh_sm + kL16HistBytes + kL16BufBytes);
  __shared__ int s_ns;
  __shared__ int s_asg[3];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < kL16HistBytes / 16; i += kLhThreads)
    reinterpret_cast<uint4*>(hb)[i] = make_uint4(0u, 0u, 0u, 0u);
  pdl_wait();
  pdl_launch();
  if (threadIdx.x == 0) {
    // items = (segment, group): expanded in place, the group in the node field's high half
    const int ns = lh_segments(cnt, layer, sib, n_sig, segs);
    for (int v = ns * ngroups - 1; v >= 0; --v) {
      const int4 sg = segs[v / ngroups];
      segs[v] = make_int4(sg.x, sg.y, sg.z | ((v % ngroups) << 16), sg.w);
    }
    s_ns = ns * ngroups;
  }
  __syncthreads();
  // One item (or a row range of one) per CTA while the items fit the grid;
  // otherwise (deep layers x many groups) the concatenated items' rows are cut
  // into gridDim.x equal contiguous parts and a CTA walks the items of its part
  // (one flush per item touched; rows, not items, are balanced).
  __shared__ long long s_part[2];  // partition mode: rows of the part still to do, -1 in item mode
  if (s_ns <= (int)gridDim.x) {
    if (warp == 0) lh_assign(segs, s_ns, (int)gridDim.x, (int)blockIdx.x, lane, s_asg);
    if (threadIdx.x == 0) s_part[0] = -1;
  } else if (threadIdx.x == 0) {
    long long tot = 0;
    for (int v = 0; v < s_ns; ++v) tot += segs[v].y;
    const long long lo = tot * (long long)blockIdx.x / gridDim.x, hi = tot * ((long long)blockIdx.x + 1) / gridDim.x;
    long long cum = 0;
    int v = 0;
    while (v < s_ns && cum + segs[v].y <= lo) cum += segs[v++].y;
    s_asg[0] = (hi > lo && v < s_ns) ? v : -1;
    s_asg[1] = (int)(lo - cum);
    s_asg[2] = v < s_ns ? (int)min((long long)segs[v].y, hi - cum) : 0;
    s_part[0] = hi - lo;
  }
  __syncthreads();
  if (s_asg[0] < 0) return;
  int item = s_asg[0], r_begin = s_asg[1], r_end = s_asg[2];
  long long part_left = s_part[0];
  const uint32_t hb_s = smem_u32(hb);
  const int w0 = lane >> 2;
  uint32_t cb[4], psel[4];
  bool hi_limb[4];
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const int hl = ((lane & 3) + b) & 3;
    const int h = hl & 1, limb = hl >> 1;
    cb[b] = (uint32_t)(8 * h + 4 * limb);
    psel[b] = h ? 0x4432u : 0x4410u;  // the half word into the low 16 bits
    hi_limb[b] = limb != 0;
  }
  uint32_t* wbuf = bufs + warp * 32 * 8;
  for (;;) {  // the items of this CTA (one in item mode)
  const int4 sg = segs[item];
  const int node = sg.z & 0xffff, grp = sg.z >> 16;
  BB_DCHECK(node < nodes && grp < ngroups);
  const int* lr = lrow + sg.x;
  const long long* lqs = lq + sg.x;
  const int fg = min(kL16Feat, d - kL16Feat * grp);  // features of this group
  for (int p0 = r_begin; p0 < r_end; p0 += kLhFlushRows) {
    const int p1 = min(r_end, p0 + kLhFlushRows);
    const int nsl = (p1 - p0 + 31) >> 5;
    const int nj = nsl > warp ? (nsl - warp + kLhWarps - 1) / kLhWarps : 0;
    constexpr int PF = 4;  // slices in flight per warp (2 x 16 bytes per lane each)
    auto entry = [&](int j, int& row, long long& qq) {
      const int sl = warp + kLhWarps * j;
      const int e = p0 + 32 * sl + lane;
      row = -1;
      qq = 0;
      if (sl < nsl && e < p1) {
        row = __ldg(lr + e);
        qq = __ldg(lqs + e);
      }
    };
    auto fetch = [&](int row, uint4& x0, uint4& x1) {  // the lane's own row: one 32-byte sector
      x0 = make_uint4(kL16Dummy2, kL16Dummy2, kL16Dummy2, kL16Dummy2);  // no row: q = 0 into the dummy bin row
      x1 = x0;
      if (row >= 0) {
        const uint4* src = rc16 + (size_t)row * pitch16 + 2 * grp;
        x0 = __ldg(src);
        x1 = __ldg(src + 1);
      }
    };
    long long qv[PF], qn[PF];
    int rn[PF];
    uint4 xa[PF], xb[PF];
#pragma unroll
    for (int u = 0; u < PF; ++u) {
      int r0;
      entry(u, r0, qv[u]);
      fetch(r0, xa[u], xb[u]);
      entry(u + PF, rn[u], qn[u]);
    }
    for (int j = 0; j < nj; j += PF) {
#pragma unroll
      for (int u = 0; u < PF; ++u) {
        if (j + u < nj) {
          uint4* rowp4 = reinterpret_cast<uint4*>(wbuf + lane * 8);
          rowp4[0] = xa[u];
          rowp4[1] = xb[u];
          __syncwarp();
          fetch(rn[u], xa[u], xb[u]);
          const long long qq = qv[u];
          qv[u] = qn[u];
          entry(j + u + 2 * PF, rn[u], qn[u]);
          const uint32_t qlo = (uint32_t)((unsigned long long)qq & 0xffffull);
          const uint32_t qhi = (uint32_t)(int)(qq >> 16);
          uint32_t val[4];
#pragma unroll
          for (int b = 0; b < 4; ++b) val[b] = hi_limb[b] ? qhi : qlo;
          const uint32_t* rowp = wbuf + lane * 8;
#pragma unroll
          for (int a = 0; a < 8; ++a) {
            const int w = (w0 + a) & 7;
            const uint32_t word = rowp[w];
            const uint32_t wpart = hb_s + 16u * (uint32_t)w;
#pragma unroll
            for (int b = 0; b < 4; ++b) {
              const uint32_t slot = __byte_perm(word, 0u, psel[b]);
              BB_DCHECK(slot <= (uint32_t)kL16Bins);
              red_shared_add_u32(slot * 128u + (wpart + cb[b]), val[b]);
            }
          }
          __syncwarp();
        }
      }
    }
    __syncthreads();
    // ---- flush in rounds of 256 bins: int64 rows [feature][bin] staged in
    // the drained buffers, one bulk reduction per feature row
    const uint32_t* hw = reinterpret_cast<const uint32_t*>(hb);
    long long* stg = reinterpret_cast<long long*>(bufs);
    for (int c0 = 0; c0 < B; c0 += kL16ChunkBins) {
      const int cn = min(kL16ChunkBins, B - c0);
      const int f = lane & 15;
      for (int bin = 2 * warp + (lane >> 4); bin < cn; bin += 2 * kLhWarps) {
        const uint2 v = *reinterpret_cast<const uint2*>(hw + (size_t)(c0 + bin) * 32 + 2 * f);
        stg[(size_t)f * kL16StagePitch + bin] = (long long)(int)v.y * 65536ll + (long long)v.x;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if ((int)threadIdx.x < fg)
        bulk_reduce_add_u64(hist + (((size_t)sg.w * nodes + node) * d + kL16Feat * grp + threadIdx.x) * B + c0,
                            stg + (size_t)threadIdx.x * kL16StagePitch, (unsigned)cn * 8u);
      if (c0 + kL16ChunkBins < B) asm volatile("cp.async.bulk.commit_group;\ncp.async.bulk.wait_group.read 0;" ::: "memory");
      else asm volatile("cp.async.bulk.commit_group;\ncp.async.bulk.wait_group 0;" ::: "memory");
      __syncthreads();
    }
    if (p1 < r_end) {
      for (int i = threadIdx.x; i < kL16HistBytes / 16; i += kLhThreads)
        reinterpret_cast<uint4*>(hb)[i] = make_uint4(0u, 0u, 0u, 0u);
      __syncthreads();
    }
  }
  // next item of the part (partition mode)
  if (part_left < 0) break;
  part_left -= r_end - r_begin;
  do ++item; while (item < s_ns && segs[item].y == 0);
  if (part_left <= 0 || item >= s_ns) break;
  r_begin = 0;
  r_end = (int)min((long long)segs[item].y, part_left);
  for (int i = threadIdx.x; i < kL16HistBytes / 16; i += kLhThreads)
    reinterpret_cast<uint4*>(hb)[i] = make_uint4(0u, 0u, 0u, 0u);
  __syncthreads();
  }
}

// Row-major copy of the tiled column-major u16 codes as histogram slots:
// rc16[row][16 * groups].  One CTA per (1024-row tile, feature group).
template <typename CodeT>  // u16 codes, or u8 codes of more than 64 features (stored code + code_off = code)
__global__ void __launch_bounds__(256) k_rowcodes16(const CodeT* __restrict__ codes, int64_t n, int d, int ngroups,
                                                    int code_off, uint16_t* __restrict__ rc16) {
  __shared__ __align__(16) CodeT col[kL16Feat][kTile];
  const int64_t tile = blockIdx.x;
  const int grp = blockIdx.y;
  const int f0 = kL16Feat * grp, fg = min(kL16Feat, d - f0);
  constexpr int kVec = kTile * (int)sizeof(CodeT) / 16;  // 16-byte vectors per column
  for (int i = threadIdx.x; i < fg * kVec; i += blockDim.x) {
    const int f = i / kVec, v = i % kVec;
    reinterpret_cast<uint4*>(&col[f][0])[v] =
        __ldg(reinterpret_cast<const uint4*>(codes + (tile * d + f0 + f) * (int64_t)kTile) + v);
  }
  __syncthreads();
  const int pitch = kL16Feat * ngroups;
  for (int r = threadIdx.x; r < kTile; r += blockDim.x) {
    const int64_t row = tile * kTile + r;
    if (row >= n) break;
    uint32_t wv[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      // slot = code - 1; missing values and padding features: the dummy bin row
      const uint32_t cl = 2 * j < fg ? (uint32_t)col[2 * j][r] + (uint32_t)code_off : 0u;
      const uint32_t ch = 2 * j + 1 < fg ? (uint32_t)col[2 * j + 1][r] + (uint32_t)code_off : 0u;
      const uint32_t lo = cl ? cl - 1u : (uint32_t)kL16Bins, hi = ch ? ch - 1u : (uint32_t)kL16Bins;
      wv[j] = lo | (hi << 16);
    }
    uint4* dst = reinterpret_cast<uint4*>(rc16 + row * pitch + f0);
    dst[0] = make_uint4(wv[0], wv[1], wv[2], wv[3]);
    dst[1] = make_uint4(wv[4], wv[5], wv[6], wv[7]);
  }
}

}  // namespace bb
