// Feature-lane layer histogram (trees.py:139-167): the bank-conflict-free
// variant of k_layer_hist, and the default histogram path.
//
// Lane layout.  A CTA type covers up to 64 features as one or two lane
// groups ("subs").  In a sub with R = 1, 2 or 4 row copies a warp handles
// R rows x 32/R features per step: lane (c = lane / FG, f = lane % FG) adds
// row (step*R + c)'s weight at feature f.  Shared-memory slots are laid out
// [node][sub][bin row][limb][lane], so the word a lane touches is always in
// bank `lane`: every warp-wide atomic is exactly one wavefront whatever the
// codes are (random, tied, all equal).  The R lanes of one feature are R
// private copies of its histogram, summed at the flush.
//
// Limbs.  A fixed-point weight q (|q| <= 2^32, oracle _fixed_scale) is added
// as two non-returning 32-bit atomics: lo16 = q & 0xffff into the lo limb and
// hi = q >> 16 (signed) into the hi limb.  Value = (int32)hi * 2^16 + lo, exact
// while a copy slot takes < 2^15 adds (flushes every kFlFlushStages stages).
// No returned values, no carries: the warps stream atomics without waiting.
//
// Rows.  Per stage (kFlRows rows of one class block) a producer warp issues
// a handful of TMA copies into a 2-3 deep ring (full/empty mbarriers): node
// ids and q as 1-D bulk copies, and the type's code columns as 2-D tensor
// boxes [features][128 bytes] with the 128-byte swizzle (few large copies:
// ~3x the throughput of per-column 512-byte bulk copies,
// profiles/r01_microbench_tma_small.txt).  The swizzle makes lane f's
// 16-byte load of its own column conflict-free.  Each of the 16 compute
// warps takes 32 rows: lane k derives row k's meta (lo16, hi, node offset)
// and the warp steps over the rows of every sub; 8-row groups without a
// contributing row are skipped, sparse groups branch per row.
//
// Flush.  The CTA's slots are combined (copies, limbs) into int64 rows
// [node][feature][bin] staged in the free ring, and each row goes to the
// global histogram with one TMA bulk reduction (cp.reduce.async.bulk .add.u64):
// scattered 64-bit global atomics cost ~1 LSU cycle per lane.
#pragma once
#include <cuda.h>

#include "common.cuh"

namespace bb {

constexpr int kFlRows = 512;          // rows per stage (half a code tile)
constexpr int kFlMaxStages = 3;       // ring depth (2 when the type's boxes are wide)
constexpr int kFlWarps = 16;          // compute warps (32 rows each per stage)
constexpr int kFlThreads = 32 * (kFlWarps + 1);
constexpr int kFlFlushStages = 63;    // copy slot adds per flush < 2^15 (at most 63 * 512 / R rows)
constexpr int kFlMaxTypes = 80;
constexpr int kFlMetaBytes = kFlWarps * 32 * 16;
#ifndef BB_FL_DENSE
#define BB_FL_DENSE 5
#endif
constexpr int kFlDenseRows = BB_FL_DENSE;  // contributing rows of 8 from which a group runs branch-free

struct FlType {
  int cta0, nctas;        // first block index, CTAs of this type
  int t0, t1;             // stage range (units of kFlRows rows) of the class block
  short cls, f0;          // class, first feature
  short fc0, r0log;       // sub 0: features, R = 1 << r0log
  short fc1, r1log;       // sub 1 (fc1 == 0: none): features f0+32 .., R = 1 << r1log
  short n0, ncount;       // built-node group
  short map, fpad;        // tensor map index, box height (fc0 + fc1 rounded up to 8)
};

struct FlPlan {
  CUtensorMap tm[2];      // codes as 2-D [tiles * d][kTile], boxes [fpad][128 bytes], 128B swizzle
  int start, nodes, sib;  // layer_start, nodes in layer, left children only
  int log2b;              // log2(B)
  int n_types;
  int smem;               // dynamic shared memory bytes (incl. 1024 alignment slack)
  int stages;             // ring depth
  int ngs;                // nodes per node group
  int stage_bytes;        // per ring slot (multiple of 1024)
  int hist_bytes;         // ncount_max * nsub_max * (B + 1) * 256
  FlType t[kFlMaxTypes];
  unsigned char cta_type[256];  // block index -> type index
  long long* partials;    // non-null: each CTA stores its rows here (k_fl_reduce sums them); null: bulk reductions into hist
  int64_t cta_stride;     // elements per CTA in partials
  int noflush;            // debug (BB_FL_NOFLUSH=1): skip the final flush (timing only)
};

// stage = [codes: fpad x kFlRows codes, swizzled boxes][q: kFlRows x 8][node]
template <typename CodeT, typename NodeT>
__host__ __device__ __forceinline__ int fl_stage_bytes(int fpad) {
  const int b = fpad * kFlRows * (int)sizeof(CodeT) + kFlRows * 8 + kFlRows * (int)sizeof(NodeT);
  return (b + 1023) & ~1023;
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* tm, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(ssrc)),
               "r"(bytes)
               : "memory");
}

// lane*4 + code*256: the lane's byte offset of the code's bin row (one PRMT;
// byte b of word w for u8, half h for u16)
template <typename CodeT>
__device__ __forceinline__ uint32_t fl_off(uint32_t w, int part, uint32_t lane4) {
  if (sizeof(CodeT) == 1) return __byte_perm(w, lane4, 0x5504u | ((uint32_t)part << 4));
  return __byte_perm(w, lane4, 0x5004u | ((uint32_t)(2 * part) << 4) | ((uint32_t)(2 * part + 1) << 8));
}

// byte offset for row s*R + c (c < R) from the lane's 32-row column registers;
// the register index is static for every R (no local-memory indexing)
template <typename CodeT, int R>
__device__ __forceinline__ uint32_t fl_code_off(const uint32_t (&cw)[8 * sizeof(CodeT)], int s, int c,
                                                uint32_t lane4) {
  if (sizeof(CodeT) == 1) return fl_off<CodeT>(cw[(s * R) >> 2], ((s * R) & 3) + c, lane4);
  if (R <= 2) return fl_off<CodeT>(cw[(s * R) >> 1], ((s * R) & 1) + c, lane4);
  return fl_off<CodeT>((c >> 1) ? cw[2 * s + 1] : cw[2 * s], c & 1, lane4);
}

// a lane's 32 codes (rows rb .. rb+31) of box line `col` (swizzled chunks)
template <typename CodeT>
__device__ __forceinline__ void fl_load_codes(uint32_t (&cw)[8 * sizeof(CodeT)], const unsigned char* line, int ch0,
                                              int col) {
#pragma unroll
  for (int v = 0; v < 2 * (int)sizeof(CodeT); ++v) {
    const uint4 x = *reinterpret_cast<const uint4*>(line + (((ch0 + v) ^ (col & 7)) << 4));
    cw[4 * v + 0] = x.x;
    cw[4 * v + 1] = x.y;
    cw[4 * v + 2] = x.z;
    cw[4 * v + 3] = x.w;
  }
}

template <bool MULTI>
__device__ __forceinline__ void fl_meta(const uint4* meta4, int k, uint32_t& ml, uint32_t& mh, uint32_t& mo) {
  if (MULTI) {
    const uint4 x = meta4[k];
    ml = x.x; mh = x.y; mo = x.z;
  } else {
    const uint2 x = reinterpret_cast<const uint2*>(meta4)[k];
    ml = x.x; mh = x.y; mo = 0u;
  }
}

// every step of one sub over the warp's 32 rows (ballot m of contributing rows)
template <typename CodeT, int R, bool MULTI>
__device__ __forceinline__ void fl_steps(const uint32_t (&cw)[8 * sizeof(CodeT)], unsigned m, const uint4* meta4,
                                         unsigned char* hb, uint32_t lane4, int c) {
  if (R == 1) {
#pragma unroll
    for (int g = 0; g < 4; ++g) {  // 8-row groups
      const unsigned mg = (m >> (8 * g)) & 0xffu;
      if (!mg) continue;
      uint32_t ml[8], mh[8], mo[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) fl_meta<MULTI>(meta4, 8 * g + j, ml[j], mh[j], mo[j]);
      if (__popc(mg) >= kFlDenseRows) {
        // dense group: every step; rows that do not contribute add zeros
        // (branch-free, so the 8 steps pipeline)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t off = fl_code_off<CodeT, 1>(cw, 8 * g + j, 0, lane4) + mo[j];
          atomicAdd(reinterpret_cast<uint32_t*>(hb + off), ml[j]);
          atomicAdd(reinterpret_cast<uint32_t*>(hb + off + 128), mh[j]);
        }
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (mg & (1u << j)) {
            const uint32_t off = fl_code_off<CodeT, 1>(cw, 8 * g + j, 0, lane4) + mo[j];
            atomicAdd(reinterpret_cast<uint32_t*>(hb + off), ml[j]);
            atomicAdd(reinterpret_cast<uint32_t*>(hb + off + 128), mh[j]);
          }
        }
      }
    }
  } else {
    // R rows per step (lane copy c takes row s*R + c); rows that do not
    // contribute add zeros, steps without any contributing row are skipped
#pragma unroll
    for (int s = 0; s < 32 / R; ++s) {
      if (!((m >> (s * R)) & ((1u << R) - 1u))) continue;
      uint32_t ml, mh, mo;
      fl_meta<MULTI>(meta4, s * R + c, ml, mh, mo);
      const uint32_t off = fl_code_off<CodeT, R>(cw, s, c, lane4) + mo;
      atomicAdd(reinterpret_cast<uint32_t*>(hb + off), ml);
      atomicAdd(reinterpret_cast<uint32_t*>(hb + off + 128), mh);
    }
  }
}

template <typename CodeT, typename NodeT, int R0LOG, int R1LOG, bool MULTI>
__device__ __forceinline__ void fl_run(int code_off, const NodeT* __restrict__ node, const long long* __restrict__ q,
                                       int64_t n_sig, int64_t n, int d, int B, const FlPlan& p, const FlType& ty,
                                       int part, unsigned long long* __restrict__ hist, unsigned char* smem) {
  constexpr int R0 = 1 << R0LOG, FG0 = 32 / R0;
  constexpr bool SUB1 = R1LOG >= 0;
  constexpr int R1 = SUB1 ? (1 << R1LOG) : 1, FG1 = 32 / R1;
  constexpr int NSUB = SUB1 ? 2 : 1;
  constexpr int BOX_ROWS = 128 / (int)sizeof(CodeT);  // rows per 128-byte box line
  constexpr int kBoxes = kFlRows / BOX_ROWS;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ncount = ty.ncount, fpad = ty.fpad, NS = p.stages;
  const int rowb = 256;                          // bytes per (bin row): 32 lo + 32 hi words
  const int subb = (B + 1) * rowb;               // bytes per (node, sub)
  const int nodeb = NSUB * subb;                 // bytes per node
  const int hist_words = ncount * nodeb / 4;
  unsigned char* stage = smem;                   // 1024-aligned (caller)
  uint4* meta_all = reinterpret_cast<uint4*>(smem + NS * p.stage_bytes);
  uint32_t* hw = reinterpret_cast<uint32_t*>(smem + NS * p.stage_bytes + kFlMetaBytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + NS * p.stage_bytes + kFlMetaBytes + p.hist_bytes);
  uint64_t* empty = full + kFlMaxStages;
  const int64_t clo = ty.cls ? n_sig : 0, chi = ty.cls ? n : n_sig;
  const int nt = ty.t1 - ty.t0;
  const int sa = ty.t0 + (int)((int64_t)nt * part / ty.nctas);
  const int sb = ty.t0 + (int)((int64_t)nt * (part + 1) / ty.nctas);
  const int s_lo = (int)(clo / kFlRows), s_hi = (int)(chi / kFlRows);  // stages that may straddle the class range
  const int cbytes = fpad * kFlRows * (int)sizeof(CodeT);  // codes region of a stage
  const int qoff = cbytes, noff = cbytes + kFlRows * 8;
  const int boxb = fpad * 128;                               // bytes per box

  for (int i = threadIdx.x; i < hist_words; i += kFlThreads) hw[i] = 0u;
  if (threadIdx.x == 0) {
    for (int b = 0; b < NS; ++b) {
      mbar_init(&full[b], 1);
      mbar_init(&empty[b], kFlWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();

  // value of slot (node nd, sub, bin, feature f of the sub): copies and limbs combined
  auto slot_value = [&](int nd, int sub, int bin, int f) -> long long {
    const int R = sub ? R1 : R0, FG = sub ? FG1 : FG0;
    const int base = (nd * nodeb + sub * subb) / 4 + (bin + 1) * 64 + f;
    long long v = 0;
    for (int c = 0; c < R; ++c) v += (long long)(int)hw[base + 32 + c * FG] * 65536ll + (long long)hw[base + c * FG];
    return v;
  };
  auto grow = [&](int nd, int sub, int f) -> unsigned long long* {  // global histogram row of (node, feature)
    const int ln = p.sib ? 2 * (ty.n0 + nd) : (ty.n0 + nd);
    return hist + (((int64_t)ty.cls * p.nodes + ln) * d + (ty.f0 + sub * 32 + f)) * B;
  };

  if (warp == kFlWarps) {
    // ---- producer: lane 0 arms the stage; lanes 0..kBoxes-1 each issue one
    // code box, the next two lanes issue q and node ids
    const CUtensorMap* tm = &p.tm[ty.map];
    int buf = 0;
    unsigned ph = 0;
    for (int k = sa; k < sb; ++k) {
      const int it = k - sa;
      if (lane == 0) {
        if (it >= NS) mbar_wait(&empty[buf], ph ^ 1u);
        mbar_expect_tx(&full[buf], (unsigned)(kBoxes * boxb + kFlRows * 8 + kFlRows * (int)sizeof(NodeT)));
      }
      __syncwarp();
      unsigned char* b = stage + buf * p.stage_bytes;
      const int64_t row0 = (int64_t)k * kFlRows;
      const int tile = (int)(row0 >> kTileLog);
      const int half = (int)(row0 & (kTile - 1));
      if (lane < kBoxes) tma_load_2d(b + lane * boxb, tm, half + lane * BOX_ROWS, tile * d + ty.f0, &full[buf]);
      else if (lane == kBoxes) tma_load_1d(b + qoff, q + row0, kFlRows * 8, &full[buf]);
      else if (lane == kBoxes + 1) tma_load_1d(b + noff, node + row0, kFlRows * sizeof(NodeT), &full[buf]);
      if (++buf == NS) { buf = 0; ph ^= 1u; }
    }
  } else {
    // ---- compute warps
    const int c0 = lane >> (5 - R0LOG), f0l = lane & (FG0 - 1);
    const int c1 = lane >> (5 - (SUB1 ? R1LOG : 0)), f1l = lane & (FG1 - 1);
    // idle lanes read line 0 and add into their own (never read) lane column
    const int col0 = f0l < ty.fc0 ? f0l : 0;
    const int col1 = f1l < ty.fc1 ? 32 + f1l : 0;
    const uint32_t lane4 = (uint32_t)lane * 4u;
    unsigned char* hb0 = reinterpret_cast<unsigned char*>(hw) + code_off * rowb;  // + node offset + lane*4 + code*256
    unsigned char* hb1 = hb0 + subb;
    uint4* meta4 = meta_all + warp * 32;
    const int rb = warp * 32;  // this warp's rows in the stage
    const int box = rb / BOX_ROWS;
    const int ch0 = ((rb % BOX_ROWS) * (int)sizeof(CodeT)) / 16;
    int buf = 0;
    unsigned ph = 0;
    for (int k = sa; k < sb; ++k) {
      const int it = k - sa;
      mbar_wait(&full[buf], ph);
      const unsigned char* b = stage + buf * p.stage_bytes;
      const NodeT* ntp = reinterpret_cast<const NodeT*>(b + noff);
      const long long* qtp = reinterpret_cast<const long long*>(b + qoff);
      // meta of row rb + lane: (lo16, hi) [, node byte offset]; zeros if the row does not contribute
      const int ln = (int)ntp[rb + lane] - p.start;
      const int nd = (ln >> p.sib) - ty.n0;
      const long long qq = qtp[rb + lane];
      bool ok = (unsigned)ln < (unsigned)p.nodes && !(p.sib & ln & 1) && (unsigned)nd < (unsigned)ncount && qq != 0;
      if (k == s_lo || k == s_hi) {  // a stage holding the class boundary
        const int64_t r = (int64_t)k * kFlRows + rb + lane;
        ok = ok && r >= clo && r < chi;
      }
      const uint32_t mlo = ok ? (uint32_t)((unsigned long long)qq & 0xffffull) : 0u;
      const uint32_t mhi = ok ? (uint32_t)(int)(qq >> 16) : 0u;
      if (MULTI) meta4[lane] = make_uint4(mlo, mhi, ok ? (unsigned)(nd * nodeb) : 0u, 0u);
      else reinterpret_cast<uint2*>(meta4)[lane] = make_uint2(mlo, mhi);
      const unsigned m = __ballot_sync(0xffffffffu, ok);
      const unsigned char* lines = b + box * boxb;
      uint32_t cw[8 * sizeof(CodeT)];
      fl_load_codes<CodeT>(cw, lines + col0 * 128, ch0, col0);
      __syncwarp();
      if (m) fl_steps<CodeT, R0, MULTI>(cw, m, meta4, hb0, lane4, c0);
      if (SUB1 && m) {
        fl_load_codes<CodeT>(cw, lines + col1 * 128, ch0, col1);
        fl_steps<CodeT, R1, MULTI>(cw, m, meta4, hb1, lane4, c1);
      }
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[buf])) : "memory");
      if (++buf == NS) { buf = 0; ph ^= 1u; }
      if ((it % kFlFlushStages) == kFlFlushStages - 1 && k + 1 < sb) {
        // mid-run flush (long row runs): 64-bit global reductions, then zero
        asm volatile("bar.sync 1, %0;" ::"n"(kFlWarps * 32) : "memory");
        for (int sub = 0; sub < NSUB; ++sub) {
          const int fc = sub ? ty.fc1 : ty.fc0, FG = sub ? FG1 : FG0;
          for (int s = threadIdx.x; s < ncount * B * FG; s += kFlWarps * 32) {
            const int f = s % FG, bin = (s / FG) & (B - 1), nd2 = (s / FG) >> p.log2b;
            if (f >= fc) continue;
            const long long v = slot_value(nd2, sub, bin, f);
            if (v != 0) atomicAdd(grow(nd2, sub, f) + bin, as_ull(v));
          }
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kFlWarps * 32) : "memory");
        for (int i = threadIdx.x; i < hist_words; i += kFlWarps * 32) hw[i] = 0u;
        asm volatile("bar.sync 1, %0;" ::"n"(kFlWarps * 32) : "memory");
      }
    }
  }
  __syncthreads();
  // ---- final flush: int64 rows [node][sub][feature][bin] staged in the ring +
  // meta area (pitch B+2 words), one bulk reduction per row
  if (p.noflush) return;
  const int pitch = B + 2;
  const int cap_rows = (NS * p.stage_bytes + kFlMetaBytes) / (pitch * 8);
  long long* st = reinterpret_cast<long long*>(smem);
  const int per_node = ty.fc0 + ty.fc1;
  const int rows = ncount * per_node;
  for (int r0 = 0; r0 < rows; r0 += cap_rows) {
    const int rn = min(cap_rows, rows - r0);
    // rows r0 .. r0+rn-1 in order (node, sub, feature): lanes take rows
    // (conflict-free slot reads), warps take bins
    for (int rl = lane; rl < rn; rl += 32) {
      const int r = r0 + rl;
      const int nd = r / per_node, fi = r - nd * per_node;
      const int sub = fi >= ty.fc0 ? 1 : 0, f = sub ? fi - ty.fc0 : fi;
      const int R = sub ? R1 : R0, FG = sub ? FG1 : FG0;
      const uint32_t* sl = hw + (nd * nodeb + sub * subb) / 4 + 64 + f;  // bin 0's slot row
      long long* dst = st + rl * pitch;
      for (int bin = warp; bin < B; bin += kFlWarps + 1) {
        const uint32_t* x = sl + bin * 64;
        long long v = (long long)(int)x[32] * 65536ll + (long long)x[0];
        for (int c = 1; c < R; ++c) v += (long long)(int)x[32 + c * FG] * 65536ll + (long long)x[c * FG];
        dst[bin] = v;
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    for (int rl = threadIdx.x; rl < rn; rl += kFlThreads) {
      const int r = r0 + rl;
      if (p.partials) {
        bulk_store(p.partials + (int64_t)blockIdx.x * p.cta_stride + (int64_t)r * B, st + rl * pitch, (unsigned)B * 8u);
      } else {
        const int nd = r / per_node, fi = r - nd * per_node;
        const int sub = fi >= ty.fc0 ? 1 : 0, f = sub ? fi - ty.fc0 : fi;
        bulk_reduce_add_u64(grow(nd, sub, f), st + rl * pitch, (unsigned)B * 8u);
      }
    }
    asm volatile("cp.async.bulk.commit_group;\ncp.async.bulk.wait_group 0;" ::: "memory");
    __syncthreads();
  }
}

template <typename CodeT, typename NodeT>
__global__ void __launch_bounds__(kFlThreads, 1)
    k_layer_hist_fl(int code_off, const NodeT* __restrict__ node, const long long* __restrict__ q, int64_t n,
                    int64_t n_sig, int d, int B, const __grid_constant__ FlPlan p,
                    unsigned long long* __restrict__ hist) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // 128B-swizzle boxes
  const FlType ty = p.t[p.cta_type[blockIdx.x]];  // one copy into registers
  const int part = (int)blockIdx.x - ty.cta0;
  const bool multi = p.ngs > 1;  // node groups of more than one node
#define BB_FL_RUN(A, C, MU) fl_run<CodeT, NodeT, A, C, MU>(code_off, node, q, n_sig, n, d, B, p, ty, part, hist, smem)
#define BB_FL_SUBS(MU)                            \
  if (ty.fc1 == 0) {                              \
    if (ty.r0log == 0) BB_FL_RUN(0, -1, MU);      \
    else if (ty.r0log == 1) BB_FL_RUN(1, -1, MU); \
    else BB_FL_RUN(2, -1, MU);                    \
  } else {                                        \
    if (ty.r1log == 0) BB_FL_RUN(0, 0, MU);       \
    else if (ty.r1log == 1) BB_FL_RUN(0, 1, MU);  \
    else BB_FL_RUN(0, 2, MU);                     \
  }
  if (multi) {
    BB_FL_SUBS(true)
  } else {
    BB_FL_SUBS(false)
  }
#undef BB_FL_SUBS
#undef BB_FL_RUN
}

// Sum of the CTAs' partial rows of each type into the layer histogram
// (adds to the built rows): grid (row within type, type), 1024 threads
// = bin pairs x CTA subsets (16-byte loads, many in flight), then a
// shared-memory sum over the subsets.
constexpr int kFlRedThreads = 1024;
__global__ void __launch_bounds__(kFlRedThreads) k_fl_reduce(int d, int B, const __grid_constant__ FlPlan p,
                                                             unsigned long long* __restrict__ hist) {
  __shared__ longlong2 red[kFlRedThreads];
  const FlType& ty = p.t[blockIdx.y];
  const int per_node = ty.fc0 + ty.fc1;
  const int r = blockIdx.x;
  if (r >= ty.ncount * per_node) return;
  const int nd = r / per_node, fi = r - nd * per_node;
  const int sub = fi >= ty.fc0 ? 1 : 0, f = sub ? fi - ty.fc0 : fi;
  const int ln = p.sib ? 2 * (ty.n0 + nd) : (ty.n0 + nd);
  unsigned long long* out = hist + (((int64_t)ty.cls * p.nodes + ln) * d + (ty.f0 + sub * 32 + f)) * B;
  const int pairs = B >> 1;  // B >= 2
  const int groups = kFlRedThreads / pairs > 0 ? kFlRedThreads / pairs : 1;
  const int bp = threadIdx.x % pairs, j = threadIdx.x / pairs;
  long long s0 = 0, s1 = 0;
  if (j < groups) {
    const longlong2* src = reinterpret_cast<const longlong2*>(p.partials + (int64_t)ty.cta0 * p.cta_stride +
                                                              (int64_t)r * B) + bp;
    const int64_t cs = p.cta_stride / 2;  // in pairs
    int c = j;
#pragma unroll 4
    for (; c < ty.nctas; c += groups) {
      const longlong2 v = __ldcg(src + (int64_t)c * cs);
      s0 += v.x;
      s1 += v.y;
    }
  }
  red[threadIdx.x] = make_longlong2(s0, s1);
  __syncthreads();
  if (threadIdx.x < pairs) {
    for (int g = 1; g < groups; ++g) {
      const longlong2 v = red[g * pairs + threadIdx.x];
      s0 += v.x;
      s1 += v.y;
    }
    out[2 * threadIdx.x] += as_ull(s0);  // + mid-run flushes (64-bit reductions) of long row runs
    out[2 * threadIdx.x + 1] += as_ull(s1);
  }
}

}  // namespace bb
