// Segment-parallel parse of the subsample draw stream (the Fisher-Yates
// step assignment of kernels_mask.cuh, reference sample.py:128-132 through
// numpy Generator.permutation; algorithm restated in bb_mask.cpp).
//
// A block job (one class block of one tree: steps i = n-1 .. 1, step i takes
// the first draw x = v & smear(i) with x <= i) consumes a data-dependent
// number of draws.  Its draw range is cut into segments at fixed offsets
// from the job's first draw (host table per block size).  For every segment
// the expected state at its first draw follows from the mean trajectory,
// (i+1)' = -(i+1)/(mask+1) per band, and the true state lies in a window
// [lo, hi] around it (the accept count is a sum of Bernoullis, sd <=
// sqrt(p)/2 after p draws; the window is 9 sd on each side).
//
//  phase 1 (k_seg_pass, func part; a warp per 512-state sub-window, a CTA
//    per 16 sub-windows of one segment, all SMs): the segment's transfer
//    function over the sub-window, inside one mask band.  Paths that start
//    at adjacent states stay ordered and at most one step apart, so the
//    sub-window is an interval [a, b] of distinct states: a draw x <= a
//    moves every path (a--, b--), x > b none, a < x <= b moves the paths at
//    states >= x and merges the groups at offsets x-a and x-a-1 (b--).  A
//    rank bitmask records which start ranks merged:
//        end(lo + r) = a_end + r - #{cleared ranks <= r},
//    valid for ranks that never fall to the band's last state h (end > h).
//  phase 2 (k_seg_compose, one CTA): warp 0 chains the functions from the
//    job's exact first state, one lookup per segment (records streamed into
//    shared memory with cp.async).  A start the records cannot answer (a
//    band crossing inside the segment, a window miss) is walked exactly by
//    the whole CTA (cta_walk); below kSegTail the CTA walks the job to its
//    end, which gives the next job's first draw.
//  phase 3 (k_seg_pass, emit part; a CTA per segment): each segment walked
//    exactly from its start state, writing J[i] = x for steps i >= k.
//
// cta_walk: 4096-draw windows, 16 warps classify draws as sure-accept
// (x <= i - r), sure-reject (x > i) or ambiguous; warp 0 resolves the
// ambiguous ones in draw order (resolve_list: accepted iff accepted-before
// <= i - x - sure-accepts-before); the band's last step ends the window so
// the next one uses the new mask.
//
// Every decision is exact: windows and records only decide how much work is
// parallel, never the result.
#pragma once
#include "kernels_mask.cuh"

namespace bb {

#ifndef BB_SEG_MAXLEN
#define BB_SEG_MAXLEN 32768
#endif
constexpr int kSegMaxLen = BB_SEG_MAXLEN;   // draws per segment (max)
constexpr int kWalkStage = 8192;            // draws per shared-memory stage of an exact walk
constexpr int kSegCrossLen = 1024; // draws per segment in band-crossing zones
constexpr int kAnchorSlackMin = 512;   // a job's segments start at its predicted first draw + a slack of
constexpr int kAnchorSlackMax = 4000;  // 5 sd of a job's draw count, clamped to this range
constexpr int kSub = 512;          // states per phase-1 sub-window (one warp)
#ifndef BB_SUB_PER_CTA
#define BB_SUB_PER_CTA 8
#endif
constexpr int kSubPerCta = BB_SUB_PER_CTA;      // sub-windows per phase-1 CTA (= warps per k_seg_pass CTA)
constexpr int kSegMaxSub = 64;     // sub-windows per segment (max)
// half-window cap (states): 5 sd of a 29M-draw stretch (a 20M-row class
// block, cfg5) is ~13.5k states; with the cap below that, a deviated path
// misses every later window and the chain degenerates into an exact walk
constexpr double kSegHalfWindowCap = 14336.0;
#ifndef BB_SEG_TAIL
#define BB_SEG_TAIL 2048
#endif
constexpr int kSegTail = BB_SEG_TAIL;     // states below this: walked by phase 2
constexpr int kSegThreads = 32 * kSubPerCta;
constexpr int kSegRing = 16;       // segments of records in flight in k_seg_compose
constexpr int kRows = 16;          // rows of 32 draws classified at once by phase 1 (512-draw chunks)
constexpr int kScalarBelow = 64;
// lean_walk for the tail (states < kSegTail: 3.8M vs 4.5M cycles per 80 cfg2
// jobs with warp_walk); warp_walk for the crossing-zone re-walks (2-4x faster
// at high states, tools/microbench/crosswalk.cu)
constexpr bool kLeanTail = true, kLeanResim = false;
constexpr bool kFuseTail = false;  // true: the tail walk runs in the chain kernel (one launch per job; masks alone -1.5%, but the fit measured 3.07 vs 3.15 G rows*trees/s)
#ifndef BB_WALK_ROWS_SHIFT
#define BB_WALK_ROWS_SHIFT 0
#endif   // walk states below this one draw at a time

__host__ __device__ __forceinline__ unsigned int smear_host(unsigned int x) {
  x |= x >> 1;
  x |= x >> 2;
  x |= x >> 4;
  x |= x >> 8;
  x |= x >> 16;
  return x;
}

struct SegTab {   // per segment of a block size (host-built)
  int off;        // first draw, relative to the job's first draw
  int len;        // draws
  int loA, nA;    // piece A: states [loA, hiA] in the band of hiA, nA sub-windows
  int hiA;
  int loB, nB;    // piece B (the band below): [loB, hiB], nB sub-windows
  int hiB;
  int rec_off;    // first sub-window record
  int pad[3];
};

// expected Fisher-Yates state after p draws from state i0 (mean trajectory,
// (i+1)' = -(i+1)/(mask+1) inside a band)
__host__ __device__ inline double seg_pred_state(int i0, double p) {
  double x = (double)i0 + 1.0;
  while (true) {
    if (x <= 1.0 + 1e-9) return 0.0;
    const unsigned M = smear_host((unsigned)fmax(1.0, floor(x - 1.0)));
    const double mp1 = (double)M + 1.0, lowx = mp1 / 2.0;
    const double pb = mp1 * log(x / lowx);
    if (p < pb) return x * exp(-p / mp1) - 1.0;
    p -= pb;
    x = lowx;
  }
}

// expected draws from state i0 to the end of the job (state 0)
__host__ __device__ inline double seg_expected_draws(int i0) {
  double x = (double)i0 + 1.0, p = 0.0;
  while (x > 1.0 + 1e-9) {
    const unsigned M = smear_host((unsigned)fmax(1.0, floor(x - 1.0)));
    const double mp1 = (double)M + 1.0, lowx = mp1 / 2.0;
    p += mp1 * log(x / lowx);
    x = lowx;
  }
  return p;
}

// half window after p draws: 5 sd (sd <= sqrt(p)/2); a start outside the
// window only costs an exact walk
#ifndef BB_SEG_WINDOW_SD
#define BB_SEG_WINDOW_SD 5.0
#endif
__host__ __device__ inline double seg_half_window(double p, double window_sd = BB_SEG_WINDOW_SD) {
  return p <= 0.0 ? 0.0 : fmin(kSegHalfWindowCap, ceil(0.5 * window_sd * sqrt(p)) + 16.0);
}

// Geometry of the segment at draw offset `off` of a stretch that starts at
// state i0: window, pieces (A: the band of the window's top, B: the band
// below, down to `floor_state`) and length (~90 paths of a 512-state
// sub-window merge at most; kSegCrossLen draws where some start may reach
// its band's last state, so the exact walk a crossing costs stays short).
// Returns false once the window lies below floor_state.
__host__ __device__ inline bool seg_geom(int i0, long long off, int floor_state, SegTab* t, long long slack = 0,
                                         int max_len = kSegMaxLen, double window_sd = BB_SEG_WINDOW_SD) {
  // the job has consumed between off and off + slack draws at this segment
  const double pi = seg_pred_state(i0, (double)off);
  const double pl = seg_pred_state(i0, (double)(off + slack));
  int lo = (int)fmax(1.0, floor(pl - seg_half_window((double)(off + slack), window_sd)));
  int hi = (int)fmin((double)i0, ceil(pi + seg_half_window((double)off, window_sd)));
  if (hi < floor_state || lo > hi) return false;
  // stop once the state is below the floor with 3 sd to spare: the window cap
  // (4096) would otherwise keep hi above a low floor forever; a job that is
  // still above the floor after the last segment walks the rest exactly
  // (the 3-sd margin is capped at half the floor: for large jobs it exceeds
  // the floor itself and the plan would never end)
  if (pi + fmin(1.5 * sqrt((double)(off + slack)), 0.5 * floor_state) < (double)floor_state) return false;
  t->off = (int)off;
  const unsigned Mh = smear_host((unsigned)hi);
  const int bbA = (int)(Mh >> 1) + 1;
  t->loA = lo > bbA ? lo : bbA;
  t->hiA = hi;
  t->nA = (t->hiA - t->loA + kSub) / kSub;
  t->loB = 1;
  t->hiB = 0;
  t->nB = 0;
  if (lo < bbA && bbA - 1 >= floor_state && bbA - 1 >= 1) {
    t->hiB = bbA - 1;
    const unsigned MB = smear_host((unsigned)t->hiB);
    const int bbB = (int)(MB >> 1) + 1;
    t->loB = lo > bbB ? lo : bbB;
    t->nB = (t->hiB - t->loB + kSub) / kSub;
  }
  // at most kSegMaxSub sub-windows (the chain's record slots): trim the far
  // ends (a start outside the window is walked exactly)
  if (t->nA > kSegMaxSub) {
    t->nA = kSegMaxSub;
    t->loA = t->hiA - kSegMaxSub * kSub + 1;
    t->loB = 1;
    t->hiB = 0;
    t->nB = 0;
  } else if (t->nA + t->nB > kSegMaxSub) {
    t->nB = kSegMaxSub - t->nA;
    t->loB = t->hiB - t->nB * kSub + 1;
    if (t->nB <= 0) {
      t->nB = 0;
      t->loB = 1;
      t->hiB = 0;
    }
  }
  const unsigned M = smear_host((unsigned)(pi > 1.0 ? (int)pi : 1));
  const double L = 0.176 * ((double)M + 1.0);
  int Lp = 256;
  while (Lp * 2 <= L && Lp < max_len) Lp *= 2;
  const double pe = seg_pred_state(i0, (double)(off + slack + Lp)) - seg_half_window((double)(off + slack + Lp), window_sd);
  if (lo < bbA || pe < (double)bbA) Lp = Lp < kSegCrossLen ? Lp : kSegCrossLen;
  t->len = Lp;
  return true;
}

struct SegRec {   // 128 B, one sub-window: end(lo + r) = a_end + pref[r/32] + popc(words[r/32] & bits <= r%32)
  int a_end, h, pad0, pad1;
  unsigned int words[16];      // rank bitmask: bit r set = rank r ends above rank r-1
  unsigned short pref[16];     // set bits in words before w
  int pad2[4];
};

struct SegJob {
  int n, k;
  int S;                       // segments in the table
  const SegTab* tab;
  const int2* tasks;           // phase-1 CTAs: (segment, first sub-window)
  int n_tasks;
  int* J;                      // J[i] for steps i >= k
  long long* pos_in;           // job's first draw (absolute index into the draw buffer)
  long long* pos_out;          // written by the tail: first draw of the next job
  long long* anchor_in;        // first draw of segment 0 (predicted first draw + this class's slack)
  long long* anchor2_out;      // written by the tail: anchor of the job after next (nullptr: none)
  long long next_draws;        // expected draws of the next job (its first draw = this job's last + 1)
  long long slack2;            // anchor slack of the job after next
  int write_rng;               // tail: update the RNG state after this job
};

struct SegArgs {
  const unsigned int* draws;
  long long n_draws;
  const PcgJump* jump;
  const RngState* rng0;        // state at draw 0 of the buffer (chunk start)
  RngState* rng;               // written by the compose of the chunk's last job
  SegRec* rec;                 // sub-window records of the job in phase 1/2
  int* seg_start;              // [S] exact start states (phase 2 -> phase 3)
  int* n_seg;                  // segments composed (phase 2 -> phase 3)
  long long* tail_p;           // chain -> tail: first draw of the tail
  int* tail_i;                 // chain -> tail: state there
  SegJob func, emit;           // k_seg_pass: phase-1 job (n_tasks = 0: none), phase-3 job
  long long* prof;
};

constexpr int kPieceWords = kSegMaxSub * 16;  // rank-mask words per piece (max)
constexpr int kPieceSmemPerWarp = 2 * kPieceWords * 4;  // words + exclusive popcount prefix
constexpr int kSegPassSmem = kSubPerCta * kPieceSmemPerWarp;  // phase 1: per-warp piece masks
constexpr int kTabChunk = 64, kTabChunks = 4;  // table entries streamed into k_seg_compose
#ifndef BB_CHAIN_SMEM_KB
#define BB_CHAIN_SMEM_KB 0
#endif
// dynamic shared memory of the chain kernel; BB_CHAIN_SMEM_KB pads it so that
// no other CTA can share the chain's SM (its single-warp dependent chains
// lose issue slots to co-resident phase-1 warps)
constexpr int kSegComposeSmemUsed = kSegRing * kSegMaxSub * 128 + kTabChunk * kTabChunks * 48 + (kWalkStage + 16) * 4;
constexpr int kSegComposeSmem =
    kSegComposeSmemUsed > BB_CHAIN_SMEM_KB * 1024 ? kSegComposeSmemUsed : BB_CHAIN_SMEM_KB * 1024;

__device__ __forceinline__ unsigned int seg_get(const SegArgs& a, const RngState& r0, long long idx) {
  return idx < a.n_draws ? __ldg(&a.draws[idx]) : draw_at(*a.jump, r0, idx);
}

// stage draws [p, p + len) into sd (all threads of the CTA)
__device__ __forceinline__ void seg_stage_cta(const SegArgs& a, const RngState& r0, long long p, int len,
                                              unsigned int* sd) {
  if (p + len <= a.n_draws) {
    for (int j = threadIdx.x; j < len; j += blockDim.x) sd[j] = __ldg(&a.draws[p + j]);
  } else {
    for (int j = threadIdx.x; j < len; j += blockDim.x) sd[j] = seg_get(a, r0, p + j);
  }
  __syncthreads();
}

// ------------------------------------------------------------- phase 1
// One warp, states [lo, lo + W) (W <= kSub) in the band of mask M.  The rank
// bitmask has 16 words; lane l < 16 owns word l (in a register, mirrored in
// smem) and keeps `incl` = set bits in words <= l up to date, so a merge
// finds its word with one ballot.
template <bool kGlobalDraws>
__device__ void seg_sub(const unsigned int* sd, int len, int lo, int W, unsigned int M, SegRec* out, int lane) {
  unsigned int wv = 0;
  if (lane < 16) wv = (lane == 0) ? 0xfffffffeu : 0xffffffffu;  // rank 0 is the base; ranks >= W sentinels
  int incl = __popc(wv);
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  int a = lo, b = lo + W - 1;
  const unsigned lt = (1u << lane) - 1u;
  for (int pos = 0; pos < len; pos += 32 * kRows) {
    // classify kRows rows against the bounds at the chunk start: every path
    // accepts if x <= a0 - r (at most r accepts before), none if x > b0
    const int a0 = a, b0 = b;
    unsigned sa[kRows], am[kRows];
    int xs[kRows];
#pragma unroll
    for (int u = 0; u < kRows; ++u) {
      const int r = 32 * u + lane;
      const bool in = pos + r < len;
      const int x = in ? (int)((kGlobalDraws ? __ldg(sd + pos + r) : sd[pos + r]) & M) : 0x7fffffff;
      xs[u] = x;
      const bool acc = in && x <= a0 - r;
      sa[u] = __ballot_sync(0xffffffffu, acc);
      am[u] = __ballot_sync(0xffffffffu, in && !acc && x <= b0);
    }
    unsigned amany = 0;
    int tot = 0;
#pragma unroll
    for (int u = 0; u < kRows; ++u) {
      amany |= am[u];
      tot += __popc(sa[u]);
    }
    if (amany == 0) {  // fast path: every path takes the same draws
      a -= tot;
      b -= tot;
      continue;
    }
    // rows in order; ambiguous draws decided exactly with the running a, b
#pragma unroll
    for (int u = 0; u < kRows; ++u) {
      unsigned acc = sa[u];
      int mrow = 0;
      unsigned rem = am[u];
      while (rem) {
        const int f = __ffs(rem) - 1;
        rem &= rem - 1u;
        const int nb = __popc(acc & ((1u << f) - 1u));
        const int ac = a - nb, bc = b - nb - mrow;
        const int xf = __shfl_sync(0xffffffffu, xs[u], f);
        if (xf <= ac) {
          acc |= 1u << f;
        } else if (xf <= bc) {
          // clear the t-th set bit of the rank bitmask, t = xf - ac (1-based)
          const int t = xf - ac;
          const unsigned own = __ballot_sync(0xffffffffu, lane < 16 && incl >= t);
          const int ow = __ffs(own) - 1;
          if (lane == ow) {
            const int tt = t - (incl - __popc(wv));
            unsigned int m = wv;
            for (int z = 1; z < tt; ++z) m &= m - 1u;
            wv &= ~(m & (0u - m));
          }
          if (lane >= ow) --incl;
          ++mrow;
        }
      }
      const int na = __popc(acc);
      a -= na;
      b -= na + mrow;
    }
  }
  (void)lt;
  // the rank bitmask and its per-word prefix counts
  const int pc = __popc(wv);
  int pi = pc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, pi, o);
    if (lane >= o) pi += y;
  }
  if (lane < 16) {
    out->words[lane] = wv;
    out->pref[lane] = (unsigned short)(pi - pc);
  }
  if (lane == 0) {
    out->a_end = a;
    out->h = (int)(M >> 1);
  }
}

// sub-window j of segment t: (lo, W, mask)
__device__ __forceinline__ void seg_sub_geom(const SegTab& t, int j, int& lo, int& W, unsigned int& M) {
  if (j < t.nA) {
    lo = t.loA + kSub * j;
    W = min(kSub, t.hiA - lo + 1);
    M = smear((unsigned)t.hiA);
  } else {
    lo = t.loB + kSub * (j - t.nA);
    W = min(kSub, t.hiB - lo + 1);
    M = smear((unsigned)t.hiB);
  }
}

// Phase 1 over a whole piece (A or B) of a segment by ONE warp: the window
// [lo, lo + W) of distinct start states is one interval [a, b] (the same
// transfer-function bookkeeping as seg_sub), its rank bitmask (nsub * 512
// ranks) in the warp's shared-memory words.  A draw is ambiguous only if it
// falls inside the whole window (not once per 512-state sub-window), so the
// piece costs one pass over the segment instead of nsub passes.  The result
// is written as the piece's nsub sub-window records (SegRec format, read by
// the chain unchanged): record j's base end = a_end + set bits of ranks
// (0, 512 j], its own rank-0 bit cleared.
__device__ void seg_piece(const SegArgs& ar, const RngState& r0, long long base, int len, int lo, int W, unsigned int M,
                          int nsub, SegRec* out, unsigned int* sw, int lane) {
  const unsigned FULL = 0xffffffffu;
  const int NWp = nsub * 16;
  const int K = (NWp + 31) >> 5;  // words per lane (contiguous)
  const int w0 = lane * K, w1 = min(NWp, w0 + K);
  int cnt = 0;
  for (int w = w0; w < w1; ++w) {
    const unsigned int v = (w == 0) ? 0xfffffffeu : 0xffffffffu;  // rank 0 is the base; ranks >= W sentinels
    sw[w] = v;
    cnt += __popc(v);
  }
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(FULL, incl, o);
    if (lane >= o) incl += y;
  }
  __syncwarp();
  const bool in_buf = base + len <= ar.n_draws;
  int a = lo, b = lo + W - 1;
  // the next 512-draw chunk is loaded while this one is classified
  unsigned int nxt[kRows];
  auto load = [&](int pos) {
#pragma unroll
    for (int u = 0; u < kRows; ++u) {
      const int r = 32 * u + lane;
      nxt[u] = (pos + r < len && in_buf) ? __ldg(ar.draws + base + pos + r) : 0u;
    }
    if (!in_buf)  // past the draw buffer (never for the configured sizes): jump-ahead per draw
      for (int u = 0; u < kRows; ++u) {
        const int r = 32 * u + lane;
        if (pos + r < len) nxt[u] = seg_get(ar, r0, base + pos + r);
      }
  };
  load(0);
  for (int pos = 0; pos < len; pos += 32 * kRows) {
    const int a0 = a, b0 = b;
    unsigned sa[kRows], am[kRows];
    int xs[kRows];
    unsigned int cur[kRows];
#pragma unroll
    for (int u = 0; u < kRows; ++u) cur[u] = nxt[u];
    if (pos + 32 * kRows < len) load(pos + 32 * kRows);
#pragma unroll
    for (int u = 0; u < kRows; ++u) {
      const int r = 32 * u + lane;
      const bool in = pos + r < len;
      const int x = in ? (int)(cur[u] & M) : 0x7fffffff;
      xs[u] = x;
      const bool acc = in && x <= a0 - r;
      sa[u] = __ballot_sync(FULL, acc);
      am[u] = __ballot_sync(FULL, in && !acc && x <= b0);
    }
    unsigned amany = 0;
    int tot = 0;
#pragma unroll
    for (int u = 0; u < kRows; ++u) {
      amany |= am[u];
      tot += __popc(sa[u]);
    }
    if (amany == 0) {
      a -= tot;
      b -= tot;
      continue;
    }
#pragma unroll
    for (int u = 0; u < kRows; ++u) {
      unsigned acc = sa[u];
      int mrow = 0;
      unsigned rem = am[u];
      while (rem) {
        const int f = __ffs(rem) - 1;
        rem &= rem - 1u;
        const int nb = __popc(acc & ((1u << f) - 1u));
        const int ac = a - nb, bc = b - nb - mrow;
        const int xf = __shfl_sync(FULL, xs[u], f);
        if (xf <= ac) {
          acc |= 1u << f;
        } else if (xf <= bc) {
          // the groups at offsets xf - ac - 1 and xf - ac merge: clear the
          // t-th set bit (1-based) of the rank mask
          const int t = xf - ac;
          const unsigned own = __ballot_sync(FULL, incl >= t);
          const int ow = __ffs(own) - 1;
          BB_DCHECK(ow >= 0 && ow < 32);
          if (lane == ow) {
            int tt = t - (incl - cnt);
            BB_DCHECK(tt >= 1 && tt <= cnt);
            for (int w = w0; w < w1; ++w) {
              unsigned int m = sw[w];
              const int pc = __popc(m);
              if (tt <= pc) {
                for (int z = 1; z < tt; ++z) m &= m - 1u;
                sw[w] &= ~(m & (0u - m));
                break;
              }
              tt -= pc;
            }
            --cnt;
          }
          if (lane >= ow) --incl;
          ++mrow;
        }
      }
      const int na = __popc(acc);
      a -= na;
      b -= na + mrow;
    }
  }
  __syncwarp();
  // exclusive popcount prefix of the words, then the sub-window records
  unsigned int* pre = sw + kPieceWords;
  {
    int run = incl - cnt;
    for (int w = w0; w < w1; ++w) {
      pre[w] = (unsigned int)run;
      run += __popc(sw[w]);
    }
  }
  __syncwarp();
  for (int j = 0; j < nsub; ++j) {
    const int wb = 16 * j;
    const unsigned int first = sw[wb];
    const unsigned int bit0 = first & 1u;
    if (lane < 16) {
      const unsigned int wv = lane == 0 ? (first & ~1u) : sw[wb + lane];
      out[j].words[lane] = wv;
      out[j].pref[lane] = (unsigned short)(pre[wb + lane] - pre[wb] - (lane > 0 ? bit0 : 0u));
    }
    if (lane == 0) {
      out[j].a_end = a + (int)(pre[wb] + bit0);
      out[j].h = (int)(M >> 1);
    }
  }
}

// bulk prefetch of [p, p + n) draws into L2 (16-byte aligned range)
__device__ __forceinline__ void seg_prefetch_l2(const unsigned int* base, long long p, long long n, long long n_draws) {
  long long a0 = p & ~3ll, a1 = min(n_draws, p + n);
  a1 &= ~3ll;
  if (a1 <= a0) return;
  const unsigned bytes = (unsigned)min((a1 - a0) * 4, (long long)1 << 20);
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base + a0), "r"(bytes) : "memory");
}

// One chunk of ROWS rows of 32 draws of the exact walk (see warp_walk),
// classified against the state i0 at the chunk start: sure accept x <= i0 - r
// (at most r accepts before draw r), sure reject x > i0.  Ambiguous draws are
// decided by Jacobi refinement over the chunk: accepted-before(r) lies in
// [A(r), A(r) + U(r)] (decided accepts / unresolved draws before r), so
// x <= i0 - A - U accepts and x > i0 - A rejects; a draw with A >= d lies
// past the band's last step (dropped).  The first unresolved draw has U = 0,
// so every pass decides at least one.  The d-th accept ends the chunk.
template <int ROWS, bool kGlobal>
__device__ __forceinline__ void walk_chunk(const unsigned int* src, int pos, int len, int i0, int d, unsigned int M,
                                           int k, int* J, int lane, int& taken, int& consumed) {
  const unsigned lt = (1u << lane) - 1u;
  unsigned acc[ROWS], ur[ROWS];
  int xs[ROWS];
  unsigned any = 0;
  int tot = 0;
#pragma unroll
  for (int u = 0; u < ROWS; ++u) {
    const int r = 32 * u + lane;
    const bool in = pos + r < len;
    const unsigned int raw = in ? (kGlobal ? __ldg(src + pos + r) : src[pos + r]) : 0u;
    const int x = in ? (int)(raw & M) : 0x7fffffff;
    xs[u] = x;
    const bool sa = in && x <= i0 - r;
    acc[u] = __ballot_sync(0xffffffffu, sa);
    ur[u] = __ballot_sync(0xffffffffu, in && !sa && x <= i0);
    any |= ur[u];
    tot += __popc(acc[u]);
  }
  consumed = min(32 * ROWS, len - pos);
  if (any == 0 && tot < d) {  // fast path: every draw decided, no band crossing
    if (J) {
      int pre = 0;
#pragma unroll
      for (int u = 0; u < ROWS; ++u) {
        if ((acc[u] >> lane) & 1u) {
          const int st = i0 - pre - __popc(acc[u] & lt);
          if (st >= k) J[st] = xs[u];
        }
        pre += __popc(acc[u]);
      }
    }
    taken = tot;
    return;
  }
  while (any) {
    unsigned na[ROWS], nr[ROWS];
    int runA = 0, runU = 0;
#pragma unroll
    for (int u = 0; u < ROWS; ++u) {
      const int A = runA + __popc(acc[u] & lt), U = runU + __popc(ur[u] & lt);
      const bool mine = (ur[u] >> lane) & 1u;
      na[u] = __ballot_sync(0xffffffffu, mine && A < d && xs[u] <= i0 - A - U);
      nr[u] = __ballot_sync(0xffffffffu, mine && (A >= d || xs[u] > i0 - A));
      runA += __popc(acc[u]);
      runU += __popc(ur[u]);
    }
    any = 0;
#pragma unroll
    for (int u = 0; u < ROWS; ++u) {
      acc[u] |= na[u];
      ur[u] &= ~(na[u] | nr[u]);
      any |= ur[u];
    }
  }
  int runA = 0, cut_row = ROWS, cut_lane = 31;
#pragma unroll
  for (int u = 0; u < ROWS; ++u) {
    const int T = __popc(acc[u]);
    if (cut_row == ROWS && runA + T >= d) {
      unsigned mm = acc[u];
      for (int z = 1; z < d - runA; ++z) mm &= mm - 1u;
      cut_row = u;
      cut_lane = __ffs(mm) - 1;
    }
    if (cut_row == ROWS) runA += T;
  }
  if (cut_row < ROWS) {
    consumed = 32 * cut_row + cut_lane + 1;
    taken = d;
  } else {
    taken = runA;
  }
  if (J) {
    int pre = 0;
#pragma unroll
    for (int u = 0; u < ROWS; ++u) {
      unsigned m = acc[u];
      if (u > cut_row) m = 0;
      if (u == cut_row) m &= (cut_lane >= 31) ? 0xffffffffu : ((2u << cut_lane) - 1u);
      if ((m >> lane) & 1u) {
        const int st = i0 - pre - __popc(m & lt);
        if (st >= k) J[st] = xs[u];
      }
      pre += __popc(m);
    }
  }
}

// Exact walk of one path by one warp, from state i over src[0 .. len-1]
// (global or shared): chunks of 32*ROWS draws with ROWS chosen per band so
// a chunk expects about one ambiguous draw ((32 ROWS)^2 <= 2(M+1)); states
// below kScalarBelow are walked draw by draw.  Stops after the draw that
// takes i to 0.  Writes J[step] = x for accepted steps >= k when J != nullptr.
template <bool kGlobal>
__device__ int warp_walk(const unsigned int* src, int len, int i, int k, int* J, int lane, int* used) {
  int pos = 0;
  while (pos < len && i >= 1) {
    if (i < kScalarBelow) {
      // 32 draws per step: taken in order from the lanes
      int ii = i, pp = pos;
      while (pp < len && ii >= 1) {
        const unsigned int v = pp + lane < len ? (kGlobal ? __ldg(src + pp + lane) : src[pp + lane]) : 0u;
        int take = 0;
        for (int q = 0; q < 32 && pp + q < len && ii >= 1; ++q) {
          const int x = (int)(__shfl_sync(0xffffffffu, v, q) & smear((unsigned)ii));
          ++take;
          if (x <= ii) {
            if (J && lane == 0 && ii >= k) J[ii] = x;
            --ii;
          }
        }
        pp += take;
      }
      i = ii;
      pos = pp;
      break;
    }
    const unsigned int M = smear((unsigned)i);
    const int d = i - (int)(M >> 1);  // accepts until the band's last step
    int taken, consumed;
    constexpr int sh = 2 * BB_WALK_ROWS_SHIFT;  // rows per chunk x 2^BB_WALK_ROWS_SHIFT at a given band
    if (M >= (1u << (17 - sh)) - 1)
      walk_chunk<16, kGlobal>(src, pos, len, i, d, M, k, J, lane, taken, consumed);
    else if (M >= (1u << (15 - sh)) - 1)
      walk_chunk<8, kGlobal>(src, pos, len, i, d, M, k, J, lane, taken, consumed);
    else if (M >= (1u << (13 - sh)) - 1)
      walk_chunk<4, kGlobal>(src, pos, len, i, d, M, k, J, lane, taken, consumed);
    else if (M >= (1u << (11 - sh)) - 1)
      walk_chunk<2, kGlobal>(src, pos, len, i, d, M, k, J, lane, taken, consumed);
    else
      walk_chunk<1, kGlobal>(src, pos, len, i, d, M, k, J, lane, taken, consumed);
    i -= taken;
    pos += consumed;
  }
  *used = pos;
  return i;
}

// Lean exact walk (one warp, one draw per lane per chunk of 32): sure accept
// x <= i - r, sure reject x > i, the few ambiguous draws resolved in draw
// order (accepted iff x <= i - accepted-before); the band's last step (or the
// job's end) cuts the chunk.  Used where the per-chunk latency is what counts
// (the tail's low states, the short crossing-zone segments of the chain):
// the next chunk's draws are loaded while this one resolves.
__device__ int lean_walk(const unsigned int* src, int len, int i, int k, int* J, int lane, int* used) {
  const unsigned FULL = 0xffffffffu, lt = (1u << lane) - 1u;
  int pos = 0;
  unsigned int raw = lane < len ? src[lane] : 0u;
  while (pos < len && i >= 1) {
    const unsigned int M = smear((unsigned)i);
    const int need = i - (int)(M >> 1);  // accepts to the band's last step
    const bool in = pos + lane < len;
    const int x = (int)(raw & M);
    const unsigned int nxt = pos + 32 + lane < len ? src[pos + 32 + lane] : 0u;
    unsigned acc = __ballot_sync(FULL, in && x <= i - lane);
    unsigned am = __ballot_sync(FULL, in && x > i - lane && x <= i);
    while (am) {
      const int r = __ffs(am) - 1;
      const int xr = __shfl_sync(FULL, x, r);
      if (xr <= i - __popc(acc & ((1u << r) - 1u))) acc |= 1u << r;
      am &= am - 1u;
    }
    const int cnt = __popc(acc);
    int consumed = min(32, len - pos), taken = cnt;
    if (cnt >= need) {
      unsigned mm = acc;
      for (int z = 1; z < need; ++z) mm &= mm - 1u;
      const int cut = __ffs(mm) - 1;
      consumed = cut + 1;
      taken = need;
      acc &= cut >= 31 ? FULL : ((2u << cut) - 1u);
    }
    if (J && i >= k) {
      const int st = i - __popc(acc & lt);
      if (((acc >> lane) & 1u) && st >= k) J[st] = x;
    }
    i -= taken;
    pos += consumed;
    raw = consumed == 32 ? nxt : (pos + lane < len ? src[pos + lane] : 0u);
  }
  *used = pos;
  return i;
}

// draws past the buffer (jump-ahead per draw): lane 0, one draw at a time
__device__ int warp_walk_slow(const SegArgs& a, const RngState& r0, long long base, int len, int i, int k, int* J,
                              int lane, int* used) {
  int pos = 0;
  if (lane == 0) {
    while (pos < len && i >= 1) {
      const int x = (int)(seg_get(a, r0, base + pos) & smear((unsigned)i));
      ++pos;
      if (x <= i) {
        if (J && i >= k) J[i] = x;
        --i;
      }
    }
  }
  i = __shfl_sync(0xffffffffu, i, 0);
  *used = __shfl_sync(0xffffffffu, pos, 0);
  return i;
}

// phase 1 (func job tasks) and phase 3 (emit job segments) in one launch:
// blocks [0, nb_func) are phase-1 tasks, the rest emit segments.
__global__ void __launch_bounds__(kSegThreads) k_seg_pass(SegArgs a, int nb_func) {
  extern __shared__ __align__(16) unsigned char ps_sm[];
  unsigned int* sd = reinterpret_cast<unsigned int*>(ps_sm);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const RngState r0 = *a.rng0;
  if ((int)blockIdx.x < nb_func) {
    // phase 1: one warp per piece (task = (segment, piece A / B))
    const SegJob& jb = a.func;
    const int task_i = (int)blockIdx.x * kSubPerCta + warp;
    if (task_i < jb.n_tasks) {
      const int2 task = jb.tasks[task_i];
      const SegTab t = jb.tab[task.x];
      const long long p0 = *jb.anchor_in;
      const long long c0 = clock64();
      unsigned int* sw = reinterpret_cast<unsigned int*>(ps_sm) + warp * (kPieceSmemPerWarp / 4);
      if (task.y == -1) {
        seg_piece(a, r0, p0 + t.off, t.len, t.loA, t.hiA - t.loA + 1, smear((unsigned)t.hiA), t.nA, a.rec + t.rec_off,
                  sw, lane);
      } else if (task.y == -2) {
        seg_piece(a, r0, p0 + t.off, t.len, t.loB, t.hiB - t.loB + 1, smear((unsigned)t.hiB), t.nB,
                  a.rec + t.rec_off + t.nA, sw, lane);
      } else {
        // a window that is a large share of its band: one warp per 512-state
        // sub-window (dense ambiguous draws are cheaper in narrow windows)
        int lo, W;
        unsigned int M;
        seg_sub_geom(t, task.y, lo, W, M);
        if (p0 + t.off + t.len <= a.n_draws)
          seg_sub<true>(a.draws + p0 + t.off, t.len, lo, W, M, a.rec + t.rec_off + task.y, lane);
        else
          seg_piece(a, r0, p0 + t.off, t.len, lo, W, M, 1, a.rec + t.rec_off + task.y, sw, lane);
      }
      if (a.prof && lane == 0) {
        atomicAdd((unsigned long long*)&a.prof[7], 1ull);
        atomicAdd((unsigned long long*)&a.prof[8], (unsigned long long)(clock64() - c0));
        atomicMax((unsigned long long*)&a.prof[9], (unsigned long long)(clock64() - c0));
      }
    }
  } else {
    const SegJob& jb = a.emit;
    const int s = (blockIdx.x - nb_func) * kSubPerCta + warp;
    if (s >= *a.n_seg) return;
    const int i0 = a.seg_start[s];
    if (i0 < jb.k) return;  // no step >= k in this segment
    const SegTab t = jb.tab[s];
    const long long base = *jb.anchor_in + t.off;
    const long long c0 = clock64();
    if (lane == 0) seg_prefetch_l2(a.draws, base, t.len, a.n_draws);
    int used;
    if (base + t.len <= a.n_draws) {
      warp_walk<true>(a.draws + base, t.len, i0, jb.k, jb.J, lane, &used);
    } else {
      // past the draw buffer (never for the configured sizes): jump-ahead per draw
      warp_walk_slow(a, r0, base, t.len, i0, jb.k, jb.J, lane, &used);
    }
    if (a.prof && lane == 0) {
      atomicAdd((unsigned long long*)&a.prof[10], 1ull);
      atomicMax((unsigned long long*)&a.prof[11], (unsigned long long)(clock64() - c0));
    }
  }
}

__device__ __forceinline__ void cp_async16_seg(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

// Exact walk by one warp over draws staged in shared memory by bulk copies
// (16-byte aligned source: copy from base & ~3, walk from base & 3).
struct StageWalk {
  unsigned int* sd;  // kWalkStage + 16 draws
  uint64_t* bar;
  unsigned phase;
  __device__ int operator()(const SegArgs& a, const RngState& r0, long long base, long long len, int i, int k, int* J,
                            int lane, long long* used, bool lean = false) {
    long long done = 0;
    while (done < len && i >= 1) {
      const long long b = base + done;
      const int n = (int)min((long long)kWalkStage, len - done);
      if (lane == 0 && len - done > n)
        seg_prefetch_l2(a.draws, b + n, min((long long)kWalkStage, len - done - n), a.n_draws);
      int u;
      if (b + n + 4 <= a.n_draws) {
        const long long ab = b & ~3ll;
        const int o = (int)(b - ab);
        const unsigned bytes = (unsigned)(((n + o + 3) / 4) * 16);
        if (lane == 0) {
          mbar_expect_tx(bar, bytes);
          tma_load_1d(sd, a.draws + ab, bytes, bar);
        }
        mbar_wait(bar, phase);
        phase ^= 1u;
        i = lean ? lean_walk(sd + o, n, i, k, J, lane, &u) : warp_walk<false>(sd + o, n, i, k, J, lane, &u);
      } else {
        i = warp_walk_slow(a, r0, b, n, i, k, J, lane, &u);
      }
      done += u;
      __syncwarp();
    }
    *used = done;
    return i;
  }
};

__device__ void seg_tail_walk(const SegArgs& a, const RngState& r0, StageWalk& walk, long long p, int i, int lane);

// phase 2a: two warps.  Warp 1 (producer) streams the table entries and
// the segments' records into shared memory with bulk copies (full/empty
// mbarriers per record slot) and prefetches the draws of band-crossing-zone
// segments into L2.  Warp 0 (consumer) walks from the job's exact first draw
// to the anchor, then chains the segments' functions down to kSegTail (an
// O(1) lookup per segment; a start the records cannot answer is walked
// exactly) and hands the tail's (draw, state) to k_seg_tail.
__global__ void __launch_bounds__(64) k_seg_chain(SegArgs a) {
  extern __shared__ __align__(16) unsigned char cs_sm[];
  SegRec* ring = reinterpret_cast<SegRec*>(cs_sm);  // [kSegRing][kSegMaxSub]
  SegTab* tring = reinterpret_cast<SegTab*>(cs_sm + (size_t)kSegRing * kSegMaxSub * sizeof(SegRec));
  unsigned int* sd = reinterpret_cast<unsigned int*>(reinterpret_cast<unsigned char*>(tring) +
                                                    (size_t)kTabChunk * kTabChunks * sizeof(SegTab));
  __shared__ __align__(16) SegTab slot_tab[kSegRing];  // the table entry of the segment in each record slot
  __shared__ __align__(8) uint64_t tab_bar[kTabChunks], full_bar[kSegRing], empty_bar[kSegRing], st_bar;
  __shared__ int s_s0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const SegJob& jb = a.func;
  const RngState r0 = *a.rng0;
  const long long p0 = *jb.pos_in;
  const long long anc = *jb.anchor_in;
  const int S = jb.S;
  if (threadIdx.x == 0) {
    for (int q = 0; q < kTabChunks; ++q) mbar_init(&tab_bar[q], 1);
    for (int q = 0; q < kSegRing; ++q) {
      mbar_init(&full_bar[q], 1);
      mbar_init(&empty_bar[q], 1);
    }
    mbar_init(&st_bar, 1);
    fence_mbar_init();
    // first segment at or after the true first draw (segment 0 unless the job
    // started more than its slack late); earlier ones are skipped
    int s0 = 0;
    while (s0 < S && anc + jb.tab[s0].off < p0) ++s0;
    s_s0 = s0;
  }
  __syncthreads();
  const int s0 = s_s0;
  if (warp == 1) {
    // ---- producer
    int tab_waited = -1;
    auto tab_issue = [&](int c) {
      const int first = c * kTabChunk, cnt = min(kTabChunk, S - first);
      if (cnt > 0 && lane == 0) {
        uint64_t* bar = &tab_bar[c % kTabChunks];
        mbar_expect_tx(bar, (unsigned)cnt * (unsigned)sizeof(SegTab));
        tma_load_1d(tring + (c % kTabChunks) * kTabChunk, jb.tab + first, (unsigned)cnt * (unsigned)sizeof(SegTab),
                    bar);
      }
    };
    if (s0 < S) {
      tab_issue(0);
      tab_issue(1);
    }
    for (int q = s0; q < S; ++q) {
      const int rq = q - s0, slot = rq % kSegRing;
      if (rq >= kSegRing) mbar_wait(&empty_bar[slot], (unsigned)(((rq / kSegRing) - 1) & 1));
      const int c = q / kTabChunk;
      while (tab_waited < c) {
        ++tab_waited;
        mbar_wait(&tab_bar[tab_waited % kTabChunks], (unsigned)((tab_waited / kTabChunks) & 1));
        tab_issue(tab_waited + 2);  // its slot held chunk tab_waited - 2 (the consumer is past it)
      }
      const SegTab& t = tring[q % (kTabChunk * kTabChunks)];
      if (lane < 12) reinterpret_cast<int*>(&slot_tab[slot])[lane] = reinterpret_cast<const int*>(&t)[lane];
      __syncwarp();
      if (lane == 0) {
        if (t.len <= kSegCrossLen) seg_prefetch_l2(a.draws, anc + t.off, t.len, a.n_draws);  // likely walked
        const unsigned bytes = (unsigned)(t.nA + t.nB) * (unsigned)sizeof(SegRec);
        mbar_expect_tx(&full_bar[slot], bytes);  // release: slot_tab visible to the consumer
        tma_load_1d(ring + slot * kSegMaxSub, a.rec + t.rec_off, bytes, &full_bar[slot]);
      }
    }
    // drain the table chunks still in flight
    if (s0 < S) {
      const int last_chunk = min((S - 1) / kTabChunk, tab_waited + 2);
      for (int c = tab_waited + 1; c <= last_chunk; ++c)
        mbar_wait(&tab_bar[c % kTabChunks], (unsigned)((c / kTabChunks) & 1));
    }
    return;
  }
  // ---- consumer (warp 0)
  StageWalk walk{sd, &st_bar, 0u};
  long long c_resim = 0, n_resim = 0;
  const long long c_start = clock64();
  for (int q = lane; q < s0; q += 32) a.seg_start[q] = -1;
  int i = jb.n - 1;
  long long p = p0;
  if (s0 < S) {
    long long used;
    // the anchor slack (up to kAnchorSlackMax draws) can exceed a short job's
    // whole draw count: the job may end inside this walk, so the position
    // is where the walk stopped, not the anchor
    i = walk(a, r0, p0, anc + jb.tab[s0].off - p0, i, jb.k, jb.J, lane, &used);
    p = p0 + used;
  }
  int s = s0;
  for (; s < S && i >= kSegTail; ++s) {
    const int rs = s - s0, slot = rs % kSegRing;
    mbar_wait(&full_bar[slot], (unsigned)((rs / kSegRing) & 1));
    if (lane == 0) a.seg_start[s] = i;
    const SegTab& t = slot_tab[slot];
    // record lookup, branch-free: piece A [loA, hiA] or B [loB, hiB] (nB > 0),
    // sub-window j = offset / kSub, rank r = offset % kSub
    const int4 ta4 = *reinterpret_cast<const int4*>(&t);                                   // off, len, loA, nA
    const int4 tb4 = *reinterpret_cast<const int4*>(reinterpret_cast<const int*>(&t) + 4);  // hiA, loB, nB, hiB
    const int dA = i - ta4.z, dB = i - tb4.y;
    const bool inA = (unsigned)dA <= (unsigned)(tb4.x - ta4.z);
    const bool inB = tb4.z > 0 && (unsigned)dB <= (unsigned)(tb4.w - tb4.y);
    const int dd = inA ? dA : dB;
    const int j = (inA ? 0 : ta4.w) + (int)((unsigned)dd / kSub);
    int next = -1;
    if (inA || inB) {
      const SegRec& R = ring[slot * kSegMaxSub + j];
      const int r = (int)((unsigned)dd % kSub), w = r >> 5, bt = r & 31;
      const unsigned int m = bt == 31 ? 0xffffffffu : ((2u << bt) - 1u);
      const int2 ah = *reinterpret_cast<const int2*>(&R.a_end);  // a_end, h
      const int e = ah.x + (int)R.pref[w] + __popc(R.words[w] & m);
      if (e > ah.y) next = e;
    }
    const int off = ta4.x, len = ta4.y;
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty_bar[slot])) : "memory");
    if (next < 0) {
      // exact walk (band crossing inside the segment, or a window miss); the
      // J values are emitted by phase 3
      const long long cr = clock64();
      long long used;
      next = walk(a, r0, anc + off, len, i, jb.k, nullptr, lane, &used, kLeanResim);
      c_resim += clock64() - cr;
      ++n_resim;
    }
    i = next;
    p = anc + off + len;
  }
  // let the producer finish: consume (release) the slots it still fills
  for (int q = s; q < S; ++q) {
    const int rq = q - s0, slot = rq % kSegRing;
    mbar_wait(&full_bar[slot], (unsigned)((rq / kSegRing) & 1));
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty_bar[slot])) : "memory");
  }
  if (lane == 0) {
    *a.n_seg = s;
    *a.tail_p = p;
    *a.tail_i = i;
    if (a.prof) {
      atomicAdd((unsigned long long*)&a.prof[0], (unsigned long long)(s - s0));
      atomicAdd((unsigned long long*)&a.prof[1], (unsigned long long)n_resim);
      atomicAdd((unsigned long long*)&a.prof[4], (unsigned long long)(clock64() - c_start - c_resim));
      atomicAdd((unsigned long long*)&a.prof[5], (unsigned long long)c_resim);
      atomicAdd((unsigned long long*)&a.prof[13], (unsigned long long)s0);
    }
  }
  if (kFuseTail) seg_tail_walk(a, r0, walk, p, i, lane);  // phase 2b in the same warp (one launch per job)
}

// phase 2b: one warp walks the tail (states below kSegTail) to the job's
// last draw, writing J for steps >= k; the next draw is the next job's first.
constexpr int kSegTailSmem = (kWalkStage + 16) * 4;
// phase 2b: walk the tail (states below kSegTail) from (p, i) to the job's
// last draw, writing J for steps >= k; the next draw is the next job's first.
__device__ void seg_tail_walk(const SegArgs& a, const RngState& r0, StageWalk& walk, long long p, int i, int lane) {
  const SegJob& jb = a.func;
  const long long ct = clock64();
  long long tail = 0;
  while (i >= 1) {
    long long used;
    i = walk(a, r0, p, 8 * kWalkStage, i, jb.k, jb.J, lane, &used, kLeanTail);
    p += used;
    tail += used;
  }
  if (lane == 0) {
    *jb.pos_out = p;
    // the job after next: first draw predicted from the next job's exact first
    // draw (p) and its expected length, so its phase 1 runs during the next
    // job's chain and tail
    if (jb.anchor2_out) *jb.anchor2_out = p + jb.next_draws + jb.slack2;
    if (a.prof) {
      atomicAdd((unsigned long long*)&a.prof[2], (unsigned long long)tail);
      atomicAdd((unsigned long long*)&a.prof[3], 1ull);
      atomicAdd((unsigned long long*)&a.prof[6], (unsigned long long)(clock64() - ct));
      // anchor error of this job: true first draw vs predicted (anchor - slack), via pos_in
    }
    if (jb.write_rng) {
      RngState r = r0;
      long long dd = p;
      if (r.has_uint32 && dd > 0) {
        r.has_uint32 = 0;
        dd -= 1;
      }
      if (dd > 0) {
        const unsigned long long outs = (unsigned long long)((dd + 1) / 2);
        const U128 st = pcg_jump(*a.jump, r0.s, outs);
        r.s = st;
        if (dd & 1) {
          r.has_uint32 = 1;
          r.uinteger = (unsigned int)(xsl_rr(st) >> 32);
        } else {
          r.has_uint32 = 0;
          r.uinteger = 0;
        }
      }
      *a.rng = r;
    }
  }
}

__global__ void __launch_bounds__(32) k_seg_tail(SegArgs a) {
  extern __shared__ __align__(16) unsigned int sd[];  // kWalkStage + 16 draws
  __shared__ __align__(8) uint64_t st_bar;
  const int lane = threadIdx.x;
  const RngState r0 = *a.rng0;
  if (lane == 0) {
    mbar_init(&st_bar, 1);
    fence_mbar_init();
  }
  __syncwarp();
  StageWalk walk{sd, &st_bar, 0u};
  seg_tail_walk(a, r0, walk, *a.tail_p, *a.tail_i, lane);
}

__global__ void k_seg_init(long long* pos, long long* anchor, long long a0, long long a1) {
  pos[0] = 0;
  anchor[0] = a0;
  anchor[1] = a1;
}

}  // namespace bb
