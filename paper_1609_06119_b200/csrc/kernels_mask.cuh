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
//  k_mask_parse    one warp assigns draws to steps: 256 draws per
//                  iteration, each classified sure-accept (v <= i - r),
//                  sure-reject (v > i) or ambiguous; a window with an
//                  ambiguous draw (or a mask-band / block boundary) is
//                  resolved serially.  Writes J[i] for steps i >= k and the
//                  PCG64 state after the tree.
//  k_bucket_*      counting sort of the steps by target position.
//  k_resolve       value moved out by step i = follow the chain of later
//                  steps that wrote its target position (see DESIGN.md
//                  §Subsample); marks it removed.
//  k_mask_bits     active bit = not removed, class-block bit order.
#pragma once
#include <cooperative_groups.h>
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

__global__ void k_pcg_draws(const PcgJump* __restrict__ Jp, const RngState* __restrict__ rs,
                            unsigned int* __restrict__ draws, long long n_draws) {
  const RngState r = *rs;
  const long long h = r.has_uint32 ? 1 : 0;
  const long long n_out = (n_draws - h + 1) / 2;
  const long long q0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * kDrawChunk;
  if (q0 >= n_out) return;
  if (q0 == 0 && h) draws[0] = r.uinteger;
  U128 s = pcg_jump(*Jp, r.s, (unsigned long long)q0);  // state before output q0
  const U128 a = Jp->A[0], c = Jp->C[0];
  const long long q1 = min(n_out, q0 + kDrawChunk);
  for (long long qq = q0; qq < q1; ++qq) {
    s = u128_add(u128_mul(a, s), c);
    const unsigned long long o = xsl_rr(s);
    const long long j = h + 2 * qq;
    if (j < n_draws) draws[j] = (unsigned int)o;
    if (j + 1 < n_draws) draws[j + 1] = (unsigned int)(o >> 32);
  }
}

__device__ __forceinline__ unsigned int smear(unsigned int x) {
  x |= x >> 1;
  x |= x >> 2;
  x |= x >> 4;
  x |= x >> 8;
  x |= x >> 16;
  return x;
}

struct ParseArgs {
  const unsigned int* draws;
  long long n_draws;
  const PcgJump* jump;
  RngState* rng;  // in: state before the tree, out: state after
  int n[2], k[2];
  int* J[2];      // J[c][i] for steps i >= k[c]; tree t of a chunk at J[c] + t * J_stride
  int n_trees;    // trees parsed by one launch (the cluster kernel parses a chunk)
  long long J_stride;
  // fast-window records, expanded into J by k_expand_windows
  int* rec_pos;            // first draw of the window
  int* rec_i;              // step of the window's first draw, class in bit 31
  int* rec_len;            // draws in the window (<= 256)
  unsigned char* rec_bits; // [w][32]: lane's 8 accept bits
  int* rec_count;          // number of records
  int rec_cap;
  long long* prof;         // optional [8] phase cycle counters (debug)
};

// One warp (launch <<<1, 32>>>).  Draws stream through a shared-memory ring
// of kRingChunks chunks filled by TMA bulk copies issued ahead of the
// consumption point, so the sequential parse never waits on HBM latency.
constexpr int kRingChunk = 4096;  // draws per chunk (16 KiB)
constexpr int kRingChunks = 8;
constexpr int kRing = kRingChunk * kRingChunks;

struct Ring {
  unsigned int* ring;
  uint64_t* bars;
  const unsigned int* src;
  int n_chunks, full;
  int issued, ready;
};

// make draws up to index `hi` (< full) readable; chunks below chunk(pos)
// are consumed and their slots may be refilled
__device__ __forceinline__ void ring_need(Ring& R, int pos, int hi, int lane) {
  const int ch = hi / kRingChunk;
  if (ch <= R.ready) return;
  const int upto = min(R.n_chunks, pos / kRingChunk + kRingChunks);
  if (lane == 0) {
    for (int x = R.issued; x < upto; ++x) {
      const int slot = x % kRingChunks;
      mbar_expect_tx(&R.bars[slot], kRingChunk * 4);
      tma_load_1d(R.ring + slot * kRingChunk, R.src + (size_t)x * kRingChunk, kRingChunk * 4, &R.bars[slot]);
    }
  }
  R.issued = max(R.issued, upto);
  for (int x = R.ready + 1; x <= ch; ++x) mbar_wait(&R.bars[x % kRingChunks], (unsigned)((x / kRingChunks) & 1));
  R.ready = ch;
}

__device__ __forceinline__ unsigned int ring_get(const Ring& R, const ParseArgs& a, const RngState& r0, int idx) {
  if (idx < R.full) return R.ring[idx & (kRing - 1)];
  return idx < a.n_draws ? __ldg(&a.draws[idx]) : draw_at(*a.jump, r0, idx);
}

__global__ void __launch_bounds__(32) k_mask_parse(ParseArgs a) {
  extern __shared__ __align__(16) unsigned int ring[];  // kRing draws
  __shared__ __align__(8) uint64_t bars[kRingChunks];
  const int lane = threadIdx.x;
  const unsigned lt = (1u << lane) - 1u;
  const RngState r0 = *a.rng;
  Ring R;
  R.ring = ring;
  R.bars = bars;
  R.src = a.draws;
  R.n_chunks = (int)(a.n_draws / kRingChunk);  // full chunks; the tail is read from global
  R.full = R.n_chunks * kRingChunk;
  R.issued = 0;   // next chunk to issue
  R.ready = -1;   // highest chunk known complete
  const int full = R.full;
  if (lane == 0) {
    for (int c = 0; c < kRingChunks; ++c) mbar_init(&bars[c], 1);
    fence_mbar_init();
  }
  __syncwarp();
  int pos = 0;
  int nrec = 0;
  ring_need(R, 0, 0, lane);
  for (int c = 0; c < 2; ++c) {
    const int n = a.n[c], k = a.k[c];
    int* J = a.J[c];
    int i = n - 1;
    while (i >= 1) {
      if (pos & 3) {
        // re-align the stream position to 4 draws (uint4 ring loads)
        if (pos + 3 < full) ring_need(R, pos, pos + 3, lane);
        while ((pos & 3) && i >= 1) {
          const unsigned int v = ring_get(R, a, r0, pos) & smear((unsigned)i);
          ++pos;
          if ((int)v <= i) {
            if (lane == 0 && i >= k) J[i] = (int)v;
            --i;
          }
        }
        continue;
      }
      const unsigned int m = smear((unsigned)i);
      const int half = (int)(m >> 1);
      if (i - 255 > half && pos + 256 <= full) {
        // ---- fast loop: 256-draw windows inside one mask band
        ring_need(R, pos, pos + 255, lane);
        // each uint4 wraps separately (pos is 4-aligned, the ring a multiple of 4)
        uint4 x0 = *reinterpret_cast<const uint4*>(ring + ((pos + lane * 8) & (kRing - 1)));
        uint4 x1 = *reinterpret_cast<const uint4*>(ring + ((pos + lane * 8 + 4) & (kRing - 1)));
        for (;;) {
          unsigned int v[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
          // prefetch the next window (consumed only if this one is sure)
          const bool more = (i - 511 > half) && (pos + 512 <= full);
          if (more) {
            ring_need(R, pos, pos + 511, lane);
            x0 = *reinterpret_cast<const uint4*>(ring + ((pos + 256 + lane * 8) & (kRing - 1)));
            x1 = *reinterpret_cast<const uint4*>(ring + ((pos + 260 + lane * 8) & (kRing - 1)));
          }
          unsigned accb = 0, ambb = 0;
          const int i0 = i - lane * 8;
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            v[u] &= m;
            const bool acc = (int)v[u] <= i0 - u;
            accb |= (acc ? 1u : 0u) << u;
            ambb |= ((!acc && (int)v[u] <= i) ? 1u : 0u) << u;
          }
          int len = 256;
          if (__any_sync(0xffffffffu, ambb != 0)) {
            // first ambiguous draw: draws before it are decided
            len = __reduce_min_sync(0xffffffffu, ambb ? lane * 8 + (__ffs(ambb) - 1) : 256);
            const int keep = len - lane * 8;
            accb &= keep >= 8 ? 0xffu : (keep <= 0 ? 0u : ((1u << keep) - 1u));
          }
          const int total = __reduce_add_sync(0xffffffffu, __popc(accb));
          if (i >= k && total > 0) {  // steps i .. i-total+1 may need J values
            if (nrec < a.rec_cap) {
              const int w = nrec++;
              a.rec_bits[(size_t)w * 32 + lane] = (unsigned char)accb;
              if (lane == 0) {
                a.rec_pos[w] = pos;
                a.rec_i[w] = i | (c << 31);
                a.rec_len[w] = len;
              }
            } else {  // record buffer full: write this window's J values directly
              const int cnt = __popc(accb);
              int incl = cnt;
              for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
              }
              int sd = i - (incl - cnt);
#pragma unroll
              for (int u = 0; u < 8; ++u) {
                if ((accb >> u) & 1u) {
                  if (sd >= k) J[sd] = (int)v[u];
                  --sd;
                }
              }
            }
          }
          i -= total;
          if (len < 256) {
            // the ambiguous draw: its step is now exact
            const unsigned int va = ring[(pos + len) & (kRing - 1)] & m;
            if ((int)va <= i) {
              if (lane == 0 && i >= k) J[i] = (int)va;
              --i;
            }
            pos += len + 1;
            break;
          }
          pos += 256;
          if (!more || i - 255 <= half) break;
        }
        continue;
      }
      if (i - 31 > half && pos + 32 <= full) {
        // 32-draw window, one draw per lane, same exact-prefix rule
        ring_need(R, pos, pos + 31, lane);
        const unsigned int v = ring[(pos + lane) & (kRing - 1)] & m;
        const bool acc = (int)v <= i - lane;
        const bool amb = !acc && (int)v <= i;
        const unsigned ambm = __ballot_sync(0xffffffffu, amb);
        const int ra = ambm ? __ffs(ambm) - 1 : 32;
        const unsigned ab = __ballot_sync(0xffffffffu, acc) & (ra >= 32 ? 0xffffffffu : ((1u << ra) - 1u));
        const int before = __popc(ab & lt);
        if (lane < ra && acc && i - before >= k) J[i - before] = (int)v;
        i -= __popc(ab);
        if (ra < 32) {
          const unsigned int va = __shfl_sync(0xffffffffu, v, ra);
          if ((int)va <= i) {
            if (lane == 0 && i >= k) J[i] = (int)va;
            --i;
          }
          pos += ra + 1;
        } else {
          pos += 32;
        }
        continue;
      }
      // serial: up to 32 draws, then re-align pos to 4; all lanes in lockstep
      if (pos + 35 < full) ring_need(R, pos, pos + 35, lane);
      for (int it = 0; (it < 32 || (pos & 3)) && i >= 1; ++it) {
        const unsigned int v = ring_get(R, a, r0, pos) & smear((unsigned)i);
        ++pos;
        if ((int)v <= i) {
          if (lane == 0 && i >= k) J[i] = (int)v;
          --i;
        }
      }
    }
  }
  // drain outstanding bulk copies before the CTA exits
  for (int x = R.ready + 1; x < R.issued; ++x) mbar_wait(&bars[x % kRingChunks], (unsigned)((x / kRingChunks) & 1));
  // state after consuming `pos` draws
  if (lane == 0) {
    *a.rec_count = nrec;
    RngState r = r0;
    long long d = pos;
    if (r.has_uint32 && d > 0) {
      r.has_uint32 = 0;
      d -= 1;
    }
    if (d > 0) {
      const unsigned long long outs = (unsigned long long)((d + 1) / 2);
      const U128 st = pcg_jump(*a.jump, r0.s, outs);
      r.s = st;
      if (d & 1) {
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

// ----------------------------------------------------------- CTA parse
// Same contract as k_mask_parse, one CTA of kPT threads (launch <<<1, kPT>>>).
// A window of W <= kPW draws inside one mask band is classified in
// parallel: sure-accept (v <= i - r), sure-reject (v > i) or ambiguous.  A
// block scan gives every draw its number of sure accepts before it; the
// ambiguous draws form a short ordered list whose acceptance
// (A_before <= key, key = i - S_before(r) - v) warp 0 resolves with the same
// sure/unsure speculation one level down; then every accepted draw's step
// s = i - S_before(r) - A_before(r) is known and J[s] is written in parallel.
// W is capped near 8*sqrt(m) so the ambiguous list stays ~32 long.
constexpr int kPT = 512;
constexpr int kPD = 16;
constexpr int kPW = kPT * kPD;        // 8192
constexpr int kPChunk = 8192;          // draws per ring chunk (32 KiB)
constexpr int kPChunks = 4;
constexpr int kPRing = kPChunk * kPChunks;
constexpr int kParseSmem = kPRing * 4 + kPW * 4 + (kPW + 1) * 4 + 64;

__device__ __forceinline__ int block_excl_scan(int v, int* s_warp, int* s_total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int w = lane < (kPT / 32) ? s_warp[lane] : 0;
    int wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    if (lane < (kPT / 32)) s_warp[lane] = wi - w;
    if (lane == 31) *s_total = wi;
  }
  __syncthreads();
  return s_warp[warp] + incl - v;
}

__global__ void __launch_bounds__(kPT, 1) k_mask_parse_cta(ParseArgs a) {
  extern __shared__ __align__(16) unsigned char psm[];
  unsigned int* ring = reinterpret_cast<unsigned int*>(psm);
  int* akey = reinterpret_cast<int*>(ring + kPRing);
  int* apref = akey + kPW;
  __shared__ __align__(8) uint64_t bars[kPChunks];
  __shared__ int s_warp[32];
  __shared__ int s_tot, s_i, s_pos, s_acc;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned lt = (1u << lane) - 1u;
  const RngState r0 = *a.rng;
  const int n_chunks = (int)(a.n_draws / kPChunk);
  const int full = n_chunks * kPChunk;
  int issued = 0, ready = -1;
  if (tid == 0) {
    for (int c = 0; c < kPChunks; ++c) mbar_init(&bars[c], 1);
    fence_mbar_init();
  }
  __syncthreads();
  // all threads: make draws [.., hi] (< full) readable; chunks below chunk(pos) are consumed
  auto need = [&](int pos, int hi) {
    const int ch = hi / kPChunk;
    if (ch <= ready) return;
    const int upto = min(n_chunks, pos / kPChunk + kPChunks);
    if (tid == 0) {
      for (int x = issued; x < upto; ++x) {
        const int slot = x % kPChunks;
        mbar_expect_tx(&bars[slot], kPChunk * 4);
        tma_load_1d(ring + slot * kPChunk, a.draws + (size_t)x * kPChunk, kPChunk * 4, &bars[slot]);
      }
    }
    issued = max(issued, upto);
    for (int x = ready + 1; x <= ch; ++x) mbar_wait(&bars[x % kPChunks], (unsigned)((x / kPChunks) & 1));
    ready = ch;
  };
  auto get = [&](int idx) -> unsigned int {
    if (idx < full) return ring[idx % kPRing];
    return idx < a.n_draws ? __ldg(&a.draws[idx]) : draw_at(*a.jump, r0, idx);
  };
  int pos = 0;
  need(0, 0);
  for (int c = 0; c < 2; ++c) {
    const int n = a.n[c], k = a.k[c];
    int* J = a.J[c];
    int i = n - 1;
    while (i >= 1) {
      const unsigned int m = smear((unsigned)i);
      const int half = (int)(m >> 1);
      int W = min(kPW, i - half);
      W = min(W, max(1024, (int)(8.0f * sqrtf((float)m))));
      W = min(W, full - pos);
      long long tq0 = clock64();
      if (W >= 64) {
        need(pos, pos + W - 1);
        long long tq1 = clock64();
        // warp w owns draws [512w, 512w+512): row u, lane l -> r = 512w + 32u + l
        const int rw = warp * 512;
        unsigned sab[16], amb[16], v[16];
        int ws = 0, wq = 0;
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const int r = rw + u * 32 + lane;
          const bool in = r < W;
          v[u] = in ? (ring[(pos + r) & (kPRing - 1)] & m) : 0u;
          const bool acc = in && (int)v[u] <= i - r;
          const bool amg = in && !acc && (int)v[u] <= i;
          sab[u] = __ballot_sync(0xffffffffu, acc);
          amb[u] = __ballot_sync(0xffffffffu, amg);
          ws += __popc(sab[u]);
          wq += __popc(amb[u]);
        }
        long long tq2 = clock64();
        if (lane == 0) {
          s_warp[warp] = ws;
          s_warp[16 + warp] = wq;
        }
        __syncthreads();
        int S_w = 0, Q_w = 0, S_tot = 0, Q_tot = 0;
#pragma unroll
        for (int w2 = 0; w2 < 16; ++w2) {
          const int a1 = s_warp[w2], a2 = s_warp[16 + w2];
          if (w2 < warp) {
            S_w += a1;
            Q_w += a2;
          }
          S_tot += a1;
          Q_tot += a2;
        }
        long long tq3 = clock64();
        // ambiguous draws in order: key = i - S_before(r) - v
        {
          int sr = S_w, qr = Q_w;
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            if ((amb[u] >> lane) & 1u) akey[qr + __popc(amb[u] & lt)] = i - (sr + __popc(sab[u] & lt)) - (int)v[u];
            sr += __popc(sab[u]);
            qr += __popc(amb[u]);
          }
        }
        if (Q_tot > 0) __syncthreads();
        long long tq4 = clock64();
        if (Q_tot > 0 && warp == 0) {
          int A = 0;
          for (int base = 0; base < Q_tot; base += 32) {
            const int j = base + lane;
            const bool valid = j < Q_tot;
            const int key = valid ? akey[j] : 0;
            const bool sacc = valid && key >= A + lane;
            const bool srej = !valid || key < A;
            if (!__any_sync(0xffffffffu, !sacc && !srej)) {
              const unsigned bal = __ballot_sync(0xffffffffu, sacc);
              if (valid) apref[j] = A + __popc(bal & lt);
              A += __popc(bal);
            } else {
              for (int l = 0; l < 32 && base + l < Q_tot; ++l) {
                const int kl = __shfl_sync(0xffffffffu, key, l);
                if (lane == l) apref[base + l] = A;
                A += (kl >= A) ? 1 : 0;
              }
            }
          }
          if (lane == 0) {
            apref[Q_tot] = A;
            s_acc = A;
          }
        }
        if (Q_tot > 0) __syncthreads();
        const int acc_amb = Q_tot > 0 ? s_acc : 0;
        long long tq5 = clock64();
        // J of every accepted draw (consecutive lanes -> consecutive steps);
        // windows entirely below k only need their accept count
        if (i >= k) {
          int sr = S_w, qr = Q_w;
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            const bool sacc = (sab[u] >> lane) & 1u;
            const bool isamb = (amb[u] >> lane) & 1u;
            if (sacc || isamb) {
              const int q = qr + __popc(amb[u] & lt);
              const int ab = apref[q];
              if (sacc || apref[q + 1] - ab == 1) {
                const int st = i - (sr + __popc(sab[u] & lt)) - ab;
                if (st >= k) J[st] = (int)v[u];
              }
            }
            sr += __popc(sab[u]);
            qr += __popc(amb[u]);
          }
        }
        i -= S_tot + acc_amb;
        pos += W;
        __syncthreads();
        if (a.prof && tid == 0) {
          long long tq6 = clock64();
          a.prof[0] += tq1 - tq0; a.prof[1] += tq2 - tq1; a.prof[2] += tq3 - tq2; a.prof[3] += tq4 - tq3;
          a.prof[4] += tq5 - tq4; a.prof[5] += tq6 - tq5; a.prof[6] += 1;
        }
      } else {
        // short stretch (band bottom, small i, buffer tail): warp 0 walks up
        // to 512 draws with 32-draw windows / serially, then broadcasts
        if (pos < full) need(pos, min(full - 1, pos + 512 + 31));
        if (warp == 0) {
          const int stop = pos + 512;
          while (i >= 1 && pos < stop) {
            const unsigned int mm = smear((unsigned)i);
            const int hf = (int)(mm >> 1);
            if (i - 31 > hf) {
              const unsigned int vv = get(pos + lane) & mm;
              const bool acc = (int)vv <= i - lane;
              const bool amb = !acc && (int)vv <= i;
              const unsigned ambm = __ballot_sync(0xffffffffu, amb);
              const int ra = ambm ? __ffs(ambm) - 1 : 32;
              const unsigned ab = __ballot_sync(0xffffffffu, acc) & (ra >= 32 ? 0xffffffffu : ((1u << ra) - 1u));
              const int before = __popc(ab & lt);
              if (lane < ra && acc && i - before >= k) J[i - before] = (int)vv;
              i -= __popc(ab);
              if (ra < 32) {
                const unsigned int va = __shfl_sync(0xffffffffu, vv, ra);
                if ((int)va <= i) {
                  if (lane == 0 && i >= k) J[i] = (int)va;
                  --i;
                }
                pos += ra + 1;
              } else {
                pos += 32;
              }
            } else {
              const unsigned int vv = get(pos) & mm;
              ++pos;
              if ((int)vv <= i) {
                if (lane == 0 && i >= k) J[i] = (int)vv;
                --i;
              }
            }
          }
          if (lane == 0) {
            s_i = i;
            s_pos = pos;
          }
        }
        __syncthreads();
        i = s_i;
        pos = s_pos;
        __syncthreads();
        if (a.prof && tid == 0) a.prof[7] += clock64() - tq0;
      }
    }
  }
  for (int x = ready + 1; x < issued; ++x) mbar_wait(&bars[x % kPChunks], (unsigned)((x / kPChunks) & 1));
  if (tid == 0) {
    *a.rec_count = 0;
    RngState r = r0;
    long long d = pos;
    if (r.has_uint32 && d > 0) {
      r.has_uint32 = 0;
      d -= 1;
    }
    if (d > 0) {
      const unsigned long long outs = (unsigned long long)((d + 1) / 2);
      const U128 st = pcg_jump(*a.jump, r0.s, outs);
      r.s = st;
      if (d & 1) {
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

// Resolve an ordered list of ambiguous draws (one warp): entry j is accepted
// iff A_before(j) <= key[j], A_before = accepted entries before j; writes
// apref[j] = A_before(j) and apref[Q] = total.  128 entries per iteration:
// an entry is a sure reject if key < A, a sure accept if key >= A + (entries
// before it in the block that are not sure rejects); on the first unsure
// entry the decided prefix is committed and that entry resolved exactly.
__device__ __forceinline__ void resolve_list(const int* __restrict__ akey, int* __restrict__ apref, int Q, int lane) {
  const unsigned lt = (1u << lane) - 1u;
  int A = 0, base = 0;
  while (base < Q) {
    int key[4];
    bool nr[4];
    unsigned bn[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = base + u * 32 + lane;
      key[u] = j < Q ? akey[j] : 0;
      nr[u] = j < Q && key[u] >= A;  // not a sure reject
      bn[u] = __ballot_sync(0xffffffffu, nr[u]);
    }
    int pre = 0;
    unsigned unsure[4];
    int bnr[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      bnr[u] = pre + __popc(bn[u] & lt);  // non-rejects before this entry
      unsure[u] = __ballot_sync(0xffffffffu, nr[u] && key[u] < A + bnr[u]);
      pre += __popc(bn[u]);
    }
    int f = 128;  // first unsure entry (block-relative)
#pragma unroll
    for (int u = 3; u >= 0; --u)
      if (unsure[u]) f = u * 32 + __ffs(unsure[u]) - 1;
    // entries before f: every non-reject is accepted
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int jl = u * 32 + lane;
      if (jl < f && base + jl < Q) apref[base + jl] = A + bnr[u];
    }
    if (f == 128) {
      A += pre;
      base += 128;
    } else {
      // exact decision for entry f
      const int uf = f >> 5, lf = f & 31;
      const int kf = __shfl_sync(0xffffffffu, key[uf], lf);
      const int bf = __shfl_sync(0xffffffffu, bnr[uf], lf);
      const int Af = A + bf;
      if (lane == 0) apref[base + f] = Af;
      A = Af + (kf >= Af ? 1 : 0);
      base += f + 1;
    }
  }
  if (lane == 0) apref[Q] = A;
}

// ----------------------------------------------------------- cluster parse
// Same contract again, spread over a cluster of kCl CTAs (8 SMs): a window
// of W <= kCl * kPW draws inside one mask band; CTA r classifies draws
// [r*kPW, (r+1)*kPW) of the window with the interleaved row layout of
// k_mask_parse_cta, the per-CTA (sure-accept, ambiguous) counts and the
// ambiguous keys meet in CTA 0 through distributed shared memory, warp 0 of
// CTA 0 resolves the ambiguous list, every CTA copies back the slice of the
// accepted-ambiguous prefix it needs and writes its J values.  Slices of
// the next window are prefetched with cp.async while the current one is
// resolved.  Short stretches (band bottoms, small i, buffer tail) are walked
// by CTA 0 alone.
constexpr int kCl = 8;
constexpr int kClW = kCl * kPW;        // 65536
constexpr int kQcap = 12288;            // ambiguous-list capacity (expected ~W^2/2m <= ~2k)
constexpr int kSlice = kPW + 16;        // slice buffer stride (room for the alignment offset)
constexpr int kClSmem = 2 * kSlice * 4 + kQcap * 4 + (kQcap + 1) * 4 + 64;

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Cluster barrier: only the threads that published shared data to other
// CTAs (DSMEM stores, or smem that other CTAs will read) pay the release
// fence (MEMBAR); everyone else arrives relaxed and waits with acquire.
__device__ __forceinline__ void csync(bool publish) {
  if (publish) asm volatile("fence.acq_rel.cluster;" ::: "memory");
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}

#define BB_PMARK(slot, t0)                                             \
  do {                                                                  \
    if (a.prof && crank == 0 && tid == 0) a.prof[slot] += clock64() - (t0); \
  } while (0)
__global__ void __cluster_dims__(kCl, 1, 1) __launch_bounds__(kPT, 1) k_mask_parse_cl(ParseArgs a) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ __align__(16) unsigned char csm[];
  unsigned int* buf0 = reinterpret_cast<unsigned int*>(csm);  // [2][kSlice] this CTA's slices
  int* akey = reinterpret_cast<int*>(buf0 + 2 * kSlice);       // CTA 0: ambiguous keys in draw order
  int* apref = akey + kQcap;                                    // CTA 0: accepted-ambiguous prefix
  __shared__ int s_warp[64];
  __shared__ int s_cnt[8 * kCl];   // CTA 0: per-CTA (sure, amb) counts (2 banks), accepted counts
  __shared__ int s_state[4];       // broadcast: i, pos, cross position
  __shared__ int s_loc[2 * kCl];    // local copy of the last exchanged counters
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned lt = (1u << lane) - 1u;
  const int crank = (int)cl.block_rank();
  const RngState r0 = *a.rng;
  const long long nd = a.n_draws;
  int* apref0 = cl.map_shared_rank(apref, 0);
  int* akey0 = cl.map_shared_rank(akey, 0);
  int* cnt0 = cl.map_shared_rank(s_cnt, 0);
  int* state0 = cl.map_shared_rank(s_state, 0);
  int cur = 0, loaded_at = -1;
  int boff[2] = {0, 0};
  if (crank == 0 && tid == 0) {
    s_state[1] = 0;
    s_state[2] = 1 << 30;  // crossing draw (min over CTAs)
    s_state[3] = 1 << 30;  // first overflowing ambiguous draw
  }
  csync(crank == 0 && tid == 0);
  auto load_slice = [&](int bsel, int wstart) {
    const long long base = (long long)wstart + (long long)crank * kPW;
    const long long abase = base & ~3ll;
    boff[bsel] = (int)(base - abase);
    unsigned int* dst = buf0 + bsel * kSlice;
    for (int j = tid; j < (kPW + 4) / 4; j += kPT) {
      const long long src = abase + 4ll * j;
      if (src + 4 <= nd) cp_async16(dst + 4 * j, a.draws + src);
    }
    cp_async_commit();
  };
  auto get = [&](long long idx) -> unsigned int {
    return idx < nd ? __ldg(&a.draws[idx]) : draw_at(*a.jump, r0, idx);
  };
  // after a cluster sync: copy cnt0[bank .. bank + cnt) into s_loc once (few
  // DSMEM loads) instead of every thread reading CTA 0's counters remotely
  auto fetch = [&](int bank, int cnt) {
    if (tid < cnt) s_loc[tid] = cnt0[bank + tid];
    __syncthreads();
  };
  int pos = 0;
  for (int tc = 0; tc < 2 * a.n_trees; ++tc) {
    const int c = tc & 1;
    const int n = a.n[c], k = a.k[c];
    int* J = a.J[c] + (long long)(tc >> 1) * a.J_stride;
    int i = n - 1;
    while (i >= 1) {
      const unsigned int m0 = smear((unsigned)i);
      // ambiguity is refined away below, so windows need no sqrt(m) cap; stop
      // near the expected band crossing (~d/p draws, p >= 1/2) to limit the
      // junk tail a crossing leaves for the next round
      int W = kClW;
      (void)m0;
      if ((long long)pos + W > nd) W = (int)max(0ll, nd - pos);
      if (i >= 64 && W >= 4096) {
        // ---- one window [pos, pos+W), processed in rounds; a round ends
        // where the band's last step is taken (mask changes) or at the
        // window end
        const long long tw0 = clock64();
        if (loaded_at != pos) {
          load_slice(cur, pos);
          loaded_at = pos;
        }
        cp_async_wait_all();
        __syncthreads();
        if (a.prof && crank == 0 && tid == 0) a.prof[13] += clock64() - tw0;  // slice wait
        load_slice(cur ^ 1, pos + W);  // prefetch (valid if the window is fully consumed)
        const unsigned int* sl = buf0 + cur * kSlice + boff[cur];
        const int rw = warp * 512, rbase = crank * kPW;
        int rs = 0;           // round start (window-relative)
        bool perm_done = false;
        while (rs < W && i >= 1) {
          const long long tR = clock64();
          const unsigned int m = smear((unsigned)i);
          const int half = (int)(m >> 1);
          const int d = i - half;  // acceptances until the band's last step
          unsigned sab[16], amb[16];
          int ws = 0, wq = 0;
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            const int rl = rw + u * 32 + lane;
            const int r = rbase + rl;
            const bool in = r >= rs && r < W;
            const unsigned int v = in ? (sl[rl] & m) : 0u;
            const int off = r - rs;
            const bool acc = in && (int)v <= i - off;
            const bool amg = in && !acc && (int)v <= i;
            sab[u] = __ballot_sync(0xffffffffu, acc);
            amb[u] = __ballot_sync(0xffffffffu, amg);
            ws += __popc(sab[u]);
            wq += __popc(amb[u]);
          }
          if (lane == 0) {
            s_warp[warp] = ws;
            s_warp[16 + warp] = wq;
          }
          __syncthreads();
          int S_w = 0, Q_w = 0, S_c = 0, Q_c = 0;
#pragma unroll
          for (int w2 = 0; w2 < 16; ++w2) {
            const int x1 = s_warp[w2], x2 = s_warp[16 + w2];
            if (w2 < warp) {
              S_w += x1;
              Q_w += x2;
            }
            S_c += x1;
            Q_c += x2;
          }
          if (tid == 0) {
            cnt0[2 * crank] = S_c;
            cnt0[2 * crank + 1] = Q_c;
          }
          long long tr1 = clock64();
          BB_PMARK(8, tR);  // classify (+warp totals)
          csync(tid == 0);  // (1) counts published by thread 0

          fetch(0, 2 * kCl);
          int S_before = 0, Q_before = 0, Q_tot = 0;
#pragma unroll
          for (int q = 0; q < kCl; ++q) {
            const int x1 = s_loc[2 * q], x2 = s_loc[2 * q + 1];
            if (q < crank) {
              S_before += x1;
              Q_before += x2;
            }
            Q_tot += x2;
          }
          int s_bank = 0;
          if (a.prof && crank == 0 && tid == 0) a.prof[4] += Q_tot;  // Q before refinement
          // refinement: accepted-before(r) lies in [S_before(r), S_before(r) + U_before(r)]
          // (sure accepts, still-ambiguous draws before r) -> re-test the
          // ambiguous draws against those bounds (Jacobi: counts of the
          // previous pass), exchange counts, repeat
          for (int pass = 0; pass < 8 && Q_tot > 768; ++pass) {
            int sr = S_before + S_w, qr = Q_before + Q_w;
            int ws2 = 0, wq2 = 0;
#pragma unroll
            for (int u = 0; u < 16; ++u) {
              const unsigned sa0 = sab[u], am0 = amb[u];
              bool na = false, nrj = false;
              if ((am0 >> lane) & 1u) {
                const int rl = rw + u * 32 + lane;
                const int v = (int)(sl[rl] & m);
                const int Sb = sr + __popc(sa0 & lt);
                const int Ub = qr + __popc(am0 & lt);
                na = v <= i - Sb - Ub;
                // Sb >= d: the band's last step was taken before this draw, so
                // it belongs to the next round (re-classified under the next
                // mask) -> drop it from this round's list
                nrj = v > i - Sb || Sb >= d;
                if (Sb >= d) na = false;
              }
              const unsigned ba = __ballot_sync(0xffffffffu, na);
              const unsigned br = __ballot_sync(0xffffffffu, nrj);
              sab[u] = sa0 | ba;
              amb[u] = am0 & ~(ba | br);
              sr += __popc(sa0);
              qr += __popc(am0);
              ws2 += __popc(sab[u]);
              wq2 += __popc(amb[u]);
            }
            __syncthreads();  // everyone has read s_warp of the previous exchange
            if (lane == 0) {
              s_warp[warp] = ws2;
              s_warp[16 + warp] = wq2;
            }
            __syncthreads();
            S_w = 0;
            Q_w = 0;
            S_c = 0;
            Q_c = 0;
#pragma unroll
            for (int w2 = 0; w2 < 16; ++w2) {
              const int x1 = s_warp[w2], x2 = s_warp[16 + w2];
              if (w2 < warp) {
                S_w += x1;
                Q_w += x2;
              }
              S_c += x1;
              Q_c += x2;
            }
            const int bank = 2 * kCl * ((pass + 1) & 1);
            if (tid == 0) {
              cnt0[bank + 2 * crank] = S_c;
              cnt0[bank + 2 * crank + 1] = Q_c;
            }
            csync(tid == 0);
            fetch(bank, 2 * kCl);
            S_before = 0;
            Q_before = 0;
            Q_tot = 0;
#pragma unroll
            for (int q = 0; q < kCl; ++q) {
              const int x1 = s_loc[2 * q], x2 = s_loc[2 * q + 1];
              if (q < crank) {
                S_before += x1;
                Q_before += x2;
              }
              Q_tot += x2;
            }
            s_bank = bank;
            if (a.prof && crank == 0 && tid == 0) {
              a.prof[15] += 1;
              if (pass < 3) a.prof[5 + pass] += Q_tot;
            }
          }
          const int Qres = min(Q_tot, kQcap);  // entries beyond the cap: resolved serially below
          bool wrote_keys = false;
          {
            int sr = S_before + S_w, qr = Q_before + Q_w;
#pragma unroll
            for (int u = 0; u < 16; ++u) {
              if ((amb[u] >> lane) & 1u) {
                const int q = qr + __popc(amb[u] & lt);
                const int rl = rw + u * 32 + lane;
                if (q < kQcap) {
                  akey0[q] = i - (sr + __popc(sab[u] & lt)) - (int)(sl[rl] & m);
                  wrote_keys = true;
                }
              }
              sr += __popc(sab[u]);
              qr += __popc(amb[u]);
            }
          }
          const long long tK = clock64();
          csync(wrote_keys);  // (2)
          BB_PMARK(9, tK);  // sync 2
          const long long tS = clock64();
          if (crank == 0) {
            // warps 1.. of CTA 0 sleep on the CTA barrier (not the cluster
            // barrier) while warp 0 resolves, leaving it the issue slots
            if (warp == 0) {
              if (a.prof && lane == 0) a.prof[14] += Qres;
              resolve_list(akey, apref, Qres, lane);
            }
            __syncthreads();
          }
          long long tr3 = clock64();
          BB_PMARK(10, tS);  // resolve
          csync(crank == 0 && warp == 0);  // (3) apref published by CTA 0 warp 0

          // S_tot from this CTA's view: S_before + own + after (all banks agree
          // only per pass, so recompute from the last exchange's bank)
          int S_tot = S_before + S_c;
          for (int q = crank + 1; q < kCl; ++q) S_tot += s_loc[2 * q];  // s_loc holds bank s_bank
          (void)s_bank;
          const int A_amb = apref0[Qres];
          BB_PMARK(13, tr3);  // sync3 + totals
          // local copy of the accepted-ambiguous prefix slice this CTA needs
          // (CTA r != 0 reuses its own, otherwise idle, apref array)
          int* apl = (crank == 0) ? apref + Q_before : akey;
          const int ncopy = min(Q_c, max(0, Qres - Q_before)) + 1;
          if (crank != 0)
            for (int q = tid; q < ncopy; q += kPT) apl[q] = apref0[min(Q_before + q, Qres)];
          __syncthreads();
          auto APF = [&](int qg) -> int {  // accepted-ambiguous before global entry qg (qg <= Qres)
            const int ql = qg - Q_before;
            return (ql >= 0 && ql < ncopy) ? apl[ql] : apref0[min(qg, Qres)];
          };
          const long long tC = clock64();
          if (Q_tot <= kQcap && S_tot + A_amb < d) {
            // common case: no band crossing in the rest of the window, every
            // draw decided -> commit all (J only needed for steps >= k)
            if (i >= k) {
              int sr = S_before + S_w, qr = Q_before + Q_w;
#pragma unroll
              for (int u = 0; u < 16; ++u) {
                const bool sacc = (sab[u] >> lane) & 1u;
                const bool isamb = (amb[u] >> lane) & 1u;
                if (sacc || isamb) {
                  const int q = qr + __popc(amb[u] & lt);
                  const int ab = APF(q);
                  if (sacc || APF(q + 1) - ab == 1) {
                    const int st = i - (sr + __popc(sab[u] & lt)) - ab;
                    if (st >= k) J[st] = (int)(sl[rw + u * 32 + lane] & m);
                  }
                }
                sr += __popc(sab[u]);
                qr += __popc(amb[u]);
              }
            }
            i -= S_tot + A_amb;
            rs = W;
            BB_PMARK(11, tC);  // common commit
            csync(false);  // (4') CTA 0 list / counters free (reads only)
            if (a.prof && crank == 0 && tid == 0) a.prof[2] += 1;
            break;
          }
          // ---- detailed path: a band crossing (or list overflow) in this round
          if (a.prof && crank == 0 && tid == 0) a.prof[3] += 1;
          const long long tD = clock64();
          unsigned accm[16];
          int wa = 0;
          {
            int qr = Q_before + Q_w;
#pragma unroll
            for (int u = 0; u < 16; ++u) {
              unsigned am_acc = 0;
              if ((amb[u] >> lane) & 1u) {
                const int q = qr + __popc(amb[u] & lt);
                const bool ok = q < Qres && APF(q + 1) - APF(q) == 1;
                am_acc = ok ? 1u : 0u;
              }
              accm[u] = sab[u] | __ballot_sync(0xffffffffu, am_acc);
              wa += __popc(accm[u]);
              qr += __popc(amb[u]);
            }
          }
          // first draw of the window that overflowed the ambiguous list
          int rcut = W;
          if (Q_tot > kQcap) {  // state0[3] holds 1<<30 until set here
            int qr = Q_before + Q_w, first = W;
#pragma unroll
            for (int u = 0; u < 16; ++u) {
              if ((amb[u] >> lane) & 1u) {
                const int q = qr + __popc(amb[u] & lt);
                if (q == kQcap) first = rbase + rw + u * 32 + lane;
              }
              qr += __popc(amb[u]);
            }
            first = __reduce_min_sync(0xffffffffu, first);
            if (lane == 0) s_warp[32 + warp] = first;
            __syncthreads();
            if (tid == 0) {
              int f = W;
              for (int w2 = 0; w2 < 16; ++w2) f = min(f, s_warp[32 + w2]);
              atomicMin(&state0[3], f);  // CTA 0's state[3] initialised to W below
            }
          }
          if (lane == 0) s_warp[48 + warp] = wa;
          __syncthreads();
          int A_w = 0, A_c = 0;
#pragma unroll
          for (int w2 = 0; w2 < 16; ++w2) {
            const int x = s_warp[48 + w2];
            if (w2 < warp) A_w += x;
            A_c += x;
          }
          if (tid == 0) cnt0[4 * kCl + crank] = A_c;
          csync(tid == 0 || (Q_tot > kQcap && lane == 0));  // (4)
          if (Q_tot > kQcap) rcut = min(W, state0[3]);
          fetch(4 * kCl, kCl);
          int A_before = 0, A_tot = 0;
#pragma unroll
          for (int q = 0; q < kCl; ++q) {
            const int x = s_loc[q];
            if (q < crank) A_before += x;
            A_tot += x;
          }
          // crossing: the d-th acceptance (band's last step) ends the round
          int rend = rcut;  // exclusive end of committed draws
          bool crossed = false;
          if (A_tot >= d) {
            // find the draw with accepted prefix count == d (1-based)
            int found = W;
            if (A_before < d && d <= A_before + A_c) {
              int run = A_before + A_w;
#pragma unroll
              for (int u = 0; u < 16; ++u) {
                const bool acc = (accm[u] >> lane) & 1u;
                const int cnt_incl = run + __popc(accm[u] & lt) + (acc ? 1 : 0);
                if (acc && cnt_incl == d) found = rbase + rw + u * 32 + lane;
                run += __popc(accm[u]);
              }
              found = __reduce_min_sync(0xffffffffu, found);
              if (lane == 0 && found < W) atomicMin(&state0[2], found);
            }
            csync(lane == 0);  // (5)
            const int rx = state0[2];
            if (rx + 1 < rend) {
              rend = rx + 1;
              crossed = true;
            } else if (rx + 1 == rend) {
              crossed = true;
            }
          }
          // overflow cut: draws at/after rcut are undecided -> round ends there
          // (the cut draw itself is resolved serially by CTA 0 below)
          // commit J for accepted draws in [rs, rend)
          int committed_acc = 0;
          {
            int run = A_before + A_w;  // accepted before this lane's row-0 draw, within the round
            int qr = Q_before + Q_w;
#pragma unroll
            for (int u = 0; u < 16; ++u) {
              const int r = rbase + rw + u * 32 + lane;
              const bool acc = (accm[u] >> lane) & 1u;
              const int before = run + __popc(accm[u] & lt);
              if (acc && r < rend) {
                const int st = i - before;
                if (st >= k) J[st] = (int)(sl[rw + u * 32 + lane] & m);
              }
              run += __popc(accm[u]);
              qr += __popc(amb[u]);
            }
            (void)qr;
          }
          // accepted count within [rs, rend): d if crossed, else all decided accepts before rend
          if (crossed) {
            committed_acc = d;
          } else if (rend == W) {
            committed_acc = A_tot;
          } else {
            // overflow cut without crossing: count accepts before rcut (cluster reduce)
            int cnt = 0;
            int run = 0;
#pragma unroll
            for (int u = 0; u < 16; ++u) {
              const int r = rbase + rw + u * 32 + lane;
              if (((accm[u] >> lane) & 1u) && r < rend) ++cnt;
              run += 0;
            }
            cnt = __reduce_add_sync(0xffffffffu, cnt);
            if (lane == 0) atomicAdd(&state0[1], cnt);
            csync(lane == 0);
            committed_acc = state0[1];
          }
          csync(false);  // (6) everyone has read state0 / cnt0
          if (crank == 0 && tid == 0) {
            state0[1] = 0;
            state0[2] = 1 << 30;
            state0[3] = 1 << 30;
          }
          i -= committed_acc;
          rs = rend;
          if (!crossed && rend < W) {
            // overflow cut: CTA 0 resolves the cut draw serially, then the round restarts after it
            if (crank == 0 && tid == 0) {
              const unsigned int v = get((long long)pos + rend) & smear((unsigned)i);
              int ii = i;
              if ((int)v <= ii) {
                if (ii >= k) J[ii] = (int)v;
                --ii;
              }
              for (int q = 0; q < kCl; ++q) cl.map_shared_rank(s_state, q)[0] = ii;
            }
            csync(crank == 0 && tid == 0);
            i = s_state[0];
            rs = rend + 1;
            csync(false);
          }
          BB_PMARK(12, tD);  // detailed path
          if (i == 0) {
            perm_done = true;
            break;
          }
        }
        if (a.prof && crank == 0 && tid == 0) {
          a.prof[0] += clock64() - tw0;
          a.prof[1] += 1;
          a.prof[4] += rs;
        }
        pos += rs;
        cur ^= 1;
        loaded_at = (rs == W) ? pos : -1;  // prefetch valid only if the whole window was consumed
        (void)perm_done;
      } else {
        // short stretch (i < 64, or the buffer tail): CTA 0 stages draws in
        // smem, warp 0 walks them serially, then broadcasts i and pos
        constexpr int kSt = 4096;
        const long long ts0 = clock64();
        cp_async_wait_all();
        __syncthreads();
        loaded_at = -1;
        if (crank == 0) {
          unsigned int* stg = buf0;
          for (int j = tid; j < kSt + 64; j += kPT) {
            const long long idx = (long long)pos + j;
            stg[j] = idx < nd ? __ldg(&a.draws[idx]) : 0u;
          }
          __syncthreads();
          if (warp == 0) {
            const int pos0 = pos;
            const int stop = pos + kSt;
            while (i >= 1 && pos < stop) {
              const int o = pos - pos0;
              const unsigned int vv = ((long long)pos < nd ? stg[o] : get((long long)pos)) & smear((unsigned)i);
              ++pos;
              if ((int)vv <= i) {
                if (lane == 0 && i >= k) J[i] = (int)vv;
                --i;
              }
            }
            if (lane == 0)
              for (int q = 0; q < kCl; ++q) {
                int* st = cl.map_shared_rank(s_state, q);
                st[0] = i;
                st[1] = pos;
              }
          }
          __syncthreads();
        }
        csync(crank == 0 && tid == 0);
        i = s_state[0];
        pos = s_state[1];
        csync(false);
        if (crank == 0 && tid == 0) {
          s_state[1] = 0;
          s_state[2] = 1 << 30;
          s_state[3] = 1 << 30;
          if (a.prof) {
            a.prof[5] += clock64() - ts0;
            a.prof[6] += 1;
          }
        }
        csync(crank == 0 && tid == 0);
      }
    }
  }
  cp_async_wait_all();
  if (crank == 0 && tid == 0) {
    *a.rec_count = 0;
    RngState r = r0;
    long long dd = pos;
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

// J values of the fast windows: one warp per record; draw r of the window is
// accepted iff its bit is set, its step is i - (accepted draws before r).
__global__ void k_expand_windows(ParseArgs a) {
  const int lane = threadIdx.x & 31;
  const int nrec = min(*a.rec_count, a.rec_cap);
  for (int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < nrec; w += (gridDim.x * blockDim.x) >> 5) {
    const int pos = a.rec_pos[w], len = a.rec_len[w];
    const int ic = a.rec_i[w];
    const int c = (ic >> 31) & 1, i = ic & 0x7fffffff;
    const unsigned int m = smear((unsigned)i);
    const unsigned accb = a.rec_bits[(size_t)w * 32 + lane];
    const int cnt = __popc(accb);
    int incl = cnt;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    int s = i - (incl - cnt);
    const int k = a.k[c];
    int* J = a.J[c];
    for (int u = 0; u < 8; ++u) {
      const int r = lane * 8 + u;
      if (r < len && ((accb >> u) & 1u)) {
        if (s >= k) J[s] = (int)(a.draws[pos + r] & m);
        --s;
      }
    }
  }
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

__global__ void k_scan_apply(const int* __restrict__ in, int n, const int* __restrict__ sums, int* __restrict__ out) {
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
    if (i < n) out[i] = run;
    run += v[j];
  }
}

}  // namespace bb
