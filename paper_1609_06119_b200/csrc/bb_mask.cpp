// Exact restatement of the reference's stratified subsample (sample.py:120-132):
// per tree, signal block then background block, active = first floor(rate*n)
// entries of numpy Generator(PCG64(seed)).permutation(n).
//
// numpy's algorithm (numpy/random, not vendored in the reference; pinned to
// the container's numpy 2.3.5):
//   permutation(n) = arange(n) shuffled by Fisher-Yates, i = n-1 .. 1:
//     j = random_interval(i)  (smallest 2^k-1 mask >= i; draw & mask until <= i;
//                              32-bit draws while i <= 0xffffffff)
//     swap(a[i], a[j])
//   32-bit draws are the low then the high half of one PCG64 64-bit output;
//   the spare half persists across calls (state has_uint32 / uinteger).
//   PCG64 = 128-bit LCG stepped before an XSL-RR output.
// Steps i < k permute positions [0, k) among themselves, so only their draws
// matter for the active SET; swaps are done for i >= k only.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

#include "bb_mask.h"

namespace bb {

static const unsigned __int128 kPcgMult =
    ((unsigned __int128)0x2360ED051FC65DA4ull << 64) | (unsigned __int128)0x4385DF649FCCF645ull;

uint64_t Pcg64::next64() {
  state = state * kPcgMult + inc;
  const uint64_t hi = (uint64_t)(state >> 64), lo = (uint64_t)state;
  const unsigned rot = (unsigned)(state >> 122);
  const uint64_t x = hi ^ lo;
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

uint32_t Pcg64::next32() {
  if (has_uint32) {
    has_uint32 = 0;
    return uinteger;
  }
  const uint64_t v = next64();
  has_uint32 = 1;
  uinteger = (uint32_t)(v >> 32);
  return (uint32_t)v;
}

uint64_t Pcg64::interval(uint64_t max) {
  if (max == 0) return 0;
  uint64_t mask = max;
  mask |= mask >> 1;
  mask |= mask >> 2;
  mask |= mask >> 4;
  mask |= mask >> 8;
  mask |= mask >> 16;
  mask |= mask >> 32;
  if (max <= 0xffffffffull) {
    uint32_t v;
    const uint32_t m32 = (uint32_t)mask;
    while ((v = (next32() & m32)) > max) {
    }
    return v;
  }
  uint64_t v;
  while ((v = (next64() & mask)) > max) {
  }
  return v;
}

int64_t subsample_count(int64_t n, double rate) { return (int64_t)std::floor(rate * (double)n); }

void subsample_block(Pcg64& g, int64_t n, double rate, uint32_t* bits, int64_t bit_off, std::vector<uint32_t>& perm) {
  const int64_t k = subsample_count(n, rate);
  if (n <= 0) return;
  perm.resize((size_t)n);
  for (int64_t i = 0; i < n; ++i) perm[(size_t)i] = (uint32_t)i;
  for (int64_t i = n - 1; i >= 1; --i) {
    const uint64_t j = g.interval((uint64_t)i);
    if (i >= k) {
      const uint32_t t = perm[(size_t)i];
      perm[(size_t)i] = perm[(size_t)j];
      perm[(size_t)j] = t;
    }
  }
  for (int64_t p = 0; p < k; ++p) {
    const int64_t b = bit_off + perm[(size_t)p];
    bits[b >> 5] |= 1u << (b & 31);
  }
}

void subsample_tree(Pcg64& g, int64_t n_sig, int64_t n_bkg, double rate, uint32_t* bits,
                    std::vector<uint32_t>& perm) {
  const int64_t n = n_sig + n_bkg;
  std::memset(bits, 0, (size_t)((n + 31) / 32) * 4);
  subsample_block(g, n_sig, rate, bits, 0, perm);
  subsample_block(g, n_bkg, rate, bits, n_sig, perm);
}

}  // namespace bb
