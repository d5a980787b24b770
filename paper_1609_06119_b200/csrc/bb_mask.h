// Host restatement of numpy's PCG64 + Fisher-Yates permutation (see bb_mask.cpp).
#pragma once
#include <cstdint>
#include <vector>

namespace bb {

struct Pcg64 {
  unsigned __int128 state;
  unsigned __int128 inc;
  int has_uint32;
  uint32_t uinteger;
  uint64_t next64();
  uint32_t next32();
  uint64_t interval(uint64_t max);
};

int64_t subsample_count(int64_t n, double rate);
// active bits of one class block at bit offset bit_off
void subsample_block(Pcg64& g, int64_t n, double rate, uint32_t* bits, int64_t bit_off, std::vector<uint32_t>& perm);
// signal block then background block (sample.py:126-132); clears bits first
void subsample_tree(Pcg64& g, int64_t n_sig, int64_t n_bkg, double rate, uint32_t* bits, std::vector<uint32_t>& perm);

}  // namespace bb
