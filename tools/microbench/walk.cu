// Microbenchmark of the single-warp exact walk (kernels_seg.cuh warp_walk):
// cycles per 512-draw chunk for a path in a given band, draws from smem.
#include <cstdio>
#include <cstdlib>
#include "../../paper_1609_06119_b200/csrc/kernels_seg.cuh"
using namespace bb;

__global__ void k_walk(const unsigned* draws, int len, int i0, long long* out) {
  __shared__ unsigned sd[kSegMaxLen + 16];
  const int lane = threadIdx.x;
  for (int j = lane; j < len; j += 32) sd[j] = draws[j];
  __syncwarp();
  const long long c0 = clock64();
  int used;
  const int i = warp_walk<false>(sd, len, i0, 1 << 30, nullptr, lane, &used);
  const long long c1 = clock64();
  if (lane == 0) {
    out[0] = c1 - c0;
    out[1] = used;
    out[2] = i;
  }
}

int main() {
  const int len = 4096;
  unsigned* h = (unsigned*)malloc(len * 4);
  unsigned s = 12345;
  for (int j = 0; j < len; ++j) { s = s * 1664525u + 1013904223u; h[j] = s ^ (s >> 13); }
  unsigned* d;
  long long* o;
  cudaMalloc(&d, len * 4);
  cudaMalloc(&o, 64);
  cudaMemcpy(d, h, len * 4, cudaMemcpyHostToDevice);
  int starts[] = {500000, 300000, 150000, 70000, 30000, 12000, 6000, 3000, 1500, 700};
  for (int st : starts) {
    for (int rep = 0; rep < 2; ++rep) {
      k_walk<<<1, 32>>>(d, len, st, o);
      long long r[3];
      cudaMemcpy(r, o, 24, cudaMemcpyDeviceToHost);
      if (rep) printf("start %7d: %lld cycles for %lld draws (%.1f cyc/draw, %.0f cyc per 512), end state %lld\n", st, r[0],
                      r[1], (double)r[0] / r[1], 512.0 * r[0] / r[1], r[2]);
    }
  }
  return 0;
}
