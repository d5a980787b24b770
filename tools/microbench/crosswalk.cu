// Crossing-zone re-walk in isolation: cycles of lean_walk and warp_walk over
// `len` random draws from state i0 (a band boundary inside the walk).
#include <cstdio>
#include <cstdlib>
#include "../../paper_1609_06119_b200/csrc/kernels_seg.cuh"
using namespace bb;
namespace bb { void set_error(const std::string&) {} }
__global__ void k(const unsigned* draws, int len, int i0, int lean, long long* out) {
  __shared__ unsigned sd[8192 + 16];
  const int lane = threadIdx.x;
  for (int j = lane; j < len; j += 32) sd[j] = draws[j];
  __syncwarp();
  const long long c0 = clock64();
  int used;
  const int i = lean ? lean_walk(sd, len, i0, 1 << 30, nullptr, lane, &used)
                     : warp_walk<false>(sd, len, i0, 1 << 30, nullptr, lane, &used);
  const long long c1 = clock64();
  if (lane == 0) { out[0] = c1 - c0; out[1] = used; out[2] = i; }
}
int main() {
  const int len = 8192;
  unsigned* h = (unsigned*)malloc(len * 4); unsigned s = 777;
  for (int j = 0; j < len; ++j) { s = s * 1664525u + 1013904223u; h[j] = s ^ (s >> 13); }
  unsigned* d; long long* o; cudaMalloc(&d, len * 4); cudaMalloc(&o, 64); cudaMemcpy(d, h, len * 4, cudaMemcpyHostToDevice);
  for (int i0 : {(1 << 19) + 300, (1 << 19) - 3000, (1 << 16) + 300, (1 << 13) + 200})
    for (int L : {1024, 8192})
      for (int lean = 0; lean < 2; ++lean) {
        k<<<1, 32>>>(d, L, i0, lean, o); cudaDeviceSynchronize();
        k<<<1, 32>>>(d, L, i0, lean, o); cudaDeviceSynchronize();
        long long r[3]; cudaMemcpy(r, o, 24, cudaMemcpyDeviceToHost);
        printf("i0=%d len=%d lean=%d: %lld cycles (%.1f/draw), end %lld\n", i0, L, lean, r[0], (double)r[0] / r[1], r[2]);
      }
  return 0;
}
