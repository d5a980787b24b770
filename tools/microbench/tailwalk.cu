// Tail walk in isolation: cycles for lean_walk and warp_walk from state i0
// to 0 over random draws in shared memory (one warp, nothing co-resident
// unless --busy launches a compute-heavy grid on the other SMs and this one).
#include <cstdio>
#include <cstdlib>
#include "../../paper_1609_06119_b200/csrc/kernels_seg.cuh"
using namespace bb;
namespace bb { void set_error(const std::string&) {} }

__global__ void k_tail(const unsigned* draws, int len, int i0, int lean, long long* out) {
  __shared__ unsigned sd[kSegMaxLen + 16];
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
__global__ void k_busy(float* x, int iters) {
  float a = x[threadIdx.x], b = 1.0001f;
  for (int k = 0; k < iters; ++k) { a = a * b + 0.5f; b = b * a - 0.25f; }
  x[threadIdx.x] = a + b;
}
int main(int argc, char** argv) {
  const int len = 8192;
  unsigned* h = (unsigned*)malloc(len * 4);
  unsigned s = 12345;
  for (int j = 0; j < len; ++j) { s = s * 1664525u + 1013904223u; h[j] = s ^ (s >> 13); }
  unsigned* d; long long* o; float* bx;
  cudaMalloc(&d, len * 4); cudaMalloc(&o, 64); cudaMalloc(&bx, 4096 * 4); cudaMemset(bx, 0, 4096 * 4);
  cudaMemcpy(d, h, len * 4, cudaMemcpyHostToDevice);
  cudaStream_t s1, s2; cudaStreamCreate(&s1); cudaStreamCreate(&s2);
  for (int busy = 0; busy < 2; ++busy)
    for (int lean = 0; lean < 2; ++lean) {
      for (int rep = 0; rep < 2; ++rep) {
        if (busy) k_busy<<<148 * 4, 256, 0, s2>>>(bx, 2000000);
        k_tail<<<1, 32, 0, s1>>>(d, len, 4095, lean, o);
        cudaDeviceSynchronize();
      }
      long long r[3]; cudaMemcpy(r, o, 24, cudaMemcpyDeviceToHost);
      printf("busy=%d lean=%d: %lld cycles, %lld draws, end state %lld  (%.1f cyc/draw)\n", busy, lean, r[0], r[1], r[2], (double)r[0] / r[1]);
    }
  return 0;
}
