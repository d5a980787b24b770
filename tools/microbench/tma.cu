// TMA 1-D bulk copy latency/throughput vs plain loads, one CTA (one warp).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_1609_06119_b200/csrc/common.cuh"
using namespace bb;
namespace bb { void set_error(const std::string&) {} }

// sequentially stream `chunks` chunks of 16 KiB through an 8-slot ring (like k_mask_parse)
__global__ void k_tma_stream(const unsigned* src, int chunks, unsigned long long* out, int depth) {
  extern __shared__ __align__(16) unsigned ring[];
  __shared__ __align__(8) uint64_t bars[8];
  const int lane = threadIdx.x;
  if (lane == 0) { for (int c = 0; c < 8; ++c) mbar_init(&bars[c], 1); fence_mbar_init(); }
  __syncwarp();
  unsigned long long t0 = clock64();
  int issued = 0; unsigned acc = 0;
  for (int c = 0; c < chunks; ++c) {
    int upto = min(chunks, c + depth);
    if (lane == 0) for (int x = issued; x < upto; ++x) { int s = x % 8; mbar_expect_tx(&bars[s], 16384); tma_load_1d(ring + s * 4096, src + (size_t)x * 4096, 16384, &bars[s]); }
    issued = upto;
    mbar_wait(&bars[c % 8], (c / 8) & 1);
    acc += ring[(c % 8) * 4096 + lane];
    __syncwarp();
  }
  unsigned long long t1 = clock64();
  if (lane == 0) { out[0] = t1 - t0; out[1] = acc; }
}
__global__ void k_ldg_stream(const uint4* src, int chunks, unsigned long long* out) {
  unsigned long long t0 = clock64(); unsigned acc = 0;
  for (int c = 0; c < chunks; ++c) {
    const uint4* p = src + (size_t)c * 1024;
    #pragma unroll 8
    for (int j = threadIdx.x; j < 1024; j += 32) { uint4 v = __ldg(p + j); acc += v.x ^ v.w; }
  }
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = acc; }
}
int main() {
  const int chunks = 400; unsigned* src; cudaMalloc(&src, (size_t)chunks * 16384); cudaMemset(src, 1, (size_t)chunks * 16384);
  unsigned long long* out; cudaMalloc(&out, 16); unsigned long long h[2];
  cudaFuncSetAttribute(k_tma_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 16384);
  for (int depth : {1, 2, 4, 8}) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a); k_tma_stream<<<1, 32, 8 * 16384>>>(src, chunks, out, depth); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
      printf("tma depth=%d: %.3f ms total, %.2f us/chunk, %.0f cycles/chunk  err=%s\n", depth, ms, ms * 1e3 / chunks, (double)h[0] / chunks, cudaGetErrorString(cudaGetLastError()));
    }
  }
  for (int rep = 0; rep < 2; ++rep) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a); k_ldg_stream<<<1, 32>>>((const uint4*)src, chunks, out); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
    printf("ldg 1 warp: %.3f ms total, %.2f us/chunk, %.0f cycles/chunk\n", ms, ms * 1e3 / chunks, (double)h[0] / chunks);
  }
  return 0;
}
