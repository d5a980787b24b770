// TMA 1-D bulk copies: chip-wide streaming throughput vs copy size, one
// producer thread per CTA, 3-stage ring, consumers only wait (no compute).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_1609_06119_b200/csrc/common.cuh"
using namespace bb;
namespace bb { void set_error(const std::string&) {} }

// each CTA streams `stages` stages of `stage_bytes`, split into copies of `copy_bytes`
__global__ void k_stream(const unsigned char* src, int64_t per_cta, int stage_bytes, int copy_bytes, int nprod,
                         unsigned long long* sink) {
  extern __shared__ __align__(16) unsigned char sm[];
  __shared__ __align__(8) uint64_t full[3], empty[3];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (threadIdx.x == 0) {
    for (int b = 0; b < 3; ++b) { mbar_init(&full[b], 1); mbar_init(&empty[b], nw - 1); }
    fence_mbar_init();
  }
  __syncthreads();
  const int stages = (int)(per_cta / stage_bytes);
  const unsigned char* base = src + (int64_t)blockIdx.x * per_cta;
  if (warp == nw - 1) {
    for (int k = 0; k < stages; ++k) {
      const int buf = k % 3;
      if (lane == 0) {
        if (k >= 3) mbar_wait(&empty[buf], (unsigned)(((k / 3) - 1) & 1));
        mbar_expect_tx(&full[buf], stage_bytes);
      }
      __syncwarp();
      const int ncopy = stage_bytes / copy_bytes;
      for (int c = lane; c < ncopy; c += nprod)
        if (lane < nprod) tma_load_1d(sm + buf * stage_bytes + c * copy_bytes, base + (int64_t)k * stage_bytes + c * copy_bytes,
                                      copy_bytes, &full[buf]);
    }
  } else {
    unsigned acc = 0;
    for (int k = 0; k < stages; ++k) {
      const int buf = k % 3;
      mbar_wait(&full[buf], (unsigned)((k / 3) & 1));
      acc += sm[buf * stage_bytes + threadIdx.x * 4];
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[buf])) : "memory");
    }
    if (acc == 12345) sink[0] = acc;
  }
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t total = 1ll << 30;
  unsigned char* src; cudaMalloc(&src, total); cudaMemset(src, 1, total);
  unsigned long long* sink; cudaMalloc(&sink, 8);
  cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int stage : {16384, 32768, 65536}) for (int cb : {512, 1024, 4096, 16384}) for (int nprod : {1, 32}) {
    if (cb > stage) continue;
    const int64_t per = (total / sms) / stage * stage;
    k_stream<<<sms, 17 * 32, 3 * stage>>>(src, per, stage, cb, nprod, sink);
    cudaEventRecord(a);
    k_stream<<<sms, 17 * 32, 3 * stage>>>(src, per, stage, cb, nprod, sink);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("stage %6d copy %6d issuers %2d : %.1f GB/s  err=%s\n", stage, cb, nprod, per * sms / ms / 1e6,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
