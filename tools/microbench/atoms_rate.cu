// Conflict-free shared atomics (lane-interleaved slots): per-SM rate with
// almost no other instructions; also broadcast LDS.128 and LDS.128 spread.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(uint32_t* out, int iters) {
  extern __shared__ uint32_t h[];  // 32K words
  for (int i = threadIdx.x; i < 32768; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  uint32_t a = (threadIdx.x * 4) & (128 * 1024 - 1);
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const uint32_t ad = (a + u * 4096) & (128 * 1024 - 1);
      if (MODE == 0) atomicAdd(&h[ad >> 2], 1u);                     // conflict-free noret
      if (MODE == 1) { uint4 x = *(uint4*)&h[((u * 64) & 32767)]; acc += x.x + x.w; }  // broadcast LDS.128
      if (MODE == 2) { uint4 x = *(uint4*)&h[(lane * 4 + u * 128) & 32767]; acc += x.x + x.w; }  // spread LDS.128 (4 wf)
      if (MODE == 3) { acc += h[(lane + u * 32) & 32767]; }                    // LDS.32 conflict-free
    }
    a += 64;
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = h[5] + acc;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* out; cudaMalloc(&out, 1 << 20);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int iters = 2048;
  auto run = [&](const char* name, auto kern, int thr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
    kern<<<sms, thr, 131072>>>(out, iters); cudaDeviceSynchronize();
    cudaEventRecord(a); kern<<<sms, thr, 131072>>>(out, iters); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double winstr = (double)thr / 32 * iters * 16;  // per SM
    printf("%-22s thr=%4d  %.3f ms  %.2f clk per warp-op per SM (at 1.965 GHz)\n", name, thr, ms, ms * 1e-3 * 1.965e9 / winstr);
  };
  for (int thr : {256, 512, 1024}) {
    run("atoms_noret_cf", k<0>, thr);
    run("lds128_broadcast", k<1>, thr);
    run("lds128_spread", k<2>, thr);
    run("lds32_cf", k<3>, thr);
  }
  return 0;
}
