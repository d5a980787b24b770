// Microbenchmark 2: shared-atomic throughput vs bank layout for the layer
// histogram.  "il32" = lane-interleaved copies (slot s of lane l at s*32+l),
// so a warp-wide atomic touches 32 distinct banks: one wavefront.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x){x^=x>>16;x*=0x7feb352d;x^=x>>15;x*=0x846ca68b;x^=x>>16;return x;}

template <int MODE>  // 0 noret random, 1 ret random, 2 noret il32, 3 ret il32, 4 ret il32 + carry, 5 noret 16-valued random, 6 2x noret il32 (16/16 split)
__global__ void k(uint32_t* out, int iters, int nslots) {
  extern __shared__ uint32_t h[];
  const int tot = MODE >= 2 && MODE != 5 ? nslots * 32 * (MODE == 6 ? 2 : 1) : nslots * 2;
  for (int i = threadIdx.x; i < tot; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  uint32_t s = hash32(blockIdx.x * blockDim.x + threadIdx.x);
  uint32_t acc = 0;
  for (int it = 0; it < iters; it += 8) {
    uint32_t sl[8], v[8], o[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      s = s * 1664525u + 1013904223u;
      uint32_t r = (s >> 8) & (uint32_t)(nslots - 1);
      if (MODE == 5) r = (r & 15) * 17 + (u << 8);
      sl[u] = (MODE >= 2 && MODE != 5) ? r * 32 + lane : r;
      v[u] = s | 0x40000000u;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (MODE == 0 || MODE == 2 || MODE == 5) atomicAdd(&h[sl[u]], v[u]);
      else if (MODE == 6) { atomicAdd(&h[sl[u]], v[u] & 0xffff); atomicAdd(&h[sl[u] + nslots * 32], v[u] >> 16); }
      else o[u] = atomicAdd(&h[sl[u]], v[u]);
    }
    if (MODE == 1 || MODE == 3) {
#pragma unroll
      for (int u = 0; u < 8; ++u) acc += o[u];
    }
    if (MODE == 4) {
#pragma unroll
      for (int u = 0; u < 8; ++u) if (o[u] + v[u] < o[u]) atomicAdd(&h[sl[u] ^ 1], 1u);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = h[5] + acc;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* out; cudaMalloc(&out, 1 << 20);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int iters = 4096; float ms;
  auto run = [&](const char* name, auto kern, int nslots, int smem, int threads) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    kern<<<sms, threads, smem>>>(out, iters, nslots); cudaDeviceSynchronize();
    cudaEventRecord(a); kern<<<sms, threads, smem>>>(out, iters, nslots); cudaEventRecord(b);
    cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
    double upd = (double)sms * threads * iters;
    printf("%-26s slots=%5d thr=%d %.3f ms %7.1f G upd/s  %.2f clk/warp-atomic/SM @1.965GHz  err=%s\n", name, nslots, threads, ms,
           upd / ms / 1e6, (ms * 1e-3 * 1.965e9) / (upd / sms / 32), cudaGetErrorString(cudaGetLastError()));
  };
  for (int thr : {512, 1024}) {
    run("noret_random", k<0>, 8192, 8192 * 8, thr);
    run("ret_random", k<1>, 8192, 8192 * 8, thr);
    run("noret_16valued", k<5>, 8192, 8192 * 8, thr);
    run("noret_il32", k<2>, 1024, 1024 * 128, thr);
    run("ret_il32", k<3>, 1024, 1024 * 128, thr);
    run("ret_il32_carry", k<4>, 1024, 1024 * 128, thr);
    run("2x_noret_il32", k<6>, 512, 512 * 256, thr);
  }
  return 0;
}
