// Cycles per 32-entry chunk of the ambiguous-list resolution loop, alone in a CTA.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(const int* keys_g, int Q, int* out, long long* cyc) {
  __shared__ int akey[4096];
  __shared__ int apref[4097];
  for (int j = threadIdx.x; j < Q; j += blockDim.x) akey[j] = keys_g[j];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  long long t0 = clock64();
  int serial = 0;
  if (warp == 0) {
    int A = 0;
    for (int base = 0; base < Q; base += 32) {
      const int j = base + lane;
      const bool valid = j < Q;
      const int key = valid ? akey[j] : 0;
      const bool sacc = valid && key >= A + lane;
      const bool srej = !valid || key < A;
      if (!__any_sync(0xffffffffu, !sacc && !srej)) {
        const unsigned bal = __ballot_sync(0xffffffffu, sacc);
        if (valid) apref[j] = A + __popc(bal & lt);
        A += __popc(bal);
      } else {
        ++serial;
        for (int l = 0; l < 32 && base + l < Q; ++l) {
          const int kl = __shfl_sync(0xffffffffu, key, l);
          if (lane == l) apref[base + l] = A;
          A += (kl >= A) ? 1 : 0;
        }
      }
    }
    if (lane == 0) { apref[Q] = A; out[0] = A; out[1] = serial; cyc[0] = clock64() - t0; }
  }
}
int main() {
  // keys like the parse's: uniform in [-0.6r, 0.4r) for growing r
  const int Q = 1408; int h[Q]; unsigned s = 12345;
  for (int j = 0; j < Q; ++j) { s = s * 1664525u + 1013904223u; int r = 64 + j * 35; h[j] = (int)(s % (unsigned)r) - (int)(0.6 * r); }
  int *kg, *o; long long* c; cudaMalloc(&kg, Q * 4); cudaMalloc(&o, 8); cudaMalloc(&c, 8);
  cudaMemcpy(kg, h, Q * 4, cudaMemcpyHostToDevice);
  for (int t : {32, 512}) {
    k<<<1, t>>>(kg, Q, o, c); cudaDeviceSynchronize();
    int ho[2]; long long hc; cudaMemcpy(ho, o, 8, cudaMemcpyDeviceToHost); cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost);
    printf("threads=%d Q=%d accepted=%d serial_chunks=%d cycles=%lld per_chunk=%.1f\n", t, Q, ho[0], ho[1], hc, (double)hc / ((Q + 31) / 32));
  }
  return 0;
}
