// Microbenchmark: shared-memory update throughput options for the level-wise
// histogram (int64 fixed-point slots).  Prints G updates/s chip-wide.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define SLOTS 4096   // 64 KB of u64 slots
__device__ __forceinline__ uint32_t hash32(uint32_t x){x^=x>>16;x*=0x7feb352d;x^=x>>15;x*=0x846ca68b;x^=x>>16;return x;}

// (a) u32 atomicAdd no return, random slots
__global__ void k_atom_u32(uint32_t* out, int iters){
  __shared__ uint32_t h[SLOTS*2];
  for(int i=threadIdx.x;i<SLOTS*2;i+=blockDim.x) h[i]=0; __syncthreads();
  uint32_t s = hash32(blockIdx.x*blockDim.x+threadIdx.x);
  for(int it=0;it<iters;it++){ s=s*1664525u+1013904223u; atomicAdd(&h[(s>>8)%(SLOTS*2)], s&0xff);}  
  __syncthreads(); if(threadIdx.x==0) out[blockIdx.x]=h[5];
}
// (b) 2-limb int64: lo atomic with return, carry into hi
__global__ void k_atom_2limb(uint32_t* out, int iters){
  __shared__ uint32_t h[SLOTS*2];
  for(int i=threadIdx.x;i<SLOTS*2;i+=blockDim.x) h[i]=0; __syncthreads();
  uint32_t s = hash32(blockIdx.x*blockDim.x+threadIdx.x);
  for(int it=0;it<iters;it++){ s=s*1664525u+1013904223u; uint32_t slot=(s>>8)%SLOTS; uint32_t v=s|0x40000000u;
     uint32_t old=atomicAdd(&h[2*slot], v); if(old+v<old) atomicAdd(&h[2*slot+1],1u);}  
  __syncthreads(); if(threadIdx.x==0) out[blockIdx.x]=h[5];
}
// (c) u64 smem atomicAdd (CAS loop on sm_100)
__global__ void k_atom_u64(uint32_t* out, int iters){
  __shared__ unsigned long long h[SLOTS];
  for(int i=threadIdx.x;i<SLOTS;i+=blockDim.x) h[i]=0; __syncthreads();
  uint32_t s = hash32(blockIdx.x*blockDim.x+threadIdx.x);
  for(int it=0;it<iters;it++){ s=s*1664525u+1013904223u; atomicAdd(&h[(s>>8)%SLOTS], (unsigned long long)(s|0x40000000u));}
  __syncthreads(); if(threadIdx.x==0) out[blockIdx.x]=(uint32_t)h[5];
}
// (d) non-atomic u64 RMW, warp-private region per warp, lane-distinct sub-histograms (lane = feature)
__global__ void k_rmw_lane(uint32_t* out, int iters){
  extern __shared__ unsigned long long hs[]; // warps * 32 lanes * 32 bins
  int w=threadIdx.x>>5, l=threadIdx.x&31; unsigned long long* h = hs + (w*32 + l)*33; // 32 bins + pad
  for(int i=0;i<33;i++) h[i]=0; __syncwarp();
  uint32_t s = hash32(blockIdx.x*blockDim.x+threadIdx.x);
  for(int it=0;it<iters;it++){ s=s*1664525u+1013904223u; uint32_t b=(s>>8)&31; h[b]+= (s|0x40000000u);}  
  __syncthreads(); if(threadIdx.x==0) out[blockIdx.x]=(uint32_t)hs[5];
}
// (e) global u64 red spread over 1M slots
__global__ void k_red_g(unsigned long long* g, int iters){
  uint32_t s = hash32(blockIdx.x*blockDim.x+threadIdx.x);
  for(int it=0;it<iters;it++){ s=s*1664525u+1013904223u; atomicAdd(&g[(s>>4)&((1<<20)-1)], (unsigned long long)(s&0xffff));}
}
// (f) u32 atomicAdd with 8-bit bins grouped by feature: lane f-> region f (like per-feature hist of 256 bins)
__global__ void k_atom_feat(uint32_t* out, int iters){
  __shared__ uint32_t h[20*257*2];
  for(int i=threadIdx.x;i<20*257*2;i+=blockDim.x) h[i]=0; __syncthreads();
  int l=threadIdx.x&31; uint32_t s = hash32(blockIdx.x*blockDim.x+threadIdx.x);
  for(int it=0;it<iters;it++){ s=s*1664525u+1013904223u; uint32_t slot=(l%20)*257+((s>>8)&255); uint32_t v=s|0x40000000u;
     uint32_t old=atomicAdd(&h[2*slot], v); if(old+v<old) atomicAdd(&h[2*slot+1],1u);}  
  __syncthreads(); if(threadIdx.x==0) out[blockIdx.x]=h[5];
}

int main(){
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* out; cudaMalloc(&out, 1<<20); unsigned long long* g; cudaMalloc(&g, 8<<20); cudaMemset(g,0,8<<20);
  cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int iters=4096; float ms;
  auto run=[&](const char* name, auto launch, int blocks, int threads){
    launch(); cudaDeviceSynchronize();
    cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);
    double upd=(double)blocks*threads*iters; printf("%-28s blocks=%d thr=%d  %.3f ms  %.1f G upd/s  err=%s\n", name, blocks, threads, ms, upd/ms/1e6, cudaGetErrorString(cudaGetLastError()));
  };
  for(int bpsm: {1,2,4}) {
    int B=sms*bpsm;
    run("atom_u32_noret", [&]{k_atom_u32<<<B,512>>>(out,iters);}, B, 512);
    run("atom_2limb_ret", [&]{k_atom_2limb<<<B,512>>>(out,iters);}, B, 512);
    run("atom_u64_cas", [&]{k_atom_u64<<<B,512>>>(out,iters);}, B, 512);
    run("atom_feat_2limb", [&]{k_atom_feat<<<B,512>>>(out,iters);}, B, 512);
  }
  cudaFuncSetAttribute(k_rmw_lane, cudaFuncAttributeMaxDynamicSharedMemorySize, 16*32*33*8);
  run("rmw_lane_private(16w)", [&]{k_rmw_lane<<<sms,512,16*32*33*8>>>(out,iters);}, sms, 512);
  run("red_global_u64", [&]{k_red_g<<<sms*4,512>>>(g,iters/8);}, sms*4, 512/8);
  return 0;
}
