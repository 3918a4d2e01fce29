// Microbenchmark: throughput of fire-and-forget global reductions to random
// bins (input to the SPA pre-filter design decision).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 mix(u64 x){x^=x>>33;x*=0xff51afd7ed558ccdULL;x^=x>>33;x*=0xc4ceb9fe1a85ec53ULL;x^=x>>33;return x;}
__global__ void fill(u64* k, u64* v, size_t n){for(size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x;i<n;i+=(size_t)gridDim.x*blockDim.x){k[i]=mix(i);v[i]=mix(i+12345);}}
template<int MODE>
__global__ void stats(const u64* __restrict__ k, const u64* __restrict__ v, size_t n, unsigned* cnt, u64* ext, unsigned nbins){
  for(size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x;i<n;i+=(size_t)gridDim.x*blockDim.x){
    u64 kk=k[i], vv=v[i]; unsigned b=(unsigned)(kk>>40)%nbins;
    if(MODE&1) atomicAdd(&cnt[b],1u);
    if(MODE&2) atomicMin(&ext[b],vv);
    if(MODE&4) { atomicAdd(&cnt[2*b],1u); atomicMin((unsigned*)&cnt[2*b+1],(unsigned)(vv>>32)); }
  }
}
__global__ void readonly(const u64* __restrict__ k, const u64* __restrict__ v, size_t n, u64* out){
  u64 acc=0; for(size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x;i<n;i+=(size_t)gridDim.x*blockDim.x){acc^=k[i]+v[i];}
  if(acc==42) out[0]=acc;
}
int main(){
  size_t n=8783067; u64 *k,*v,*ext; unsigned* cnt;
  cudaMalloc(&k,n*8);cudaMalloc(&v,n*8);cudaMalloc(&ext,(1<<20)*8*2);cudaMalloc(&cnt,(1<<20)*4*2);
  fill<<<1184,256>>>(k,v,n); cudaDeviceSynchronize();
  cudaEvent_t a,b; cudaEventCreate(&a);cudaEventCreate(&b);
  for(unsigned nbins: {1u<<16, 1u<<18, 1u<<20}){
   for(int mode: {0,1,2,3,4}){
    float best=1e9;
    for(int r=0;r<5;r++){
      cudaEventRecord(a);
      if(mode==0) readonly<<<148*8,256>>>(k,v,n,ext); 
      else if(mode==1) stats<1><<<148*8,256>>>(k,v,n,cnt,ext,nbins);
      else if(mode==2) stats<2><<<148*8,256>>>(k,v,n,cnt,ext,nbins);
      else if(mode==3) stats<3><<<148*8,256>>>(k,v,n,cnt,ext,nbins);
      else stats<4><<<148*8,256>>>(k,v,n,cnt,ext,nbins);
      cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms,a,b); if(ms<best)best=ms;
    }
    printf("nbins=%u mode=%d (0=read,1=add,2=min64,3=add+min64,4=add+min32 adjacent) best=%.1f us  -> %.1f Gatom/s\n",nbins,mode,best*1e3, (mode==3||mode==4?2:1)*n/(best*1e-3)/1e9);
   }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
