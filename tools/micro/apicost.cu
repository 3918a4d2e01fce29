#include <cstdio>
#include <chrono>
#include <cuda_runtime.h>
__global__ void k(){}
int main(){
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t ev[12]; for (auto& e: ev) cudaEventCreate(&e);
  void* d; cudaMalloc(&d, 1<<22);
  for (int rep=0; rep<5; ++rep){
    for (int i=0;i<12;++i){ k<<<1,1,0,s>>>(); cudaEventRecord(ev[i], s);}
    cudaStreamSynchronize(s);
    auto t0=std::chrono::steady_clock::now();
    float ms, acc=0; for (int i=0;i<10;++i){ cudaEventElapsedTime(&ms, ev[i], ev[i+1]); acc+=ms;}
    auto t1=std::chrono::steady_clock::now();
    cudaMemsetAsync(d, 0, 1<<22, s);
    auto t2=std::chrono::steady_clock::now();
    cudaEventRecord(ev[0], s);
    auto t3=std::chrono::steady_clock::now();
    k<<<1,1,0,s>>>();
    auto t4=std::chrono::steady_clock::now();
    cudaStreamSynchronize(s);
    auto t5=std::chrono::steady_clock::now();
    printf("10x elapsed %.2f us, memset %.2f us, record %.2f us, launch %.2f us, sync(idle) %.2f us\n",
      std::chrono::duration<double,std::micro>(t1-t0).count(), std::chrono::duration<double,std::micro>(t2-t1).count(),
      std::chrono::duration<double,std::micro>(t3-t2).count(), std::chrono::duration<double,std::micro>(t4-t3).count(),
      std::chrono::duration<double,std::micro>(t5-t4).count());
  }
}
