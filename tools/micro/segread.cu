// Micro-benchmark: reading K2-style survivor segments (256 slots of 8 B,
// ~44% filled) in different orders, to find the floor of k_filter's key
// stream. nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o segread segread.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
typedef unsigned long long u64;
typedef unsigned int u32;

template <int MODE>
__global__ void k_read(const u64* __restrict__ seg, const u64* __restrict__ cnt, u32 nseg, u64* out) {
  const int lane = threadIdx.x & 31;
  const u32 nw = gridDim.x * (blockDim.x / 32);
  const u32 w = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  u64 acc = 0;
  if (MODE == 0) {  // warp stride, 4 rounds in flight
    for (u32 s = w; s < nseg; s += nw) {
      const u32 tot = (u32)cnt[s];
      u64 k[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) k[j] = (32 * j + lane < tot) ? __ldcs(seg + (u64)s * 256 + 32 * j + lane) : 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) acc += k[j];
      for (u32 i = 128 + lane; i < tot; i += 32) acc += __ldcs(seg + (u64)s * 256 + i);
    }
  } else if (MODE == 1) {  // contiguous partition per warp
    const u32 per = (nseg + nw - 1) / nw;
    for (u32 s = w * per; s < min(nseg, (w + 1) * per); ++s) {
      const u32 tot = (u32)cnt[s];
      u64 k[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) k[j] = (32 * j + lane < tot) ? __ldcs(seg + (u64)s * 256 + 32 * j + lane) : 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) acc += k[j];
      for (u32 i = 128 + lane; i < tot; i += 32) acc += __ldcs(seg + (u64)s * 256 + i);
    }
  } else {  // dense stream of the whole array (grid stride, 16 B per lane)
    const uint4* p = reinterpret_cast<const uint4*>(seg);
    const u64 n4 = (u64)nseg * 256 * 8 / 16;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (u64)gridDim.x * blockDim.x) {
      const uint4 v = __ldcs(p + i);
      acc += v.x ^ v.w;
    }
  }
  if (acc == 0x1234567) out[0] = acc;
}

int main() {
  const u32 nseg = 78125;
  std::vector<u64> cnt(nseg);
  srand(1);
  for (auto& c : cnt) c = 100 + rand() % 27;
  u64 *d_seg, *d_cnt, *d_out, *d_flush;
  cudaMalloc(&d_seg, (size_t)nseg * 256 * 8);
  cudaMalloc(&d_cnt, nseg * 8);
  cudaMalloc(&d_out, 8);
  cudaMalloc(&d_flush, 512 << 20);
  cudaMemset(d_seg, 1, (size_t)nseg * 256 * 8);
  cudaMemcpy(d_cnt, cnt.data(), nseg * 8, cudaMemcpyHostToDevice);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const char* names[] = {"stride4", "contig4", "dense"};
  for (int mode = 0; mode < 3; ++mode)
    for (int occ : {8, 16, 32, 64}) {
      float best = 1e9;
      for (int rep = 0; rep < 5; ++rep) {
        cudaMemset(d_flush, rep, 512 << 20);  // flush L2
        cudaEventRecord(a);
        const int blocks = sms * occ / 8;
        if (mode == 0) k_read<0><<<blocks, 256>>>(d_seg, d_cnt, nseg, d_out);
        if (mode == 1) k_read<1><<<blocks, 256>>>(d_seg, d_cnt, nseg, d_out);
        if (mode == 2) k_read<2><<<blocks, 256>>>(d_seg, d_cnt, nseg, d_out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
      }
      printf("%-8s warps/SM %2d: %7.1f us\n", names[mode], occ, best * 1e3);
    }
  return 0;
}
