// Micro-benchmark: streaming-read bandwidth of a 320 MB double2 array on
// B200 (the K1 access pattern), plain loads vs 1D TMA bulk copies into a
// shared-memory ring. nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o readbw readbw.cu
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;

__device__ __forceinline__ double2 ldg_nc(const double2* p) {
  double2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}

// warp tiles of 32*U points, grid-strided (K1's loop), a min/max fold
template <int U>
__global__ void k_plain(const double2* __restrict__ p, u64 n, double* out) {
  const int ln = threadIdx.x & 31;
  const u64 tw = (u64)gridDim.x * (blockDim.x / 32);
  double a = 1e300, b = -1e300;
  for (u64 t = (u64)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); (t + 1) * 32 * U <= n; t += tw) {
    double2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ldg_nc(p + t * 32 * U + ln + 32 * u);
#pragma unroll
    for (int u = 0; u < U; ++u) { a = fmin(a, v[u].x); b = fmax(b, v[u].y); }
  }
  if (a == 12345.0) out[0] = b;
}

// contiguous partition per CTA, 1D bulk copies (cp.async.bulk) into a ring of
// S stages of B bytes, one mbarrier per stage; every thread folds from smem
template <int S, int B>
__global__ void k_tma(const double2* __restrict__ p, u64 n, double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) u64 bar[S];
  const u64 bytes = n * 16;
  const u64 per = ((bytes / gridDim.x) + B - 1) / B * B;
  const u64 beg = (u64)blockIdx.x * per;
  const u64 end = beg + per < bytes ? beg + per : bytes;
  const int nchunks = beg < end ? (int)((end - beg + B - 1) / B) : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      unsigned a = (unsigned)__cvta_generic_to_shared(&bar[s]);
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(a));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int c) {
    const int s = c % S;
    const u64 off = beg + (u64)c * B;
    const unsigned len = (unsigned)((end - off) < (u64)B ? (end - off) : (u64)B);
    unsigned a = (unsigned)__cvta_generic_to_shared(&bar[s]);
    unsigned d = (unsigned)__cvta_generic_to_shared(sm + (size_t)s * B);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(a), "r"(len) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(d), "l"(reinterpret_cast<const unsigned char*>(p) + off), "r"(len), "r"(a) : "memory");
  };
  if (threadIdx.x == 0)
    for (int c = 0; c < S && c < nchunks; ++c) issue(c);
  double a = 1e300, b = -1e300;
  for (int c = 0; c < nchunks; ++c) {
    const int s = c % S;
    const unsigned ph = (unsigned)((c / S) & 1);
    unsigned ba = (unsigned)__cvta_generic_to_shared(&bar[s]);
    asm volatile("{\n .reg .pred P;\n W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n @!P bra W;\n}" :: "r"(ba), "r"(ph) : "memory");
    const u64 off = beg + (u64)c * B;
    const unsigned len = (unsigned)((end - off) < (u64)B ? (end - off) : (u64)B);
    const double2* q = reinterpret_cast<const double2*>(sm + (size_t)s * B);
    for (unsigned i = threadIdx.x; i < len / 16; i += blockDim.x) { const double2 v = q[i]; a = fmin(a, v.x); b = fmax(b, v.y); }
    __syncthreads();
    if (threadIdx.x == 0 && c + S < nchunks) issue(c + S);
  }
  if (a == 12345.0) out[0] = b;
}

int main() {
  const u64 n = 20000000;
  double2* p; double* o;
  cudaMalloc(&p, n * 16); cudaMalloc(&o, 8);
  {
    double2* h = (double2*)malloc(n * 16);
    unsigned long long z = 88172645463325252ull;
    for (u64 i = 0; i < n; ++i) {
      z ^= z << 13; z ^= z >> 7; z ^= z << 17; double a = (z >> 11) * 0x1.0p-53;
      z ^= z << 13; z ^= z >> 7; z ^= z << 17; double b = (z >> 11) * 0x1.0p-53;
      h[i] = make_double2(a, b);
    }
    cudaMemcpy(p, h, n * 16, cudaMemcpyHostToDevice);
    free(h);
  }
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto bench = [&](const char* name, auto launch) {
    for (int i = 0; i < 3; ++i) launch();
    cudaEventRecord(e0);
    for (int i = 0; i < 20; ++i) launch();
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 20;
    printf("%-36s %7.2f us  %6.0f GB/s  %s\n", name, ms * 1e3, n * 16 / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  };
  for (int bps : {2, 3, 4, 6, 8}) {
    char nm[64];
    sprintf(nm, "plain U=8 256thr x %d/SM", bps);
    bench(nm, [&] { k_plain<8><<<sms * bps, 256>>>(p, n, o); });
    sprintf(nm, "plain U=4 256thr x %d/SM", bps);
    bench(nm, [&] { k_plain<4><<<sms * bps, 256>>>(p, n, o); });
  }
  {
    constexpr int S = 4, B = 32768;
    cudaFuncSetAttribute(k_tma<S, B>, cudaFuncAttributeMaxDynamicSharedMemorySize, S * B);
    for (int bps : {1, 2}) { char nm[64]; sprintf(nm, "tma 4x32KB 256thr x %d/SM", bps);
      bench(nm, [&] { k_tma<S, B><<<sms * bps, 256, S * B>>>(p, n, o); }); }
  }
  {
    constexpr int S = 6, B = 16384;
    cudaFuncSetAttribute(k_tma<S, B>, cudaFuncAttributeMaxDynamicSharedMemorySize, S * B);
    for (int bps : {1, 2}) { char nm[64]; sprintf(nm, "tma 6x16KB 256thr x %d/SM", bps);
      bench(nm, [&] { k_tma<S, B><<<sms * bps, 256, S * B>>>(p, n, o); }); }
  }
  {
    constexpr int S = 8, B = 24576;
    cudaFuncSetAttribute(k_tma<S, B>, cudaFuncAttributeMaxDynamicSharedMemorySize, S * B);
    bench("tma 8x24KB 512thr x 1/SM", [&] { k_tma<S, B><<<sms, 512, S * B>>>(p, n, o); });
  }
  // copy for reference
  double2* q; cudaMalloc(&q, n * 16);
  bench("cudaMemcpy D2D (read+write, /2)", [&] { cudaMemcpyAsync(q, p, n * 16, cudaMemcpyDeviceToDevice); });
  return 0;
}
