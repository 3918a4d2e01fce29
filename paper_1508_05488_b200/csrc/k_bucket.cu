// K3 main path: the region sort as a bucket sort with no inter-tile scan.
//
// sort_region (reference spa.cpp:59-81) orders each region by
// region_less. Every record carries q = quantize(primary) (a monotone map of
// the primary onto [0, 2^qbits), chgpu_internal.cuh / k_sort.cu), split as
//   bucket = q >> kLocalBits   (2^bbits buckets per region)
//   local  = q & (2^kLocalBits - 1)
// Three kernels, all without look-back chains:
//   k_bucket_hist    per-bucket counts (shared-memory histograms per CTA)
//   k_bucket_scan    exclusive scan -> bucket bases and scatter cursors
//   k_bucket_scatter a CTA bins a 16384-record tile in shared memory,
//                    reserves each bucket's slice with one atomicAdd, and
//                    scatters the records there (order inside a bucket is
//                    free: the next kernel sorts it completely)
//   k_bucket_sort    one CTA per bucket: counting sort on `local` in shared
//                    memory, then equal-q groups insertion-sorted by the
//                    total order (canon k, v, k); written back in place.
// Buckets larger than kBucketCap records are listed for the host, which
// sorts them with the onesweep engine (k_sort.cu).

#include <algorithm>

#include "chgpu_internal.cuh"
#include "kernels.h"

namespace chgpu {

__device__ __forceinline__ u32 bq_quantize(const BucketPlan& P, int s, u64 k) {
  const int region = P.region[s];
  const double p = primary_of(region, k);
  double t = __dmul_rn(__dsub_rn(p, P.qlo[s]), P.qscale[s]);
  t = fmin(fmax(t, 0.0), P.qmax);
  const u32 q = (u32)__double2ull_rz(t);
  return (region == 3 || region == 4) ? (u32)((u64)P.qmax - q) : q;
}

__device__ __forceinline__ int seg_of(const BucketPlan& P, u64 i) {
  int s = 0;
  while (s + 1 < P.nseg && i >= P.cum[s + 1]) ++s;
  return s;
}

__device__ __forceinline__ u64 canon_key(int region, u64 k) {
  const bool desc = (region == 3 || region == 4);
  const u64 neg0 = desc ? ~0x7FFFFFFFFFFFFFFFull : 0x7FFFFFFFFFFFFFFFull;
  const u64 pos0 = desc ? ~0x8000000000000000ull : 0x8000000000000000ull;
  return k == neg0 ? pos0 : k;
}

__device__ __forceinline__ bool total_less(int region, u64 ka, u64 va, u64 kb, u64 vb) {
  const u64 ca = canon_key(region, ka), cb = canon_key(region, kb);
  return ca < cb || (ca == cb && (va < vb || (va == vb && ka < kb)));
}

// ------------------------------------------------------------------ histogram

// Each CTA owns a contiguous slice of the concatenated segments and keeps a
// shared-memory histogram of the current segment's buckets, flushing the
// non-zero bins with global atomics when the segment changes.
__global__ __launch_bounds__(512) void k_bucket_hist(const u64* __restrict__ kbuf, BucketPlan P,
                                                     u32* __restrict__ hist) {
  extern __shared__ u32 sh[];  // [nbuckets]
  const u32 nb = 1u << P.bbits;
  const u64 total = P.cum[P.nseg];
  const u64 per = (total + gridDim.x - 1) / gridDim.x;
  const u64 i0 = (u64)blockIdx.x * per;
  const u64 i1 = min(total, i0 + per);
  if (i0 >= i1) return;
  for (u32 b = threadIdx.x; b < nb; b += blockDim.x) sh[b] = 0;
  __syncthreads();
  int s = seg_of(P, i0);
  u64 i = i0;
  while (i < i1) {
    const u64 seg_end = min(i1, P.cum[s + 1]);
    const u64 src = P.src_off[s] - P.cum[s];
    // Loads are batched ahead of the shared atomics so each thread keeps
    // kBatch requests in flight.
    constexpr int kBatch = 8;
    for (u64 j0 = i + threadIdx.x; j0 < seg_end; j0 += (u64)kBatch * blockDim.x) {
      u64 kk[kBatch];
#pragma unroll
      for (int u = 0; u < kBatch; ++u) {
        const u64 j = j0 + (u64)u * blockDim.x;
        kk[u] = j < seg_end ? kbuf[src + j] : 0ull;
      }
#pragma unroll
      for (int u = 0; u < kBatch; ++u)
        if (j0 + (u64)u * blockDim.x < seg_end)
          atomicAdd(&sh[bq_quantize(P, s, kk[u]) >> kLocalBits], 1u);
    }
    __syncthreads();
    for (u32 b = threadIdx.x; b < nb; b += blockDim.x) {
      const u32 c = sh[b];
      if (c) {
        atomicAdd(&hist[(size_t)s * nb + b], c);
        sh[b] = 0;
      }
    }
    __syncthreads();
    i = seg_end;
    ++s;
  }
}

// One CTA per segment: bucket bases (absolute destination offsets) and the
// scatter cursors, plus the list of buckets too large for k_bucket_sort.
__global__ __launch_bounds__(1024) void k_bucket_scan(const u32* __restrict__ hist, BucketPlan P,
                                                      u64* __restrict__ base, u32* __restrict__ cursor,
                                                      u32* __restrict__ big, u32* __restrict__ nbig) {
  const int s = blockIdx.x;
  const u32 nb = 1u << P.bbits;
  const u32* h = hist + (size_t)s * nb;
  __shared__ u32 wsum[32];
  __shared__ u32 carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (u32 b0 = 0; b0 < nb; b0 += blockDim.x) {
    const u32 b = b0 + threadIdx.x;
    const u32 c = b < nb ? h[b] : 0u;
    u32 x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const u32 y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    u32 pre = 0;
    for (int w = 0; w < warp; ++w) pre += wsum[w];
    u32 tot = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += wsum[w];
    const u32 excl = carry + pre + x - c;
    if (b < nb) {
      base[(size_t)s * nb + b] = P.dst_off[s] + excl;
      cursor[(size_t)s * nb + b] = excl;
      if (c > kBucketCap) big[atomicAdd(nbig, 1u)] = (u32)(s * nb + b);
    }
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
}

// ------------------------------------------------------------------ scatter

constexpr int kScatterThreads = 512;
constexpr int kScatterTile = 16384;

__global__ __launch_bounds__(kScatterThreads, 3) void k_bucket_scatter(
    const u64* __restrict__ kin, const u64* __restrict__ vin, u64* __restrict__ kout,
    u64* __restrict__ vout, BucketPlan P, u32* __restrict__ cursor) {
  extern __shared__ __align__(16) u32 sm[];
  const u32 nb = 1u << P.bbits;
  u32* cnt = sm;                                                   // [nb] counts, then slice bases
  unsigned short* bid = reinterpret_cast<unsigned short*>(sm + nb);  // [kScatterTile]
  // Tiles never straddle segments: tile t of segment s covers
  // [t * kScatterTile, ...) of that segment (tile_begin in P).
  const u32 tile = blockIdx.x;
  int s = 0;
  while (s + 1 < P.nseg && tile >= P.tile_begin[s + 1]) ++s;
  const u64 e0 = (u64)(tile - P.tile_begin[s]) * kScatterTile;
  const u64 m = P.cum[s + 1] - P.cum[s];
  if (e0 >= m) return;
  const u32 n = (u32)min((u64)kScatterTile, m - e0);
  const u64 src = P.src_off[s] + e0;
  for (u32 b = threadIdx.x; b < nb; b += blockDim.x) cnt[b] = 0;
  __syncthreads();
  constexpr int kBatch = 8;
  for (u32 i0 = threadIdx.x; i0 < n; i0 += kBatch * blockDim.x) {
    u64 kk[kBatch];
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      const u32 i = i0 + u * blockDim.x;
      kk[u] = i < n ? kin[src + i] : 0ull;
    }
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      const u32 i = i0 + u * blockDim.x;
      if (i < n) {
        const u32 b = bq_quantize(P, s, kk[u]) >> kLocalBits;
        bid[i] = (unsigned short)b;
        atomicAdd(&cnt[b], 1u);
      }
    }
  }
  __syncthreads();
  u32* cur = cursor + (size_t)s * nb;
  for (u32 b = threadIdx.x; b < nb; b += blockDim.x) {
    const u32 c = cnt[b];
    if (c) cnt[b] = atomicAdd(&cur[b], c);  // this tile's slice of bucket b
  }
  __syncthreads();
  const u64 dst = P.dst_off[s];
  for (u32 i0 = threadIdx.x; i0 < n; i0 += kBatch * blockDim.x) {
    u64 kk[kBatch], vv[kBatch];
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      const u32 i = i0 + u * blockDim.x;
      if (i < n) {
        kk[u] = kin[src + i];
        vv[u] = vin[src + i];
      }
    }
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      const u32 i = i0 + u * blockDim.x;
      if (i < n) {
        const u32 pos = atomicAdd(&cnt[bid[i]], 1u);
        kout[dst + pos] = kk[u];
        vout[dst + pos] = vv[u];
      }
    }
  }
}

// ------------------------------------------------------------------ local sort

constexpr int kSortThreadsB = 128;
constexpr int kSortBinBits = 8;  // counting-sort bins: the top bits of the local key
constexpr u32 kLocalBins = 1u << kSortBinBits;

struct BucketSmem {
  u64 k[kBucketCap];
  u64 v[kBucketCap];
  unsigned short lk[kBucketCap];    // local key of record i
  unsigned short perm[kBucketCap];  // sorted position -> record
  u32 bin[kLocalBins];
  u32 wsum[kSortThreadsB / 32];
};

// One CTA per bucket: the records are loaded once (coalesced), their local
// keys computed once, and the sort moves 16-bit indices only: a counting
// sort on the local key, then equal-q groups insertion-sorted by the total
// order. The bucket is written back in sorted order.
__global__ __launch_bounds__(kSortThreadsB, 4) void k_bucket_sort(
    u64* __restrict__ k, u64* __restrict__ v, BucketPlan P, const u64* __restrict__ base,
    const u32* __restrict__ hist, unsigned long long* __restrict__ ngroups) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  BucketSmem& S = *reinterpret_cast<BucketSmem*>(smem_raw);
  const u32 nb = 1u << P.bbits;
  const u32 gb = blockIdx.x;  // global bucket id: s * nb + b
  const int s = (int)(gb / nb);
  const u32 n = hist[gb];
  if (n <= 1 || n > kBucketCap) return;
  const u64 b0 = base[gb];
  const int region = P.region[s];
  const int tid = threadIdx.x;

  for (u32 i = tid; i < kLocalBins; i += blockDim.x) S.bin[i] = 0;
  __syncthreads();
  constexpr int kBatch = 8;
  for (u32 i0 = tid; i0 < n; i0 += kBatch * blockDim.x) {
    u64 kk[kBatch], vv[kBatch];
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      const u32 i = i0 + u * blockDim.x;
      if (i < n) {
        kk[u] = k[b0 + i];
        vv[u] = v[b0 + i];
      }
    }
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      const u32 i = i0 + u * blockDim.x;
      if (i < n) {
        S.k[i] = kk[u];
        S.v[i] = vv[u];
        const u32 l = (bq_quantize(P, s, kk[u]) & ((1u << kLocalBits) - 1)) >> (kLocalBits - kSortBinBits);
        S.lk[i] = (unsigned short)l;
        atomicAdd(&S.bin[l], 1u);
      }
    }
  }
  __syncthreads();
  // Exclusive scan of the local bins (two per thread).
  constexpr int per = kLocalBins / kSortThreadsB;
  u32 loc[per];
  u32 sum = 0;
#pragma unroll
  for (int j = 0; j < per; ++j) {
    loc[j] = S.bin[tid * per + j];
    sum += loc[j];
  }
  const int lane = tid & 31, warp = tid >> 5;
  u32 x = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const u32 y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) S.wsum[warp] = x;
  __syncthreads();
  u32 pre = 0;
  for (int w = 0; w < warp; ++w) pre += S.wsum[w];
  u32 run = pre + x - sum;
#pragma unroll
  for (int j = 0; j < per; ++j) {
    S.bin[tid * per + j] = run;
    run += loc[j];
  }
  __syncthreads();
  for (u32 i = tid; i < n; i += blockDim.x) S.perm[atomicAdd(&S.bin[S.lk[i]], 1u)] = (unsigned short)i;
  __syncthreads();
  // After the counting sort, bin[l] is the end of local key l's run; a run
  // of length >= 2 is a group of equal q, ordered here by the total order.
  u32 found = 0;
  for (u32 l = tid; l < kLocalBins; l += blockDim.x) {
    const u32 end = S.bin[l];
    const u32 beg = l ? S.bin[l - 1] : 0u;
    if (end - beg < 2) continue;
    ++found;
    for (u32 j = beg + 1; j < end; ++j) {
      const unsigned short rx = S.perm[j];
      const u64 kx = S.k[rx], vx = S.v[rx];
      u32 t = j;
      while (t > beg && total_less(region, kx, vx, S.k[S.perm[t - 1]], S.v[S.perm[t - 1]])) {
        S.perm[t] = S.perm[t - 1];
        --t;
      }
      S.perm[t] = rx;
    }
  }
  __syncthreads();
  for (u32 i = tid; i < n; i += blockDim.x) {
    const unsigned short rx = S.perm[i];
    k[b0 + i] = S.k[rx];
    v[b0 + i] = S.v[rx];
  }
  if (found) atomicAdd(ngroups, (unsigned long long)found);
}

// ------------------------------------------------------------------ launchers

void launch_bucket_hist(const u64* kbuf, const BucketPlan& P, u32* hist, cudaStream_t st) {
  const size_t smem = sizeof(u32) << P.bbits;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_bucket_hist, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    configured = true;
  }
  const u64 total = P.cum[P.nseg];
  const u32 grid = (u32)std::min<u64>(148 * 2, (total + 4095) / 4096);
  if (grid) k_bucket_hist<<<grid, 512, smem, st>>>(kbuf, P, hist);
}

void launch_bucket_scan(const u32* hist, const BucketPlan& P, u64* base, u32* cursor, u32* big,
                        u32* nbig, cudaStream_t st) {
  k_bucket_scan<<<P.nseg, 1024, 0, st>>>(hist, P, base, cursor, big, nbig);
}

u32 bucket_scatter_tiles(BucketPlan& P) {
  u32 t = 0;
  for (int s = 0; s < P.nseg; ++s) {
    P.tile_begin[s] = t;
    t += (u32)((P.cum[s + 1] - P.cum[s] + kScatterTile - 1) / kScatterTile);
  }
  P.tile_begin[P.nseg] = t;
  return t;
}

void launch_bucket_scatter(const u64* kin, const u64* vin, u64* kout, u64* vout, const BucketPlan& P,
                           u32 tiles, u32* cursor, cudaStream_t st) {
  const size_t smem = (sizeof(u32) << P.bbits) + kScatterTile * sizeof(unsigned short);
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_bucket_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    configured = true;
  }
  if (tiles) k_bucket_scatter<<<tiles, kScatterThreads, smem, st>>>(kin, vin, kout, vout, P, cursor);
}

void launch_bucket_sort(u64* k, u64* v, const BucketPlan& P, const u64* base, const u32* hist,
                        unsigned long long* ngroups, cudaStream_t st) {
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_bucket_sort, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sizeof(BucketSmem));
    configured = true;
  }
  const u32 nbuckets = (u32)P.nseg << P.bbits;
  k_bucket_sort<<<nbuckets, kSortThreadsB, sizeof(BucketSmem), st>>>(k, v, P, base, hist, ngroups);
}

}  // namespace chgpu
