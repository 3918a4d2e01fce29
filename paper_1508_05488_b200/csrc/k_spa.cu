// K4 + K5: SPA second-round discard and chain compaction.
//
// spa_filter (reference spa.cpp:109-163) scans each chunk of a sorted
// region sequentially with a running threshold t that only moves when a
// point is kept. Since a kept point always satisfies g <= t (LL/UL) or
// g >= t (LR/UR), t after any step equals the running min (resp. max) of
// the chunk's seed and every guarded value seen so far, whether kept or
// not. The filter is therefore an exclusive segmented prefix-min/max:
//   keep(i)  <=>  !steps_back(g_i, op(seed_c, g_begin .. g_{i-1}))
// with seed_0 = guarded(anchors.first) (:130-132) and seed_c = the op's
// identity for c > 0, which keeps every later chunk's first point (:134-138).
// One CTA owns one chunk: a block-wide scan per 4096-record tile with the
// carry in registers. Kept records are then compacted, stably and in
// region order, into decoded points with a decoupled look-back over chunks
// (the serial compaction of spa.cpp:158-161).

#include <math.h>

#include "chgpu_internal.cuh"
#include "kernels.h"

namespace chgpu {

constexpr int kSpaThreads = 256;
constexpr int kSpaItems = 16;
constexpr int kSpaTile = kSpaThreads * kSpaItems;


// Block-wide exclusive scan with op_ext; returns the exclusive value for
// this thread and the block aggregate in *agg.
__device__ __forceinline__ double block_excl_ext(bool is_min, double x, double ident, double* sw,
                                                 double* agg) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double incl = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl = op_ext(is_min, y, incl);
  }
  double excl_w = __shfl_up_sync(0xffffffffu, incl, 1);
  if (lane == 0) excl_w = ident;
  if (lane == 31) sw[warp] = incl;
  __syncthreads();
  double pre = ident;
  for (int w = 0; w < warp; ++w) pre = op_ext(is_min, pre, sw[w]);
  double tot = ident;
  for (int w = 0; w < kSpaThreads / 32; ++w) tot = op_ext(is_min, tot, sw[w]);
  *agg = tot;
  __syncthreads();
  return op_ext(is_min, pre, excl_w);
}

__device__ __forceinline__ u32 block_excl_sum(u32 x, u32* sw, u32* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  u32 incl = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const u32 y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) sw[warp] = incl;
  __syncthreads();
  u32 pre = 0, tot = 0;
  for (int w = 0; w < kSpaThreads / 32; ++w) {
    if (w < warp) pre += sw[w];
    tot += sw[w];
  }
  *total = tot;
  __syncthreads();
  return pre + incl - x;
}

// Degenerate branch: unique over the lexicographically sorted survivors
// (oracle.cpp:16-17 std::sort + std::unique), compacted in order.
__global__ __launch_bounds__(kSpaThreads) void k_unique(const u64* __restrict__ k,
                                                        const u64* __restrict__ v, u64 n,
                                                        double2* __restrict__ out,
                                                        u64* __restrict__ status, u32 tag,
                                                        u32* __restrict__ tile_ctr,
                                                        unsigned long long* __restrict__ total) {
  __shared__ u32 swu[kSpaThreads / 32];
  __shared__ u32 s_tile, s_excl;
  const int tid = threadIdx.x;
  if (tid == 0) s_tile = atomicAdd(tile_ctr, 1u);
  __syncthreads();
  const u32 tile = s_tile;
  const u64 t0 = (u64)tile * kSpaTile;
  unsigned char f[kSpaItems];
  u32 mine = 0;
#pragma unroll
  for (int j = 0; j < kSpaItems; ++j) {
    const u64 i = t0 + tid * kSpaItems + j;
    f[j] = 0;
    if (i < n) {
      if (i == 0) {
        f[j] = 1;
      } else {
        double x0, y0, x1, y1;
        decode_point(0, k[i - 1], v[i - 1], x0, y0);
        decode_point(0, k[i], v[i], x1, y1);
        f[j] = (x0 == x1 && y0 == y1) ? 0 : 1;
      }
    }
    mine += f[j];
  }
  u32 tile_cnt;
  const u32 lpos = block_excl_sum(mine, swu, &tile_cnt);
  if (tid < 32) {
    u32 excl = 0;
    if (tile == 0) {
      if (tid == 0) store_status(status, make_status(tag, kFlagPrefix, tile_cnt));
    } else {
      if (tid == 0) store_status(status + tile, make_status(tag, kFlagAgg, tile_cnt));
      excl = warp_lookback(status, 1, (int)tile, 0, tag);
      if (tid == 0) store_status(status + tile, make_status(tag, kFlagPrefix, excl + tile_cnt));
    }
    if (tid == 0) {
      s_excl = excl;
      if (tile_cnt) atomicAdd(total, (unsigned long long)tile_cnt);
    }
  }
  __syncthreads();
  u32 pos = s_excl + lpos;
#pragma unroll
  for (int j = 0; j < kSpaItems; ++j) {
    if (f[j]) {
      const u64 i = t0 + tid * kSpaItems + j;
      double x, y;
      decode_point(0, k[i], v[i], x, y);
      out[pos++] = make_double2(x, y);
    }
  }
}

void launch_unique(const u64* k, const u64* v, u64 n, double2* out, u64* status, u32 tag,
                   u32* tile_ctr, unsigned long long* total, cudaStream_t st) {
  const u64 tiles = (n + kSpaTile - 1) / kSpaTile;
  if (tiles == 0) return;
  k_unique<<<(unsigned)tiles, kSpaThreads, 0, st>>>(k, v, n, out, status, tag, tile_ctr, total);
}

}  // namespace chgpu

namespace chgpu {

// ------------------------------------------------------------------ SPA, warp per chunk
//
// One warp scans one chunk, 256 records per step (8 coalesced rows of 32),
// with a shuffle scan per row and the carry in a register: no block
// barriers and no inter-chunk dependency. Kept records are written,
// decoded, compactly at the start of the chunk's own range of a scratch
// array (ranges never overlap); k_spa_offsets scans the per-chunk counts and
// k_spa_gather moves each chunk's run to its final, region-ordered place.

constexpr int kSpaPer = 8;                  // consecutive records per lane and step
constexpr int kSpaStep = 32 * kSpaPer;      // records per warp step

// Lane L of a step owns records [t0 + 8L, t0 + 8L + 8): it folds them
// sequentially, one warp scan combines the 32 lane aggregates, and the lane
// replays its 8 records against the exclusive prefix. The next step's loads
// are issued before the current step is scanned.
__global__ __launch_bounds__(256) void k_spa_warp(const u64* __restrict__ k,
                                                  const u64* __restrict__ v,
                                                  const SpaPlan* __restrict__ plan_p,
                                                  double2* __restrict__ scratch,
                                                  u32* __restrict__ chunk_kept) {
  const SpaPlan& plan = *plan_p;
  const int lane = threadIdx.x & 31;
  const u32 c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (c >= plan.total_chunks) return;
  int r = 0;
  while (r < 3 && c >= plan.chunk_begin[r + 1]) ++r;
  const int region = r + 1;
  const u64 cl = c - plan.chunk_begin[r];
  const u64 begin = plan.off[r] + cl * plan.chunk_size[r];
  const u64 len = min((u64)plan.chunk_size[r], (u64)plan.m[r] - cl * plan.chunk_size[r]);
  const bool is_min = (region == 1 || region == 4);
  const double ident = is_min ? INFINITY : -INFINITY;
  double carry = (cl == 0) ? plan.seed[r] : ident;
  u32 kept = 0;

  u64 nv[kSpaPer];
  auto fetch = [&](u64 t0) {
#pragma unroll
    for (int j = 0; j < kSpaPer; ++j) {
      const u64 idx = t0 + (u64)lane * kSpaPer + j;
      nv[j] = idx < len ? v[begin + idx] : 0ull;
    }
  };
  fetch(0);
  for (u64 t0 = 0; t0 < len; t0 += kSpaStep) {
    double g[kSpaPer];
    double agg = ident;
#pragma unroll
    for (int j = 0; j < kSpaPer; ++j) {
      const u64 idx = t0 + (u64)lane * kSpaPer + j;
      g[j] = idx < len ? guarded_of(region, nv[j]) : ident;
      agg = op_ext(is_min, agg, g[j]);
    }
    if (t0 + kSpaStep < len) fetch(t0 + kSpaStep);
    double x = agg;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x = op_ext(is_min, y, x);
    }
    double ex = __shfl_up_sync(0xffffffffu, x, 1);
    if (lane == 0) ex = ident;
    double t = op_ext(is_min, carry, ex);
    carry = op_ext(is_min, carry, __shfl_sync(0xffffffffu, x, 31));
    u32 kmask = 0;
#pragma unroll
    for (int j = 0; j < kSpaPer; ++j) {
      const u64 idx = t0 + (u64)lane * kSpaPer + j;
      if (idx < len && !steps_back(is_min, g[j], t)) kmask |= 1u << j;
      t = op_ext(is_min, t, g[j]);
    }
    const u32 nk = __popc(kmask);
    u32 pre = nk;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const u32 y = __shfl_up_sync(0xffffffffu, pre, o);
      if (lane >= o) pre += y;
    }
    u32 pos = kept + pre - nk;
    kept += __shfl_sync(0xffffffffu, pre, 31);
    while (kmask) {
      const int j = __ffs(kmask) - 1;
      kmask &= kmask - 1;
      const u64 a = begin + t0 + (u64)lane * kSpaPer + j;
      double px, py;
      decode_point(region, k[a], v[a], px, py);
      scratch[begin + pos++] = make_double2(px, py);
    }
  }
  if (lane == 0) chunk_kept[c] = kept;
}

// Exclusive scan of the per-chunk kept counts (one block); per-region
// totals follow from the offsets at the region boundaries.
__global__ __launch_bounds__(1024) void k_spa_offsets(const u32* __restrict__ chunk_kept,
                                                      const SpaPlan* __restrict__ plan_p,
                                                      u32* __restrict__ offs,
                                                      unsigned long long* __restrict__ kept_counts) {
  const SpaPlan& plan = *plan_p;
  __shared__ u32 wsum[32];
  __shared__ u32 carry;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const u32 total = plan.total_chunks;
  for (u32 c0 = 0; c0 < total; c0 += blockDim.x) {
    const u32 c = c0 + threadIdx.x;
    const u32 x0 = c < total ? chunk_kept[c] : 0u;
    u32 x = x0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const u32 y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    u32 pre = 0, tot = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      const u32 ws = wsum[w];
      pre += (w < warp) ? ws : 0u;
      tot += ws;
    }
    if (c < total) offs[c] = carry + pre + x - x0;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const u32 grand = carry;
    for (int r = 0; r < 4; ++r) {
      const u32 a = plan.chunk_begin[r];
      const u32 b = r < 3 ? plan.chunk_begin[r + 1] : total;
      const u32 oa = a < total ? offs[a] : grand;
      const u32 ob = b < total ? offs[b] : grand;
      kept_counts[r] = (unsigned long long)(ob - oa);
    }
  }
}

__global__ __launch_bounds__(256) void k_spa_gather(const double2* __restrict__ scratch,
                                                    const SpaPlan* __restrict__ plan_p,
                                                    const u32* __restrict__ chunk_kept,
                                                    const u32* __restrict__ offs,
                                                    double2* __restrict__ out) {
  const SpaPlan& plan = *plan_p;
  const int lane = threadIdx.x & 31;
  const u32 c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (c >= plan.total_chunks) return;
  const u32 kc = chunk_kept[c];
  if (!kc) return;
  int r = 0;
  while (r < 3 && c >= plan.chunk_begin[r + 1]) ++r;
  const u64 begin = plan.off[r] + (u64)(c - plan.chunk_begin[r]) * plan.chunk_size[r];
  const u32 o = offs[c];
  for (u32 i = lane; i < kc; i += 32) out[o + i] = scratch[begin + i];
}


void launch_spa_warp(const u64* k, const u64* v, const SpaPlan* plan, u32 max_chunks,
                     double2* scratch, u32* chunk_kept, u32* offs,
                     unsigned long long* kept_counts, double2* out, cudaStream_t st) {
  if (max_chunks == 0) return;
  const u32 blocks = (max_chunks + 7) / 8;
  k_spa_warp<<<blocks, 256, 0, st>>>(k, v, plan, scratch, chunk_kept);
  k_spa_offsets<<<1, 1024, 0, st>>>(chunk_kept, plan, offs, kept_counts);
  k_spa_gather<<<blocks, 256, 0, st>>>(scratch, plan, chunk_kept, offs, out);
}

}  // namespace chgpu
