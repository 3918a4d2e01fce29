// K3: region sort. Replaces sort_region's per-region std::sort
// (reference spa.cpp:59-81) with a segmented onesweep LSD radix sort.
//
// * Records are (k, v) 64-bit pairs (chgpu_internal.cuh codec); ascending
//   (k, v) order is region_less (spa.cpp:38-52).
// * All four regions sort in the same launches: each region is a segment,
//   tiles never straddle segments, and each (segment, digit) bin has its own
//   decoupled look-back chain, so one pass moves every region at once.
// * One histogram pass computes the digit counts of all 8 digit positions;
//   positions where every segment has a single populated bin are skipped.
// * LSD on k alone leaves equal-primary runs in input order; k_tie_detect /
//   k_tie_fix then order each run by v (short runs in shared memory, long
//   runs through the same onesweep engine keyed on v). prim_eq merges -0.0
//   and +0.0 into one run, which is exactly the reference's `==` tie.

#include "chgpu_internal.cuh"
#include "kernels.h"

namespace chgpu {

__device__ __forceinline__ int find_segment(const SegDesc* segs, int nseg, u32 tile) {
  int lo = 0, hi = nseg - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (segs[mid].tile_begin <= tile) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// ------------------------------------------------------------------ histogram

constexpr int kHistThreads = 256;

__global__ __launch_bounds__(kHistThreads) void k_hist(const u64* __restrict__ kin,
                                                       const u64* __restrict__ vin,
                                                       const SegDesc* __restrict__ segs, int nseg,
                                                       u32 total_tiles, int from_v, int use_src,
                                                       u32* __restrict__ hist) {
  __shared__ u32 sh[kPasses][kDigits];
  const u32 per = (total_tiles + gridDim.x - 1) / gridDim.x;
  const u32 t0 = blockIdx.x * per;
  const u32 t1 = min(total_tiles, t0 + per);
  if (t0 >= t1) return;
  for (int i = threadIdx.x; i < kPasses * kDigits; i += blockDim.x) (&sh[0][0])[i] = 0;
  __syncthreads();
  const u64* src = from_v ? vin : kin;
  int seg = find_segment(segs, nseg, t0);
  for (u32 t = t0; t < t1; ++t) {
    while (seg + 1 < nseg && segs[seg + 1].tile_begin <= t) {
      // flush the finished segment
      __syncthreads();
      for (int i = threadIdx.x; i < kPasses * kDigits; i += blockDim.x) {
        const u32 c = (&sh[0][0])[i];
        if (c) {
          atomicAdd(&hist[(size_t)seg * kPasses * kDigits + i], c);
          (&sh[0][0])[i] = 0;
        }
      }
      __syncthreads();
      ++seg;
    }
    const SegDesc sd = segs[seg];
    const u64 e0 = (u64)(t - sd.tile_begin) * kSortTile;
    const u32 cnt = (u32)min((u64)kSortTile, (u64)sd.len - e0);
    const u64 base = (use_src ? sd.src_off : sd.dst_off) + e0;
    for (u32 i = threadIdx.x; i < cnt; i += blockDim.x) {
      const u64 key = src[base + i];
#pragma unroll
      for (int p = 0; p < kPasses; ++p) atomicAdd(&sh[p][(key >> (8 * p)) & 0xFF], 1u);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kPasses * kDigits; i += blockDim.x) {
    const u32 c = (&sh[0][0])[i];
    if (c) atomicAdd(&hist[(size_t)seg * kPasses * kDigits + i], c);
  }
}

// One block per (segment, pass): exclusive digit prefix and the
// "this pass moves something" mask.
__global__ void k_hist_scan(const u32* __restrict__ hist, const SegDesc* __restrict__ segs,
                            u32* __restrict__ digit_excl, u32* __restrict__ needed_mask) {
  const int seg = blockIdx.x / kPasses, pass = blockIdx.x % kPasses;
  const u32* h = hist + ((size_t)seg * kPasses + pass) * kDigits;
  u32* out = digit_excl + ((size_t)seg * kPasses + pass) * kDigits;
  __shared__ u32 s[kDigits];
  __shared__ int s_trivial;
  const int b = threadIdx.x;
  const u32 c = h[b];
  if (b == 0) s_trivial = 0;
  __syncthreads();
  if (c == segs[seg].len) s_trivial = 1;  // every record has the same digit
  s[b] = c;
  __syncthreads();
  // Hillis-Steele inclusive scan over 256 bins.
  for (int o = 1; o < kDigits; o <<= 1) {
    const u32 add = b >= o ? s[b - o] : 0u;
    __syncthreads();
    s[b] += add;
    __syncthreads();
  }
  out[b] = s[b] - c;
  if (b == 0 && !s_trivial && segs[seg].len > 0) atomicOr(needed_mask, 1u << pass);
}

// ------------------------------------------------------------------ onesweep pass

template <bool kFromV>
__global__ __launch_bounds__(kSortThreads, 2) void k_onesweep(
    const u64* __restrict__ kin, const u64* __restrict__ vin, u64* __restrict__ kout,
    u64* __restrict__ vout, const SegDesc* __restrict__ segs, int nseg, int use_src,
    const u32* __restrict__ digit_excl, int pass, u64* __restrict__ status, u32 tag,
    u32* __restrict__ tile_ctr) {
  __shared__ u32 whist[kSortThreads / 32][kDigits];
  __shared__ u32 bin_excl[kDigits];
  __shared__ u64 bin_base[kDigits];
  __shared__ u64 stage[kSortTile];
  __shared__ unsigned char sdig[kSortTile];
  __shared__ u32 s_tile;
  __shared__ int s_seg;
  __shared__ u32 s_wsum[kSortThreads / 32];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    const u32 t = atomicAdd(tile_ctr, 1u);
    s_tile = t;
    s_seg = find_segment(segs, nseg, t);
  }
  for (int i = tid; i < (kSortThreads / 32) * kDigits; i += kSortThreads) (&whist[0][0])[i] = 0;
  __syncthreads();

  const u32 tile = s_tile;
  const int segi = s_seg;
  const SegDesc sd = segs[segi];
  const u64 e0 = (u64)(tile - sd.tile_begin) * kSortTile;
  const u32 cnt = (u32)min((u64)kSortTile, (u64)sd.len - e0);
  const u64 src = (use_src ? sd.src_off : sd.dst_off) + e0;
  const int shift = 8 * pass;

  u64 kk[kSortItems], vv[kSortItems];
  u32 rank[kSortItems];
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const u32 li = warp * (kSortItems * 32) + j * 32 + lane;
    kk[j] = vv[j] = 0;
    if (li < cnt) {
      kk[j] = kin[src + li];
      vv[j] = vin[src + li];
    }
  }
  // Warp-local multisplit: items are ranked in (warp, item, lane) order,
  // which is the input order inside the tile, so the pass is stable.
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const u32 li = warp * (kSortItems * 32) + j * 32 + lane;
    const bool valid = li < cnt;
    const u32 d = (u32)(((kFromV ? vv[j] : kk[j]) >> shift) & 0xFF);
    const u32 key = valid ? d : (0x100u | (u32)lane);
    const unsigned peers = __match_any_sync(0xffffffffu, key);
    const int leader = __ffs(peers) - 1;
    u32 old = 0;
    if (valid && lane == leader) {
      old = whist[warp][d];
      whist[warp][d] = old + __popc(peers);
    }
    old = __shfl_sync(0xffffffffu, old, leader);
    rank[j] = old + __popc(peers & lanemask_lt());
  }
  __syncthreads();

  // Per-bin totals and per-warp exclusive offsets (thread = bin).
  const int b = tid;
  u32 tile_cnt = 0;
#pragma unroll
  for (int w = 0; w < kSortThreads / 32; ++w) {
    const u32 c = whist[w][b];
    whist[w][b] = tile_cnt;
    tile_cnt += c;
  }
  // Block exclusive scan of tile_cnt over bins.
  u32 incl = tile_cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const u32 y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_wsum[warp] = incl;
  __syncthreads();
  u32 wpre = 0;
  for (int w = 0; w < warp; ++w) wpre += s_wsum[w];
  bin_excl[b] = wpre + incl - tile_cnt;

  // Decoupled look-back, one chain per (segment, bin).
  u64* col = status + b;
  u32 before = 0;
  if (tile == sd.tile_begin) {
    store_status(col + (size_t)tile * kDigits, make_status(tag, kFlagPrefix, tile_cnt));
  } else {
    store_status(col + (size_t)tile * kDigits, make_status(tag, kFlagAgg, tile_cnt));
    int j = (int)tile - 1;
    while (true) {
      u64 w;
      u32 f;
      do {
        w = load_status(col + (size_t)j * kDigits);
        f = status_flag(w, tag);
      } while (f == kFlagNone);
      before += (u32)w;
      if (f == kFlagPrefix || j == (int)sd.tile_begin) break;
      --j;
    }
    store_status(col + (size_t)tile * kDigits, make_status(tag, kFlagPrefix, before + tile_cnt));
  }
  bin_base[b] = sd.dst_off + digit_excl[((size_t)segi * kPasses + pass) * kDigits + b] + before -
                bin_excl[b];
  __syncthreads();

  // Scatter through shared memory so global writes of a bin are contiguous.
  u32 lpos[kSortItems];
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const u32 li = warp * (kSortItems * 32) + j * 32 + lane;
    if (li < cnt) {
      const u32 d = (u32)(((kFromV ? vv[j] : kk[j]) >> shift) & 0xFF);
      lpos[j] = bin_excl[d] + whist[warp][d] + rank[j];
      stage[lpos[j]] = kk[j];
      sdig[lpos[j]] = (unsigned char)d;
    }
  }
  __syncthreads();
  for (u32 i = tid; i < cnt; i += kSortThreads) kout[bin_base[sdig[i]] + i] = stage[i];
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const u32 li = warp * (kSortItems * 32) + j * 32 + lane;
    if (li < cnt) stage[lpos[j]] = vv[j];
  }
  __syncthreads();
  for (u32 i = tid; i < cnt; i += kSortThreads) vout[bin_base[sdig[i]] + i] = stage[i];
}

// Moves segments between layouts without reordering (used when every
// digit pass is trivial, and to return tie runs after an odd pass count).
__global__ void k_seg_copy(const u64* __restrict__ kin, const u64* __restrict__ vin,
                           u64* __restrict__ kout, u64* __restrict__ vout,
                           const SegDesc* __restrict__ segs, int nseg, int use_src) {
  const u32 tile = blockIdx.x;
  const int s = find_segment(segs, nseg, tile);
  const SegDesc sd = segs[s];
  const u64 e0 = (u64)(tile - sd.tile_begin) * kSortTile;
  if (e0 >= sd.len) return;
  const u32 cnt = (u32)min((u64)kSortTile, (u64)sd.len - e0);
  const u64 src = (use_src ? sd.src_off : sd.dst_off) + e0, dst = sd.dst_off + e0;
  for (u32 i = threadIdx.x; i < cnt; i += blockDim.x) {
    kout[dst + i] = kin[src + i];
    vout[dst + i] = vin[src + i];
  }
}

// ------------------------------------------------------------------ tie runs

struct TieRun {
  u64 start;
  u32 len;
  int region;
};

// Marks the start of every maximal run (length >= 2) of ==-equal primaries
// inside a segment. One block per 4096-element tile of the region layout.
__global__ void k_tie_detect(const u64* __restrict__ k, const SegDesc* __restrict__ segs,
                             int nseg, u64* __restrict__ starts, u32* __restrict__ nstarts,
                             u32 cap) {
  const u32 tile = blockIdx.x;
  const int s = find_segment(segs, nseg, tile);
  const SegDesc sd = segs[s];
  const u64 e0 = (u64)(tile - sd.tile_begin) * kSortTile;
  if (e0 >= sd.len) return;
  const u32 cnt = (u32)min((u64)kSortTile, (u64)sd.len - e0);
  for (u32 i = threadIdx.x; i < cnt; i += blockDim.x) {
    const u64 pos = e0 + i;  // position inside the segment
    if (pos + 1 >= sd.len) continue;
    const u64 a = sd.dst_off + pos;
    if (!prim_eq(sd.region, k[a], k[a + 1])) continue;
    if (pos > 0 && prim_eq(sd.region, k[a - 1], k[a])) continue;  // not the first of its run
    const u32 slot = atomicAdd(nstarts, 1u);
    if (slot < cap) starts[slot] = ((u64)s << 40) | pos;
  }
}

constexpr int kTieSmem = 2048;

// Orders each run by v. Runs up to kTieSmem records are bitonic-sorted in
// shared memory; longer runs are handed back for the onesweep engine.
__global__ __launch_bounds__(256) void k_tie_fix(u64* __restrict__ k, u64* __restrict__ v,
                                                 const SegDesc* __restrict__ segs,
                                                 const u64* __restrict__ starts, u32 nstarts,
                                                 TieRun* __restrict__ long_runs,
                                                 u32* __restrict__ nlong) {
  __shared__ u64 sk[kTieSmem], sv[kTieSmem];
  __shared__ u32 s_len;
  for (u32 r = blockIdx.x; r < nstarts; r += gridDim.x) {
    const u64 code = starts[r];
    const int s = (int)(code >> 40);
    const u64 pos = code & ((1ull << 40) - 1);
    const SegDesc sd = segs[s];
    const u64 a = sd.dst_off + pos;
    const u64 k0 = k[a];
    // Run length: first index past the run, found 256 at a time.
    if (threadIdx.x == 0) s_len = 0;
    __syncthreads();
    u64 probe = 1;
    while (true) {
      const u64 q = probe + threadIdx.x;
      const bool stop = (pos + q >= sd.len) || !prim_eq(sd.region, k0, k[a + q]);
      const unsigned m = __ballot_sync(0xffffffffu, stop);
      __shared__ u32 s_stop[8];
      if ((threadIdx.x & 31) == 0) s_stop[threadIdx.x >> 5] = m ? (u32)(__ffs(m) - 1) : 0xFFFFFFFFu;
      __syncthreads();
      u32 found = 0xFFFFFFFFu;
      for (int w = 0; w < 8; ++w)
        if (s_stop[w] != 0xFFFFFFFFu) { found = w * 32 + s_stop[w]; break; }
      __syncthreads();
      if (found != 0xFFFFFFFFu) {
        if (threadIdx.x == 0) s_len = (u32)(probe + found);
        break;
      }
      probe += blockDim.x;
    }
    __syncthreads();
    const u32 len = s_len;
    if (len > kTieSmem) {
      if (threadIdx.x == 0) {
        const u32 slot = atomicAdd(nlong, 1u);
        long_runs[slot] = TieRun{a, len, sd.region};
      }
      __syncthreads();
      continue;
    }
    u32 P = 1;
    while (P < len) P <<= 1;
    for (u32 i = threadIdx.x; i < P; i += blockDim.x) {
      sk[i] = i < len ? k[a + i] : ~0ull;
      sv[i] = i < len ? v[a + i] : ~0ull;
    }
    __syncthreads();
    for (u32 size = 2; size <= P; size <<= 1) {
      for (u32 stride = size >> 1; stride > 0; stride >>= 1) {
        for (u32 i = threadIdx.x; i < P; i += blockDim.x) {
          const u32 jx = i ^ stride;
          if (jx > i) {
            const bool up = (i & size) == 0;
            const bool gt = sv[i] > sv[jx] || (sv[i] == sv[jx] && sk[i] > sk[jx]);
            if (gt == up) {
              const u64 tk = sk[i]; sk[i] = sk[jx]; sk[jx] = tk;
              const u64 tv = sv[i]; sv[i] = sv[jx]; sv[jx] = tv;
            }
          }
        }
        __syncthreads();
      }
    }
    for (u32 i = threadIdx.x; i < len; i += blockDim.x) {
      k[a + i] = sk[i];
      v[a + i] = sv[i];
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ launchers

void launch_hist(const u64* kin, const u64* vin, const SegDesc* segs, int nseg, u32 total_tiles,
                 int from_v, int use_src, u32* hist, cudaStream_t st) {
  if (total_tiles == 0) return;
  const int blocks = (int)min(total_tiles, 148u * 4u);
  k_hist<<<blocks, kHistThreads, 0, st>>>(kin, vin, segs, nseg, total_tiles, from_v, use_src, hist);
}

void launch_hist_scan(const u32* hist, const SegDesc* segs, int nseg, u32* digit_excl,
                      u32* needed_mask, cudaStream_t st) {
  if (nseg == 0) return;
  k_hist_scan<<<nseg * kPasses, kDigits, 0, st>>>(hist, segs, digit_excl, needed_mask);
}

void launch_onesweep(const u64* kin, const u64* vin, u64* kout, u64* vout, const SegDesc* segs,
                     int nseg, u32 total_tiles, int use_src, int from_v, const u32* digit_excl,
                     int pass, u64* status, u32 tag, u32* tile_ctr, cudaStream_t st) {
  if (total_tiles == 0) return;
  if (from_v)
    k_onesweep<true><<<total_tiles, kSortThreads, 0, st>>>(kin, vin, kout, vout, segs, nseg, use_src,
                                                           digit_excl, pass, status, tag, tile_ctr);
  else
    k_onesweep<false><<<total_tiles, kSortThreads, 0, st>>>(kin, vin, kout, vout, segs, nseg,
                                                            use_src, digit_excl, pass, status, tag,
                                                            tile_ctr);
}

void launch_seg_copy(const u64* kin, const u64* vin, u64* kout, u64* vout, const SegDesc* segs,
                     int nseg, u32 total_tiles, int use_src, cudaStream_t st) {
  if (total_tiles == 0) return;
  k_seg_copy<<<total_tiles, 256, 0, st>>>(kin, vin, kout, vout, segs, nseg, use_src);
}

void launch_tie_detect(const u64* k, const SegDesc* segs, int nseg, u32 total_tiles, u64* starts,
                       u32* nstarts, u32 cap, cudaStream_t st) {
  if (total_tiles == 0) return;
  k_tie_detect<<<total_tiles, 256, 0, st>>>(k, segs, nseg, starts, nstarts, cap);
}

void launch_tie_fix(u64* k, u64* v, const SegDesc* segs, const u64* starts, u32 nstarts,
                    void* long_runs, u32* nlong, cudaStream_t st) {
  if (nstarts == 0) return;
  const u32 blocks = nstarts < 148u * 8u ? nstarts : 148u * 8u;
  k_tie_fix<<<blocks, 256, 0, st>>>(k, v, segs, starts, nstarts, (TieRun*)long_runs, nlong);
}

size_t tie_run_record_bytes() { return sizeof(TieRun); }

}  // namespace chgpu
