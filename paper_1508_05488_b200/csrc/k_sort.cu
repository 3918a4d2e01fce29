// K3: region sort. Replaces sort_region's per-region std::sort
// (reference spa.cpp:59-81).
//
// Records are (k, v) 64-bit pairs (chgpu_internal.cuh codec): ascending
// (k, v) with -0.0/+0.0 merged is region_less (spa.cpp:38-52). The sort
// runs in two phases, both over all four regions at once (one segment per
// region, tiles never straddle segments, one decoupled look-back chain per
// (segment, digit)):
//
//  1. Bucket phase: a segmented onesweep LSD radix sort keyed on
//     q = quantize(primary) with 24 or 32 bits, a monotone map of the
//     region's primary coordinate onto [0, 2^bits) (monotone because
//     subtraction, multiplication by a positive constant, clamping and
//     truncation are all monotone in IEEE round-to-nearest). It moves each
//     record to its final bucket in 3-4 passes instead of the 8 a 64-bit
//     key needs.
//  2. Group phase: runs of equal q (a few percent of records for smooth
//     inputs) are ordered by the full key (kc, v) in place: a thread per
//     run up to 16 records, a block-wide bitonic sort up to 2048, and the
//     same onesweep engine keyed on k then v beyond that.
//
// Every launch uses (segment, bin) tagged look-back words, so the status
// array never needs clearing.

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

// Monotone quantizer of the primary coordinate (see header comment).
__device__ __forceinline__ u32 quantize(const SegDesc& s, u64 k) {
  const double p = primary_of(s.region, k);
  const double qmax = s.qmax;
  double t = __dmul_rn(__dsub_rn(p, s.qlo), s.qscale);
  t = fmin(fmax(t, 0.0), qmax);
  const u32 q = (u32)__double2ull_rz(t);
  return (s.region == 3 || s.region == 4) ? (u32)((u64)qmax - q) : q;
}


template <int kMode>
__device__ __forceinline__ u32 digit_of(const SegDesc& s, u64 k, u64 v, int pass) {
  if (kMode == kDigitQ) return (quantize(s, k) >> (8 * pass)) & 0xFFu;
  if (kMode == kDigitV) return (u32)(v >> (8 * pass)) & 0xFFu;
  return (u32)(k >> (8 * pass)) & 0xFFu;
}

// ------------------------------------------------------------------ histogram

constexpr int kHistThreads = 256;

template <int kMode>
__global__ __launch_bounds__(kHistThreads) void k_hist(const u64* __restrict__ kin,
                                                       const u64* __restrict__ vin,
                                                       const SegDesc* __restrict__ segs, int nseg,
                                                       u32 total_tiles, int npasses, int use_src,
                                                       u32* __restrict__ hist) {
  __shared__ u32 sh[kPasses][kDigits];
  const u32 per = (total_tiles + gridDim.x - 1) / gridDim.x;
  const u32 t0 = blockIdx.x * per;
  const u32 t1 = min(total_tiles, t0 + per);
  if (t0 >= t1) return;
  for (int i = threadIdx.x; i < kPasses * kDigits; i += blockDim.x) (&sh[0][0])[i] = 0;
  __syncthreads();
  int seg = find_segment(segs, nseg, t0);
  for (u32 t = t0; t < t1; ++t) {
    while (seg + 1 < nseg && segs[seg + 1].tile_begin <= t) {
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
      const u64 k = kMode == kDigitV ? 0 : kin[base + i];
      const u64 v = kMode == kDigitV ? vin[base + i] : 0;
      if (kMode == kDigitQ) {
        const u32 q = quantize(sd, k);
        for (int p = 0; p < npasses; ++p) atomicAdd(&sh[p][(q >> (8 * p)) & 0xFF], 1u);
      } else {
        const u64 key = kMode == kDigitV ? v : k;
        for (int p = 0; p < npasses; ++p) atomicAdd(&sh[p][(key >> (8 * p)) & 0xFF], 1u);
      }
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
                            int npasses, u32* __restrict__ digit_excl, u32* __restrict__ needed_mask) {
  const int seg = blockIdx.x / kPasses, pass = blockIdx.x % kPasses;
  if (pass >= npasses) return;
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

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gmem) : "memory");
}

struct OnesweepSmem {
  u32 whist[kSortThreads / 32][kDigits];  // per-warp digit counters, then offsets
  u32 bin_excl[kDigits];                  // tile-local exclusive prefix over digits
  u64 bin_base[kDigits];                  // global destination base per digit
  u64 kstage[kSortTile];                  // keys in tile-sorted order
  u64 vraw[kSortTile];                    // values in load order (cp.async)
  unsigned short perm[kSortTile];         // tile-sorted position -> load position
  unsigned char sdig[kSortTile];          // digit of each tile-sorted record
  u32 wsum[kSortThreads / 32];
  u32 tile;
  int seg;
};

// One LSD pass. Keys stay in registers for the ranking; values travel
// global -> shared with cp.async and are only touched again by the scatter,
// so a thread holds kSortItems keys and nothing else across the pass.
//
// kScan = false: one-pass ("onesweep") with a decoupled look-back for the
// per-(tile, digit) global offsets. kScan = true: the downsweep of a
// reduce-then-scan pass, reading those offsets from tile_prefix (written by
// k_upsweep + k_colscan), so tiles never wait on each other.
template <int kMode, bool kScan>
#ifndef CHGPU_SORT_MINB
#define CHGPU_SORT_MINB 3
#endif
__global__ __launch_bounds__(kSortThreads, CHGPU_SORT_MINB) void k_onesweep(
    const u64* __restrict__ kin, const u64* __restrict__ vin, u64* __restrict__ kout,
    u64* __restrict__ vout, const SegDesc* __restrict__ segs, int nseg, int use_src,
    const u32* __restrict__ digit_excl, int pass, u64* __restrict__ status, u32 tag,
    u32* __restrict__ tile_ctr, u32 total_tiles, u32* __restrict__ rows) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  OnesweepSmem& S = *reinterpret_cast<OnesweepSmem*>(smem_raw);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // reduce-then-scan: this (tile, digit)'s offset from k_colscan (digit-
  // major), loaded now so its latency hides behind the tile load and ranking
  const u32 scan_before = kScan ? __ldcg(rows + (size_t)tid * total_tiles + blockIdx.x) : 0u;
  if (tid == 0) {
    const u32 t = kScan ? blockIdx.x : atomicAdd(tile_ctr, 1u);
    S.tile = t;
    S.seg = find_segment(segs, nseg, t);
  }
  for (int i = tid; i < (kSortThreads / 32) * kDigits; i += kSortThreads) (&S.whist[0][0])[i] = 0;
  __syncthreads();

  const u32 tile = S.tile;
  const int segi = S.seg;
  const SegDesc sd = segs[segi];
  const u64 e0 = (u64)(tile - sd.tile_begin) * kSortTile;
  const u32 cnt = (u32)min((u64)kSortTile, (u64)sd.len - e0);
  const u64 src = (use_src ? sd.src_off : sd.dst_off) + e0;
  const u32 wbase = warp * (kSortItems * 32);

  // The digit source word (v for kDigitV, else k) stays in registers; the
  // other word rides along through shared memory.
  const u64* rin = kMode == kDigitV ? vin : kin;
  const u64* oin = kMode == kDigitV ? kin : vin;
  u64 kk[kSortItems];
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const u32 li = wbase + j * 32 + lane;
    kk[j] = 0;
    if (li < cnt) {
      kk[j] = rin[src + li];
      cp_async8(&S.vraw[li], oin + src + li);
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");

  // Warp-local multisplit: items are ranked in (warp, item, lane) order,
  // which is the input order inside the tile, so the pass is stable. The
  // peer masks are independent of each other and are computed first; only
  // the per-warp counter updates form a chain.
  unsigned peers[kSortItems];
  u32 dig[kSortItems];
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const u32 li = wbase + j * 32 + lane;
    const bool valid = li < cnt;
    dig[j] = digit_of<kMode>(sd, kk[j], kk[j], pass);
    peers[j] = __match_any_sync(0xffffffffu, valid ? dig[j] : (0x100u | (u32)lane));
  }
  u32 code[kSortItems];  // digit | rank << 8
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const u32 li = wbase + j * 32 + lane;
    const bool valid = li < cnt;
    const u32 d = dig[j];
    const int leader = __ffs(peers[j]) - 1;
    u32 old = 0;
    if (valid && lane == leader) {
      old = S.whist[warp][d];
      S.whist[warp][d] = old + __popc(peers[j]);
    }
    old = __shfl_sync(0xffffffffu, old, leader);
    code[j] = d | ((old + __popc(peers[j] & lanemask_lt())) << 8);
    __syncwarp();  // (orders this leader's counter write before the next item's leader reads it)
  }
  __syncthreads();

  // Per-bin totals and per-warp exclusive offsets (thread = bin).
  const int b = tid;
  u32 tile_cnt = 0;
#pragma unroll
  for (int w = 0; w < kSortThreads / 32; ++w) {
    const u32 c = S.whist[w][b];
    S.whist[w][b] = tile_cnt;
    tile_cnt += c;
  }
  u32 incl = tile_cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const u32 y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) S.wsum[warp] = incl;
  __syncthreads();
  u32 wpre = 0;
  for (int w = 0; w < warp; ++w) wpre += S.wsum[w];
  const u32 bexcl = wpre + incl - tile_cnt;
  S.bin_excl[b] = bexcl;

  // Tile-level decoupled look-back. status[0, T) holds one flag word per
  // tile; agg[T][256] and inc[T][256] (u32, after the flags) hold the
  // per-digit tile counts and inclusive prefixes. A tile publishes its whole
  // row at once, so the look-back finds the nearest predecessor with a
  // prefix using one warp over 32 flags at a time and then reads the rows in
  // between with independent loads: a few round trips whatever the depth.
  // rows: kScan = the per-(tile, digit) offsets from k_colscan; onesweep =
  // the published per-tile counts (agg) and inclusive prefixes (inc), raw
  // words kept apart from the tagged status words
  u32* agg = rows;
  u32* inc = agg + (size_t)total_tiles * kDigits;
  u32 before = 0;
  // Publication is the release pattern "row stores; bar.sync; one thread:
  // fence.acq_rel.gpu + flag store"; readers acquire the flag in one warp
  // and bar.sync before touching rows.
  if (kScan) {
    before = scan_before;
  } else if (tile == sd.tile_begin) {
    __stcg(inc + (size_t)tile * kDigits + b, tile_cnt);
    __syncthreads();
    if (tid == 0) {
      fence_acq_rel_gpu();
      store_status(status + tile, make_status(tag, kFlagPrefix, 0));
    }
  } else {
    __stcg(agg + (size_t)tile * kDigits + b, tile_cnt);
    __syncthreads();
    if (warp == 0) {
      if (lane == 0) {
        fence_acq_rel_gpu();
        store_status(status + tile, make_status(tag, kFlagAgg, 0));
      }
      int base = (int)tile - 1;
      int front;
      while (true) {
        const int j = base - lane;
        u32 f = kFlagPrefix;  // the segment's first tile always holds a prefix
        if (j >= (int)sd.tile_begin) {
          do {
            f = status_flag(load_status(status + j), tag);
          } while (f == kFlagNone);
        }
        const unsigned pm = __ballot_sync(0xffffffffu, f == kFlagPrefix);
        if (pm) {
          front = base - (__ffs(pm) - 1);
          break;
        }
        base -= 32;
      }
      if (lane == 0) S.seg = front;  // reuse: frontier tile
      fence_acq_rel_gpu();            // acquire for the flags observed above
    }
    __syncthreads();
    const int front = S.seg;
    before = __ldcg(inc + (size_t)front * kDigits + b);
    int j = front + 1;
    for (; j + 3 < (int)tile; j += 4) {
      const u32 a0 = __ldcg(agg + (size_t)j * kDigits + b);
      const u32 a1 = __ldcg(agg + (size_t)(j + 1) * kDigits + b);
      const u32 a2 = __ldcg(agg + (size_t)(j + 2) * kDigits + b);
      const u32 a3 = __ldcg(agg + (size_t)(j + 3) * kDigits + b);
      before += a0 + a1 + a2 + a3;
    }
    for (; j < (int)tile; ++j) before += __ldcg(agg + (size_t)j * kDigits + b);
    __stcg(inc + (size_t)tile * kDigits + b, before + tile_cnt);
    __syncthreads();
    if (tid == 0) {
      fence_acq_rel_gpu();
      store_status(status + tile, make_status(tag, kFlagPrefix, 0));
    }
  }
  u32 dex = digit_excl[((size_t)segi * kPasses + pass) * kDigits + b];
  if (kScan) {
    // reduce-then-scan: k_colscan left the segment's raw digit totals of
    // this pass there; their exclusive scan over digits is the digit base
    u32 incl = dex;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const u32 y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    __syncthreads();  // (S.wsum was read above for the tile's bin offsets)
    if (lane == 31) S.wsum[warp] = incl;
    __syncthreads();
    u32 wp = 0;
    for (int w = 0; w < warp; ++w) wp += S.wsum[w];
    dex = wp + incl - dex;
  }
  S.bin_base[b] = sd.dst_off + dex + before - bexcl;
  __syncthreads();

  // Tile-sorted staging: keys, load positions and digits.
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const u32 li = wbase + j * 32 + lane;
    if (li < cnt) {
      const u32 d = code[j] & 0xFF;
      const u32 lp = S.bin_excl[d] + S.whist[warp][d] + (code[j] >> 8);
      S.kstage[lp] = kk[j];
      S.perm[lp] = (unsigned short)li;
      S.sdig[lp] = (unsigned char)d;
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  // Scatter: consecutive sorted positions of a digit are consecutive in
  // global memory, so warps write contiguous runs.
  u64* rout = kMode == kDigitV ? vout : kout;
  u64* oout = kMode == kDigitV ? kout : vout;
#pragma unroll 4
  for (u32 i = tid; i < cnt; i += kSortThreads) {
    const u64 dst = S.bin_base[S.sdig[i]] + i;
    rout[dst] = S.kstage[i];
    oout[dst] = S.vraw[S.perm[i]];
  }
}

// Moves segments between layouts without reordering (used when every
// digit pass is trivial, and to return runs after an odd pass count).
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

// ------------------------------------------------------------------ groups

// Group = maximal run (length >= 2) of records that compare equal under
//   kEqQ:    equal quantized primary (bucket-phase leftovers), or
//   kEqPrim: ==-equal primary (after a full sort on k).
// Both are then ordered by (canon_k, v), which is region_less.
__device__ __forceinline__ bool group_eq(int eqmode, const SegDesc& s, u64 a, u64 b) {
  return eqmode == kEqQ ? quantize(s, a) == quantize(s, b) : prim_eq(s.region, a, b);
}


struct GroupRun {
  u64 start;  // absolute record index
  u32 len;
  int seg;
};

constexpr int kSmallGroup = 16;
constexpr int kMediumGroup = 2048;

// Group key: equal keys <=> same group (q for kEqQ; canonical k, i.e. the
// primary under ==, for kEqPrim).
__device__ __forceinline__ u64 group_key(int eqmode, const SegDesc& s, u64 k) {
  return eqmode == kEqQ ? (u64)quantize(s, k) : canon_k(s.region, k);
}

// Detects group starts tile by tile and fixes each group on the spot: the
// group keys of the tile's records plus a kSmallGroup halo are computed
// once (coalesced k reads) into shared memory, the thread owning a group
// start insertion-sorts it in registers when it holds at most kSmallGroup
// records (reading and writing only that group's k and v); longer groups
// are queued for k_group_fix_medium.
constexpr int kGroupWin = kSortTile + kSmallGroup + 1;
struct GroupSmem {
  u64 g[kGroupWin + 1];  // g[0]: group key of the record before the tile
};

__global__ __launch_bounds__(256) void k_group_scan(u64* __restrict__ k, u64* __restrict__ v,
                                                    const SegDesc* __restrict__ segs, int nseg,
                                                    int eqmode, GroupRun* __restrict__ medium,
                                                    u32* __restrict__ nmedium,
                                                    unsigned long long* __restrict__ ngroups) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  GroupSmem& S = *reinterpret_cast<GroupSmem*>(smem_raw);
  __shared__ u32 s_found;
  const u32 tile = blockIdx.x;
  const int s = find_segment(segs, nseg, tile);
  const SegDesc sd = segs[s];
  const u64 e0 = (u64)(tile - sd.tile_begin) * kSortTile;
  if (e0 >= sd.len) return;
  const u32 cnt = (u32)min((u64)kSortTile, (u64)sd.len - e0);
  const u32 win = (u32)min((u64)cnt + kSmallGroup + 1, (u64)sd.len - e0);
  const u64 base = sd.dst_off + e0;
  if (threadIdx.x == 0) {
    s_found = 0;
    S.g[0] = e0 > 0 ? group_key(eqmode, sd, k[base - 1]) : ~0ull;
  }
  for (u32 i = threadIdx.x; i < win; i += blockDim.x) S.g[i + 1] = group_key(eqmode, sd, k[base + i]);
  __syncthreads();
  u32 found = 0;
  for (u32 i = threadIdx.x; i < cnt; i += blockDim.x) {
    if (i + 1 >= win || S.g[i + 1] != S.g[i + 2]) continue;  // no successor in the group
    if (S.g[i] == S.g[i + 1]) continue;                        // not the first of its group
    ++found;
    const u64 g0 = S.g[i + 1];
    u32 len = 2;
    while (i + len < win && S.g[i + len + 1] == g0) ++len;
    if (len > kSmallGroup || (i + len == win && e0 + win < sd.len)) {
      // Longer than the halo: measure it in global memory, queue it.
      const u64 a = base + i;
      while (e0 + i + len < sd.len && group_key(eqmode, sd, k[a + len]) == g0) ++len;
      if (len <= kSmallGroup) goto small;  // ended right at the window edge
      medium[atomicAdd(nmedium, 1u)] = GroupRun{a, len, s};
      continue;
    }
  small : {
    // (a few percent of the records: the group is sorted in registers,
    // read and written back in global memory)
    u64 gk[kSmallGroup], gv[kSmallGroup];
    for (u32 j = 0; j < len; ++j) {
      const u64 kx = k[base + i + j], vx = v[base + i + j];
      u32 t = j;
      while (t > 0 && rec_less(sd.region, kx, vx, gk[t - 1], gv[t - 1])) {
        gk[t] = gk[t - 1];
        gv[t] = gv[t - 1];
        --t;
      }
      gk[t] = kx;
      gv[t] = vx;
    }
    for (u32 j = 0; j < len; ++j) {
      k[base + i + j] = gk[j];
      v[base + i + j] = gv[j];
    }
  }
  }
  if (found) atomicAdd(&s_found, found);
  __syncthreads();
  if (threadIdx.x == 0 && s_found) atomicAdd(ngroups, (unsigned long long)s_found);
}

// One block per medium group: bitonic sort in shared memory; groups longer
// than kMediumGroup are handed back for the onesweep engine.
__global__ __launch_bounds__(256) void k_group_fix_medium(u64* __restrict__ k, u64* __restrict__ v,
                                                          const SegDesc* __restrict__ segs,
                                                          const GroupRun* __restrict__ medium,
                                                          const u32* __restrict__ nmedium_p,
                                                          GroupRun* __restrict__ longr,
                                                          u32* __restrict__ nlong) {
  __shared__ u64 sk[kMediumGroup], sv[kMediumGroup], sc[kMediumGroup];
  const u32 nmedium = *nmedium_p;
  for (u32 r = blockIdx.x; r < nmedium; r += gridDim.x) {
    const GroupRun g = medium[r];
    if (g.len > kMediumGroup) {
      if (threadIdx.x == 0) longr[atomicAdd(nlong, 1u)] = g;
      continue;
    }
    const int region = segs[g.seg].region;
    u32 P = 1;
    while (P < g.len) P <<= 1;
    for (u32 i = threadIdx.x; i < P; i += blockDim.x) {
      if (i < g.len) {
        sk[i] = k[g.start + i];
        sv[i] = v[g.start + i];
        sc[i] = canon_k(region, sk[i]);
      } else {
        sk[i] = sv[i] = sc[i] = ~0ull;
      }
    }
    __syncthreads();
    for (u32 size = 2; size <= P; size <<= 1) {
      for (u32 stride = size >> 1; stride > 0; stride >>= 1) {
        for (u32 i = threadIdx.x; i < P; i += blockDim.x) {
          const u32 jx = i ^ stride;
          if (jx > i) {
            const bool up = (i & size) == 0;
            const bool gt = sc[i] > sc[jx] ||
                            (sc[i] == sc[jx] && (sv[i] > sv[jx] || (sv[i] == sv[jx] && sk[i] > sk[jx])));
            if (gt == up) {
              u64 t = sk[i]; sk[i] = sk[jx]; sk[jx] = t;
              t = sv[i]; sv[i] = sv[jx]; sv[jx] = t;
              t = sc[i]; sc[i] = sc[jx]; sc[jx] = t;
            }
          }
        }
        __syncthreads();
      }
    }
    for (u32 i = threadIdx.x; i < g.len; i += blockDim.x) {
      k[g.start + i] = sk[i];
      v[g.start + i] = sv[i];
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ launchers

void launch_hist(const u64* kin, const u64* vin, const SegDesc* segs, int nseg, u32 total_tiles,
                 int mode, int npasses, int use_src, u32* hist, cudaStream_t st) {
  if (total_tiles == 0) return;
  const int blocks = (int)min(total_tiles, 148u * 4u);
  switch (mode) {
    case kDigitQ:
      k_hist<kDigitQ><<<blocks, kHistThreads, 0, st>>>(kin, vin, segs, nseg, total_tiles, npasses,
                                                       use_src, hist);
      break;
    case kDigitV:
      k_hist<kDigitV><<<blocks, kHistThreads, 0, st>>>(kin, vin, segs, nseg, total_tiles, npasses,
                                                       use_src, hist);
      break;
    default:
      k_hist<kDigitK><<<blocks, kHistThreads, 0, st>>>(kin, vin, segs, nseg, total_tiles, npasses,
                                                       use_src, hist);
  }
}

void launch_hist_scan(const u32* hist, const SegDesc* segs, int nseg, int npasses, u32* digit_excl,
                      u32* needed_mask, cudaStream_t st) {
  if (nseg == 0) return;
  k_hist_scan<<<nseg * kPasses, kDigits, 0, st>>>(hist, segs, npasses, digit_excl, needed_mask);
}

template <int kMode, bool kScan>
static void onesweep_launch(const u64* kin, const u64* vin, u64* kout, u64* vout,
                            const SegDesc* segs, int nseg, u32 total_tiles, int use_src,
                            const u32* digit_excl, int pass, u64* status, u32 tag, u32* tile_ctr,
                            u32* rows, cudaStream_t st) {
  k_onesweep<kMode, kScan><<<total_tiles, kSortThreads, sizeof(OnesweepSmem), st>>>(
      kin, vin, kout, vout, segs, nseg, use_src, digit_excl, pass, status, tag, tile_ctr,
      total_tiles, rows);
}

void launch_onesweep(const u64* kin, const u64* vin, u64* kout, u64* vout, const SegDesc* segs,
                     int nseg, u32 total_tiles, int use_src, int mode, const u32* digit_excl,
                     int pass, u64* status, u32 tag, u32* tile_ctr, u32* rows, cudaStream_t st) {
  if (total_tiles == 0) return;
  switch (mode) {
    case kDigitQ:
      onesweep_launch<kDigitQ, false>(kin, vin, kout, vout, segs, nseg, total_tiles, use_src,
                                      digit_excl, pass, status, tag, tile_ctr, rows, st);
      break;
    case kDigitV:
      onesweep_launch<kDigitV, false>(kin, vin, kout, vout, segs, nseg, total_tiles, use_src,
                                      digit_excl, pass, status, tag, tile_ctr, rows, st);
      break;
    default:
      onesweep_launch<kDigitK, false>(kin, vin, kout, vout, segs, nseg, total_tiles, use_src,
                                      digit_excl, pass, status, tag, tile_ctr, rows, st);
  }
}

// ------------------------------------------------------------------ reduce-then-scan pass

// Upsweep: the digit histogram of every tile (same tiling as the downsweep).
template <int kMode>
__global__ __launch_bounds__(kSortThreads) void k_upsweep(const u64* __restrict__ kin,
                                                          const u64* __restrict__ vin,
                                                          const SegDesc* __restrict__ segs,
                                                          int nseg, int use_src, int pass,
                                                          u32* __restrict__ counts) {
  __shared__ u32 h[kDigits];
  const u32 tile = blockIdx.x;
  const int s = find_segment(segs, nseg, tile);
  const SegDesc sd = segs[s];
  const u64 e0 = (u64)(tile - sd.tile_begin) * kSortTile;
  const u32 cnt = (u32)min((u64)kSortTile, (u64)sd.len - e0);
  const u64 src = (use_src ? sd.src_off : sd.dst_off) + e0;
  const u64* rin = kMode == kDigitV ? vin : kin;
  h[threadIdx.x] = 0;
  __syncthreads();
  u64 kk[kSortItems];
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const u32 i = j * kSortThreads + threadIdx.x;
    kk[j] = i < cnt ? rin[src + i] : 0ull;
  }
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const u32 i = j * kSortThreads + threadIdx.x;
    if (i < cnt) atomicAdd(&h[digit_of<kMode>(sd, kk[j], kk[j], pass)], 1u);
  }
  __syncthreads();
  counts[(size_t)threadIdx.x * gridDim.x + tile] = h[threadIdx.x];  // column-major: [digit][tile]
}

// Column scan: for digit d and segment s (one block each), the exclusive
// prefix of counts[d][t] over the segment's tiles, in place, and the
// segment's digit total (into totals, slot [s][pass][d]). The column is
// contiguous (k_upsweep writes digit-major) and each thread scans kColItems
// consecutive tiles, so a segment of up to 2048 tiles is one block scan.
constexpr int kColItems = 8;
__global__ __launch_bounds__(256) void k_colscan(u32* __restrict__ counts,
                                                 const SegDesc* __restrict__ segs, int nseg,
                                                 u32 total_tiles, u32* __restrict__ totals,
                                                 int pass) {
  u32* const col = counts + (size_t)blockIdx.x * total_tiles;
  __shared__ u32 wsum[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int s = blockIdx.y; s < nseg; s += gridDim.y) {
    const u32 tb = segs[s].tile_begin;
    const u32 te = (s + 1 < nseg) ? segs[s + 1].tile_begin : total_tiles;
    u32 carry = 0;
    for (u32 t0 = tb; t0 < te; t0 += blockDim.x * kColItems) {
      const u32 t = t0 + threadIdx.x * kColItems;
      u32 x[kColItems];
      u32 sum = 0;
#pragma unroll
      for (int j = 0; j < kColItems; ++j) {
        x[j] = t + j < te ? col[t + j] : 0u;
        sum += x[j];
      }
      u32 incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const u32 y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (lane == 31) wsum[warp] = incl;
      __syncthreads();
      u32 pre = 0, tot = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
        const u32 ws = wsum[w];
        pre += (w < warp) ? ws : 0u;
        tot += ws;
      }
      u32 run = carry + pre + incl - sum;
#pragma unroll
      for (int j = 0; j < kColItems; ++j) {
        if (t + j < te) col[t + j] = run;
        run += x[j];
      }
      carry += tot;
      __syncthreads();
    }
    if (threadIdx.x == 0) totals[((size_t)s * kPasses + pass) * kDigits + blockIdx.x] = carry;
  }
}

template <int kMode>
static void lsd_pass_launch(const u64* kin, const u64* vin, u64* kout, u64* vout,
                            const SegDesc* segs, int nseg, u32 total_tiles, int use_src,
                            const u32* digit_excl, int pass, u32* counts, cudaStream_t st) {
  k_upsweep<kMode><<<total_tiles, kSortThreads, 0, st>>>(kin, vin, segs, nseg, use_src, pass,
                                                         counts);
  // (the segment totals go where the downsweep reads its digit bases)
  k_colscan<<<dim3(kDigits, (unsigned)nseg), 256, 0, st>>>(counts, segs, nseg, total_tiles,
                                                           const_cast<u32*>(digit_excl), pass);
  onesweep_launch<kMode, true>(kin, vin, kout, vout, segs, nseg, total_tiles, use_src, digit_excl,
                               pass, nullptr, 0, nullptr, counts, st);
}

void launch_lsd_pass(const u64* kin, const u64* vin, u64* kout, u64* vout, const SegDesc* segs,
                     int nseg, u32 total_tiles, int use_src, int mode, const u32* digit_excl,
                     int pass, u32* counts, cudaStream_t st) {
  if (total_tiles == 0) return;
  switch (mode) {
    case kDigitQ:
      lsd_pass_launch<kDigitQ>(kin, vin, kout, vout, segs, nseg, total_tiles, use_src, digit_excl,
                               pass, counts, st);
      break;
    case kDigitV:
      lsd_pass_launch<kDigitV>(kin, vin, kout, vout, segs, nseg, total_tiles, use_src, digit_excl,
                               pass, counts, st);
      break;
    default:
      lsd_pass_launch<kDigitK>(kin, vin, kout, vout, segs, nseg, total_tiles, use_src, digit_excl,
                               pass, counts, st);
  }
}

void launch_seg_copy(const u64* kin, const u64* vin, u64* kout, u64* vout, const SegDesc* segs,
                     int nseg, u32 total_tiles, int use_src, cudaStream_t st) {
  if (total_tiles == 0) return;
  k_seg_copy<<<total_tiles, 256, 0, st>>>(kin, vin, kout, vout, segs, nseg, use_src);
}

void launch_group_scan(u64* k, u64* v, const SegDesc* segs, int nseg, u32 total_tiles, int eqmode,
                       void* medium, u32* nmedium, unsigned long long* ngroups, cudaStream_t st) {
  if (total_tiles == 0) return;
  k_group_scan<<<total_tiles, 256, sizeof(GroupSmem), st>>>(k, v, segs, nseg, eqmode,
                                                           (GroupRun*)medium, nmedium,
                                            ngroups);
}

void launch_group_fix_medium(u64* k, u64* v, const SegDesc* segs, const void* medium,
                             const u32* nmedium, void* longr, u32* nlong, cudaStream_t st) {
  k_group_fix_medium<<<148 * 2, 256, 0, st>>>(k, v, segs, (const GroupRun*)medium, nmedium,
                                              (GroupRun*)longr, nlong);
}

size_t group_run_bytes() { return sizeof(GroupRun); }

// Dynamic shared memory opt-ins of the sort kernels (per device: called by
// device_limits() once for each device).
cudaError_t configure_sort_kernels() {
  const int os = (int)sizeof(OnesweepSmem);
  const void* fns[] = {(const void*)k_onesweep<kDigitQ, false>, (const void*)k_onesweep<kDigitV, false>,
                       (const void*)k_onesweep<kDigitK, false>, (const void*)k_onesweep<kDigitQ, true>,
                       (const void*)k_onesweep<kDigitV, true>, (const void*)k_onesweep<kDigitK, true>};
  for (const void* f : fns) {
    const cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, os);
    if (e != cudaSuccess) return e;
  }
  return cudaFuncSetAttribute((const void*)k_group_scan, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)sizeof(GroupSmem));
}

}  // namespace chgpu
