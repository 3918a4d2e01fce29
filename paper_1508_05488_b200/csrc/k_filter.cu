// SPA pre-filter: the region sort restricted to the records the SPA can
// keep. Replaces, on the hull path, sort_region over every survivor
// (reference spa.cpp:59-81) followed by spa_filter (spa.cpp:109-163), with
// the same kept chains.
//
// Why it is exact. spa_filter keeps record i of chunk c iff its guarded key
// w_i (chgpu_internal.cuh wkey) is >= the running max of the chunk's seed
// and every earlier w of the chunk (k_spa.cu header). Cut each region's
// sorted sequence into bins of its primary coordinate (bin_of, monotone, so
// bins are contiguous runs in sorted order), and let T_b be the max of the
// chunk's seed and of w over every bin lying entirely inside the chunk
// before bin b. T_b never exceeds the true running max at any record of b,
// so a record with w < T_b steps back: it is not kept and, being below the
// running max, does not move it. Dropping it therefore changes nothing for
// any other record. What survives ("candidates") is sorted and scanned
// exactly like the full sequence, provided every candidate knows its chunk:
//   * a bin inside one chunk: the bin's chunk (from exact per-bin counts);
//   * a bin straddling a chunk boundary: T = 0, every record is a candidate,
//     so after sorting a record's rank inside the bin is its position.
// The first bin of every chunk c > 0 has T = 0 (seed = identity) as well,
// so each chunk's first candidate sits at a known rank.
//
// Kernels:
//   K2 (k_discard.cu)  per survivor: bin count += 1, bin max(w); the
//                      survivor point into its warp's segment
//   k_bin_scan         one cooperative launch: the plan, bin starts (ranks),
//                      each chunk's first bin, T_b: segmented exclusive max
//                      (segments = chunks)
//   k_filter           survivors with w >= T_b -> their bin's slots of a
//                      sparse region-ordered layout (unordered in the bin),
//                      and a bit per bin holding a candidate
//   k_bin_sort_warp/_big  bins above 32 candidates sorted in place
//   k_spa_chunks       one warp per chunk: its candidate bins from the
//                      bitmap, small bins batched and ordered in registers,
//                      the SPA scan; kept records to scratch
//   k_spa_emit         kept records at their output offsets, decoded
//
// Algorithmic traffic: the filter reads 16 B per survivor and writes 16 B
// per candidate (a few percent of survivors for spread-out inputs); the
// bin tables are ~40 B per bin and stay in L2.

#include <algorithm>
#include <cstdio>

#include "chgpu_internal.cuh"
#include "kernels.h"

namespace chgpu {

// ------------------------------------------------------------------ bin scan

// Segmented running max over bins: (seg, val) pairs, seg = chunk id,
// kNone = empty prefix.
constexpr u32 kNone = 0xFFFFFFFFu;
struct SegMax {
  u32 seg;
  u64 val;
};
__device__ __forceinline__ SegMax seg_combine(SegMax a, SegMax b) {
  if (b.seg == kNone) return a;
  if (a.seg == kNone || b.seg != a.seg) return b;
  return SegMax{b.seg, a.val > b.val ? a.val : b.val};
}
__device__ __forceinline__ SegMax shfl_up_seg(SegMax x, int o) {
  return SegMax{__shfl_up_sync(0xffffffffu, x.seg, o), __shfl_up_sync(0xffffffffu, x.val, o)};
}

constexpr int kBinThreads = 256;
constexpr int kBinPer = 8;
// Bins per entry of the coarse threshold table (min T of the group), which
// the filter keeps in shared memory: kCoarseBins / kBinPer bin-scan
// threads' bins.
#ifndef CHGPU_COARSE_LOG2
#define CHGPU_COARSE_LOG2 5
#endif
constexpr int kCoarseLog2 = CHGPU_COARSE_LOG2;
constexpr int kCoarseBins = 1 << kCoarseLog2;
static_assert(kCoarseBins >= kBinPer && kCoarseBins <= 32 * kBinPer, "coarse group = whole threads of a warp");
constexpr int kBinTile = kBinThreads * kBinPer;  // 2048 bins

__device__ __forceinline__ u32 bin_tiles(int log2nb) { return max(1u, (1u << log2nb) / kBinTile); }

__device__ __forceinline__ void load8(const u32* p, u32* c) {
  const uint4 a = reinterpret_cast<const uint4*>(p)[0], d = reinterpret_cast<const uint4*>(p)[1];
  c[0] = a.x; c[1] = a.y; c[2] = a.z; c[3] = a.w;
  c[4] = d.x; c[5] = d.y; c[6] = d.z; c[7] = d.w;
}

// Block-wide exclusive sum (kBinThreads threads); *total gets the sum.
__device__ __forceinline__ u32 block_excl_sum(u32 x, u32* sh, u32* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  u32 incl = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const u32 y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) sh[warp] = incl;
  __syncthreads();
  u32 pre = 0, tot = 0;
#pragma unroll
  for (int w = 0; w < kBinThreads / 32; ++w) {
    pre += (w < warp) ? sh[w] : 0u;
    tot += sh[w];
  }
  *total = tot;
  return pre + incl - x;
}

// Block-wide exclusive segmented max; *total gets the block aggregate.
__device__ __forceinline__ SegMax block_excl_segmax(SegMax x, u32* sseg, u64* sval, SegMax* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  SegMax inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const SegMax y = shfl_up_seg(inc, o);
    if (lane >= o) inc = seg_combine(y, inc);
  }
  if (lane == 31) {
    sseg[warp] = inc.seg;
    sval[warp] = inc.val;
  }
  __syncthreads();
  SegMax pre{kNone, 0}, tot{kNone, 0};
#pragma unroll
  for (int w = 0; w < kBinThreads / 32; ++w) {
    const SegMax a{sseg[w], sval[w]};
    if (w < warp) pre = seg_combine(pre, a);
    tot = seg_combine(tot, a);
  }
  *total = tot;
  SegMax ex = shfl_up_seg(inc, 1);
  if (lane == 0) ex = SegMax{kNone, 0};
  return seg_combine(pre, ex);
}

// Chunk of a rank, s / cs, for a thread walking increasing ranks: one
// division on entry and one per chunk boundary crossed, not one per bin.
struct ChunkCursor {
  u32 cur;   // chunk of the last rank asked for
  u64 next;  // first rank of chunk cur + 1
  u32 cs;
  __device__ __forceinline__ ChunkCursor(u32 s, u32 chunk_size) : cs(chunk_size) {
    cur = s / cs;
    next = (u64)(cur + 1) * cs;
  }
  __device__ __forceinline__ u32 at(u32 s) {  // s no smaller than the last rank asked for
    if (s >= next) {
      cur = s / cs;
      next = (u64)(cur + 1) * cs;
    }
    return cur;
  }
  __device__ __forceinline__ u32 peek(u32 s) const { return s < next ? cur : s / cs; }
};

// Segmented-max elements of 8 consecutive bins starting at rank s: a bin
// inside one chunk contributes (chunk, w); a straddling bin restarts its
// last chunk with nothing known; an empty bin contributes nothing.
// *straddle bit j: whether bin j crosses a chunk boundary.
__device__ __forceinline__ void seg_elems(const u32* c, const u64* w, u32 s, u32 cs, SegMax* e,
                                          u32* straddle) {
  ChunkCursor cc(s, cs);
  u32 sm = 0;
#pragma unroll
  for (int j = 0; j < kBinPer; ++j) {
    if (c[j] == 0) {
      e[j] = SegMax{kNone, 0};
    } else {
      const u32 clo = cc.at(s), chi = cc.peek(s + c[j] - 1);
      sm |= (u32)(clo != chi) << j;
      e[j] = clo != chi ? SegMax{chi, 0} : SegMax{clo, w[j]};
    }
    s += c[j];
  }
  *straddle = sm;
}

// The plan of the filter path, computed on the device from K2's region
// counts and the quad, so the host enqueues the whole path without waiting
// for K2. A degenerate frame (no SPA, pipeline.cpp:53-71) leaves every
// region empty and the path idle.
__device__ void make_filter_plan(const QuadInfo& qi, const u32* __restrict__ counts,
                                 u64 chunk_count, int log2nb, FilterPlan& P) {
  P.log2nb = log2nb;
  u64 m[4];
  for (int r = 0; r < 4; ++r) m[r] = qi.degenerate ? 0ull : (u64)counts[r];
  u64 off = 0;
  u32 chunks = 0;
  for (int r = 0; r < 4; ++r) {
    P.spa.off[r] = off;
    off += m[r];
    P.spa.m[r] = m[r];
    P.spa.chunk_begin[r] = chunks;
    const u64 cs = m[r] ? (m[r] + chunk_count - 1) / chunk_count : 1;  // spa.cpp:121
    P.spa.chunk_size[r] = cs;
    if (m[r]) chunks += (u32)((m[r] + cs - 1) / cs);                   // spa.cpp:122
    // guarded(region, anchors.first): LL left.y, LR bottom.x, UR right.y, UL top.x
    const double seed = (r == 0 || r == 2) ? qi.q[2 * r + 1] : qi.q[2 * r];
    P.spa.seed[r] = seed;
    const int reg = r + 1;
    // (w >> kWShift, like the filter keys and the bin maxima)
    P.seed_w[r] = wkey(reg, (reg == 1 || reg == 4) ? ~ord_enc(seed) : ord_enc(seed)) >> kWShift;
  }
  P.spa.total_chunks = chunks;
}

__device__ __forceinline__ u32 ld_acquire_u32(const u32* p) {
  u32 v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Grid-wide barrier of a cooperative launch (every CTA resident): arrival
// count in *ctr (zero at launch); barrier g releases at (g + 1) * gridDim.x.
__device__ __forceinline__ void grid_barrier(u32* ctr, u32 g) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(ctr, 1u);
    const u32 target = (g + 1) * gridDim.x;
    while (ld_acquire_u32(ctr) < target) __nanosleep(20);
  }
  __syncthreads();
}

// The whole bin scan in one cooperative launch (one CTA per tile of 2048
// bins, at most 512 CTAs, all resident), bins held in registers across two
// grid barriers:
//   plan      every CTA derives the FilterPlan from K2's region counts
//             (CTA 0 publishes it for the later kernels);
//   phase 1   records per tile;
//   phase 2   bin starts (ranks inside the region) from the earlier tiles'
//             sums, and the tile's segmented-max aggregate;
//   phase 3   T_b = max(seed of its chunk, exclusive segmented max of w over
//             the chunk's inner bins), 0 for straddling and empty bins; the
//             carry into a tile folds the aggregates of the region's earlier
//             tiles.
__global__ __launch_bounds__(kBinThreads, 4) void k_bin_scan(
    const QuadInfo* __restrict__ qinfo, u32* __restrict__ counts, u64 chunk_count,
    int log2nb, const u32* __restrict__ bcnt, const u32* __restrict__ bw,
    FilterPlan* __restrict__ plan_out, u32* __restrict__ bstart, u32* __restrict__ bthr,
    u32* __restrict__ tcoarse, u32* __restrict__ first_bin, u32* __restrict__ tsum,
    u32* __restrict__ agg_seg, u64* __restrict__ agg_val, u32* __restrict__ bar,
    u32* __restrict__ overflow) {
  __shared__ FilterPlan sP;
  __shared__ u32 s_m[4];
  __shared__ u32 sh[kBinThreads / 32];
  __shared__ u32 sseg[kBinThreads / 32];
  __shared__ u64 sval[kBinThreads / 32];
  __shared__ u32 s_base;
  __shared__ u32 c_seg;
  __shared__ u64 c_val;
  const u32 nb = 1u << log2nb;
  const u32 tiles = bin_tiles(log2nb);
  const u32 r = blockIdx.x / tiles, t = blockIdx.x % tiles;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const u32 b0 = t * kBinTile + threadIdx.x * kBinPer;
  const size_t boff = (size_t)r << log2nb;
  // the bins (an empty region's bins are all zero)
  u32 c[kBinPer] = {0, 0, 0, 0, 0, 0, 0, 0};
  u64 w[kBinPer] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (b0 < nb) {
    load8(bcnt + boff + b0, c);
    u32 w32[kBinPer];
    load8(bw + boff + b0, w32);
#pragma unroll
    for (int j = 0; j < kBinPer; ++j) w[j] = w32[j];
  }
  // phase 1
  u32 x = 0;
#pragma unroll
  for (int j = 0; j < kBinPer; ++j) x += c[j];
  u32 tot;
  const u32 ex = block_excl_sum(x, sh, &tot);
  if (threadIdx.x == 0) tsum[blockIdx.x] = tot;
  grid_barrier(bar, 0);
  // phase 2: this tile's first rank, the region sizes (sums of the bin
  // counts: K2 keeps no region totals of its own), then the plan
  if (warp == 0) {
    u32 y = 0;
    for (u32 i = lane; i < t; i += 32) y += __ldcg(tsum + r * tiles + i);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) y += __shfl_xor_sync(0xffffffffu, y, o);
    if (lane == 0) s_base = y;
  } else if (warp <= 4) {
    const u32 rr = warp - 1;
    u32 y = 0;
    for (u32 i = lane; i < tiles; i += 32) y += __ldcg(tsum + rr * tiles + i);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) y += __shfl_xor_sync(0xffffffffu, y, o);
    if (lane == 0) s_m[rr] = y;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const QuadInfo qi = *qinfo;
    make_filter_plan(qi, s_m, chunk_count, log2nb, sP);
    if (blockIdx.x == 0) {
      *plan_out = sP;
      if (!qi.degenerate)  // (a degenerate frame's K2 counted its LEX stream itself)
        for (int q = 0; q < 4; ++q) counts[q] = s_m[q];
    }
  }
  __syncthreads();
  const bool active = sP.spa.m[r] != 0;  // CTA-uniform; idle CTAs still meet the barriers
  const bool in = active && b0 < nb;
  const u32 s0 = s_base + ex;
  const u32 cs = (u32)sP.spa.chunk_size[r];  // ranks and sizes fit 32 bits (n < 2^32)
  SegMax e[kBinPer];
  u32 straddle;
  seg_elems(c, w, s0, cs, e, &straddle);
  SegMax agg{kNone, 0};
#pragma unroll
  for (int j = 0; j < kBinPer; ++j) agg = seg_combine(agg, e[j]);
  SegMax tagg;
  SegMax run = block_excl_segmax(agg, sseg, sval, &tagg);
  if (threadIdx.x == 0) {
    agg_seg[blockIdx.x] = tagg.seg;
    agg_val[blockIdx.x] = tagg.val;
  }
  if (in) {
    // bin starts, and the bin holding each chunk's first rank
    const u32 cbase = sP.spa.chunk_begin[r];
    ChunkCursor cc(s0, cs);
    u32 so[kBinPer];
    u32 q = s0;
#pragma unroll
    for (int j = 0; j < kBinPer; ++j) {
      so[j] = q;
      if (c[j]) {
        const u32 clo = cc.at(q), chi = cc.peek(q + c[j] - 1);
        for (u32 k = ((u64)clo * cs == q) ? clo : clo + 1; k <= chi; ++k) first_bin[cbase + k] = b0 + j;
      }
      q += c[j];
    }
    uint4* o = reinterpret_cast<uint4*>(bstart + boff + b0);
    o[0] = make_uint4(so[0], so[1], so[2], so[3]);
    o[1] = make_uint4(so[4], so[5], so[6], so[7]);
  }
  grid_barrier(bar, 1);
  // phase 3
  if (warp == 0) {
    // ordered fold of tiles [0, t): lane L folds its contiguous share, then
    // an ordered warp scan
    const u32 per = (t + 31) / 32;
    SegMax a{kNone, 0};
    for (u32 i = lane * per; i < min(t, (lane + 1) * per); ++i)
      a = seg_combine(a, SegMax{__ldcg(agg_seg + r * tiles + i), __ldcg(agg_val + r * tiles + i)});
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const SegMax y = shfl_up_seg(a, o);
      if (lane >= o) a = seg_combine(y, a);
    }
    if (lane == 31) {
      c_seg = a.seg;
      c_val = a.val;
    }
  }
  __syncthreads();
  run = seg_combine(SegMax{c_seg, c_val}, run);
  const u64 seedw = sP.seed_w[r];
  u64 th[kBinPer];
  ChunkCursor cc(s0, cs);
  u32 q = s0;
  u32 gmin = ~0u;  // min T over this thread's bins holding records
#pragma unroll
  for (int j = 0; j < kBinPer; ++j) {
    th[j] = 0;
    if (c[j] && !((straddle >> j) & 1u)) {
      const u32 clo = cc.at(q);
      u64 tv = clo == 0 ? seedw : 0ull;
      if (run.seg == clo && run.val > tv) tv = run.val;
      th[j] = tv;
    }
    if (c[j]) gmin = min(gmin, (u32)th[j]);
    run = seg_combine(run, e[j]);
    q += c[j];
  }
  // the coarse table: min T over each group of kCoarseBins bins
#pragma unroll
  for (int o = 1; o < kCoarseBins / kBinPer; o <<= 1) gmin = min(gmin, __shfl_xor_sync(0xffffffffu, gmin, o));
  if (in && (threadIdx.x & (kCoarseBins / kBinPer - 1)) == 0) tcoarse[(boff + b0) >> kCoarseLog2] = gmin;
  if (!in) return;
  uint4* const to = reinterpret_cast<uint4*>(bthr + boff + b0);
  to[0] = make_uint4((u32)th[0], (u32)th[1], (u32)th[2], (u32)th[3]);
  to[1] = make_uint4((u32)th[4], (u32)th[5], (u32)th[6], (u32)th[7]);
  // T = 0 passes every record: such a bin above kBinSortMax records is
  // certain to overflow the bin sorts, so the filter can stand down now
  bool certain = false;
#pragma unroll
  for (int j = 0; j < kBinPer; ++j) certain |= th[j] == 0 && c[j] > (u32)kBinSortMax;
  if (certain) atomicOr(overflow, 1u);
}

// ------------------------------------------------------------------ filter

#ifndef CHGPU_SPA_CLOCKS
#define CHGPU_SPA_CLOCKS 0
#endif
#ifndef CHGPU_FINISH_CLOCKS
#define CHGPU_FINISH_CLOCKS 0
#endif
#if CHGPU_FINISH_CLOCKS  // (diagnostic build: phase clocks of k_spa_finish)
__device__ unsigned long long g_fin_clk[9];
__global__ void k_fin_clocks_report() {
  printf("spa_finish max clocks: warp sorts %llu | big sorts %llu | barrier %llu | chunk SPA %llu | "
         "barrier %llu ; lists: warp %llu big %llu deferred %llu\n",
         g_fin_clk[1], g_fin_clk[2], g_fin_clk[3], g_fin_clk[4], g_fin_clk[5], g_fin_clk[6],
         g_fin_clk[7], g_fin_clk[8]);
  for (int i = 0; i < 9; ++i) g_fin_clk[i] = 0;
}
#endif
#if CHGPU_SPA_CLOCKS  // (diagnostic build: per-chunk clocks of k_spa_chunks)
__device__ unsigned long long g_spa_clk[40];
#endif
#ifndef CHGPU_FILTER_DIST
#define CHGPU_FILTER_DIST 1
#endif
#ifndef CHGPU_FILTER_ABL
#define CHGPU_FILTER_ABL 0
#endif
constexpr int kFilterThreads = 1024;  // one CTA per SM (the coarse table fills shared memory)

// Bytes of k_filter's dynamic shared memory (the coarse threshold table).
size_t filter_smem_bytes(int log2nb) { return ((size_t)4 << log2nb) / kCoarseBins * sizeof(u32); }

// Warp-stride over K2's survivor segments (k_classify_survivors: 256
// slots each): per survivor one 8-byte key, its global bin over w >> kWShift
// (filter_key). A survivor with (w >> kWShift) < T_b is dropped: since the
// shift is monotone, that implies w < the bin's lower bound of the running
// max. The bins' thresholds are random 4-byte lookups, so they are tested in
// two steps: first against the min T of the bin's group of kCoarseBins bins,
// from a copy of the coarse table in shared memory (a key below it is below
// T_b: dropped without touching L2), and only the rest against T_b itself.
// A candidate fetches its point from the input (its index from K2), takes
// the next slot of its bin and writes its sort record; the bin's 33rd
// candidate queues it for k_bin_sort_warp, its 257th for k_bin_sort_big.
__global__ __launch_bounds__(kFilterThreads, 1) void k_filter(
    const u64* __restrict__ seg, const u64* __restrict__ segcnt,
    u32 nseg, const double2* __restrict__ pts, const FilterPlan* __restrict__ P_p,
    const QuadInfo* __restrict__ qinfo, const u32* __restrict__ bstart,
    const u32* __restrict__ bthr, const u32* __restrict__ tcoarse, u32* __restrict__ bcur,
    u32* __restrict__ bmap, u64* __restrict__ kout, u64* __restrict__ vout, u32* __restrict__ big,
    u32* __restrict__ nbig, unsigned long long* __restrict__ ncand, const u32* __restrict__ overflow) {
  extern __shared__ __align__(16) u32 s_tc[];  // coarse thresholds, (4 << log2nb) / kCoarseBins
  __shared__ u64 s_off[4];
  __shared__ u32 s_lg, s_nseg;
  __shared__ u32 s_cand;
  // candidate queue, per warp (see push)
  __shared__ u64 s_qkey[kFilterThreads / 32][64];
  __shared__ u32 s_qat[kFilterThreads / 32][64];
  if (threadIdx.x < 4) {
    const int r = threadIdx.x;
    s_off[r] = P_p->spa.off[r];
    if (r == 0) {
      s_lg = (u32)P_p->log2nb;
      // no segments on a degenerate frame (K2 wrote LEX records), nothing to
      // do once the bin scan saw a certain overflow
      s_nseg = (qinfo->degenerate || *overflow) ? 0u : nseg;
      s_cand = 0;
    }
  }
  __syncthreads();
  const u32 lg = s_lg;
  nseg = s_nseg;
  if (nseg) {
    const u32 ntc4 = (u32)(((size_t)4 << lg) / kCoarseBins / 4);  // uint4 words
    const uint4* src = reinterpret_cast<const uint4*>(tcoarse);
    uint4* dst = reinterpret_cast<uint4*>(s_tc);
    for (u32 i = threadIdx.x; i < ntc4; i += kFilterThreads) dst[i] = __ldcg(src + i);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const u32 wstride = gridDim.x * (kFilterThreads / 32);
  u32 mine = 0;
  // One candidate's work (its point, bin slot, sort record, big-bin queue);
  // `at` = its survivor slot in K2's segments.
  auto take = [&](u64 key, u32 at) {
    const u32 bi = key_bin(key);
    const u32 r = bi >> lg;
    const int reg = (int)r + 1;
    const u32 bs = bstart[bi];
    // the input index: the segment's first point + the position in the key
    const double2 p = __ldg(pts + ((at & ~(u32)(kSegPts - 1)) | key_pos(key)));
    const u32 pos = atomicAdd(bcur + bi, 1u);
    if (pos == 0) atomicOr(bmap + (bi >> 5), 1u << (bi & 31));  // k_spa_chunks' index
    const u64 dst = s_off[r] + bs + pos;
    kout[dst] = k_of(reg, p.x, p.y);
    vout[dst] = v_of(reg, p.x, p.y);
    if (pos == 32) big[atomicAdd(nbig, 1u)] = bi;                       // > 32: by a warp
    if (pos == kWarpSortMax) big[kBigListB + atomicAdd(nbig + 1, 1u)] = bi;  // > 256: a CTA
#if !(CHGPU_FILTER_ABL & 1)
    ++mine;
#endif
  };
  // Candidates are rare (~1.6% of survivors on spread-out inputs): the scan
  // queues them in a warp-private list and takes them 32 at a time, every
  // lane busy, instead of stalling a whole round on one lane's
  // index -> point -> slot chain.
  u32 qn = 0;  // warp-uniform queue length (< 32 between rounds)
  auto push = [&](bool cand, u64 key, u32 at) {
    const unsigned m = __ballot_sync(0xffffffffu, cand);
    if (!m) return;
    if (cand) {
      const u32 q = qn + __popc(m & lanemask_lt());
      s_qkey[warp][q] = key;
      s_qat[warp][q] = at;
    }
    qn += __popc(m);
    if (qn < 32) return;
    __syncwarp();
    take(s_qkey[warp][lane], s_qat[warp][lane]);
    const u32 rest = qn - 32;
    u64 k2 = 0;
    u32 a2 = 0;
    if ((u32)lane < rest) {
      k2 = s_qkey[warp][32 + lane];
      a2 = s_qat[warp][32 + lane];
    }
    __syncwarp();
    if ((u32)lane < rest) {
      s_qkey[warp][lane] = k2;
      s_qat[warp][lane] = a2;
    }
    __syncwarp();
    qn = rest;
  };
  // A segment at a time, software-pipelined: while one segment's keys are
  // tested (coarse table, then the exact threshold of the few that pass),
  // the next segment's keys (up to kR rounds of 32) and the count of the one
  // after are in flight. K2 fills ~44% of a segment's 256 slots on uniform
  // inputs; rounds beyond kR (fuller segments) are loaded on the spot.
  constexpr int kR = 4;
  auto load_keys = [&](u32 g, u32 t, u64* k) {
#pragma unroll
    for (int j = 0; j < kR; ++j) {
      const u32 sl = 32 * j + lane;
      k[j] = (g < nseg && sl < t) ? __ldcs(seg + (u64)g * kSegPts + sl) : 0ull;
    }
  };
  auto test = [&](u32 g, u32 sl, u32 t, u64 key, u32 th) {
    push(sl < t && (u32)key >= th, key, g * kSegPts + sl);
  };
  auto coarse = [&](u32 sl, u32 t, u64 key) -> u32 {
    const u32 bi = key_bin(key);
    const bool pass = sl < t && (u32)key >= s_tc[bi >> kCoarseLog2];
#if CHGPU_FILTER_ABL & 1  // (diagnostic: count the coarse passes instead of the candidates)
    mine += pass;
#endif
    return pass ? __ldcg(bthr + bi) : ~0u;
  };
  // kDist segments of keys in flight ahead of the one being tested (a
  // register ring), each segment's count loaded one step before its keys.
  constexpr int kDist = CHGPU_FILTER_DIST;
  u32 sg = blockIdx.x * (kFilterThreads / 32) + warp;
  u64 kr[kDist + 1][kR];
  u32 tr[kDist + 2];
#pragma unroll
  for (int d = 0; d <= kDist + 1; ++d) {
    const u32 g = sg + d * wstride;
    tr[d] = g < nseg ? (u32)__ldg(segcnt + g) : 0u;
  }
#pragma unroll
  for (int d = 0; d < kDist; ++d) load_keys(sg + d * wstride, tr[d], kr[d]);
  for (; sg < nseg; sg += wstride) {
    const u32 gl = sg + (kDist + 2) * wstride;
    const u32 tl = gl < nseg ? (u32)__ldg(segcnt + gl) : 0u;
    load_keys(sg + kDist * wstride, tr[kDist], kr[kDist]);
    const u32 tot = tr[0];
    u32 th[kR];
#pragma unroll
    for (int j = 0; j < kR; ++j) th[j] = coarse(32 * j + lane, tot, kr[0][j]);
#pragma unroll
    for (int j = 0; j < kR; ++j) test(sg, 32 * j + lane, tot, kr[0][j], th[j]);
    for (u32 s0 = 32 * kR; s0 < tot; s0 += 32) {  // a fuller segment's remaining rounds
      const u32 sl = s0 + lane;
      const u64 key = sl < tot ? __ldcs(seg + (u64)sg * kSegPts + sl) : 0ull;
      test(sg, sl, tot, key, coarse(sl, tot, key));
    }
#pragma unroll
    for (int d = 0; d < kDist; ++d)
#pragma unroll
      for (int j = 0; j < kR; ++j) kr[d][j] = kr[d + 1][j];
#pragma unroll
    for (int d = 0; d <= kDist; ++d) tr[d] = tr[d + 1];
    tr[kDist + 1] = tl;
  }
  __syncwarp();
  if ((u32)lane < qn) take(s_qkey[warp][lane], s_qat[warp][lane]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
  if ((threadIdx.x & 31) == 0 && mine) atomicAdd(&s_cand, mine);
  __syncthreads();
  if (threadIdx.x == 0 && s_cand) atomicAdd(ncand, (unsigned long long)s_cand);
}

// ------------------------------------------------------------------ big bins
//
// Bins above 32 candidates are sorted in place, by (canon k, v, k) =
// rec_less: up to kWarpSortMax by one warp in its own shared memory, above
// that by a CTA, above kBinSortMax not at all (*overflow: the caller re-runs
// the SPA over the full region sort).

__device__ __forceinline__ bool key_gt(u64 ci, u64 vi, u64 ki, u64 cj, u64 vj, u64 kj) {
  return ci > cj || (ci == cj && (vi > vj || (vi == vj && ki > kj)));
}

// Bitonic network over sc/sv/sk[0, Pn) executed by `nthreads` threads
// (index `me`); `sync` separates the stages. A stage of stride <= 32 keeps
// every warp inside its own 64-element blocks (thread t's pair starts at
// 2t - (t & (stride - 1))), so two such stages in a row need only `wsync`
// (a warp barrier) between them; `sync` runs where a stride >= 64 ends or
// begins.
template <typename Sync, typename WSync>
__device__ __forceinline__ void bitonic_smem(u64* sc, u64* sv, u64* sk, u32 Pn, u32 me, u32 nthreads,
                                             Sync sync, WSync wsync) {
  for (u32 size = 2; size <= Pn; size <<= 1) {
    for (u32 stride = size >> 1; stride > 0; stride >>= 1) {
      for (u32 t = me; t < Pn / 2; t += nthreads) {
        const u32 i = 2 * t - (t & (stride - 1));  // lower index of the pair
        const u32 jx = i + stride;
        const bool up = (i & size) == 0;
        const u64 ci = sc[i], cj = sc[jx], vi = sv[i], vj = sv[jx], ki = sk[i], kj = sk[jx];
        if (key_gt(ci, vi, ki, cj, vj, kj) == up) {
          sc[i] = cj; sc[jx] = ci;
          sv[i] = vj; sv[jx] = vi;
          sk[i] = kj; sk[jx] = ki;
        }
      }
      const u32 next = stride > 1 ? stride >> 1 : size;  // the next stage's stride
      if (stride >= 64 || next >= 64)
        sync();
      else
        wsync();
    }
  }
}

constexpr int kWarpSortWarps = 8;

// Bins of 33..kWarpSortMax candidates, one warp each (sh: the warp's 3 x
// kWarpSortMax words of shared memory); items strided over nvb virtual
// blocks of kWarpSortWarps warps.
__device__ void bin_sort_warp_body(u64* __restrict__ k, u64* __restrict__ v, const FilterPlan& P,
                                   const u32* __restrict__ bstart, const u32* __restrict__ bcur,
                                   const u32* __restrict__ big, u32 nbig, u64* sh, u32 vb, u32 nvb) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  u64* sc = sh;
  u64* sv = sh + kWarpSortMax;
  u64* sk = sh + 2 * kWarpSortMax;
  for (u32 item = vb * kWarpSortWarps + wid; item < nbig; item += nvb * kWarpSortWarps) {
    const u32 bi = big[item];
    const u32 len = bcur[bi];
    if (len > (u32)kWarpSortMax) continue;  // the CTA sort's
    const int r = (int)(bi >> P.log2nb);
    const u64 base = P.spa.off[r] + bstart[bi];
    u32 Pn = 64;
    while (Pn < len) Pn <<= 1;
    for (u32 i = lane; i < Pn; i += 32) {
      if (i < len) {
        const u64 kk = k[base + i];
        sk[i] = kk;
        sv[i] = v[base + i];
        sc[i] = canon_k(r + 1, kk);
      } else {
        sk[i] = sv[i] = sc[i] = ~0ull;
      }
    }
    __syncwarp();
    bitonic_smem(sc, sv, sk, Pn, lane, 32, [] { __syncwarp(); }, [] { __syncwarp(); });
    for (u32 i = lane; i < len; i += 32) {
      k[base + i] = sk[i];
      v[base + i] = sv[i];
    }
    __syncwarp();
  }
}

constexpr int kBigThreads = 256;

struct BigSmem {
  u64 c[kBinSortMax], v[kBinSortMax], k[kBinSortMax];
};

// Bins of kWarpSortMax+1..kBinSortMax candidates, one CTA each; above that
// *overflow (the caller falls back to the full region sort).
__device__ void bin_sort_big_body(u64* __restrict__ k, u64* __restrict__ v, const FilterPlan& P,
                                  const u32* __restrict__ bstart, const u32* __restrict__ bcur,
                                  const u32* __restrict__ big, u32 nbig, u32* __restrict__ overflow,
                                  BigSmem& S, u32 vb, u32 nvb) {
  for (u32 item = vb; item < nbig; item += nvb) {
    const u32 bi = big[item];
    const int r = (int)(bi >> P.log2nb);
    const u32 len = bcur[bi];
    if (len > (u32)kBinSortMax) {
      if (threadIdx.x == 0) atomicOr(overflow, 1u);
      continue;
    }
    const u64 base = P.spa.off[r] + bstart[bi];
    u32 Pn = 64;
    while (Pn < len) Pn <<= 1;
    for (u32 i = threadIdx.x; i < Pn; i += kBigThreads) {
      if (i < len) {
        const u64 kk = k[base + i];
        S.k[i] = kk;
        S.v[i] = v[base + i];
        S.c[i] = canon_k(r + 1, kk);
      } else {
        S.k[i] = S.v[i] = S.c[i] = ~0ull;
      }
    }
    __syncthreads();
    bitonic_smem(S.c, S.v, S.k, Pn, threadIdx.x, kBigThreads, [] { __syncthreads(); },
                 [] { __syncwarp(); });
    for (u32 i = threadIdx.x; i < len; i += kBigThreads) {
      k[base + i] = S.k[i];
      v[base + i] = S.v[i];
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ in-register batch order

// Ascending bitonic sort of one record per lane by (g, canon k, v, k), g a
// small group id (the bin's lane); lanes without a record carry g = ~0 and
// sort last.
__device__ __forceinline__ void warp_sort_records(int region, u32& g, u64& k, u64& v) {
  const int lane = threadIdx.x & 31;
  u64 c = g == ~0u ? ~0ull : canon_k(region, k);
#pragma unroll
  for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      const u32 og = __shfl_xor_sync(0xffffffffu, g, stride);
      const u64 oc = __shfl_xor_sync(0xffffffffu, c, stride);
      const u64 ov = __shfl_xor_sync(0xffffffffu, v, stride);
      const u64 ok = __shfl_xor_sync(0xffffffffu, k, stride);
      const bool other_less =
          og < g || (og == g && (oc < c || (oc == c && (ov < v || (ov == v && ok < k)))));
      const bool mine_less =
          g < og || (g == og && (c < oc || (c == oc && (v < ov || (v == ov && k < ok)))));
      const bool want_min = ((lane & stride) == 0) == ((lane & size) == 0);
      if (want_min ? other_less : mine_less) {
        g = og;
        c = oc;
        v = ov;
        k = ok;
      }
    }
  }
}

// ------------------------------------------------------------------ chunk SPA, small chunks
//
// One warp per SPA chunk whose candidates fit kSmallCap (every chunk of a
// spread-out input): spa_filter (spa.cpp:109-163) over the chunk's
// candidates without any bin having been sorted. The chunk's candidate bins
// are listed in order from the filter's bitmap and their candidates
// gathered bin after bin into shared memory; a candidate's rank inside its
// bin, #{y in the bin: rec_less(y, x)} (ties by slot), places it at its
// sorted position (bins are contiguous runs of the sorted order). In a bin
// straddling a chunk boundary (T = 0 there: all its records are
// candidates) the bin's start rank + that rank decides whether it belongs to
// this chunk, exactly as in k_spa_chunks. The scan then keeps a record iff
// its w is >= the running max (the seed's for chunk 0): spa_filter's
// threshold is the max over every earlier record of the chunk, and the
// record holding it is never dropped by the filter. Kept records go to the
// chunk's scratch range and counters exactly like k_spa_chunks. A chunk with
// more candidates (or more than 32 x kSmallRounds candidate bins) is listed
// for k_spa_chunks, which then runs after the bin sorts.
constexpr int kSmallCap = kSpaSmallCap;
static_assert(kSmallCap <= 256, "bin slots are bytes");
constexpr int kSmallWarps = 8;
struct SmallSmem {
  u64 c[kSmallCap], v[kSmallCap], k[kSmallCap];  // gathered records
  u64 ok[kSmallCap], ov[kSmallCap];              // sorted records
  u32 bex[kSmallCap], bn[kSmallCap], bst[kSmallCap];
  u32 list[32];
  unsigned char b[kSmallCap], oin[kSmallCap];
};
constexpr size_t kSmallSmem = kSmallWarps * sizeof(SmallSmem);

__global__ __launch_bounds__(32 * kSmallWarps) void k_spa_small(
    const u64* __restrict__ k, const u64* __restrict__ v, const u32* __restrict__ bcur,
    const u32* __restrict__ bstart, const u32* __restrict__ bmap, const u32* __restrict__ first_bin,
    const FilterPlan* __restrict__ P_p, u64* __restrict__ sk, u64* __restrict__ sv,
    u32* __restrict__ chunk_kept, u32* __restrict__ group_kept,
    unsigned long long* __restrict__ kept_counts, u32* __restrict__ defer, u32* __restrict__ ndefer,
    u32 cap) {
  const SpaPlan& plan = P_p->spa;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const u32 c = blockIdx.x * kSmallWarps + warp;
  if (c >= plan.total_chunks) return;
#if CHGPU_SPA_CLOCKS
  const long long t0 = clock64();
#endif
  int r = 0;
  while (r < 3 && c >= plan.chunk_begin[r + 1]) ++r;
  const int region = r + 1;
  const int log2nb = P_p->log2nb;
  const u32 cl = c - plan.chunk_begin[r];
  const u32 nchunks = (r < 3 ? plan.chunk_begin[r + 1] : plan.total_chunks) - plan.chunk_begin[r];
  const u32 cs = (u32)plan.chunk_size[r];
  const u32 lo = cl * cs, hi = (u32)min((u64)lo + cs, plan.m[r]);
  const size_t boff = (size_t)r << log2nb;
  const u64 rbase = plan.off[r];
  const u32 b_first = first_bin[c];
  const u32 b_last = cl + 1 < nchunks ? first_bin[c + 1] : (1u << log2nb) - 1u;

  extern __shared__ __align__(16) unsigned char small_smem[];
  SmallSmem& S = reinterpret_cast<SmallSmem*>(small_smem)[warp];
  u64* const C = S.c;  // gathered records (bin after bin): canon k, v, k, bin slot
  u64* const V = S.v;
  u64* const K = S.k;
  unsigned char* const B = S.b;
  u32* const BEX = S.bex;  // per bin (in order): first gathered slot, candidates, start rank
  u32* const BN = S.bn;
  u32* const BST = S.bst;

  // 1. the chunk's candidate bins in order, 32 bitmap words per round
  u32 m = 0, nbins = 0;
  bool over = cap == 0;
  const u32 gb0 = (u32)boff + b_first, gb1 = (u32)boff + b_last;  // inclusive
  for (u32 w0 = gb0 >> 5; w0 <= (gb1 >> 5) && !over; w0 += 32) {
    const u32 wi = w0 + lane;
    u32 word = wi <= (gb1 >> 5) ? bmap[wi] : 0u;
    if (wi == (gb0 >> 5)) word &= ~0u << (gb0 & 31);
    if (wi == (gb1 >> 5) && (gb1 & 31) != 31) word &= (2u << (gb1 & 31)) - 1u;
    const u32 cntw = __popc(word);
    u32 at = cntw;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const u32 y = __shfl_up_sync(0xffffffffu, at, o);
      if (lane >= o) at += y;
    }
    const u32 nlist = __shfl_sync(0xffffffffu, at, 31);
    if (nbins + nlist > (u32)kSmallCap) {
      over = true;
      break;
    }
    // this round's bins in order, 32 at a time: their counts and starts
    for (u32 lb = 0; lb < nlist; lb += 32) {
      // list the bins [lb, lb + 32) of this round (lanes holding them write)
      {
        u32 idx = at - cntw;
        u32 wd = word;
        while (wd) {
          const u32 b = (wi << 5) + (u32)(__ffs(wd) - 1);
          if (idx >= lb && idx < lb + 32) S.list[idx - lb] = b;
          ++idx;
          wd &= wd - 1;
        }
      }
      __syncwarp();
      const bool listed = lb + lane < nlist;
      const u32 gb = listed ? S.list[lane] : 0u;
      u32 n = 0, st = 0;
      if (listed) {
        n = bcur[gb];
        st = bstart[gb];
      }
      u32 incl = n;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const u32 y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const u32 tot = __shfl_sync(0xffffffffu, incl, 31);
      if (m + tot > cap) {
        over = true;
        break;
      }
      const u32 bi = nbins + lane;
      if (listed) {
        BEX[bi] = m + incl - n;
        BN[bi] = n;
        BST[bi] = st;
      }
      __syncwarp();
      // gather: slot e of this batch belongs to the first listed lane whose
      // end exceeds it
      for (u32 e = m + lane; e < m + tot; e += 32) {
        int a = 0, z = (int)min(31u, nlist - lb - 1);
        while (a < z) {
          const int mid = (a + z) >> 1;
          if (BEX[nbins + mid] + BN[nbins + mid] > e) z = mid; else a = mid + 1;
        }
        const u64 src = rbase + BST[nbins + a] + (e - BEX[nbins + a]);
        const u64 kk = k[src];
        K[e] = kk;
        V[e] = v[src];
        C[e] = canon_k(region, kk);
        B[e] = (unsigned char)(nbins + a);  // < kSmallCap <= 256
      }
      __syncwarp();
      m += tot;
      nbins += min(32u, nlist - lb);
    }
  }
  if (__any_sync(0xffffffffu, over)) {
    if (lane == 0) defer[atomicAdd(ndefer, 1u)] = c;
#if CHGPU_SPA_CLOCKS
    if (lane == 0) atomicAdd(&g_spa_clk[7], 1ull);
#endif
    return;
  }
#if CHGPU_SPA_CLOCKS
  const long long t1 = clock64();
#endif
  // 2. each record's rank inside its bin -> its sorted position; the
  // in-chunk test of straddling bins' records
  for (u32 e = lane; e < m; e += 32) {
    const u32 b = B[e];
    const u32 ex = BEX[b], n = BN[b], st = BST[b];
    const u64 ce = C[e];
    u32 rank = 0;
    bool tie = false;
    for (u32 y = ex; y < ex + n; ++y) {
      const u64 cy = C[y];
      rank += cy < ce;
      tie |= cy == ce && y != e;
    }
    if (tie) {  // (rare: an equal primary coordinate in the bin) the rest of rec_less
      const u64 ve = V[e], ke = K[e];
      for (u32 y = ex; y < ex + n; ++y) {
        const u64 vy = V[y], ky = K[y];
        rank += C[y] == ce && (vy < ve || (vy == ve && (ky < ke || (ky == ke && y < e))));
      }
    }
    const bool partial = st < lo || st + n > hi;
    const u32 rk = st + rank;
    S.ok[ex + rank] = K[e];
    S.ov[ex + rank] = V[e];
    S.oin[ex + rank] = (unsigned char)(!partial || (rk >= lo && rk < hi));
  }
  __syncwarp();
#if CHGPU_SPA_CLOCKS
  const long long t2 = clock64();
#endif
  // 3. the scan in sorted order, 32 records per round
  const u64 seedw = (cl == 0) ? wkey(region, (region == 1 || region == 4) ? ~ord_enc(plan.seed[r])
                                                                          : ord_enc(plan.seed[r]))
                              : 0ull;  // (no finite point has w = 0)
  u64 carry = seedw;
  u64* const kd = sk + rbase + lo;
  u64* const vd = sv + rbase + lo;
  u32 kept = 0;
  for (u32 base = 0; base < m; base += 32) {
    const u32 e = base + lane;
    const bool in = e < m && S.oin[e];
    u64 kk = 0, vv = 0, w = 0;
    if (e < m) {
      kk = S.ok[e];
      vv = S.ov[e];
      w = in ? wkey(region, vv) : 0ull;
    }
    u64 incl = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const u64 y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl = y > incl ? y : incl;
    }
    u64 ex = __shfl_up_sync(0xffffffffu, incl, 1);
    if (lane == 0) ex = 0ull;
    const u64 before = ex > carry ? ex : carry;
    const bool keep = in && w >= before;
    const unsigned km = __ballot_sync(0xffffffffu, keep);
    if (keep) {
      const u32 at = kept + __popc(km & lanemask_lt());
      kd[at] = kk;
      vd[at] = vv;
    }
    kept += __popc(km);
    const u64 rmax = __shfl_sync(0xffffffffu, incl, 31);
    carry = rmax > carry ? rmax : carry;
  }
  if (lane == 0) {
    chunk_kept[c] = kept;
    if (kept) {
      atomicAdd(&group_kept[c >> 8], kept);
      atomicAdd(&kept_counts[r], (unsigned long long)kept);
    }
  }
#if CHGPU_SPA_CLOCKS
  if (lane == 0) {
    const long long t3 = clock64();
    atomicMax(&g_spa_clk[20], (u64)(t1 - t0));
    atomicMax(&g_spa_clk[21], (u64)(t2 - t1));
    atomicMax(&g_spa_clk[22], (u64)(t3 - t2));
    atomicAdd(&g_spa_clk[23], (u64)(t1 - t0));
    atomicAdd(&g_spa_clk[24], (u64)(t2 - t1));
    atomicAdd(&g_spa_clk[25], (u64)(t3 - t2));
    atomicAdd(&g_spa_clk[26], 1ull);
    atomicMax(&g_spa_clk[27], (u64)m);
    atomicAdd(&g_spa_clk[28], (u64)m);
  }
#endif
}

// ------------------------------------------------------------------ chunk SPA
//
// One warp per SPA chunk (spa.cpp:109-163 over the chunk's candidates),
// chunks taken in order from an atomic counter for the look-back. The
// chunk's ranks [lo, hi) cover bins first_bin[c] .. first_bin[c + 1]; each
// bin's candidates sit at its sparse slots (region offset + bin start),
// sorted in place when above 32 (k_bin_sort_warp / _big), else batched with
// their neighbours and sorted in registers by (bin, record). A candidate's
// index inside its sorted bin is its rank offset whenever the bin straddles
// a chunk boundary (T = 0 there: every record is a candidate), so clipping
// to [lo - start, hi - start) gives the chunk's share; inner bins lie
// wholly inside. The running extremum starts at the seed for chunk 0 and at
// the identity otherwise; kept records go to scratch at the chunk's own
// rank range, their count to chunk_kept[c] and to the sum of its group of
// 256 chunks; k_spa_emit places them. (Chunks all finish their scans at
// about the same time, so a decoupled look-back here would walk back
// through thousands of aggregates before any prefix appears.)
// Smem of one warp of spa_chunk_warp.
struct SpaWarpSmem {
  u32 list[1024];
  u64 pk[32], pv[32], pc[32];
  int mark[32];
};

__device__ void spa_chunk_warp(
    u32 c, const u64* __restrict__ k, const u64* __restrict__ v, const u32* __restrict__ bcur,
    const u32* __restrict__ bstart, const u32* __restrict__ bmap, const u32* __restrict__ first_bin,
    const FilterPlan* __restrict__ P_p, u64* __restrict__ sk, u64* __restrict__ sv,
    u32* __restrict__ chunk_kept, u32* __restrict__ group_kept,
    unsigned long long* __restrict__ kept_counts, SpaWarpSmem& W) {
  const SpaPlan& plan = P_p->spa;
  const int lane = threadIdx.x & 31;
  if (c >= plan.total_chunks) return;
#if CHGPU_SPA_CLOCKS
  const long long t_start = clock64();
  u32 n_batches = 0, n_listed = 0;
#endif
  int r = 0;
  while (r < 3 && c >= plan.chunk_begin[r + 1]) ++r;
  const int region = r + 1;
  const int log2nb = P_p->log2nb;
  const u32 cl = c - plan.chunk_begin[r];
  const u32 nchunks = (r < 3 ? plan.chunk_begin[r + 1] : plan.total_chunks) - plan.chunk_begin[r];
  const u32 cs = (u32)plan.chunk_size[r];
  const u32 lo = cl * cs, hi = (u32)min((u64)lo + cs, plan.m[r]);
  const size_t boff = (size_t)r << log2nb;
  const u64 rbase = plan.off[r];
  const u32 b_first = first_bin[c];
  const u32 b_last = cl + 1 < nchunks ? first_bin[c + 1] : (1u << log2nb) - 1u;
  const bool is_min = (region == 1 || region == 4);
  const double ident = is_min ? INFINITY : -INFINITY;
  double carry = (cl == 0) ? plan.seed[r] : ident;
  u64* const kd = sk + rbase + lo;
  u64* const vd = sv + rbase + lo;
  u32 kept = 0;

  // one SPA step over 32 lanes in lane order; inactive lanes are neutral
  auto step = [&](bool active, u64 kk, u64 vv) {
    const double g = active ? guarded_of(region, vv) : ident;
    double incl = g;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl = op_ext(is_min, y, incl);
    }
    double ex = __shfl_up_sync(0xffffffffu, incl, 1);
    if (lane == 0) ex = ident;
    const bool keep = active && !steps_back(is_min, g, op_ext(is_min, carry, ex));
    carry = op_ext(is_min, carry, __shfl_sync(0xffffffffu, incl, 31));
    const unsigned km = __ballot_sync(0xffffffffu, keep);
    if (keep) {
      const u32 at = kept + __popc(km & lanemask_lt());
      kd[at] = kk;
      vd[at] = vv;
    }
    kept += __popc(km);
  };

  // The chunk's bins holding candidates, in order, from the filter's
  // bitmap: 1024 bins per load round (a sparse stretch of a region can put
  // thousands of empty bins in one chunk), then 32 of them per window.
  const u32 gb0 = (u32)boff + b_first, gb1 = (u32)boff + b_last;  // inclusive
  for (u32 w0 = gb0 >> 5; w0 <= (gb1 >> 5); w0 += 32) {
    const u32 wi = w0 + lane;
    u32 word = wi <= (gb1 >> 5) ? bmap[wi] : 0u;
    if (wi == (gb0 >> 5)) word &= ~0u << (gb0 & 31);
    if (wi == (gb1 >> 5) && (gb1 & 31) != 31) word &= (2u << (gb1 & 31)) - 1u;
    const u32 cntw = __popc(word);
    u32 at = cntw;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const u32 y = __shfl_up_sync(0xffffffffu, at, o);
      if (lane >= o) at += y;
    }
    const u32 nlist = __shfl_sync(0xffffffffu, at, 31);
#if CHGPU_SPA_CLOCKS
    n_listed += nlist;
#endif
    at -= cntw;
    while (word) {
      W.list[at++] = (wi << 5) + (u32)(__ffs(word) - 1) - (u32)boff;
      word &= word - 1;
    }
    __syncwarp();
   for (u32 lb = 0; lb < nlist; lb += 32) {
    const bool listed = lb + lane < nlist;
    const u32 b = listed ? W.list[lb + lane] : 0u;
    u32 n = 0, s = 0;
    if (listed) {
      n = bcur[boff + b];
      s = bstart[boff + b];
    }
    // the chunk's share of the bin, as indices into its sorted candidates
    const u32 i0 = lo > s ? lo - s : 0u;
    const u32 i1 = min(n, hi > s ? hi - s : 0u);
    const bool act = n > 0 && i1 > i0;
    const bool small = n <= 32;
    unsigned todo = __ballot_sync(0xffffffffu, act);
    while (todo) {
#if CHGPU_SPA_CLOCKS
      ++n_batches;
#endif
      const int p = __ffs(todo) - 1;
      if (!__shfl_sync(0xffffffffu, small, p)) {
        // a bin sorted in place: its share in slices of 32
        const u64 src = rbase + __shfl_sync(0xffffffffu, s, p);
        const u32 a0 = __shfl_sync(0xffffffffu, i0, p), a1 = __shfl_sync(0xffffffffu, i1, p);
        for (u32 t = a0; t < a1; t += 32) {
          const bool on = t + lane < a1;
          u64 kk = 0, vv = 0;
          if (on) {
            kk = k[src + t + lane];
            vv = v[src + t + lane];
          }
          step(on, kk, vv);
        }
        todo &= todo - 1;
        continue;
      }
      // consecutive small bins from p with at most 32 candidates in all
      const u32 xx = (lane >= p && act) ? (small ? n : 64u) : 0u;
      u32 incl = xx;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const u32 y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const unsigned over = __ballot_sync(0xffffffffu, incl > 32);
      const int e = over ? __ffs(over) - 1 : 32;  // batch = active bins in [p, e)
      const bool inb = lane >= p && lane < e && act;
      const u32 excl = incl - xx;
      const u32 total = __shfl_sync(0xffffffffu, incl, e - 1);
      W.mark[lane] = -1;
      __syncwarp();
      if (inb) W.mark[excl] = lane;
      __syncwarp();
      int jj = W.mark[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, jj, o);
        if (lane >= o && y > jj) jj = y;
      }
      __syncwarp();
      const bool has = (u32)lane < total;
      const int src = has ? jj : 0;
      const u32 bs = __shfl_sync(0xffffffffu, s, src);
      const u32 bex = __shfl_sync(0xffffffffu, excl, src);
      u64 kk = 0, vv = 0;
      u32 g = ~0u;
      if (has) {
        const u64 a = rbase + bs + (lane - bex);
        kk = k[a];
        vv = v[a];
        g = (u32)jj;
      }
      // bin g's records occupy lanes [gex, gex + gn); order each bin by
      // (canon k, v, k) = rec_less: a record's new lane is gex + the number
      // of its bin's records below it (ties by lane), gn compares each
      const int gs = has ? (int)g : 0;
      const u32 gex = __shfl_sync(0xffffffffu, excl, gs);
      const u32 gn_all = __shfl_sync(0xffffffffu, n, gs);  // (all lanes shuffle)
      const u32 gn = has ? gn_all : 1u;
      u32 maxn = gn;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) maxn = max(maxn, __shfl_xor_sync(0xffffffffu, maxn, o));
      if (maxn > 8) {
        // a bin of many records: one bitonic pass over the batch, by (bin, record)
        warp_sort_records(region, g, kk, vv);
      } else if (maxn > 1) {
        // few records per bin: rank by counting (canonical k first, the
        // rest of rec_less only on a tie)
        const u64 cc = canon_k(region, kk);
        W.pc[lane] = cc;
        W.pk[lane] = kk;
        W.pv[lane] = vv;
        __syncwarp();
        u32 rank = 0;
        if (has) {
          for (u32 j = 0; j < gn; ++j) {
            const u32 o = gex + j;
            const u64 oc = W.pc[o];
            bool less = oc < cc;
            if (oc == cc && o != (u32)lane) {
              const u64 ov = W.pv[o], ok = W.pk[o];
              less = ov < vv || (ov == vv && (ok < kk || (ok == kk && o < (u32)lane)));
            }
            rank += less;
          }
        }
        __syncwarp();
        if (has) {
          W.pk[gex + rank] = kk;
          W.pv[gex + rank] = vv;
        }
        __syncwarp();
        if (has) {
          kk = W.pk[lane];
          vv = W.pv[lane];
        }
        __syncwarp();
      }
      // lane order is now (bin, record); keep each bin's share
      const u32 g0 = __shfl_sync(0xffffffffu, i0, gs), g1 = __shfl_sync(0xffffffffu, i1, gs);
      const u32 idx = (u32)lane - gex;
      step(has && idx >= g0 && idx < g1, kk, vv);
      todo &= ~__ballot_sync(0xffffffffu, inb);
    }
   }
    __syncwarp();  // s_list is rewritten next round
  }

  if (lane == 0) {
    chunk_kept[c] = kept;
    if (kept) {
      atomicAdd(&group_kept[c >> 8], kept);
      atomicAdd(&kept_counts[r], (unsigned long long)kept);
    }
  }
#if CHGPU_SPA_CLOCKS
  if (lane == 0) {
    const u64 d = (u64)(clock64() - t_start);
    atomicMax(&g_spa_clk[0], d);
    atomicAdd(&g_spa_clk[1], d);
    atomicAdd(&g_spa_clk[2], 1ull);
    atomicAdd(&g_spa_clk[8 + min(31, (int)(d / 2000))], 1ull);
    if (d == g_spa_clk[0]) { g_spa_clk[3] = c; g_spa_clk[4] = n_batches; g_spa_clk[5] = n_listed; g_spa_clk[6] = kept; }
  }
#endif
}

#if CHGPU_SPA_CLOCKS
__global__ void k_spa_clocks_report() {
  printf("spa_chunks clocks: max %llu mean %llu chunks %llu | slowest c=%llu batches %llu listed %llu kept %llu\n",
         g_spa_clk[0], g_spa_clk[1] / max(1ull, g_spa_clk[2]), g_spa_clk[2], g_spa_clk[3], g_spa_clk[4], g_spa_clk[5], g_spa_clk[6]);
  printf("  hist(2000 clk buckets):");
  for (int i = 0; i < 32; ++i) printf(" %llu", g_spa_clk[8 + i]);
  printf("\n");
  const unsigned long long ns = max(1ull, g_spa_clk[26]);
  printf("spa_small: chunks %llu deferred %llu | gather max %llu mean %llu | sort max %llu mean %llu | scan max %llu mean %llu | m max %llu mean %llu\n",
         g_spa_clk[26], g_spa_clk[7], g_spa_clk[20], g_spa_clk[23] / ns, g_spa_clk[21], g_spa_clk[24] / ns,
         g_spa_clk[22], g_spa_clk[25] / ns, g_spa_clk[27], g_spa_clk[28] / ns);
  for (int i = 0; i < 40; ++i) g_spa_clk[i] = 0;
}
#endif

// Places each chunk's kept records (from k_spa_chunks' scratch) at its
// output offset: the kept counts of the earlier groups of 256 chunks plus
// those of the earlier chunks of its own group. Decoded to points.
__device__ void spa_emit_warp(u32 c, const FilterPlan* __restrict__ P_p, const u64* __restrict__ sk,
                              const u64* __restrict__ sv, const u32* __restrict__ chunk_kept,
                              const u32* __restrict__ group_kept, double2* __restrict__ out,
                              double2* hout, u32 hcap) {
  const SpaPlan& plan = P_p->spa;
  const int lane = threadIdx.x & 31;
  if (c >= plan.total_chunks) return;
  const u32 kept = chunk_kept[c];
  if (kept == 0) return;
  int r = 0;
  while (r < 3 && c >= plan.chunk_begin[r + 1]) ++r;
  const int region = r + 1;
  const u32 lo = (c - plan.chunk_begin[r]) * (u32)plan.chunk_size[r];
  const u32 g = c >> 8;
  u32 x = 0;
  for (u32 i = lane; i < g; i += 32) x += group_kept[i];
  for (u32 i = (g << 8) + lane; i < c; i += 32) x += chunk_kept[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  const u64 src = plan.off[r] + lo;
  for (u32 i = lane; i < kept; i += 32) {
    double px, py;
    decode_point(region, sk[src + i], sv[src + i], px, py);
    out[x + i] = make_double2(px, py);
    // (the host's copy, straight over PCIe while the emit runs)
    if (x + i < hcap) hout[x + i] = make_double2(px, py);
  }
}

// ------------------------------------------------------------------ device-side plan
//
// The plan of the filter path, computed on the device from K2's region
// counts and the quad, so the host enqueues the whole path without waiting
// for K2. A degenerate frame (no SPA, pipeline.cpp:53-71) leaves every
// region empty and the path idle.
// ------------------------------------------------------------------ chunk SPA finish

constexpr int kFinishThreads = 256;
constexpr size_t kFinishSmem =
    sizeof(BigSmem) > 8 * sizeof(SpaWarpSmem) ? sizeof(BigSmem) : 8 * sizeof(SpaWarpSmem);
static_assert(kFinishSmem >= (size_t)kWarpSortWarps * 3 * kWarpSortMax * sizeof(u64), "warp sorts fit");

// Everything after k_spa_small in one cooperative launch (every CTA
// resident): if it deferred any chunk, the bin sorts (bins of 33..256
// candidates by a warp, up to kBinSortMax by a CTA), a grid barrier, the
// sorted chunk SPA (spa_chunk_warp) over the deferred chunks, a grid
// barrier; then always the emit (spa_emit_warp) of every chunk. With no
// deferred chunk this is a single pass of the emit.
__global__ __launch_bounds__(kFinishThreads) void k_spa_finish(
    u64* __restrict__ k, u64* __restrict__ v, const u32* __restrict__ bcur,
    const u32* __restrict__ bstart, const u32* __restrict__ bmap, const u32* __restrict__ first_bin,
    const FilterPlan* __restrict__ P_p, const u32* __restrict__ big, const u32* __restrict__ nbig_p,
    u32* __restrict__ overflow, const u32* __restrict__ defer, const u32* __restrict__ ndefer_p,
    u64* __restrict__ sk, u64* __restrict__ sv, u32* __restrict__ chunk_kept,
    u32* __restrict__ group_kept, unsigned long long* __restrict__ kept_counts,
    double2* __restrict__ out, u32* __restrict__ bar, ReadbackArgs rb) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5;
  const u32 nwarps = gridDim.x * (kFinishThreads / 32);
  const u32 gw = blockIdx.x * (kFinishThreads / 32) + warp;
  const u32 nd = *ndefer_p;
#if CHGPU_FINISH_CLOCKS
  long long fc[6] = {clock64(), 0, 0, 0, 0, 0};
#endif
  if (nd) {
    const FilterPlan& P = *P_p;
    bin_sort_warp_body(k, v, P, bstart, bcur, big, nbig_p[0],
                       reinterpret_cast<u64*>(smem) + (size_t)warp * 3 * kWarpSortMax, blockIdx.x,
                       gridDim.x);
    __syncthreads();
#if CHGPU_FINISH_CLOCKS
    fc[1] = clock64();
#endif
    bin_sort_big_body(k, v, P, bstart, bcur, big + kBigListB, nbig_p[1], overflow,
                      *reinterpret_cast<BigSmem*>(smem), blockIdx.x, gridDim.x);
#if CHGPU_FINISH_CLOCKS
    fc[2] = clock64();
#endif
    grid_barrier(bar, 0);
#if CHGPU_FINISH_CLOCKS
    fc[3] = clock64();
#endif
    SpaWarpSmem& W = reinterpret_cast<SpaWarpSmem*>(smem)[warp];
    for (u32 i = gw; i < nd; i += nwarps)
      spa_chunk_warp(defer[i], k, v, bcur, bstart, bmap, first_bin, P_p, sk, sv, chunk_kept,
                     group_kept, kept_counts, W);
#if CHGPU_FINISH_CLOCKS
    fc[4] = clock64();
#endif
    grid_barrier(bar, 1);
  }
#if CHGPU_FINISH_CLOCKS
  fc[5] = clock64();
  if (threadIdx.x == 0) {
    for (int q = 1; q < 6; ++q) atomicMax(&g_fin_clk[q], (u64)(fc[q] - fc[q - 1]));
    if (blockIdx.x == 0) {
      g_fin_clk[6] = nbig_p[0];
      g_fin_clk[7] = nbig_p[1];
      g_fin_clk[8] = nd;
    }
  }
#endif
  const u32 total = P_p->spa.total_chunks;
  for (u32 c = gw; c < total; c += nwarps)
    spa_emit_warp(c, P_p, sk, sv, chunk_kept, group_kept, out, rb.h_chains, rb.h_chains_cap);
  if (rb.h_done) __threadfence_system();  // this CTA's host chain writes, before the flag
  // every CTA is done with the counters: CTA 0 hands them to the host and
  // clears them (no separate read-back launch), then raises the call's flag
  grid_barrier(bar, nd ? 2u : 0u);
  if (blockIdx.x == 0) {
    readback_block(rb);
    if (rb.h_done) {
      __threadfence_system();
      __syncthreads();
      if (threadIdx.x == 0) *reinterpret_cast<volatile u32*>(rb.h_done) = rb.seq;
    }
  }
}

// ------------------------------------------------------------------ launchers

cudaError_t launch_bin_scan(const QuadInfo* qinfo, u32* counts, u64 chunk_count, int log2nb,
                     const u32* bcnt, const u32* bw, FilterPlan* plan, u32* bstart, u32* bthr,
                     u32* tcoarse, u32* first_bin, FilterAux aux, u32* bar, u32* overflow,
                     cudaStream_t st) {
  const u32 tiles = std::max(1u, (1u << log2nb) / kBinTile);
  dim3 grid(4 * tiles), block(kBinThreads);
  void* args[] = {(void*)&qinfo, (void*)&counts, (void*)&chunk_count, (void*)&log2nb,
                  (void*)&bcnt, (void*)&bw, (void*)&plan, (void*)&bstart, (void*)&bthr,
                  (void*)&tcoarse, (void*)&first_bin, (void*)&aux.tsum, (void*)&aux.agg_seg, (void*)&aux.agg_val, (void*)&bar,
                  (void*)&overflow};
  // cooperative: the launch fails rather than run with a CTA not resident
  // (the caller checked bin_scan_blocks against the device's residency and
  // checks the launch status)
  return cudaLaunchCooperativeKernel((const void*)k_bin_scan, grid, block, args, 0, st);
}

u32 bin_scan_blocks(int log2nb) { return 4 * std::max(1u, (1u << log2nb) / kBinTile); }

void launch_filter(const u64* seg, const u64* segcnt, u32 nseg,
                   const double2* pts, const FilterPlan* P, const QuadInfo* qinfo,
                   const u32* bstart, const u32* bthr, const u32* tcoarse, int log2nb, u32* bcur,
                   u32* bmap, u64* kout, u64* vout, u32* big, u32* nbig, unsigned long long* ncand,
                   const u32* overflow, cudaStream_t st) {
  if (nseg == 0) return;
  // one persistent CTA per SM (the warp-stride loop then has no partial
  // last wave)
  const u32 blocks = std::min<u32>((nseg + kFilterThreads / 32 - 1) / (kFilterThreads / 32),
                                   (u32)device_limits().filter_resident);
  k_filter<<<blocks, kFilterThreads, filter_smem_bytes(log2nb), st>>>(
      seg, segcnt, nseg, pts, P, qinfo, bstart, bthr, tcoarse, bcur, bmap, kout, vout, big,
      nbig, ncand, overflow);
}

// The chunk SPA: k_spa_small over every chunk, then (after the caller's
// bin sorts) k_spa_chunks over the chunks it deferred, then k_spa_emit.
void launch_spa_small(const u64* k, const u64* v, const u32* bcur, const u32* bstart,
                      const u32* bmap, const u32* first_bin, const FilterPlan* P, u32 max_chunks,
                      u64* sk, u64* sv, u32* chunk_kept, u32* group_kept,
                      unsigned long long* kept_counts, u32* defer, u32* ndefer, u32 cap,
                      cudaStream_t st) {
  if (max_chunks == 0) return;
  cudaMemsetAsync(group_kept, 0, ((max_chunks + 255) / 256) * sizeof(u32), st);
  k_spa_small<<<(max_chunks + kSmallWarps - 1) / kSmallWarps, 32 * kSmallWarps, kSmallSmem, st>>>(
      k, v, bcur, bstart, bmap, first_bin, P, sk, sv, chunk_kept, group_kept, kept_counts, defer,
      ndefer, std::min<u32>(cap, (u32)kSmallCap));
}

cudaError_t launch_spa_finish(u64* k, u64* v, const u32* bcur, const u32* bstart, const u32* bmap,
                              const u32* first_bin, const FilterPlan* P, const u32* big,
                              const u32* nbig, u32* overflow, const u32* defer, const u32* ndefer,
                              u64* sk, u64* sv, u32* chunk_kept, u32* group_kept,
                              unsigned long long* kept_counts, double2* out, u32* bar,
                              u32 max_chunks, const ReadbackArgs& rb_in, cudaStream_t st) {
  ReadbackArgs rb = rb_in;
  if (max_chunks == 0) return cudaSuccess;
  const u32 blocks = std::max(1u, std::min<u32>((u32)device_limits().finish_coop,
                                                (max_chunks + 7) / 8));
  void* args[] = {(void*)&k, (void*)&v, (void*)&bcur, (void*)&bstart, (void*)&bmap,
                  (void*)&first_bin, (void*)&P, (void*)&big, (void*)&nbig, (void*)&overflow,
                  (void*)&defer, (void*)&ndefer, (void*)&sk, (void*)&sv, (void*)&chunk_kept,
                  (void*)&group_kept, (void*)&kept_counts, (void*)&out, (void*)&bar, (void*)&rb};
  const cudaError_t e = cudaLaunchCooperativeKernel((const void*)k_spa_finish, dim3(blocks),
                                                    dim3(kFinishThreads), args, kFinishSmem, st);
#if CHGPU_SPA_CLOCKS
  k_spa_clocks_report<<<1, 1, 0, st>>>();
#endif
#if CHGPU_FINISH_CLOCKS
  k_fin_clocks_report<<<1, 1, 0, st>>>();
#endif
  return e;
}


// Dynamic shared memory opt-in and residency of the filter kernels for the
// current device (device_limits()).
cudaError_t configure_filter_kernels(DeviceLimits* lim) {
  cudaError_t e = cudaFuncSetAttribute((const void*)k_spa_small,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmallSmem);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute((const void*)k_spa_finish,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFinishSmem);
  if (e != cudaSuccess) return e;
  int fo = 0;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&fo, k_spa_finish, kFinishThreads, kFinishSmem)) !=
      cudaSuccess)
    return e;
  lim->finish_coop = fo * lim->sms;
  const int fsm = (int)filter_smem_bytes(kMaxFilterLog2);
  if ((e = cudaFuncSetAttribute((const void*)k_filter, cudaFuncAttributeMaxDynamicSharedMemorySize, fsm)) !=
      cudaSuccess)
    return e;
  int occ = 0;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_filter, kFilterThreads, fsm)) != cudaSuccess)
    return e;
  lim->filter_resident = std::max(occ, 1) * lim->sms;
  occ = 0;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_bin_scan, kBinThreads, 0)) != cudaSuccess)
    return e;
  lim->binscan_coop = occ * lim->sms;
  return cudaSuccess;
}

}  // namespace chgpu
