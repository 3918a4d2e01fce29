// K1 (extreme quad) and K2 (classify + round-1 discard + 4-way compaction).
//
// K1 follows find_extremes/fold (reference extremes.cpp:12-47): four
// lexicographic min/max reductions with the earliest index winning among
// ==-equal points. It streams the input once (16 B/point).
//
// K2 fuses classify_point (classify.hpp:42-48), the per-region counting of
// classify (classify.cpp:9-33) and discard_round1's partition
// (classify.cpp:40-87) into one pass: every point is read once, labelled in
// registers, and survivors are written straight into per-region output
// streams as sort-ready (k, v) records (chgpu_internal.cuh key codec).
// Stream offsets come from a single-pass decoupled look-back with four
// independent chains (one per region). Interior points are never written.

#include <algorithm>

#include "chgpu_internal.cuh"
#include "kernels.h"

namespace chgpu {

// ------------------------------------------------------------------ K1

__device__ __forceinline__ bool beats_left(const Cand& a, const Cand& b) {
  if (less_xy(a.x, a.y, b.x, b.y)) return true;
  if (less_xy(b.x, b.y, a.x, a.y)) return false;
  return a.i < b.i;
}
__device__ __forceinline__ bool beats_bottom(const Cand& a, const Cand& b) {
  if (less_yx(a.x, a.y, b.x, b.y)) return true;
  if (less_yx(b.x, b.y, a.x, a.y)) return false;
  return a.i < b.i;
}
__device__ __forceinline__ bool beats_right(const Cand& a, const Cand& b) {
  if (less_xy(b.x, b.y, a.x, a.y)) return true;
  if (less_xy(a.x, a.y, b.x, b.y)) return false;
  return a.i < b.i;
}
__device__ __forceinline__ bool beats_top(const Cand& a, const Cand& b) {
  if (less_yx(b.x, b.y, a.x, a.y)) return true;
  if (less_yx(a.x, a.y, b.x, b.y)) return false;
  return a.i < b.i;
}

// Empty candidates carry +-inf sentinels (index ~0) and lose to any point.
__device__ __forceinline__ void merge_quad(QuadCand& acc, const QuadCand& o) {
  if (beats_left(o.c[0], acc.c[0])) acc.c[0] = o.c[0];
  if (beats_bottom(o.c[1], acc.c[1])) acc.c[1] = o.c[1];
  if (beats_right(o.c[2], acc.c[2])) acc.c[2] = o.c[2];
  if (beats_top(o.c[3], acc.c[3])) acc.c[3] = o.c[3];
}

__device__ __forceinline__ Cand shfl_cand(const Cand& c, int src) {
  Cand r;
  r.x = __shfl_down_sync(0xffffffffu, c.x, src);
  r.y = __shfl_down_sync(0xffffffffu, c.y, src);
  r.i = __shfl_down_sync(0xffffffffu, c.i, src);
  return r;
}

// Folds one point visited in increasing index order: strict comparisons
// keep the earliest of ==-equal points, exactly like fold() (:12-17).
// A point strictly inside the running box on a corner's axis cannot win that
// corner, so each corner costs one compare on the common path; the full
// lexicographic test only runs on the rare boundary hits. Empty corners
// hold +-inf sentinels (inputs are finite), so no emptiness test is needed.
__device__ __forceinline__ void fold_point(QuadCand& a, double x, double y, u64 i) {
  if (!(x > a.c[0].x) && less_xy(x, y, a.c[0].x, a.c[0].y)) a.c[0] = Cand{x, y, i};
  if (!(y > a.c[1].y) && less_yx(x, y, a.c[1].x, a.c[1].y)) a.c[1] = Cand{x, y, i};
  if (!(x < a.c[2].x) && less_xy(a.c[2].x, a.c[2].y, x, y)) a.c[2] = Cand{x, y, i};
  if (!(y < a.c[3].y) && less_yx(a.c[3].x, a.c[3].y, x, y)) a.c[3] = Cand{x, y, i};
}

__device__ __forceinline__ void empty_quad(QuadCand& a) {
  a.c[0] = Cand{INFINITY, INFINITY, ~0ull};
  a.c[1] = Cand{INFINITY, INFINITY, ~0ull};
  a.c[2] = Cand{-INFINITY, -INFINITY, ~0ull};
  a.c[3] = Cand{-INFINITY, -INFINITY, ~0ull};
}

constexpr int kK1Threads = 256;
#ifndef CHGPU_K1_UNROLL
#define CHGPU_K1_UNROLL 8
#endif
constexpr int kK1Unroll = CHGPU_K1_UNROLL;  // points per lane per warp tile
#ifndef CHGPU_K1_MINB
#define CHGPU_K1_MINB 3
#endif

// Block-wide merge of nparts partials and the QuadInfo (with
// frame_vertices, extremes.cpp:49-57). Ties fall back to the global index,
// so the result is independent of the merge order.
__device__ void merge_partials_block(const QuadCand* __restrict__ partials, int nparts,
                                     QuadInfo* __restrict__ out, QuadCand* __restrict__ raw_out,
                                     int log2nb) {
  QuadCand acc;
  empty_quad(acc);
  for (int p = threadIdx.x; p < nparts; p += blockDim.x) merge_quad(acc, partials[p]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    QuadCand other;
#pragma unroll
    for (int c = 0; c < 4; ++c) other.c[c] = shfl_cand(acc.c[c], o);
    merge_quad(acc, other);
  }
  __shared__ QuadCand sacc[32];
  if ((threadIdx.x & 31) == 0) sacc[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int t = 1; t < (int)(blockDim.x >> 5); ++t) merge_quad(acc, sacc[t]);
    if (raw_out) *raw_out = acc;
    if (out) {
      QuadInfo qi;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        qi.q[2 * c] = acc.c[c].x;
        qi.q[2 * c + 1] = acc.c[c].y;
        qi.idx[c] = acc.c[c].i;
      }
      // frame_vertices (extremes.cpp:49-57): consecutive and wrap duplicates
      // collapse; compared by == like Point2::operator==.
      u32 k = 1;
      double lx = qi.q[0], ly = qi.q[1];
#pragma unroll
      for (int c = 1; c < 4; ++c) {
        const double x = qi.q[2 * c], y = qi.q[2 * c + 1];
        if (!(lx == x && ly == y)) {
          ++k;
          lx = x;
          ly = y;
        }
      }
      if (k > 1 && qi.q[0] == lx && qi.q[1] == ly) --k;
      qi.frame_size = k;
      qi.degenerate = k <= 2 ? 1u : 0u;
      quad_derive(qi, log2nb);
      *out = qi;
    }
  }
}

// Grid-stride pass: thread t visits t, t+T, t+2T, ... in increasing order,
// so its running fold is the sequential fold of its subsequence. With a
// ticket counter, the last block to finish (over every launch of the call:
// total_parts blocks) merges all partials itself, so no final launch is
// needed.
//
// kCheck (file ingestion): also flags any non-finite coordinate
// (io.cpp:38-42 require_finite; the reference rejects them before hulling).
template <bool kCheck>
__global__ __launch_bounds__(kK1Threads, CHGPU_K1_MINB) void k_extremes_partial(
    const double2* __restrict__ pts, u64 n, u64 base_index, QuadCand* __restrict__ partials,
    u32 part_base, u32* __restrict__ ticket, u32 total_parts, QuadInfo* __restrict__ out,
    u32* __restrict__ nonfinite, int log2nb) {
  // a programmatically launched K2 may start as K1's CTAs retire (it waits
  // for K1's completion before reading the quad)
  asm volatile("griddepcontrol.launch_dependents;");
  QuadCand acc;
  empty_quad(acc);
  bool finite = true;
  // Warp tiles of 32 * kK1Unroll contiguous points (every load of a tile
  // in flight before the fold), grid-strided over the warps; a lane visits
  // its points in increasing index order, as the fold requires.
  constexpr u64 kTile = 32 * kK1Unroll;
  const int ln = threadIdx.x & 31;
  const u64 tw = (u64)gridDim.x * (kK1Threads / 32);
  u64 t = (u64)blockIdx.x * (kK1Threads / 32) + (threadIdx.x >> 5);
  for (; (t + 1) * kTile <= n; t += tw) {
    const u64 i0 = t * kTile + ln;
    double2 p[kK1Unroll];
#pragma unroll
    for (int u = 0; u < kK1Unroll; ++u) p[u] = ldg_stream(pts + i0 + 32 * u);
#pragma unroll
    for (int u = 0; u < kK1Unroll; ++u) {
      if (kCheck) finite &= isfinite(p[u].x) && isfinite(p[u].y);
      fold_point(acc, p[u].x, p[u].y, base_index + i0 + 32 * u);
    }
  }
  if (t * kTile < n) {  // the one partial tile
    for (u64 i = t * kTile + ln; i < n; i += 32) {
      const double2 p = ldg_stream(pts + i);
      if (kCheck) finite &= isfinite(p.x) && isfinite(p.y);
      fold_point(acc, p.x, p.y, base_index + i);
    }
  }
  if (kCheck && !__all_sync(0xffffffffu, finite) && (threadIdx.x & 31) == 0) atomicOr(nonfinite, 1u);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    QuadCand other;
#pragma unroll
    for (int c = 0; c < 4; ++c) other.c[c] = shfl_cand(acc.c[c], o);
    merge_quad(acc, other);
  }
  __shared__ QuadCand warp_acc[kK1Threads / 32];
  __shared__ int s_last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) warp_acc[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < kK1Threads / 32; ++w) merge_quad(acc, warp_acc[w]);
    partials[part_base + blockIdx.x] = acc;
    s_last = 0;
    if (ticket) {
      __threadfence();
      s_last = atomicAdd(ticket, 1u) == total_parts - 1;
    }
  }
  __syncthreads();
  if (s_last) {
    __threadfence();
    merge_partials_block(partials, (int)total_parts, out, nullptr, log2nb);
  }
}

__global__ __launch_bounds__(1024) void k_extremes_final(const QuadCand* __restrict__ partials, int nparts,
                                 QuadInfo* __restrict__ out, QuadCand* __restrict__ raw_out) {
  merge_partials_block(partials, nparts, out, raw_out, 0);
}

// ------------------------------------------------------------------ K2

// classify_point (classify.hpp:42-48): the first CCW quad edge the point is
// strictly right of, else Interior.
struct QuadEdges {
  double ax[4], ay[4], ex[4], ey[4];
};

// All four predicates are evaluated and the first Right one selected, so the
// warp never diverges on the data; evaluating a predicate the reference would
// have skipped has no effect on the result.
__device__ __forceinline__ int classify(const QuadEdges& e, double px, double py) {
  // The four Right flags as a bit mask, the region as its lowest set bit:
  // no select chain the compiler could turn into divergent early exits.
  const u32 m = (u32)(cross_edge(e.ax[0], e.ay[0], e.ex[0], e.ey[0], px, py) < 0.0) |
                (u32)(cross_edge(e.ax[1], e.ay[1], e.ex[1], e.ey[1], px, py) < 0.0) << 1 |
                (u32)(cross_edge(e.ax[2], e.ay[2], e.ex[2], e.ey[2], px, py) < 0.0) << 2 |
                (u32)(cross_edge(e.ax[3], e.ay[3], e.ex[3], e.ey[3], px, py) < 0.0) << 3;
  // lowest set bit + 1 (0: no edge has the point on its right, Interior):
  // an 8-entry table of 3-bit fields for the low three flags (one 32-bit
  // shift, not the XU pipe's FLO), edge 4 when only it is set
  return (int)((0x28b28c28b288ull >> (3 * m)) & 7u);
}

// Two-ended stream layout: streams 1 and 2 share kbuf[0, ncap) growing
// from both ends, streams 3 and 4 share kbuf[ncap, 2*ncap).
__device__ __forceinline__ u64 stream_slot(int s, u64 pos, u64 ncap) {
  switch (s) {
    case 1: return pos;
    case 2: return ncap - 1 - pos;
    case 3: return ncap + pos;
    default: return 2 * ncap - 1 - pos;
  }
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  const int bytes = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(gmem), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// One tile (2048 points) per CTA, streamed into shared memory with
// cp.async. The region sort that follows canonically orders each region by
// its full key, so the order of records inside a stream is free: a tile
// reserves its output range per stream with one global atomicAdd each,
// instead of an ordered (look-back) scan. Per point the work is the
// classification, a register counter increment and one record store.
template <bool kGivenLabels>
__global__ __launch_bounds__(kK2Threads, 3) void k_classify_compact(
    const double2* __restrict__ pts, u32 n, const QuadInfo* __restrict__ qinfo,
    const unsigned char* __restrict__ given_labels, int force_lex, u64* __restrict__ kbuf,
    u64* __restrict__ vbuf, u64 ncap, u32* __restrict__ counts_out) {
  extern __shared__ __align__(16) double2 sbuf[];  // [kK2Tile]
  __shared__ u32 s_wtot[kK2Threads / 32][4];
  __shared__ u32 s_base[4];
  __shared__ QuadEdges s_edges;
  __shared__ int s_lex;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const u64 tile_base = (u64)blockIdx.x * kK2Tile;
#pragma unroll
  for (int j = 0; j < kK2Items; ++j) {
    const u64 idx = tile_base + (u64)j * kK2Threads + tid;
    const bool ok = idx < n;
    cp_async16(sbuf + j * kK2Threads + tid, ok ? (const void*)(pts + idx) : (const void*)pts, ok);
  }
  cp_async_commit();
  if (tid == 0) {
    const QuadInfo qi = *qinfo;
    for (int c = 0; c < 4; ++c) {
      const int d = (c + 1) & 3;
      s_edges.ax[c] = qi.q[2 * c];
      s_edges.ay[c] = qi.q[2 * c + 1];
      s_edges.ex[c] = __dsub_rn(qi.q[2 * d], qi.q[2 * c]);
      s_edges.ey[c] = __dsub_rn(qi.q[2 * d + 1], qi.q[2 * c + 1]);
    }
    // Degenerate frame: survivors all go to stream 1 in lexicographic
    // encoding for the hull_oracle-style finish (pipeline.cpp:53-71).
    s_lex = force_lex || (!kGivenLabels && qi.degenerate);
  }
  __syncthreads();
  const bool lex = s_lex != 0;
  const QuadEdges e = s_edges;
  cp_async_wait<0>();  // each thread reads back only its own copies

  u64 codes = 0;  // 3 bits of stream id per item
  u32 cnt[4] = {0, 0, 0, 0};
#pragma unroll
  for (int j = 0; j < kK2Items; ++j) {
    const u64 idx = tile_base + (u64)j * kK2Threads + tid;
    int r = 0;
    if (idx < n) {
      if (kGivenLabels) {
        r = (int)given_labels[idx];
      } else {
        const double2 p = sbuf[j * kK2Threads + tid];
        r = classify(e, p.x, p.y);
      }
      if (lex && r != 0) r = 1;
    }
    codes |= (u64)r << (3 * j);
#pragma unroll
    for (int s = 0; s < 4; ++s) cnt[s] += (r == s + 1);
  }
  // Warp-exclusive prefix of the per-thread counts, per stream.
  u32 excl[4];
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    u32 x = cnt[s];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const u32 y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    excl[s] = x - cnt[s];
    if (lane == 31) s_wtot[warp][s] = x;
  }
  __syncthreads();
  if (tid < 4) {
    u32 tot = 0;
    for (int w = 0; w < kK2Threads / 32; ++w) {
      const u32 c = s_wtot[w][tid];
      s_wtot[w][tid] = tot;
      tot += c;
    }
    s_base[tid] = tot ? atomicAdd(&counts_out[tid + 1], tot) : 0u;
  }
  __syncthreads();
  u32 pos0 = s_base[0] + s_wtot[warp][0] + excl[0];
  u32 pos1 = s_base[1] + s_wtot[warp][1] + excl[1];
  u32 pos2 = s_base[2] + s_wtot[warp][2] + excl[2];
  u32 pos3 = s_base[3] + s_wtot[warp][3] + excl[3];
  // Straight-line per item (selects, one predicated store pair): the key
  // codec of chgpu_internal.cuh written as swap + complement masks, and the
  // two-ended stream slot as base +/- position.
#pragma unroll
  for (int j = 0; j < kK2Items; ++j) {
    const u32 r = (codes >> (3 * j)) & 7;
    const double2 p = sbuf[j * kK2Threads + tid];
    const u64 ox = ord_enc(p.x), oy = ord_enc(p.y);
    const bool sw = !lex && !(r & 1u);
    const u64 kmask = (!lex && r >= 3) ? ~0ull : 0ull;
    const u64 vmask = (!lex && (r == 1 || r == 4)) ? ~0ull : 0ull;
    const u64 k = (sw ? oy : ox) ^ kmask;
    const u64 v = (sw ? ox : oy) ^ vmask;
    const u32 pp = r == 1 ? pos0 : (r == 2 ? pos1 : (r == 3 ? pos2 : pos3));
    pos0 += (r == 1);
    pos1 += (r == 2);
    pos2 += (r == 3);
    pos3 += (r == 4);
    const u64 base = r == 1 ? 0ull : (r == 2 ? ncap - 1 : (r == 3 ? ncap : 2 * ncap - 1));
    const u64 slot = (r & 1u) ? base + pp : base - pp;
    if (r) {
      kbuf[slot] = k;
      vbuf[slot] = v;
    }
  }
}

#ifndef CHGPU_K2_MINB
#define CHGPU_K2_MINB 4
#endif
#ifndef CHGPU_K2_ABL  // ablation bits, A/B timing only (results are invalid when set)
#define CHGPU_K2_ABL 0
#endif
// K2 of the pre-filtered path (k_filter.cu): classify, count, and for
// every survivor one fire-and-forget increment of its SPA bin's count and
// (for one record in 2^k, wmask) a running max of its guarded key w.
//
// Survivor layout: each warp owns the 256-slot segment of its 256 input
// points (seg + 256 * warp index) and writes its survivors there in any
// order (the filter re-establishes the order inside a bin by the bin sort,
// and a key names its region through its bin), with the survivor count in
// segcnt[warp index]. Positions come from one 32-bit warp scan, so no CTA
// barrier or global reservation sits between the loads and the stores. A
// degenerate frame (pipeline.cpp:53-71) writes LEX records into dense
// stream 1 of (kbuf, vbuf) instead, exactly like k_classify_compact.
__global__ __launch_bounds__(kK2Threads, CHGPU_K2_MINB) void k_classify_survivors(
    const double2* __restrict__ pts, u32 n, const QuadInfo* __restrict__ qinfo,
    u64* __restrict__ seg, u64* __restrict__ segcnt, u64* __restrict__ kbuf,
    u64* __restrict__ vbuf, u32* __restrict__ counts_out, int log2nb, u32* __restrict__ bcnt,
    u32* __restrict__ bw, u32 wmask) {
  __shared__ u32 s_segT[kK2Threads / 32];  // (degenerate frame only)
  __shared__ u32 s_base;
  __shared__ __align__(16) double2 s_seg[kK2Threads / 32 * kSegPts];
  __shared__ unsigned short s_stag[kK2Threads / 32 * kSegPts];  // segment position << 2 | region
  __shared__ double2 s_bmap[kK2Threads / 32][4];  // (lo, scale) per region, per warp

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const u32 sidx = blockIdx.x * (kK2Threads / 32) + warp;
  const u32 base = sidx * kSegPts;  // n < 2^32
  double2 p[kSegItems];
#pragma unroll
  for (int j = 0; j < kSegItems; ++j) {
    const u32 idx = base + j * 32 + lane;
    p[j] = idx < n ? ldg_stream(pts + idx) : make_double2(0.0, 0.0);
  }
  // (launched programmatically behind K1: the point loads above are in
  // flight; K1's quad is complete and visible past this point)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // the quad's edges by uniform loads (one transaction per warp, L1 hits
  // after the first warp), the bin map of region `lane` in lanes 0..3 into
  // the warp's own table: no CTA barrier between the point loads and the
  // classification
  // (K1 may still be running when this CTA starts: its output is read with
  // ordinary cached loads kept below the wait, not as read-only data)
  QuadEdges e;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    e.ax[c] = ld_after_wait_f64(&qinfo->q[2 * c]);
    e.ay[c] = ld_after_wait_f64(&qinfo->q[2 * c + 1]);
    e.ex[c] = ld_after_wait_f64(&qinfo->ex[c]);
    e.ey[c] = ld_after_wait_f64(&qinfo->ey[c]);
  }
  const bool lex = ld_after_wait_u32(&qinfo->degenerate) != 0;
  // (the bin map's scale comes precomputed: quad_derive at the call's bin count)
  if (lane < 4)
    s_bmap[warp][lane] = make_double2(ld_after_wait_f64(&qinfo->blo[lane]), ld_after_wait_f64(&qinfo->bscale[lane]));

  u32 codes = 0;  // 3 bits of stream id per item
  u32 cnt = 0;    // survivors of this lane
#pragma unroll
  for (int j = 0; j < kSegItems; ++j) {
    const u32 idx = base + j * 32 + lane;
    int r = classify(e, p[j].x, p[j].y);  // unconditional: no per-item branch
    r = idx < n ? r : 0;  // (a degenerate frame only asks r != 0)
    codes |= (u32)r << (3 * j);
    cnt += r != 0;
  }
  u32 incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const u32 y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  const u32 tot = __shfl_sync(0xffffffffu, incl, 31);  // the segment's survivors

  if (lex) {  // uniform: dense stream 1 through a CTA reservation
    if (lane == 0) s_segT[warp] = tot;
    __syncthreads();
    if (tid == 0) {
      u32 sum = 0;
      for (int w = 0; w < kK2Threads / 32; ++w) sum += s_segT[w];
      s_base = sum ? atomicAdd(&counts_out[1], sum) : 0u;
    }
    __syncthreads();
    u32 pp = s_base + (incl - cnt);
    for (int w = 0; w < warp; ++w) pp += s_segT[w];
#pragma unroll
    for (int j = 0; j < kSegItems; ++j) {
      if (!((codes >> (3 * j)) & 7)) continue;
      kbuf[pp] = ord_enc(p[j].x);
      vbuf[pp] = ord_enc(p[j].y);
      ++pp;
    }
    return;
  }

  if (lane == 0) segcnt[sidx] = tot;
  // Stage the segment in shared memory in slot order, then work on it with
  // every lane busy: ~44% of the items survive, so the per-survivor code
  // runs in ceil(count / 32) rounds instead of once per item, and the
  // segment's global stores are coalesced.
  double2* const ss = s_seg + warp * kSegPts;
  unsigned short* const stg = s_stag + warp * kSegPts;
  {
    // shared-window addresses held in registers and predicated stores:
    // no per-item branch and no re-derived shared base per item
    const u32 a_pt = (u32)__cvta_generic_to_shared(ss), a_tg = (u32)__cvta_generic_to_shared(stg);
    u32 pos = incl - cnt;
#pragma unroll
    for (int j = 0; j < kSegItems; ++j) {
      const u32 r = (codes >> (3 * j)) & 7;
      asm volatile(
          "{\n\t.reg .pred q;\n\t"
          "setp.ne.u32 q, %0, 0;\n\t"
          "@q st.shared.v2.f64 [%1], {%2, %3};\n\t"
          "@q st.shared.u16 [%4], %5;\n\t}" ::"r"(r),
          "r"(a_pt + 16 * pos), "d"(p[j].x), "d"(p[j].y), "r"(a_tg + 2 * pos),
          "h"((unsigned short)(((j * 32 + lane) << 2) | (r - 1)))
          : "memory");
      pos += r != 0;
    }
  }
  __syncwarp();
  if (CHGPU_K2_ABL & 8) return;
  u64* const out = seg + (u64)base;
  const u32 top = (1u << log2nb) - 1u;
  for (u32 slot = lane; slot < tot; slot += 32) {
    const double2 q = ss[slot];
    const u32 tg = stg[slot];
    const u32 ri = tg & 3u;
    const bool odd = (ri & 1u) == 0;  // LL, UR (ri 0, 2): primary x
    const double prim = odd ? q.x : q.y;
    const double2 bm = s_bmap[warp][ri];
    const u32 b = (ri << log2nb) | bin_of(bm.x, bm.y, top, ri, prim);
    if (!(CHGPU_K2_ABL & 1)) atomicAdd(bcnt + b, 1u);
    // w = wkey(v): the guarded coordinate with -0.0 folded onto +0.0,
    // complemented for the min-regions LL and UL; kept as w >> kWShift
    const double g = odd ? q.y : q.x;
    const u64 key = filter_key(b, tg >> 2, ord_enc_z(g) ^ ((ri == 0 || ri == 3) ? ~0ull : 0ull));
    // any subset of a bin's records gives a valid (lower) max: sample
    if (!(CHGPU_K2_ABL & 2) && (slot & wmask) == 0) atomicMax(bw + b, (u32)key);
    if (!(CHGPU_K2_ABL & 4)) out[slot] = key;  // the filter reads 8 B per survivor

  }
  // (region totals: the bin scan sums the bin counts)
}

// Labels only (the classify() stage tap, classify.cpp:9-33).
__global__ void k_classify_labels(const double2* __restrict__ pts, u64 n,
                                  const QuadInfo* __restrict__ qinfo,
                                  unsigned char* __restrict__ labels,
                                  unsigned long long* __restrict__ counts) {
  __shared__ QuadEdges s_edges;
  __shared__ unsigned long long s_cnt[5];
  if (threadIdx.x < 5) s_cnt[threadIdx.x] = 0;
  if (threadIdx.x == 0) {
    const QuadInfo qi = *qinfo;
    for (int c = 0; c < 4; ++c) {
      const int d = (c + 1) & 3;
      s_edges.ax[c] = qi.q[2 * c];
      s_edges.ay[c] = qi.q[2 * c + 1];
      s_edges.ex[c] = __dsub_rn(qi.q[2 * d], qi.q[2 * c]);
      s_edges.ey[c] = __dsub_rn(qi.q[2 * d + 1], qi.q[2 * c + 1]);
    }
  }
  __syncthreads();
  const QuadEdges e = s_edges;
  u32 local[5] = {0, 0, 0, 0, 0};
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
    const double2 p = ldg_stream(pts + i);
    const int r = classify(e, p.x, p.y);
    labels[i] = (unsigned char)r;
    ++local[r];
  }
  for (int r = 0; r < 5; ++r) {
    u32 c = local[r];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(&s_cnt[r], (unsigned long long)c);
  }
  __syncthreads();
  if (threadIdx.x < 5 && s_cnt[threadIdx.x]) atomicAdd(&counts[threadIdx.x], s_cnt[threadIdx.x]);
}

// ------------------------------------------------------------------ launchers

int extremes_blocks(int requested) {
  // One resident wave at most: a grid-stride kernel gains nothing from a
  // second partial wave, it only adds a tail.
  return std::max(1, std::min(requested, device_limits().k1_wave));
}

int extremes_wave(int sms) {
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_extremes_partial<true>, kK1Threads, 0);
  return std::max(1, occ) * std::max(1, sms);
}

int launch_extremes_partial(const double2* pts, u64 n, u64 base_index, QuadCand* partials,
                            int blocks, cudaStream_t st, u32 part_base, u32* ticket,
                            u32 total_parts, QuadInfo* out, u32* nonfinite, int log2nb) {
  blocks = extremes_blocks(blocks);
  if (nonfinite)
    k_extremes_partial<true><<<blocks, kK1Threads, 0, st>>>(pts, n, base_index, partials, part_base,
                                                            ticket, total_parts, out, nonfinite,
                                                            log2nb);
  else
    k_extremes_partial<false><<<blocks, kK1Threads, 0, st>>>(pts, n, base_index, partials, part_base,
                                                             ticket, total_parts, out, nullptr,
                                                             log2nb);
  return blocks;
}

void launch_extremes_final(const QuadCand* partials, int nparts, QuadInfo* out,
                           QuadCand* raw_out, cudaStream_t st) {
  k_extremes_final<<<1, 1024, 0, st>>>(partials, nparts, out, raw_out);
}

// Dynamic shared memory opt-in of the record-writing K2 (its point tile).
cudaError_t configure_k2_kernels() {
  const int smem = (int)(kK2Tile * sizeof(double2));
  cudaError_t e = cudaFuncSetAttribute((const void*)k_classify_compact<false>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute((const void*)k_classify_compact<true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  return e;
}

void launch_classify_compact(const double2* pts, u32 n, const QuadInfo* qinfo,
                             const unsigned char* given_labels, int force_lex, u64* kbuf,
                             u64* vbuf, u64 ncap, u32* counts_out, cudaStream_t st) {
  const u32 tiles = (n + kK2Tile - 1) / kK2Tile;
  if (tiles == 0) return;
  constexpr size_t smem = kK2Tile * sizeof(double2);
  if (given_labels)
    k_classify_compact<true><<<tiles, kK2Threads, smem, st>>>(pts, n, qinfo, given_labels,
                                                              force_lex, kbuf, vbuf, ncap, counts_out);
  else
    k_classify_compact<false><<<tiles, kK2Threads, smem, st>>>(pts, n, qinfo, nullptr, force_lex,
                                                               kbuf, vbuf, ncap, counts_out);
}

void launch_classify_survivors(const double2* pts, u32 n, const QuadInfo* qinfo, u64* seg,
                               u64* segcnt, u64* kbuf, u64* vbuf, u32* counts_out, int log2nb,
                               u32* bcnt, u32* bw, u32 wmask, bool programmatic, cudaStream_t st) {
  constexpr u32 tile = kK2Threads / 32 * kSegPts;  // one segment per warp
  const u32 tiles = (n + tile - 1) / tile;
  if (tiles == 0) return;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(tiles);
  cfg.blockDim = dim3(kK2Threads);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = programmatic ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k_classify_survivors, pts, n, qinfo, seg, segcnt, kbuf, vbuf,
                     counts_out, log2nb, bcnt, bw, wmask);
}

void launch_classify_labels(const double2* pts, u64 n, const QuadInfo* qinfo,
                            unsigned char* labels, unsigned long long* counts, int blocks,
                            cudaStream_t st) {
  k_classify_labels<<<blocks, 256, 0, st>>>(pts, n, qinfo, labels, counts);
}

}  // namespace chgpu

namespace chgpu {

// Stage-tap helpers: raw points <-> sort records for one region codec.
__global__ void k_encode(const double2* __restrict__ pts, u64 n, int region, u64* __restrict__ k,
                         u64* __restrict__ v) {
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
    const double2 p = pts[i];
    encode_point(region, p.x, p.y, k[i], v[i]);
  }
}

__global__ void k_decode(const u64* __restrict__ k, const u64* __restrict__ v, u64 n, int region,
                         double2* __restrict__ out) {
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
    double x, y;
    decode_point(region, k[i], v[i], x, y);
    out[i] = make_double2(x, y);
  }
}

void launch_encode(const double2* pts, u64 n, int region, u64* k, u64* v, cudaStream_t st) {
  if (!n) return;
  const u64 blocks = (n + 255) / 256 < 148 * 16 ? (n + 255) / 256 : 148 * 16;
  k_encode<<<(unsigned)blocks, 256, 0, st>>>(pts, n, region, k, v);
}

void launch_decode(const u64* k, const u64* v, u64 n, int region, double2* out, cudaStream_t st) {
  if (!n) return;
  const u64 blocks = (n + 255) / 256 < 148 * 16 ? (n + 255) / 256 : 148 * 16;
  k_decode<<<(unsigned)blocks, 256, 0, st>>>(k, v, n, region, out);
}

}  // namespace chgpu
