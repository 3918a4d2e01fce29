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

// ------------------------------------------------------------------ SPA, tile scan
//
// The same filter as one pass over the sorted records, whatever the chunk
// sizes: a CTA takes 4096 consecutive records (16 per thread), and the
// running threshold is a segmented prefix-max over the guarded key w
// (wkey: every region's SPA is a running MAX of w, steps_back <=> w < t),
// reset at every chunk head to the chunk's seed. Across tiles it is carried
// by a decoupled look-back over (any head, max w) pairs; a second look-back
// over the kept counts places the tile's kept points, which are decoded,
// staged in shared memory and written once, coalesced, to their final,
// region-ordered place: no scratch copy and no gather pass.

constexpr int kTileThreads = 256;
#ifndef CHGPU_SPA_TILE_ITEMS
#define CHGPU_SPA_TILE_ITEMS 16
#endif
constexpr int kTileItems = CHGPU_SPA_TILE_ITEMS;
constexpr int kTileRecs = kTileThreads * kTileItems;

struct SpaTileSmem {
  unsigned short kidx[kTileRecs];  // the tile's kept records (tile offsets), in order
  u64 wx[kTileThreads / 32];
  u32 wf[kTileThreads / 32];
  u32 wk[kTileThreads / 32];
  u64 carry_x;
  u64 rend[4], cs[4], wseed[4];  // region ends, chunk sizes, seeds as w
  u32 tile, kept_excl, last;
};

// (F, X) pairs: F = a chunk head was seen, X = max w since the last head.
__device__ __forceinline__ void seg_max(u32& fa, u64& xa, u32 fb, u64 xb) {
  xa = fb ? xb : (xb > xa ? xb : xa);
  fa |= fb;
}

__device__ __forceinline__ u64 ld_cg_u64(const u64* p) { return __ldcg(p); }

#ifndef CHGPU_SPA_TILE_MINB
#define CHGPU_SPA_TILE_MINB 4
#endif
__global__ __launch_bounds__(kTileThreads, CHGPU_SPA_TILE_MINB) void k_spa_tile(
    const u64* __restrict__ k, const u64* __restrict__ v, const SpaPlan plan, u64 total,
    u64* __restrict__ status, u32 tag, u32 ntiles, u64* __restrict__ pay, u32* __restrict__ ticket,
    double2* __restrict__ out, unsigned long long* __restrict__ kept_counts) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SpaTileSmem& S = *reinterpret_cast<SpaTileSmem*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) S.tile = atomicAdd(ticket, 1u);
  if (tid < 4) {
    S.rend[tid] = plan.off[tid] + plan.m[tid];
    S.cs[tid] = plan.chunk_size[tid];
    S.wseed[tid] = wkey(tid + 1, (tid == 0 || tid == 3) ? ~ord_enc(plan.seed[tid])
                                                         : ord_enc(plan.seed[tid]));
  }
  __syncthreads();
  u64* const pay_agg = pay;
  u64* const pay_inc = pay + ntiles;
  // tiles in ticket order: a tile only waits on lower tickets, all taken by
  // CTAs that are already running
  const u32 tile = S.tile;
  const u64 i0 = (u64)tile * kTileRecs + (u64)tid * kTileItems;

  // region (0-based) and chunk position of the thread's first record
  int r = 0;
  while (r < 3 && i0 >= S.rend[r]) ++r;
  u64 cs = S.cs[r], rend = S.rend[r];
  const u64 roff = r ? S.rend[r - 1] : 0;
  const u64 rel = i0 >= roff ? i0 - roff : 0;
  u64 pos = rel % cs;
  bool first_chunk = rel < cs;

  u64 w[kTileItems];
  if (i0 + kTileItems <= total) {
    const ulonglong2* vp = reinterpret_cast<const ulonglong2*>(v + i0);
#pragma unroll
    for (int j = 0; j < kTileItems / 2; ++j) {
      const ulonglong2 t = vp[j];
      w[2 * j] = t.x;
      w[2 * j + 1] = t.y;
    }
  } else {
#pragma unroll
    for (int j = 0; j < kTileItems; ++j) w[j] = i0 + j < total ? v[i0 + j] : 0ull;
  }
  // per record: head bit, first-chunk bit, region (2 bits)
  u32 heads = 0, firsts = 0, regs = 0, F = 0;
  u64 X = 0;
#pragma unroll
  for (int j = 0; j < kTileItems; ++j) {
    const u64 i = i0 + j;
    if (i < total) {
      if (i == rend) {  // next non-empty region
        while (r < 3 && i >= S.rend[r]) ++r;
        cs = S.cs[r];
        rend = S.rend[r];
        pos = 0;
        first_chunk = true;
      } else if (pos == cs) {
        pos = 0;
        first_chunk = false;
      }
      w[j] = wkey(r + 1, w[j]);
      regs |= (u32)r << (2 * j);
      if (pos == 0) {
        heads |= 1u << j;
        if (first_chunk) firsts |= 1u << j;
        const u64 seed = first_chunk ? S.wseed[r] : 0ull;
        X = w[j] > seed ? w[j] : seed;
        F = 1;
      } else {
        X = w[j] > X ? w[j] : X;
      }
      ++pos;
    }
  }
  // block scan of the (F, X) pairs: warp shuffles, then the warp totals
  u32 fi = F;
  u64 xi = X;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const u32 fy = __shfl_up_sync(0xffffffffu, fi, o);
    const u64 xy = __shfl_up_sync(0xffffffffu, xi, o);
    if (lane >= o) {
      u32 f2 = fy;
      u64 x2 = xy;
      seg_max(f2, x2, fi, xi);
      fi = f2;
      xi = x2;
    }
  }
  if (lane == 31) {
    S.wf[warp] = fi;
    S.wx[warp] = xi;
  }
  u32 fe = __shfl_up_sync(0xffffffffu, fi, 1);  // warp-exclusive
  u64 xe = __shfl_up_sync(0xffffffffu, xi, 1);
  if (lane == 0) fe = 0, xe = 0;
  __syncthreads();
  u32 fw = 0, ft = 0;  // block-exclusive for this warp; tile aggregate
  u64 xw = 0, xt = 0;
  for (int q = 0; q < kTileThreads / 32; ++q) {
    if (q == warp) fw = ft, xw = xt;
    seg_max(ft, xt, S.wf[q], S.wx[q]);
  }
  seg_max(fw, xw, fe, xe);  // this thread's block-exclusive prefix

  // look-back 1: the carry into the tile
  if (warp == 0) {
    u64 carry = 0;
    if (tile == 0) {
      if (lane == 0) {
        __stcg(pay_inc, xt);
        fence_acq_rel_gpu();
        store_status(status, make_status(tag, kFlagPrefix, ft));
      }
    } else {
      if (lane == 0) {
        __stcg(pay_agg + tile, xt);
        fence_acq_rel_gpu();
        store_status(status + tile, make_status(tag, kFlagAgg, ft));
      }
      int base = (int)tile - 1;
      while (true) {
        const int j = base - lane;
        u32 flag = kFlagPrefix, fj = 1;
        if (j >= 0) {
          u64 st;
          do {
            st = load_status(status + j);
            flag = status_flag(st, tag);
          } while (flag == kFlagNone);
          fj = (u32)st;
        }
        const unsigned stopm = __ballot_sync(0xffffffffu, flag == kFlagPrefix || fj != 0);
        const int stop = stopm ? __ffs(stopm) - 1 : 31;
        fence_acq_rel_gpu();  // acquire for the payloads of the flags seen
        u64 xj = 0;
        if (j >= 0 && lane <= stop) xj = ld_cg_u64((flag == kFlagPrefix ? pay_inc : pay_agg) + j);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const u64 y = __shfl_xor_sync(0xffffffffu, xj, o);
          xj = y > xj ? y : xj;
        }
        carry = xj > carry ? xj : carry;
        if (stopm) break;
        base -= 32;
      }
      if (lane == 0) {
        u32 fin = 1;
        u64 xin = carry;
        seg_max(fin, xin, ft, xt);
        __stcg(pay_inc + tile, xin);
        fence_acq_rel_gpu();
        store_status(status + tile, make_status(tag, kFlagPrefix, 1));
      }
    }
    if (lane == 0) S.carry_x = carry;
  }
  __syncthreads();
  // the thread's exclusive threshold, then the keep test per record
  u64 t = fw ? xw : (xw > S.carry_x ? xw : S.carry_x);
  u32 kmask = 0;
#pragma unroll
  for (int j = 0; j < kTileItems; ++j) {
    if (i0 + j < total) {
      if (heads & (1u << j)) {
        const int rj = (regs >> (2 * j)) & 3;
        t = (firsts & (1u << j)) ? S.wseed[rj] : 0ull;
      }
      if (w[j] >= t) kmask |= 1u << j;
      t = w[j] > t ? w[j] : t;
    }
  }
  // block-exclusive kept positions
  const u32 nk = __popc(kmask);
  u32 ki = nk;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const u32 y = __shfl_up_sync(0xffffffffu, ki, o);
    if (lane >= o) ki += y;
  }
  if (lane == 31) S.wk[warp] = ki;
  __syncthreads();
  u32 kw = 0, kt = 0;
  for (int q = 0; q < kTileThreads / 32; ++q) {
    if (q == warp) kw = kt;
    kt += S.wk[q];
  }
  const u32 kex = kw + ki - nk;
  // look-back 2: the kept points before the tile
  if (warp == 0) {
    u64* const col = status + ntiles;
    u32 excl = 0;
    if (tile == 0) {
      if (lane == 0) store_status(col, make_status(tag, kFlagPrefix, kt));
    } else {
      if (lane == 0) store_status(col + tile, make_status(tag, kFlagAgg, kt));
      excl = warp_lookback(col, 1, (int)tile, 0, tag);
      if (lane == 0) store_status(col + tile, make_status(tag, kFlagPrefix, excl + kt));
    }
    if (lane == 0) S.kept_excl = excl;
  }
  // the kept records' tile offsets, in order
  {
    u32 o = kex;
#pragma unroll
    for (int j = 0; j < kTileItems; ++j)
      if (kmask & (1u << j)) S.kidx[o++] = (unsigned short)(tid * kTileItems + j);
  }
  __syncthreads();
  const u64 gbase = S.kept_excl;
  // per-region kept counts: + the kept position after the region's last
  // record, - the one before its first (kept_counts starts at zero)
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    if (!plan.m[q]) continue;
    const u64 a = plan.off[q], e = S.rend[q] - 1;
    if (a >= i0 && a < i0 + kTileItems)
      atomicAdd(kept_counts + q,
                0ull - (gbase + kex + __popc(kmask & ((1u << (int)(a - i0)) - 1u))));
    if (e >= i0 && e < i0 + kTileItems)
      atomicAdd(kept_counts + q, gbase + kex + __popc(kmask & ((2u << (int)(e - i0)) - 1u)));
  }
  // decoded and written in order, coalesced: consecutive threads take
  // consecutive kept records (their k and v words re-read: L1/L2 hits)
  // (four records per thread in flight: the loads are the latency here)
  const u64 tbase = (u64)tile * kTileRecs;
  for (u32 i0c = tid; i0c < kt; i0c += 4 * kTileThreads) {
    u64 rec[4], kw[4], vw[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const u32 i = i0c + q * kTileThreads;
      rec[q] = tbase + (i < kt ? S.kidx[i] : 0u);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const bool ok = i0c + q * kTileThreads < kt;
      kw[q] = ok ? k[rec[q]] : 0ull;
      vw[q] = ok ? v[rec[q]] : 0ull;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const u32 i = i0c + q * kTileThreads;
      if (i < kt) {
        int rq = 0;
        while (rq < 3 && rec[q] >= S.rend[rq]) ++rq;
        double px, py;
        decode_point(rq + 1, kw[q], vw[q], px, py);
        out[gbase + i] = make_double2(px, py);
      }
    }
  }
}

void launch_spa_tile(const u64* k, const u64* v, const SpaPlan& plan, u64 total, u64* status,
                     u32 tag, u64* pay, u32* ticket, double2* out,
                     unsigned long long* kept_counts, cudaStream_t st) {
  const u64 tiles = (total + kTileRecs - 1) / kTileRecs;
  if (tiles == 0) return;
  k_spa_tile<<<(unsigned)tiles, kTileThreads, sizeof(SpaTileSmem), st>>>(
      k, v, plan, total, status, tag, (u32)tiles, pay, ticket, out, kept_counts);
}

cudaError_t configure_spa_kernels() {
  return cudaFuncSetAttribute((const void*)k_spa_tile, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)sizeof(SpaTileSmem));
}


}  // namespace chgpu
