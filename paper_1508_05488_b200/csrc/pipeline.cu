// Orchestration of the hull path behind the C ABI (include/chgpu.h).
//
// Mirrors convex_hull (reference pipeline.cpp:25-106) stage for stage:
//   K1 extremes -> frame -> K2 classify+discard -> [degenerate branch]
//   -> K3 region sort (+ tie runs) -> K4/K5 SPA + chain compaction
//   -> D2H chains -> host assemble + Melkman (finisher.cpp).
// Host syncs happen only where the host must size the next launch: after
// K2 (region counts), after the histogram (which digit passes move data),
// after the tie scan, and after the SPA (how many chain points to copy).

#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <string>
#include <vector>

#include "chgpu.h"
#include "chgpu_internal.cuh"
#include "finisher.h"
#include "kernels.h"

using namespace chgpu;
using chgpu::host::Pt;

namespace {

constexpr int kMaxPartials = 148 * 8 * 16;
constexpr int kPartialBlocks = 148 * 8;
constexpr size_t kH2DChunk = size_t(1) << 21;  // points per staged copy (32 MB)

// Counter slots (u32) cleared once per call.
enum Ctr : int {
  kCtrK2 = 0,
  kCtrPass = 1,       // 8 slots: region sort passes
  kCtrLongPass = 9,   // 8 slots: tie-run passes
  kCtrSpa = 17,
  kCtrUnique = 18,
  kCtrMask = 19,
  kCtrMaskLong = 20,
  kCtrNStarts = 21,
  kCtrNLong = 22,
  kCtrCounts = 24,    // 5 slots: K2 stream counts
  kCtrSlots = 64
};

struct Pinned {
  QuadInfo qi;
  u32 ctr[kCtrSlots];
  unsigned long long kept[4];
  unsigned long long uniq;
  unsigned long long counts5[5];
};

double ms_between(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  return (double)ms;
}

}  // namespace

struct chgpu_ctx {
  int device = 0;
  cudaStream_t st = nullptr, st_copy = nullptr;
  std::string err;
  u32 tag = 0;

  size_t cap = 0;               // points
  double2* d_pts = nullptr;     // cap
  u64* d_kbuf = nullptr;        // 2*cap (K2 streams, then ping-pong B)
  u64* d_vbuf = nullptr;        // 2*cap
  u64* d_ka = nullptr;          // cap (ping-pong A)
  u64* d_va = nullptr;          // cap
  unsigned char* d_flags = nullptr;  // cap
  double2* d_kept = nullptr;    // cap
  u64* d_status = nullptr;      // status words
  size_t status_words = 0;
  u64* d_tie_starts = nullptr;  // cap/2+16
  void* d_long_runs = nullptr;  // cap/2049+16 records

  QuadCand* d_partials = nullptr;
  QuadInfo* d_qinfo = nullptr;
  QuadCand* d_rawquad = nullptr;
  u32* d_ctr = nullptr;
  unsigned long long* d_u64 = nullptr;  // [0..3] kept counts, [4] unique total, [5..9] label counts
  u32* d_hist = nullptr;
  u32* d_digit_excl = nullptr;
  SegDesc* d_segs = nullptr;
  size_t seg_cap = 0;

  Pinned* h = nullptr;
  SegDesc* h_segs = nullptr;
  double2* h_out = nullptr;  // pinned chain / survivor staging
  size_t h_out_cap = 0;

  std::vector<Pt> hull, ring, chains;
  int launches = 0;
  cudaEvent_t ev[12] = {};
  std::vector<cudaEvent_t> ev_copy;
};

namespace {

u32 next_tag(chgpu_ctx* c) {
  c->tag = (c->tag + 1) & 0x3FFFFFFFu;
  if (c->tag == 0) c->tag = 1;
  return c->tag;
}

#define CK(call)                                                          \
  do {                                                                    \
    cudaError_t e_ = (call);                                              \
    if (e_ != cudaSuccess) {                                              \
      ctx->err = std::string(#call) + ": " + cudaGetErrorString(e_);      \
      return CHGPU_CUDA_ERR;                                              \
    }                                                                     \
  } while (0)

int fail(chgpu_ctx* ctx, int code, const char* msg) {
  ctx->err = msg;
  return code;
}

void free_ws(chgpu_ctx* c) {
  cudaFree(c->d_pts);
  cudaFree(c->d_kbuf);
  cudaFree(c->d_vbuf);
  cudaFree(c->d_ka);
  cudaFree(c->d_va);
  cudaFree(c->d_flags);
  cudaFree(c->d_kept);
  cudaFree(c->d_status);
  cudaFree(c->d_tie_starts);
  cudaFree(c->d_long_runs);
  c->d_pts = nullptr;
  c->d_kbuf = c->d_vbuf = c->d_ka = c->d_va = nullptr;
  c->d_flags = nullptr;
  c->d_kept = nullptr;
  c->d_status = nullptr;
  c->d_tie_starts = nullptr;
  c->d_long_runs = nullptr;
  c->cap = 0;
}

int ensure_segs(chgpu_ctx* ctx, size_t nseg) {
  if (nseg <= ctx->seg_cap) return CHGPU_OK;
  size_t want = std::max<size_t>(nseg, 64);
  cudaFree(ctx->d_segs);
  cudaFree(ctx->d_hist);
  cudaFree(ctx->d_digit_excl);
  cudaFreeHost(ctx->h_segs);
  CK(cudaMalloc(&ctx->d_segs, want * sizeof(SegDesc)));
  CK(cudaMalloc(&ctx->d_hist, want * kPasses * kDigits * sizeof(u32)));
  CK(cudaMalloc(&ctx->d_digit_excl, want * kPasses * kDigits * sizeof(u32)));
  CK(cudaMallocHost(&ctx->h_segs, want * sizeof(SegDesc)));
  ctx->seg_cap = want;
  return CHGPU_OK;
}

int ensure_host_out(chgpu_ctx* ctx, size_t pts) {
  if (pts <= ctx->h_out_cap) return CHGPU_OK;
  size_t want = std::max<size_t>(pts, size_t(1) << 16);
  want += want / 4;
  cudaFreeHost(ctx->h_out);
  ctx->h_out = nullptr;
  CK(cudaMallocHost(&ctx->h_out, want * sizeof(double2)));
  ctx->h_out_cap = want;
  return CHGPU_OK;
}

int ensure_cap(chgpu_ctx* ctx, size_t n) {
  if (n <= ctx->cap) return CHGPU_OK;
  free_ws(ctx);
  size_t cap = std::max<size_t>(n, 4096);
  cap = (cap + 4095) & ~size_t(4095);
  CK(cudaMalloc(&ctx->d_pts, cap * sizeof(double2)));
  CK(cudaMalloc(&ctx->d_kbuf, 2 * cap * sizeof(u64)));
  CK(cudaMalloc(&ctx->d_vbuf, 2 * cap * sizeof(u64)));
  CK(cudaMalloc(&ctx->d_ka, cap * sizeof(u64)));
  CK(cudaMalloc(&ctx->d_va, cap * sizeof(u64)));
  CK(cudaMalloc(&ctx->d_flags, cap));
  CK(cudaMalloc(&ctx->d_kept, cap * sizeof(double2)));
  // Status words: K2 needs 4 per 2048-point tile, a sort pass 256 per
  // 4096-record tile (+1 tile per segment), the SPA one per chunk (<= cap).
  ctx->status_words = std::max(cap + 4096, (cap / kSortTile + 4096) * (size_t)kDigits);
  CK(cudaMalloc(&ctx->d_status, ctx->status_words * sizeof(u64)));
  CK(cudaMemset(ctx->d_status, 0, ctx->status_words * sizeof(u64)));
  CK(cudaMalloc(&ctx->d_tie_starts, (cap / 2 + 16) * sizeof(u64)));
  CK(cudaMalloc(&ctx->d_long_runs, (cap / 2049 + 16) * tie_run_record_bytes()));
  ctx->cap = cap;
  return CHGPU_OK;
}

int sync(chgpu_ctx* ctx) {
  CK(cudaStreamSynchronize(ctx->st));
  return CHGPU_OK;
}

// Fills tile_begin for host segment descriptors and returns the tile count.
u32 plan_tiles(SegDesc* segs, int nseg) {
  u32 t = 0;
  for (int s = 0; s < nseg; ++s) {
    segs[s].tile_begin = t;
    t += (u32)((segs[s].len + kSortTile - 1) / kSortTile);
  }
  return t;
}

// Segmented LSD radix sort of (k, v) records.
// First executed pass reads (ksrc, vsrc) at src_off; passes alternate
// between (kA, vA) and (kB, vB) at dst_off. *in_a reports where the result
// landed. from_v selects v as the key (tie runs), k riding along.
int radix_sort(chgpu_ctx* ctx, int nseg, const u64* ksrc, const u64* vsrc, u64* kA, u64* vA,
               u64* kB, u64* vB, int from_v, int ctr_base, int mask_slot, bool* in_a,
               int* passes_run, bool timed = false) {
  const u32 tiles = plan_tiles(ctx->h_segs, nseg);
  *passes_run = 0;
  *in_a = true;
  if (tiles == 0) return CHGPU_OK;
  CK(cudaMemcpyAsync(ctx->d_segs, ctx->h_segs, nseg * sizeof(SegDesc), cudaMemcpyHostToDevice,
                     ctx->st));
  CK(cudaMemsetAsync(ctx->d_hist, 0, (size_t)nseg * kPasses * kDigits * sizeof(u32), ctx->st));
  launch_hist(ksrc, vsrc, ctx->d_segs, nseg, tiles, from_v, 1, ctx->d_hist, ctx->st);
  launch_hist_scan(ctx->d_hist, ctx->d_segs, nseg, ctx->d_digit_excl, ctx->d_ctr + mask_slot,
                   ctx->st);
  ctx->launches += 2;
  if (timed) CK(cudaEventRecord(ctx->ev[3], ctx->st));
  CK(cudaMemcpyAsync(&ctx->h->ctr[mask_slot], ctx->d_ctr + mask_slot, sizeof(u32),
                     cudaMemcpyDeviceToHost, ctx->st));
  if (int e = sync(ctx)) return e;
  const u32 mask = ctx->h->ctr[mask_slot];
  const u64* kin = ksrc;
  const u64* vin = vsrc;
  int use_src = 1, done = 0;
  if (timed) CK(cudaEventRecord(ctx->ev[4], ctx->st));
  for (int p = 0; p < kPasses; ++p) {
    if (!(mask & (1u << p))) continue;
    u64* ko = (done % 2 == 0) ? kA : kB;
    u64* vo = (done % 2 == 0) ? vA : vB;
    launch_onesweep(kin, vin, ko, vo, ctx->d_segs, nseg, tiles, use_src, from_v,
                    ctx->d_digit_excl, p, ctx->d_status, next_tag(ctx), ctx->d_ctr + ctr_base + p,
                    ctx->st);
    kin = ko;
    vin = vo;
    use_src = 0;
    ++done;
    ++ctx->launches;
  }
  if (done == 0) {
    if (!(ksrc == kA && vsrc == vA)) {
      launch_seg_copy(ksrc, vsrc, kA, vA, ctx->d_segs, nseg, tiles, 1, ctx->st);
      ++ctx->launches;
    }
    *in_a = true;
  } else {
    *in_a = (done % 2 == 1);
  }
  *passes_run = done;
  if (timed) CK(cudaEventRecord(ctx->ev[5], ctx->st));
  CK(cudaGetLastError());
  return CHGPU_OK;
}

// Orders every equal-primary run of the sorted region layout by v.
int fix_ties(chgpu_ctx* ctx, int nseg, u64* kF, u64* vF, u64* kS, u64* vS, size_t* nruns) {
  const u32 tiles = plan_tiles(ctx->h_segs, nseg);
  *nruns = 0;
  if (tiles == 0) return CHGPU_OK;
  const u32 cap = (u32)(ctx->cap / 2 + 16);
  CK(cudaMemcpyAsync(ctx->d_segs, ctx->h_segs, nseg * sizeof(SegDesc), cudaMemcpyHostToDevice,
                     ctx->st));
  launch_tie_detect(kF, ctx->d_segs, nseg, tiles, ctx->d_tie_starts, ctx->d_ctr + kCtrNStarts, cap,
                    ctx->st);
  ++ctx->launches;
  CK(cudaMemcpyAsync(&ctx->h->ctr[kCtrNStarts], ctx->d_ctr + kCtrNStarts, sizeof(u32),
                     cudaMemcpyDeviceToHost, ctx->st));
  if (int e = sync(ctx)) return e;
  const u32 nstarts = std::min(ctx->h->ctr[kCtrNStarts], cap);
  *nruns = nstarts;
  if (nstarts == 0) return CHGPU_OK;
  launch_tie_fix(kF, vF, ctx->d_segs, ctx->d_tie_starts, nstarts, ctx->d_long_runs,
                 ctx->d_ctr + kCtrNLong, ctx->st);
  ++ctx->launches;
  CK(cudaMemcpyAsync(&ctx->h->ctr[kCtrNLong], ctx->d_ctr + kCtrNLong, sizeof(u32),
                     cudaMemcpyDeviceToHost, ctx->st));
  if (int e = sync(ctx)) return e;
  const u32 nlong = ctx->h->ctr[kCtrNLong];
  if (nlong == 0) return CHGPU_OK;

  // Long runs: sort each by v with the onesweep engine, in place.
  struct Run {
    u64 start;
    u32 len;
    int region;
  };
  std::vector<Run> runs(nlong);
  CK(cudaMemcpyAsync(runs.data(), ctx->d_long_runs, nlong * sizeof(Run), cudaMemcpyDeviceToHost,
                     ctx->st));
  if (int e = sync(ctx)) return e;
  std::sort(runs.begin(), runs.end(), [](const Run& a, const Run& b) { return a.start < b.start; });
  if (int e = ensure_segs(ctx, nlong)) return e;
  for (u32 i = 0; i < nlong; ++i) {
    ctx->h_segs[i] = SegDesc{runs[i].start, runs[i].start, runs[i].len, 0, runs[i].region, 0};
  }
  bool in_a = true;
  int passes = 0;
  // A = scratch, B = F: an even pass count ends back in F.
  if (int e = radix_sort(ctx, (int)nlong, kF, vF, kS, vS, kF, vF, 1, kCtrLongPass, kCtrMaskLong,
                         &in_a, &passes))
    return e;
  if (passes % 2 == 1) {
    const u32 tiles2 = plan_tiles(ctx->h_segs, (int)nlong);
    launch_seg_copy(kS, vS, kF, vF, ctx->d_segs, (int)nlong, tiles2, 0, ctx->st);
    ++ctx->launches;
  }
  CK(cudaGetLastError());
  return CHGPU_OK;
}

// Core of chgpu_hull / chgpu_hull_device. pts_dev must already hold the
// input unless h_src != nullptr (then the copy is staged here, overlapped
// with K1 on a second stream).
int run_pipeline(chgpu_ctx* ctx, const double* h_src, const double2* pts_dev, size_t n,
                 size_t chunk_count, int fallback, const double** hull_xy, size_t* n_hull,
                 chgpu_stats* stats, chgpu_diag* diag) {
  const auto t_wall0 = std::chrono::steady_clock::now();
  chgpu_stats S{};
  chgpu_diag D{};
  S.n_input = n;
  cudaStream_t st = ctx->st;
  ctx->launches = 0;

  CK(cudaMemsetAsync(ctx->d_ctr, 0, kCtrSlots * sizeof(u32), st));
  CK(cudaMemsetAsync(ctx->d_u64, 0, 16 * sizeof(unsigned long long), st));
  CK(cudaEventRecord(ctx->ev[0], st));

  // ---- K1: extremes (extremes.cpp:28-47), overlapped with the H2D copy.
  int nparts = 0;
  if (h_src) {
    const size_t nchunks = (n + kH2DChunk - 1) / kH2DChunk;
    const int per = std::max(1, std::min(kPartialBlocks, kMaxPartials / (int)nchunks));
    if (ctx->ev_copy.size() < nchunks) {
      size_t old = ctx->ev_copy.size();
      ctx->ev_copy.resize(nchunks);
      for (size_t i = old; i < nchunks; ++i)
        CK(cudaEventCreateWithFlags(&ctx->ev_copy[i], cudaEventDisableTiming));
    }
    CK(cudaEventRecord(ctx->ev[11], st));
    CK(cudaStreamWaitEvent(ctx->st_copy, ctx->ev[11], 0));
    for (size_t c = 0; c < nchunks; ++c) {
      const size_t off = c * kH2DChunk, cnt = std::min(kH2DChunk, n - off);
      CK(cudaMemcpyAsync(ctx->d_pts + off, h_src + 2 * off, cnt * sizeof(double2),
                         cudaMemcpyHostToDevice, ctx->st_copy));
      CK(cudaEventRecord(ctx->ev_copy[c], ctx->st_copy));
      CK(cudaStreamWaitEvent(st, ctx->ev_copy[c], 0));
      const int blocks = (int)std::min<size_t>(per, (cnt + 255) / 256);
      launch_extremes_partial(ctx->d_pts + off, cnt, off, ctx->d_partials + nparts, blocks, st);
      nparts += blocks;
      ++ctx->launches;
    }
    CK(cudaEventRecord(ctx->ev[10], ctx->st_copy));
  } else {
    const int blocks = (int)std::min<size_t>(kPartialBlocks, (n + 255) / 256);
    launch_extremes_partial(pts_dev, n, 0, ctx->d_partials, blocks, st);
    nparts = blocks;
    ++ctx->launches;
  }
  const double2* pts = h_src ? ctx->d_pts : pts_dev;
  launch_extremes_final(ctx->d_partials, nparts, ctx->d_qinfo, nullptr, st);
  CK(cudaEventRecord(ctx->ev[1], st));
  ctx->launches += 2;  // final + K2 below

  // ---- K2: classify + round-1 discard (classify.cpp:9-87).
  launch_classify_compact(pts, (u32)n, ctx->d_qinfo, nullptr, 0, ctx->d_kbuf, ctx->d_vbuf,
                          ctx->cap, ctx->d_status, next_tag(ctx), ctx->d_ctr + kCtrK2,
                          ctx->d_ctr + kCtrCounts, st);
  CK(cudaGetLastError());
  CK(cudaEventRecord(ctx->ev[2], st));
  CK(cudaMemcpyAsync(&ctx->h->qi, ctx->d_qinfo, sizeof(QuadInfo), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&ctx->h->ctr[kCtrCounts], ctx->d_ctr + kCtrCounts, 5 * sizeof(u32),
                     cudaMemcpyDeviceToHost, st));
  if (int e = sync(ctx)) return e;

  const QuadInfo qi = ctx->h->qi;
  u64 m[4];
  for (int s = 0; s < 4; ++s) m[s] = ctx->h->ctr[kCtrCounts + 1 + s];
  const u64 s1 = m[0] + m[1] + m[2] + m[3];
  std::memcpy(D.quad, qi.q, sizeof D.quad);
  D.frame_size = qi.frame_size;
  S.n_after_round1 = s1 + qi.frame_size;  // pipeline.cpp:51

  const Pt* corners = reinterpret_cast<const Pt*>(qi.q);
  double t_sort_ms = 0, t_spa_ms = 0;
  auto t_fin0 = std::chrono::steady_clock::now();

  if (qi.degenerate) {
    // ---- pipeline.cpp:53-71: no quad to scan around.
    D.degenerate_branch = 1;
    D.region_counts[0] = n - s1;
    D.region_counts[1] = s1;  // all survivors travel in stream 1 (LEX codec)
    if (!fallback) return fail(ctx, CHGPU_DEGENERATE, "convex_hull: degenerate extreme quadrilateral");
    S.n_after_spa = S.n_after_round1;
    // GPU lexicographic sort + unique of the survivors (oracle.cpp:16-17).
    if (int e = ensure_segs(ctx, 1)) return e;
    ctx->h_segs[0] = SegDesc{0, 0, (u32)s1, 0, 0, 0};
    bool in_a = true;
    int passes = 0;
    if (int e = radix_sort(ctx, 1, ctx->d_kbuf, ctx->d_vbuf, ctx->d_ka, ctx->d_va, ctx->d_kbuf,
                           ctx->d_vbuf, 0, kCtrPass, kCtrMask, &in_a, &passes))
      return e;
    D.sort_passes = passes;
    u64* kF = in_a ? ctx->d_ka : ctx->d_kbuf;
    u64* vF = in_a ? ctx->d_va : ctx->d_vbuf;
    u64* kS = in_a ? ctx->d_kbuf : ctx->d_ka;
    u64* vS = in_a ? ctx->d_vbuf : ctx->d_va;
    ctx->h_segs[0] = SegDesc{0, 0, (u32)s1, 0, 0, 0};
    if (int e = fix_ties(ctx, 1, kF, vF, kS, vS, &D.tie_runs)) return e;
    ++ctx->launches;
    launch_unique(kF, vF, s1, ctx->d_kept, ctx->d_status, next_tag(ctx), ctx->d_ctr + kCtrUnique,
                  ctx->d_u64 + 4, st);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(&ctx->h->uniq, ctx->d_u64 + 4, sizeof(unsigned long long),
                       cudaMemcpyDeviceToHost, st));
    if (int e = sync(ctx)) return e;
    const size_t nu = (size_t)ctx->h->uniq;
    if (int e = ensure_host_out(ctx, nu + 4)) return e;
    CK(cudaMemcpyAsync(ctx->h_out, ctx->d_kept, nu * sizeof(double2), cudaMemcpyDeviceToHost, st));
    if (int e = sync(ctx)) return e;
    t_fin0 = std::chrono::steady_clock::now();
    const Pt* up = reinterpret_cast<const Pt*>(ctx->h_out);
    ctx->chains.assign(up, up + nu);
    // frame_vertices(quad) joins the survivors (pipeline.cpp:63-64).
    Pt fr[4];
    int nf = 0;
    for (int c = 0; c < 4; ++c) {
      const Pt p = corners[c];
      if (nf == 0 || !(fr[nf - 1].x == p.x && fr[nf - 1].y == p.y)) fr[nf++] = p;
    }
    if (nf > 1 && fr[0].x == fr[nf - 1].x && fr[0].y == fr[nf - 1].y) --nf;
    for (int f = 0; f < nf; ++f) chgpu::host::insert_sorted_unique(ctx->chains, fr[f]);
    chgpu::host::monotone_chain(ctx->chains.data(), ctx->chains.size(), ctx->hull);
  } else {
    for (int s = 0; s < 4; ++s) D.region_counts[s + 1] = m[s];
    D.region_counts[0] = n - s1;
    // ---- K3: region sort (spa.cpp:59-81).
    if (int e = ensure_segs(ctx, 4)) return e;
    const u64 cap = ctx->cap;
    const u64 src_off[4] = {0, cap - m[1], cap, 2 * cap - m[3]};
    u64 dst = 0;
    for (int s = 0; s < 4; ++s) {
      ctx->h_segs[s] = SegDesc{src_off[s], dst, (u32)m[s], 0, s + 1, 0};
      dst += m[s];
    }
    bool in_a = true;
    int passes = 0;
    if (int e = radix_sort(ctx, 4, ctx->d_kbuf, ctx->d_vbuf, ctx->d_ka, ctx->d_va, ctx->d_kbuf,
                           ctx->d_vbuf, 0, kCtrPass, kCtrMask, &in_a, &passes, true))
      return e;
    D.sort_passes = passes;
    const bool sort_timed = plan_tiles(ctx->h_segs, 4) > 0;
    u64* kF = in_a ? ctx->d_ka : ctx->d_kbuf;
    u64* vF = in_a ? ctx->d_va : ctx->d_vbuf;
    u64* kS = in_a ? ctx->d_kbuf : ctx->d_ka;
    u64* vS = in_a ? ctx->d_vbuf : ctx->d_va;
    dst = 0;
    for (int s = 0; s < 4; ++s) {
      ctx->h_segs[s] = SegDesc{dst, dst, (u32)m[s], 0, s + 1, 0};
      dst += m[s];
    }
    if (int e = fix_ties(ctx, 4, kF, vF, kS, vS, &D.tie_runs)) return e;
    CK(cudaEventRecord(ctx->ev[6], st));

    // ---- K4/K5: SPA (spa.cpp:109-163). chunk_count == 0 raises here, on
    // the non-degenerate branch only, exactly like the reference.
    if (chunk_count == 0) return fail(ctx, CHGPU_INVALID_ARG, "spa_filter: chunk_count must be >= 1");
    SpaPlan plan{};
    u32 chunks = 0;
    u64 off = 0;
    for (int r = 0; r < 4; ++r) {
      plan.off[r] = off;
      plan.m[r] = m[r];
      plan.chunk_begin[r] = chunks;
      if (m[r]) {
        const u64 cs = (m[r] + chunk_count - 1) / chunk_count;
        plan.chunk_size[r] = cs;
        chunks += (u32)((m[r] + cs - 1) / cs);
      } else {
        plan.chunk_size[r] = 1;
      }
      off += m[r];
      // guarded(region, anchors.first): LL left.y, LR bottom.x, UR right.y, UL top.x
      plan.seed[r] = (r == 0 || r == 2) ? qi.q[2 * r + 1] : qi.q[2 * r];
    }
    plan.total_chunks = chunks;
    launch_spa(kF, vF, plan, ctx->d_flags, ctx->d_kept, ctx->d_u64, ctx->d_status, next_tag(ctx),
               ctx->d_ctr + kCtrSpa, st);
    if (plan.total_chunks) ++ctx->launches;
    CK(cudaGetLastError());
    CK(cudaEventRecord(ctx->ev[8], st));
    CK(cudaMemcpyAsync(ctx->h->kept, ctx->d_u64, 4 * sizeof(unsigned long long),
                       cudaMemcpyDeviceToHost, st));
    if (int e = sync(ctx)) return e;
    size_t kept_counts[4], kept = 0;
    for (int r = 0; r < 4; ++r) {
      kept_counts[r] = (size_t)ctx->h->kept[r];
      D.kept_counts[r] = kept_counts[r];
      kept += kept_counts[r];
    }
    S.n_after_spa = kept + qi.frame_size;  // pipeline.cpp:96
    t_sort_ms = ms_between(ctx->ev[2], ctx->ev[6]);
    t_spa_ms = ms_between(ctx->ev[6], ctx->ev[8]);
    D.t_spa_kernel_ms = t_spa_ms;
    if (sort_timed) {
      D.t_hist_ms = ms_between(ctx->ev[2], ctx->ev[3]);
      D.t_passes_ms = ms_between(ctx->ev[4], ctx->ev[5]);
      D.t_ties_ms = ms_between(ctx->ev[5], ctx->ev[6]);
    }

    // ---- D2H of the chains, then polygon.cpp + melkman.cpp on the host.
    t_fin0 = std::chrono::steady_clock::now();
    if (int e = ensure_host_out(ctx, kept + 4)) return e;
    CK(cudaMemcpyAsync(ctx->h_out, ctx->d_kept, kept * sizeof(double2), cudaMemcpyDeviceToHost,
                       st));
    CK(cudaEventRecord(ctx->ev[9], st));
    if (int e = sync(ctx)) return e;
    D.t_d2h_ms = ms_between(ctx->ev[8], ctx->ev[9]);
    const auto t_host0 = std::chrono::steady_clock::now();
    const int a = chgpu::host::assemble_ring(reinterpret_cast<const Pt*>(ctx->h_out), kept_counts,
                                             corners, ctx->ring);
    if (a) return fail(ctx, CHGPU_DEGENERATE, "assemble_polygon: fewer than 3 distinct vertices");
    const int mk = chgpu::host::melkman(ctx->ring.data(), ctx->ring.size(), ctx->hull);
    if (mk) return fail(ctx, CHGPU_DEGENERATE, "melkman: degenerate polygon");
    D.t_host_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_host0).count();
  }
  const auto t_end = std::chrono::steady_clock::now();

  S.n_hull = ctx->hull.size();
  S.t_extremes_ms = ms_between(ctx->ev[0], ctx->ev[1]);
  S.t_classify_ms = ms_between(ctx->ev[1], ctx->ev[2]);
  S.t_partition_ms = 0.0;
  S.t_sort_ms = t_sort_ms;
  S.t_spa_ms = t_spa_ms;
  S.t_melkman_ms = std::chrono::duration<double, std::milli>(t_end - t_fin0).count();
  S.t_total_ms = std::chrono::duration<double, std::milli>(t_end - t_wall0).count();
  D.t_k1_ms = S.t_extremes_ms;
  D.t_k2_ms = S.t_classify_ms;
  if (h_src) D.t_h2d_ms = ms_between(ctx->ev[0], ctx->ev[10]);
  D.launches = ctx->launches;

  *hull_xy = reinterpret_cast<const double*>(ctx->hull.data());
  *n_hull = ctx->hull.size();
  if (stats) *stats = S;
  if (diag) *diag = D;
  return CHGPU_OK;
}

}  // namespace

// ====================================================================== C ABI

extern "C" {

int chgpu_ctx_create(int device, chgpu_ctx** out) {
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return CHGPU_NO_DEVICE;
  chgpu_ctx* ctx = new chgpu_ctx();
  if (device < 0) cudaGetDevice(&device);
  ctx->device = device;
  if (cudaSetDevice(device) != cudaSuccess) {
    delete ctx;
    return CHGPU_NO_DEVICE;
  }
  auto bad = [&](cudaError_t e) {
    ctx->err = cudaGetErrorString(e);
    return e != cudaSuccess;
  };
  if (bad(cudaStreamCreateWithFlags(&ctx->st, cudaStreamNonBlocking)) ||
      bad(cudaStreamCreateWithFlags(&ctx->st_copy, cudaStreamNonBlocking)) ||
      bad(cudaMalloc(&ctx->d_partials, kMaxPartials * sizeof(QuadCand))) ||
      bad(cudaMalloc(&ctx->d_qinfo, sizeof(QuadInfo))) ||
      bad(cudaMalloc(&ctx->d_rawquad, sizeof(QuadCand))) ||
      bad(cudaMalloc(&ctx->d_ctr, kCtrSlots * sizeof(u32))) ||
      bad(cudaMalloc(&ctx->d_u64, 16 * sizeof(unsigned long long))) ||
      bad(cudaMallocHost(&ctx->h, sizeof(Pinned)))) {
    chgpu_ctx_destroy(ctx);
    return CHGPU_CUDA_ERR;
  }
  for (auto& e : ctx->ev) cudaEventCreate(&e);
  if (ensure_segs(ctx, 64) != CHGPU_OK) {
    chgpu_ctx_destroy(ctx);
    return CHGPU_CUDA_ERR;
  }
  *out = ctx;
  return CHGPU_OK;
}

void chgpu_ctx_destroy(chgpu_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->st) cudaStreamSynchronize(ctx->st);
  free_ws(ctx);
  cudaFree(ctx->d_partials);
  cudaFree(ctx->d_qinfo);
  cudaFree(ctx->d_rawquad);
  cudaFree(ctx->d_ctr);
  cudaFree(ctx->d_u64);
  cudaFree(ctx->d_segs);
  cudaFree(ctx->d_hist);
  cudaFree(ctx->d_digit_excl);
  cudaFreeHost(ctx->h);
  cudaFreeHost(ctx->h_segs);
  cudaFreeHost(ctx->h_out);
  for (auto& e : ctx->ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : ctx->ev_copy) cudaEventDestroy(e);
  if (ctx->st) cudaStreamDestroy(ctx->st);
  if (ctx->st_copy) cudaStreamDestroy(ctx->st_copy);
  delete ctx;
}

const char* chgpu_last_error(const chgpu_ctx* ctx) { return ctx ? ctx->err.c_str() : "no context"; }

void* chgpu_ctx_stream(chgpu_ctx* ctx) { return ctx ? (void*)ctx->st : nullptr; }

int chgpu_reserve(chgpu_ctx* ctx, size_t n) {
  cudaSetDevice(ctx->device);
  return ensure_cap(ctx, n);
}

int chgpu_hull(chgpu_ctx* ctx, const double* xy, size_t n, size_t chunk_count,
               int degenerate_fallback, const double** hull_xy, size_t* n_hull, chgpu_stats* stats,
               chgpu_diag* diag) {
  *n_hull = 0;
  if (n == 0) return fail(ctx, CHGPU_EMPTY, "convex_hull: no points");
  if (n >= (size_t(1) << 32)) return fail(ctx, CHGPU_TOO_LARGE, "more than 2^32-1 points per call");
  cudaSetDevice(ctx->device);
  if (int e = ensure_cap(ctx, n)) return e;
  return run_pipeline(ctx, xy, nullptr, n, chunk_count, degenerate_fallback, hull_xy, n_hull, stats,
                      diag);
}

int chgpu_hull_device(chgpu_ctx* ctx, const double* d_xy, size_t n, size_t chunk_count,
                      int degenerate_fallback, const double** hull_xy, size_t* n_hull,
                      chgpu_stats* stats, chgpu_diag* diag) {
  *n_hull = 0;
  if (n == 0) return fail(ctx, CHGPU_EMPTY, "convex_hull: no points");
  if (n >= (size_t(1) << 32)) return fail(ctx, CHGPU_TOO_LARGE, "more than 2^32-1 points per call");
  if (reinterpret_cast<uintptr_t>(d_xy) % 16 != 0)
    return fail(ctx, CHGPU_INVALID_ARG, "device input must be 16-byte aligned");
  cudaSetDevice(ctx->device);
  if (int e = ensure_cap(ctx, n)) return e;
  return run_pipeline(ctx, nullptr, reinterpret_cast<const double2*>(d_xy), n, chunk_count,
                      degenerate_fallback, hull_xy, n_hull, stats, diag);
}

// ---------------------------------------------------------------- stage taps

static int upload_points(chgpu_ctx* ctx, const double* xy, size_t n) {
  if (int e = ensure_cap(ctx, n)) return e;
  CK(cudaMemcpyAsync(ctx->d_pts, xy, n * sizeof(double2), cudaMemcpyHostToDevice, ctx->st));
  return CHGPU_OK;
}

static int upload_quad(chgpu_ctx* ctx, const double* quad) {
  QuadInfo qi{};
  std::memcpy(qi.q, quad, sizeof qi.q);
  Pt fr[4];
  int nf = 0;
  for (int c = 0; c < 4; ++c) {
    const Pt p{quad[2 * c], quad[2 * c + 1]};
    if (nf == 0 || !(fr[nf - 1].x == p.x && fr[nf - 1].y == p.y)) fr[nf++] = p;
  }
  if (nf > 1 && fr[0].x == fr[nf - 1].x && fr[0].y == fr[nf - 1].y) --nf;
  qi.frame_size = (u32)nf;
  qi.degenerate = nf <= 2;
  ctx->h->qi = qi;
  CK(cudaMemcpyAsync(ctx->d_qinfo, &ctx->h->qi, sizeof(QuadInfo), cudaMemcpyHostToDevice, ctx->st));
  return CHGPU_OK;
}

int chgpu_find_extremes(chgpu_ctx* ctx, const double* xy, size_t n, double* quad_out) {
  if (n == 0) return fail(ctx, CHGPU_EMPTY, "find_extremes: no points");
  if (n >= (size_t(1) << 32)) return fail(ctx, CHGPU_TOO_LARGE, "too many points");
  cudaSetDevice(ctx->device);
  if (int e = upload_points(ctx, xy, n)) return e;
  const int blocks = (int)std::min<size_t>(kPartialBlocks, (n + 255) / 256);
  launch_extremes_partial(ctx->d_pts, n, 0, ctx->d_partials, blocks, ctx->st);
  launch_extremes_final(ctx->d_partials, blocks, ctx->d_qinfo, nullptr, ctx->st);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(&ctx->h->qi, ctx->d_qinfo, sizeof(QuadInfo), cudaMemcpyDeviceToHost, ctx->st));
  if (int e = sync(ctx)) return e;
  std::memcpy(quad_out, ctx->h->qi.q, 8 * sizeof(double));
  return CHGPU_OK;
}

int chgpu_classify(chgpu_ctx* ctx, const double* xy, size_t n, const double* quad, uint8_t* labels,
                   size_t* counts) {
  for (int r = 0; r < 5; ++r) counts[r] = 0;
  if (n == 0) return CHGPU_OK;
  cudaSetDevice(ctx->device);
  if (int e = upload_points(ctx, xy, n)) return e;
  if (int e = upload_quad(ctx, quad)) return e;
  CK(cudaMemsetAsync(ctx->d_u64 + 5, 0, 5 * sizeof(unsigned long long), ctx->st));
  const int blocks = (int)std::min<size_t>(148 * 8, (n + 255) / 256);
  launch_classify_labels(ctx->d_pts, n, ctx->d_qinfo, ctx->d_flags, ctx->d_u64 + 5, blocks, ctx->st);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(labels, ctx->d_flags, n, cudaMemcpyDeviceToHost, ctx->st));
  CK(cudaMemcpyAsync(ctx->h->counts5, ctx->d_u64 + 5, 5 * sizeof(unsigned long long),
                     cudaMemcpyDeviceToHost, ctx->st));
  if (int e = sync(ctx)) return e;
  for (int r = 0; r < 5; ++r) counts[r] = (size_t)ctx->h->counts5[r];
  return CHGPU_OK;
}

int chgpu_discard_round1(chgpu_ctx* ctx, const double* xy, const uint8_t* labels, size_t n,
                         double* out_xy, uint8_t* out_labels, size_t* counts) {
  for (int r = 0; r < 5; ++r) counts[r] = 0;
  if (n == 0) return CHGPU_OK;
  if (n >= (size_t(1) << 32)) return fail(ctx, CHGPU_TOO_LARGE, "too many points");
  cudaSetDevice(ctx->device);
  if (int e = upload_points(ctx, xy, n)) return e;
  CK(cudaMemcpyAsync(ctx->d_flags, labels, n, cudaMemcpyHostToDevice, ctx->st));
  CK(cudaMemsetAsync(ctx->d_ctr, 0, kCtrSlots * sizeof(u32), ctx->st));
  launch_classify_compact(ctx->d_pts, (u32)n, ctx->d_qinfo, ctx->d_flags, 0, ctx->d_kbuf,
                          ctx->d_vbuf, ctx->cap, ctx->d_status, next_tag(ctx),
                          ctx->d_ctr + kCtrK2, ctx->d_ctr + kCtrCounts, ctx->st);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(&ctx->h->ctr[kCtrCounts], ctx->d_ctr + kCtrCounts, 5 * sizeof(u32),
                     cudaMemcpyDeviceToHost, ctx->st));
  if (int e = sync(ctx)) return e;
  const u64 cap = ctx->cap;
  u64 m[4], s1 = 0;
  for (int s = 0; s < 4; ++s) {
    m[s] = ctx->h->ctr[kCtrCounts + 1 + s];
    s1 += m[s];
  }
  // Decode each stream on the device into contiguous block order.
  const u64 src_off[4] = {0, cap - m[1], cap, 2 * cap - m[3]};
  u64 dst = 0;
  for (int s = 0; s < 4; ++s) {
    launch_decode(ctx->d_kbuf + src_off[s], ctx->d_vbuf + src_off[s], m[s], s + 1,
                  ctx->d_kept + dst, ctx->st);
    dst += m[s];
  }
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out_xy, ctx->d_kept, s1 * sizeof(double2), cudaMemcpyDeviceToHost, ctx->st));
  if (int e = sync(ctx)) return e;
  dst = 0;
  for (int s = 0; s < 4; ++s) {
    std::memset(out_labels + dst, s + 1, m[s]);
    counts[s + 1] = m[s];
    dst += m[s];
  }
  counts[0] = 0;
  return CHGPU_OK;
}

int chgpu_sort_region(chgpu_ctx* ctx, int region, double* xy, size_t m) {
  if (region < 1 || region > 4)
    return fail(ctx, CHGPU_INVALID_ARG, "sort_region: interior segments are never sorted");
  if (m <= 1) return CHGPU_OK;
  if (m >= (size_t(1) << 32)) return fail(ctx, CHGPU_TOO_LARGE, "too many points");
  cudaSetDevice(ctx->device);
  if (int e = upload_points(ctx, xy, m)) return e;
  CK(cudaMemsetAsync(ctx->d_ctr, 0, kCtrSlots * sizeof(u32), ctx->st));
  launch_encode(ctx->d_pts, m, region, ctx->d_kbuf, ctx->d_vbuf, ctx->st);
  if (int e = ensure_segs(ctx, 1)) return e;
  ctx->h_segs[0] = SegDesc{0, 0, (u32)m, 0, region, 0};
  bool in_a = true;
  int passes = 0;
  if (int e = radix_sort(ctx, 1, ctx->d_kbuf, ctx->d_vbuf, ctx->d_ka, ctx->d_va, ctx->d_kbuf,
                         ctx->d_vbuf, 0, kCtrPass, kCtrMask, &in_a, &passes))
    return e;
  u64* kF = in_a ? ctx->d_ka : ctx->d_kbuf;
  u64* vF = in_a ? ctx->d_va : ctx->d_vbuf;
  u64* kS = in_a ? ctx->d_kbuf : ctx->d_ka;
  u64* vS = in_a ? ctx->d_vbuf : ctx->d_va;
  ctx->h_segs[0] = SegDesc{0, 0, (u32)m, 0, region, 0};
  size_t runs = 0;
  if (int e = fix_ties(ctx, 1, kF, vF, kS, vS, &runs)) return e;
  launch_decode(kF, vF, m, region, ctx->d_kept, ctx->st);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(xy, ctx->d_kept, m * sizeof(double2), cudaMemcpyDeviceToHost, ctx->st));
  return sync(ctx);
}

int chgpu_spa_filter(chgpu_ctx* ctx, int region, const double* xy, size_t m, const double* anchors,
                     size_t chunk_count, double* out, size_t* n_out) {
  *n_out = 0;
  if (chunk_count == 0) return fail(ctx, CHGPU_INVALID_ARG, "spa_filter: chunk_count must be >= 1");
  if (m == 0) return CHGPU_OK;
  if (region < 1 || region > 4) {
    // spa.cpp:92-105: an Interior "region" never steps back; all kept.
    std::memcpy(out, xy, m * sizeof(double2));
    *n_out = m;
    return CHGPU_OK;
  }
  if (m >= (size_t(1) << 32)) return fail(ctx, CHGPU_TOO_LARGE, "too many points");
  cudaSetDevice(ctx->device);
  if (int e = upload_points(ctx, xy, m)) return e;
  CK(cudaMemsetAsync(ctx->d_ctr, 0, kCtrSlots * sizeof(u32), ctx->st));
  CK(cudaMemsetAsync(ctx->d_u64, 0, 4 * sizeof(unsigned long long), ctx->st));
  launch_encode(ctx->d_pts, m, region, ctx->d_ka, ctx->d_va, ctx->st);
  SpaPlan plan{};
  const int r = region - 1;
  const u64 cs = (m + chunk_count - 1) / chunk_count;
  for (int q = 0; q < 4; ++q) {
    plan.off[q] = 0;
    plan.m[q] = q == r ? m : 0;
    plan.chunk_size[q] = q == r ? cs : 1;
    plan.chunk_begin[q] = q <= r ? 0 : (u32)((m + cs - 1) / cs);
  }
  plan.total_chunks = (u32)((m + cs - 1) / cs);
  plan.seed[r] = (region == 1 || region == 3) ? anchors[1] : anchors[0];
  launch_spa(ctx->d_ka, ctx->d_va, plan, ctx->d_flags, ctx->d_kept, ctx->d_u64, ctx->d_status,
             next_tag(ctx), ctx->d_ctr + kCtrSpa, ctx->st);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(ctx->h->kept, ctx->d_u64, 4 * sizeof(unsigned long long),
                     cudaMemcpyDeviceToHost, ctx->st));
  if (int e = sync(ctx)) return e;
  const size_t k = (size_t)ctx->h->kept[r];
  CK(cudaMemcpyAsync(out, ctx->d_kept, k * sizeof(double2), cudaMemcpyDeviceToHost, ctx->st));
  if (int e = sync(ctx)) return e;
  *n_out = k;
  return CHGPU_OK;
}

// ---------------------------------------------------------------- sharded path

int chgpu_shard_extremes(chgpu_ctx* ctx, const double* d_xy, size_t n, uint64_t base_index,
                         double* quad_out, uint64_t* idx_out) {
  if (n == 0) return fail(ctx, CHGPU_EMPTY, "find_extremes: no points");
  cudaSetDevice(ctx->device);
  const int blocks = (int)std::min<size_t>(kPartialBlocks, (n + 255) / 256);
  launch_extremes_partial(reinterpret_cast<const double2*>(d_xy), n, base_index, ctx->d_partials,
                          blocks, ctx->st);
  launch_extremes_final(ctx->d_partials, blocks, nullptr, ctx->d_rawquad, ctx->st);
  CK(cudaGetLastError());
  QuadCand qc;
  CK(cudaMemcpyAsync(&qc, ctx->d_rawquad, sizeof qc, cudaMemcpyDeviceToHost, ctx->st));
  if (int e = sync(ctx)) return e;
  for (int c = 0; c < 4; ++c) {
    quad_out[2 * c] = qc.c[c].x;
    quad_out[2 * c + 1] = qc.c[c].y;
    idx_out[c] = qc.c[c].i;
  }
  return CHGPU_OK;
}

void chgpu_fold_extremes(const double* quads, const uint64_t* idxs, size_t k, double* quad_out) {
  // extremes.cpp:39-46 with an explicit global-index tie-break.
  struct C {
    double x, y;
    uint64_t i;
  } best[4];
  auto lxy = [](const C& a, const C& b) { return a.x < b.x || (a.x == b.x && a.y < b.y); };
  auto lyx = [](const C& a, const C& b) { return a.y < b.y || (a.y == b.y && a.x < b.x); };
  for (size_t r = 0; r < k; ++r) {
    for (int c = 0; c < 4; ++c) {
      const C cand{quads[8 * r + 2 * c], quads[8 * r + 2 * c + 1], idxs[4 * r + c]};
      if (r == 0) {
        best[c] = cand;
        continue;
      }
      bool take;
      switch (c) {
        case 0: take = lxy(cand, best[c]) || (!lxy(best[c], cand) && cand.i < best[c].i); break;
        case 1: take = lyx(cand, best[c]) || (!lyx(best[c], cand) && cand.i < best[c].i); break;
        case 2: take = lxy(best[c], cand) || (!lxy(cand, best[c]) && cand.i < best[c].i); break;
        default: take = lyx(best[c], cand) || (!lyx(cand, best[c]) && cand.i < best[c].i); break;
      }
      if (take) best[c] = cand;
    }
  }
  for (int c = 0; c < 4; ++c) {
    quad_out[2 * c] = best[c].x;
    quad_out[2 * c + 1] = best[c].y;
  }
}

int chgpu_shard_chains(chgpu_ctx* ctx, const double* d_xy, size_t n, const double* quad,
                       size_t chunk_count, const double** chains_xy, size_t* kept_counts) {
  for (int r = 0; r < 4; ++r) kept_counts[r] = 0;
  *chains_xy = nullptr;
  if (n == 0) return CHGPU_OK;
  if (n >= (size_t(1) << 32)) return fail(ctx, CHGPU_TOO_LARGE, "shard too large");
  cudaSetDevice(ctx->device);
  if (int e = ensure_cap(ctx, n)) return e;
  cudaStream_t st = ctx->st;
  CK(cudaMemsetAsync(ctx->d_ctr, 0, kCtrSlots * sizeof(u32), st));
  CK(cudaMemsetAsync(ctx->d_u64, 0, 16 * sizeof(unsigned long long), st));
  if (int e = upload_quad(ctx, quad)) return e;
  const bool degenerate = ctx->h->qi.degenerate != 0;
  launch_classify_compact(reinterpret_cast<const double2*>(d_xy), (u32)n, ctx->d_qinfo, nullptr,
                          degenerate ? 1 : 0, ctx->d_kbuf, ctx->d_vbuf, ctx->cap, ctx->d_status,
                          next_tag(ctx), ctx->d_ctr + kCtrK2, ctx->d_ctr + kCtrCounts, st);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(&ctx->h->ctr[kCtrCounts], ctx->d_ctr + kCtrCounts, 5 * sizeof(u32),
                     cudaMemcpyDeviceToHost, st));
  if (int e = sync(ctx)) return e;
  u64 m[4], s1 = 0;
  for (int s = 0; s < 4; ++s) {
    m[s] = ctx->h->ctr[kCtrCounts + 1 + s];
    s1 += m[s];
  }
  const u64 cap = ctx->cap;
  if (int e = ensure_segs(ctx, 4)) return e;
  if (degenerate) {
    // Survivors go back sorted and unique; the merge re-runs the
    // degenerate branch on their union.
    ctx->h_segs[0] = SegDesc{0, 0, (u32)s1, 0, 0, 0};
    bool in_a = true;
    int passes = 0;
    if (int e = radix_sort(ctx, 1, ctx->d_kbuf, ctx->d_vbuf, ctx->d_ka, ctx->d_va, ctx->d_kbuf,
                           ctx->d_vbuf, 0, kCtrPass, kCtrMask, &in_a, &passes))
      return e;
    u64* kF = in_a ? ctx->d_ka : ctx->d_kbuf;
    u64* vF = in_a ? ctx->d_va : ctx->d_vbuf;
    u64* kS = in_a ? ctx->d_kbuf : ctx->d_ka;
    u64* vS = in_a ? ctx->d_vbuf : ctx->d_va;
    ctx->h_segs[0] = SegDesc{0, 0, (u32)s1, 0, 0, 0};
    size_t runs = 0;
    if (int e = fix_ties(ctx, 1, kF, vF, kS, vS, &runs)) return e;
    launch_unique(kF, vF, s1, ctx->d_kept, ctx->d_status, next_tag(ctx), ctx->d_ctr + kCtrUnique,
                  ctx->d_u64 + 4, st);
    CK(cudaMemcpyAsync(&ctx->h->uniq, ctx->d_u64 + 4, sizeof(unsigned long long),
                       cudaMemcpyDeviceToHost, st));
    if (int e = sync(ctx)) return e;
    kept_counts[0] = (size_t)ctx->h->uniq;
  } else {
    if (chunk_count == 0) return fail(ctx, CHGPU_INVALID_ARG, "spa_filter: chunk_count must be >= 1");
    const u64 src_off[4] = {0, cap - m[1], cap, 2 * cap - m[3]};
    u64 dst = 0;
    for (int s = 0; s < 4; ++s) {
      ctx->h_segs[s] = SegDesc{src_off[s], dst, (u32)m[s], 0, s + 1, 0};
      dst += m[s];
    }
    bool in_a = true;
    int passes = 0;
    if (int e = radix_sort(ctx, 4, ctx->d_kbuf, ctx->d_vbuf, ctx->d_ka, ctx->d_va, ctx->d_kbuf,
                           ctx->d_vbuf, 0, kCtrPass, kCtrMask, &in_a, &passes))
      return e;
    u64* kF = in_a ? ctx->d_ka : ctx->d_kbuf;
    u64* vF = in_a ? ctx->d_va : ctx->d_vbuf;
    u64* kS = in_a ? ctx->d_kbuf : ctx->d_ka;
    u64* vS = in_a ? ctx->d_vbuf : ctx->d_va;
    dst = 0;
    for (int s = 0; s < 4; ++s) {
      ctx->h_segs[s] = SegDesc{dst, dst, (u32)m[s], 0, s + 1, 0};
      dst += m[s];
    }
    size_t runs = 0;
    if (int e = fix_ties(ctx, 4, kF, vF, kS, vS, &runs)) return e;
    SpaPlan plan{};
    u32 chunks = 0;
    u64 off = 0;
    for (int r = 0; r < 4; ++r) {
      plan.off[r] = off;
      plan.m[r] = m[r];
      plan.chunk_begin[r] = chunks;
      const u64 cs = m[r] ? (m[r] + chunk_count - 1) / chunk_count : 1;
      plan.chunk_size[r] = cs;
      if (m[r]) chunks += (u32)((m[r] + cs - 1) / cs);
      off += m[r];
      plan.seed[r] = (r == 0 || r == 2) ? quad[2 * r + 1] : quad[2 * r];
    }
    plan.total_chunks = chunks;
    launch_spa(kF, vF, plan, ctx->d_flags, ctx->d_kept, ctx->d_u64, ctx->d_status, next_tag(ctx),
               ctx->d_ctr + kCtrSpa, st);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(ctx->h->kept, ctx->d_u64, 4 * sizeof(unsigned long long),
                       cudaMemcpyDeviceToHost, st));
    if (int e = sync(ctx)) return e;
    for (int r = 0; r < 4; ++r) kept_counts[r] = (size_t)ctx->h->kept[r];
  }
  const size_t total = kept_counts[0] + kept_counts[1] + kept_counts[2] + kept_counts[3];
  if (int e = ensure_host_out(ctx, total + 4)) return e;
  CK(cudaMemcpyAsync(ctx->h_out, ctx->d_kept, total * sizeof(double2), cudaMemcpyDeviceToHost, st));
  if (int e = sync(ctx)) return e;
  *chains_xy = reinterpret_cast<const double*>(ctx->h_out);
  return CHGPU_OK;
}

}  // extern "C"
