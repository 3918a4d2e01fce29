// Orchestration of the hull path behind the C ABI (include/chgpu.h).
//
// Mirrors convex_hull (reference pipeline.cpp:25-106) stage for stage:
//   K1 extremes -> frame -> K2 classify+discard -> [degenerate branch]
//   -> K3 region sort (quantised LSD passes + group fix-up) -> K4/K5 SPA + chain
//   compaction -> D2H chains -> host assemble + Melkman (finisher.cpp).
// Host syncs happen only where the host must size the next launch: after
// K2 (region counts), after the histogram (which digit passes move data),
// after the group scan, and after the SPA (how many chain points to copy).

#include <cuda_runtime.h>

#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>
#include <emmintrin.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
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
constexpr size_t kFileSlots = 4;               // pinned file-ingestion chunks in flight
constexpr int kCtrSlots = 256;                 // u32 counters, cleared once per call

struct Pinned {
  QuadInfo qi;
  u32 ctr[kCtrSlots];
  unsigned long long kept[4];
  unsigned long long uniq;
  unsigned long long counts5[5];
  unsigned long long ncand;
  u32 done;  // k_spa_finish's completion flag (the call's sequence number)
};

// The per-call counters the host reads after K2 and the filter path: the
// quad, K2's region counts (cnt_slot + 1 .. 4), the overflow and
// non-finite flags, the kept counts and the candidate count. ctx->h is
// pinned host memory, mapped into the device address space (UVA).
__global__ void k_readback(const QuadInfo* __restrict__ qinfo, u32* __restrict__ ctr,
                           int cnt_slot, int ovf_slot, int nonfinite_slot,
                           unsigned long long* __restrict__ u64s, Pinned* h) {
  const int t = threadIdx.x;
  const u32* q = reinterpret_cast<const u32*>(qinfo);
  u32* hq = reinterpret_cast<u32*>(&h->qi);
  for (int i = t; i < (int)(sizeof(QuadInfo) / 4); i += blockDim.x) hq[i] = q[i];
  if (t < 5) h->ctr[cnt_slot + t] = ctr[cnt_slot + t];
  if (t == 5 && ovf_slot >= 0) h->ctr[ovf_slot] = ctr[ovf_slot];
  if (t == 6 && nonfinite_slot >= 0) h->ctr[nonfinite_slot] = ctr[nonfinite_slot];
  if (t >= 8 && t < 12) h->kept[t - 8] = u64s[t - 8];
  if (t == 12) h->ncand = u64s[11];
  // ... then clear every counter for what follows (later stages of this
  // call take fresh slots; a call that ends here leaves them clean for the
  // next one, which then skips its clearing memsets)
  __syncthreads();
  for (int i = t; i < kCtrSlots; i += blockDim.x) ctr[i] = 0;
  if (t < 16) u64s[t] = 0;
}

constexpr int kMaxFilterBits = kMaxFilterLog2;
constexpr size_t kConvexMin = size_t(1) << 16;  // ring size from which k_convex.cu is tried  // SPA pre-filter: at most 2^18 bins per region

// The bin tables must be zero when K2 starts. They are cleared right after
// a call's counters come back (the GPU is otherwise idle while the host
// finishes the hull), so the next call usually finds them clean.
int ftab_prepare(chgpu_ctx* ctx, int log2nb, cudaStream_t st);
int ftab_clear_behind(chgpu_ctx* ctx);

// d_ftab: per bin a max w (u64), a record count and a candidate count
// (u32 each), then the candidate-bin bitmap.
size_t filter_tab_bytes(int log2nb) { return (size_t(4) << log2nb) * 16 + (size_t(4) << log2nb) / 8; }

double ms_between(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  return (double)ms;
}

}  // namespace

struct chgpu_ctx {
  int device = 0;
  // chgpu_hull_sharded: this context's shards' chains (device), and on the
  // merging context the union of every shard's chains + the frame
  double2* d_store = nullptr;
  size_t store_cap = 0, store_n = 0;
  double2* d_union = nullptr;
  size_t union_cap = 0;
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
  u64* d_status = nullptr;      // tagged look-back status words, nothing else
  u32* d_raw = nullptr;         // raw per-tile / per-chunk scratch (never tagged)
  size_t raw_words = 0;
  size_t status_words = 0;
  u64* d_starts = nullptr;      // group starts (cap/2+16)
  void* d_medium = nullptr;     // medium groups (cap/2+16)
  void* d_long = nullptr;       // long groups (cap/2049+16)

  QuadCand* d_partials = nullptr;
  QuadInfo* d_qinfo = nullptr;
  QuadCand* d_rawquad = nullptr;
  u32* d_ctr = nullptr;
  int ctr_used = 0;
  unsigned long long* d_u64 = nullptr;  // [0..3] kept counts, [4] unique total, [5..9] label counts
  u32* d_hist = nullptr;
  u32* d_digit_excl = nullptr;
  SegDesc* d_segs = nullptr;
  size_t seg_cap = 0;
  // SPA pre-filter tables (k_filter.cu), nbt = 4 << log2nb bins per call:
  // d_ftab holds [max w: u64 x nbt][count: u32 x nbt][candidates: u32 x nbt],
  // cleared by one memset per call.
  unsigned char* d_ftab = nullptr;
  size_t ftab_zero = 0;   // leading bytes of d_ftab known to be zero
  bool counters_clean = false;  // d_ctr and d_u64 are all zero
  size_t ftab_dirty = 0;  // bytes the current call's K2 may have written
  u32* d_fstart = nullptr;   // per-bin first rank          [4 << kMaxFilterBits]
  u64* d_fthr = nullptr;     // per-bin threshold            [4 << kMaxFilterBits]
  u32* d_fbig = nullptr;     // bins queued for the big sorts [2 * kBigListB]
  unsigned char* d_faux = nullptr;  // FilterAux scratch (bin-tile sums and aggregates)
  u64* d_ck = nullptr;       // kept records per chunk, k words (scratch) [cap]
  u64* d_cv = nullptr;       // ... v words                             [cap]
  u32* d_ffirst = nullptr;   // per-chunk first bin
  u32* d_fdefer = nullptr;   // chunks k_spa_small deferred to k_spa_chunks
  size_t ffirst_cap = 0;
  int spa_mode = 0;          // CHGPU_SPA_AUTO / _SORT / _FILTER
  bool chains_tap = false;   // CHGPU_OPT_CHAINS_TAP
  bool pdl = true;           // CHGPU_OPT_PDL: K2 launched programmatically behind K1
  bool stage_times = false;  // CHGPU_OPT_STAGE_TIMES: per-kernel events (chgpu_diag)
  std::vector<Pt> tap;       // the last call's chains (tap on)
  size_t tap_counts[4] = {0, 0, 0, 0};
  FilterPlan* d_plan = nullptr;  // device-side plan (FilterPlan; .spa alone on the sort path)
  size_t kept_hint = 0;          // chain points of the previous call (speculative D2H size)
  // AUTO mode: the previous call of about this size overflowed the
  // pre-filter (or, sent to the sort by this hint, kept a dense chain set),
  // so this one goes straight to the full region sort instead of running
  // K2 twice. Performance only: both paths give the same hull.
  bool sort_hint = false;
  size_t sort_hint_n = 0;
  u32 call_seq = 0;  // the filter path's completion flag value (Pinned::done)
  // Pinned staging arena for host->device uploads of small host-built
  // tables (segments, plans, quads): every upload gets its own slice, so a
  // host buffer can be rewritten while earlier copies are still queued.
  unsigned char* h_stage = nullptr;
  size_t stage_cap = 0, stage_used = 0;
  // File ingestion (chgpu_hull_xy_binary): pinned ring of kFileSlots chunks.
  double2* h_fslots = nullptr;

  Pinned* h = nullptr;
  SegDesc* h_segs = nullptr;
  double2* h_out = nullptr;  // pinned chain / survivor staging
  size_t h_out_cap = 0;

  std::vector<Pt> hull, ring, chains;
  const Pt* hull_ptr = nullptr;  // the last call's hull (hull.data() or h_out)
  size_t hull_n = 0;
  int launches = 0;
  cudaEvent_t ev[12] = {};
  std::vector<cudaEvent_t> ev_copy;
};

namespace {

// Look-back tags are drawn from one process-wide counter, so no two
// launches (of any context) share a tag until it wraps after 2^30.
u32 next_tag(chgpu_ctx* c) {
  static std::atomic<u32> counter{0};
  u32 t;
  do {
    t = (counter.fetch_add(1, std::memory_order_relaxed) + 1) & 0x3FFFFFFFu;
  } while (t == 0);
  c->tag = t;
  return t;
}

#define CK(call)                                                     \
  do {                                                               \
    cudaError_t e_ = (call);                                         \
    if (e_ != cudaSuccess) {                                         \
      ctx->err = std::string(#call) + ": " + cudaGetErrorString(e_); \
      return CHGPU_CUDA_ERR;                                         \
    }                                                                \
  } while (0)

#define TRY(expr)               \
  do {                          \
    if (int e_ = (expr)) return e_; \
  } while (0)

int fail(chgpu_ctx* ctx, int code, const char* msg) {
  ctx->err = msg;
  return code;
}

// A fresh zeroed device counter for this call.
int ftab_prepare(chgpu_ctx* ctx, int log2nb, cudaStream_t st) {
  const size_t need = filter_tab_bytes(log2nb);
  if (ctx->ftab_zero < need) CK(cudaMemsetAsync(ctx->d_ftab, 0, need, st));
  ctx->ftab_zero = 0;
  ctx->ftab_dirty = need;
  return CHGPU_OK;
}

int ftab_clear_behind(chgpu_ctx* ctx) {
  if (ctx->ftab_dirty) {
    CK(cudaMemsetAsync(ctx->d_ftab, 0, ctx->ftab_dirty, ctx->st));
    ctx->ftab_zero = ctx->ftab_dirty;
    ctx->ftab_dirty = 0;
  }
  return CHGPU_OK;
}

int take_ctr(chgpu_ctx* ctx) {
  if (ctx->ctr_used >= kCtrSlots) return kCtrSlots - 1;  // never reached for sane inputs
  return ctx->ctr_used++;
}

void free_ws(chgpu_ctx* c) {
  cudaFree(c->d_pts);
  cudaFree(c->d_kbuf);
  cudaFree(c->d_vbuf);
  cudaFree(c->d_ka);
  cudaFree(c->d_va);
  cudaFree(c->d_flags);
  cudaFree(c->d_kept);
  cudaFree(c->d_ck);
  cudaFree(c->d_cv);
  cudaFree(c->d_status);
  cudaFree(c->d_raw);
  cudaFree(c->d_starts);
  cudaFree(c->d_medium);
  cudaFree(c->d_long);
  c->d_pts = nullptr;
  c->d_kbuf = c->d_vbuf = c->d_ka = c->d_va = nullptr;
  c->d_flags = nullptr;
  c->d_kept = nullptr;
  c->d_ck = c->d_cv = nullptr;
  c->d_status = nullptr;
  c->d_raw = nullptr;
  c->d_starts = nullptr;
  c->d_medium = c->d_long = nullptr;
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
  CK(cudaMalloc(&ctx->d_pts, (cap + 64) * sizeof(double2)));  // + the convex path's hull
  CK(cudaMalloc(&ctx->d_kbuf, 2 * cap * sizeof(u64)));
  CK(cudaMalloc(&ctx->d_vbuf, 2 * cap * sizeof(u64)));
  CK(cudaMalloc(&ctx->d_ka, cap * sizeof(u64)));
  CK(cudaMalloc(&ctx->d_va, cap * sizeof(u64)));
  CK(cudaMalloc(&ctx->d_flags, cap));
  CK(cudaMalloc(&ctx->d_kept, cap * sizeof(double2)));
  CK(cudaMalloc(&ctx->d_ck, cap * sizeof(u64)));
  CK(cudaMalloc(&ctx->d_cv, cap * sizeof(u64)));
  // Tagged status words only (a raw value there could decode as a live word
  // of a later look-back): one per sort tile, unique tile or SPA chunk.
  ctx->status_words = cap + 4096;
  CK(cudaMalloc(&ctx->d_status, ctx->status_words * sizeof(u64)));
  // Ordered on the context stream: a stale word from recycled memory must
  // never be mistaken for a current one.
  CK(cudaMemsetAsync(ctx->d_status, 0, ctx->status_words * sizeof(u64), ctx->st));
  // Raw scratch: onesweep agg + inc rows (2 x 256 per tile), LSD tile
  // counts, SPA per-chunk counts and offsets (2 per chunk, chunks <= cap).
  ctx->raw_words = std::max((cap / kSortTile + 4096) * 2 * (size_t)kDigits, 2 * cap + 64);
  CK(cudaMalloc(&ctx->d_raw, ctx->raw_words * sizeof(u32)));
  CK(cudaMalloc(&ctx->d_starts, (cap / 2 + 16) * sizeof(u64)));
  CK(cudaMalloc(&ctx->d_medium, (cap / 2 + 16) * group_run_bytes()));
  CK(cudaMalloc(&ctx->d_long, (cap / 2049 + 16) * group_run_bytes()));
  ctx->cap = cap;
  return CHGPU_OK;
}

int sync(chgpu_ctx* ctx) {
  CK(cudaStreamSynchronize(ctx->st));
  return CHGPU_OK;
}

// Whether the filter path's emit writes the chains straight into pinned
// host memory (CHGPU_EMIT_MAPPED=1) instead of a DMA read-back after it.
// Off by default: the saving (~13 µs) depends on the host. On some B200
// hosts the finisher reads PCIe-written lines far slower than DMA-written
// ones (its worker segments 50 -> 95 µs), a net loss of ~30 µs.
bool emit_mapped() {
  static const bool on = [] {
    const char* e = std::getenv("CHGPU_EMIT_MAPPED");
    return e && std::atoi(e) != 0;
  }();
  return on;
}

// The filter path's results are in host memory once k_spa_finish raises
// the call's flag (its last act): the host starts on them without waiting
// for the stream to drain. The stream is polled now and then, so a failed
// launch ends the wait (sync() then reports it).
int wait_filter_flag(chgpu_ctx* ctx) {
  static const bool on = [] {
    const char* e = std::getenv("CHGPU_FLAG_WAIT");  // A/B knob: 0 = stream sync
    return !e || std::atoi(e) != 0;
  }();
  if (!on) return sync(ctx);
  const volatile u32* f = &ctx->h->done;
  for (unsigned i = 1; *f != ctx->call_seq; ++i) {
    if ((i & 255) == 0) {
      const cudaError_t q = cudaStreamQuery(ctx->st);
      if (q != cudaErrorNotReady) {
        if (*f == ctx->call_seq) break;
        return sync(ctx);  // done without the flag (an error, or a path that skips it)
      }
    }
#if defined(__x86_64__) || defined(__i386__)
    __builtin_ia32_pause();
#endif
  }
  std::atomic_thread_fence(std::memory_order_acquire);
  return CHGPU_OK;
}

// Enqueues the upload of `bytes` of host memory `src` to device `dst` on the
// context stream through a fresh slice of the pinned staging arena. The
// source may be modified as soon as this returns (an async copy from pinned
// memory reads it only when the stream reaches the copy).
int upload(chgpu_ctx* ctx, void* dst, const void* src, size_t bytes) {
  size_t off = (ctx->stage_used + 255) & ~size_t(255);
  if (off + bytes > ctx->stage_cap) {
    TRY(sync(ctx));  // queued copies out of the arena are done: reuse it
    off = 0;
    if (bytes > ctx->stage_cap) {
      cudaFreeHost(ctx->h_stage);
      ctx->h_stage = nullptr;
      ctx->stage_cap = 0;
      const size_t want = std::max<size_t>(bytes * 2, size_t(1) << 20);
      CK(cudaMallocHost(&ctx->h_stage, want));
      ctx->stage_cap = want;
    }
  }
  std::memcpy(ctx->h_stage + off, src, bytes);
  ctx->stage_used = off + bytes;
  CK(cudaMemcpyAsync(dst, ctx->h_stage + off, bytes, cudaMemcpyHostToDevice, ctx->st));
  return CHGPU_OK;
}

// Reads one device counter (synchronising the stream).
int read_ctr(chgpu_ctx* ctx, int slot, u32* out) {
  CK(cudaMemcpyAsync(&ctx->h->ctr[slot], ctx->d_ctr + slot, sizeof(u32), cudaMemcpyDeviceToHost,
                     ctx->st));
  TRY(sync(ctx));
  *out = ctx->h->ctr[slot];
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

SegDesc make_seg(u64 src, u64 dst, u64 len, int region) {
  SegDesc s{};
  s.src_off = src;
  s.dst_off = dst;
  s.len = (u32)len;
  s.region = region;
  return s;
}

// Quantizer over the primary range [lo, hi] of a region (chgpu_internal.cuh).
void set_quantizer(SegDesc& s, double lo, double hi, int bits) {
  s.qbits = bits;
  s.qmax = std::ldexp(1.0, bits) - 1.0;
  s.qlo = lo;
  const double span = hi - lo;
  double scale = (span > 0.0) ? s.qmax / span : 0.0;
  if (!std::isfinite(scale)) scale = 0.0;
  s.qscale = scale;
}

// Primary range of each region between its anchors (exact arithmetic puts
// every region survivor inside it; rounding stragglers clamp).
void region_range(const double* q, int region, double* lo, double* hi) {
  switch (region) {
    case 1: *lo = q[0]; *hi = q[2]; break;  // LL: x in [left.x, bottom.x]
    case 2: *lo = q[3]; *hi = q[5]; break;  // LR: y in [bottom.y, right.y]
    case 3: *lo = q[6]; *hi = q[4]; break;  // UR: x in [top.x, right.x]
    case 4: *lo = q[1]; *hi = q[7]; break;  // UL: y in [left.y, top.y]
    default: *lo = q[0]; *hi = q[4]; break; // LEX: x in [left.x, right.x]
  }
}

// LSD passes as reduce-then-scan (default) or onesweep look-back
// (CHGPU_LSD=onesweep).
bool lsd_scan_passes() {
  static const bool b = [] {
    const char* e = std::getenv("CHGPU_LSD");
    return !(e && std::strcmp(e, "onesweep") == 0);
  }();
  return b;
}

// Segmented LSD radix sort of (k, v) records over the segments in
// ctx->h_segs. The first executed pass reads (ksrc, vsrc) at src_off;
// passes alternate between (kA, vA) and (kB, vB) at dst_off. *in_a tells
// where the result landed.
int radix_sort(chgpu_ctx* ctx, int nseg, const u64* ksrc, const u64* vsrc, u64* kA, u64* vA,
               u64* kB, u64* vB, int mode, int npasses, bool* in_a, int* passes_run,
               bool timed = false, bool all_passes = false) {
  const u32 tiles = plan_tiles(ctx->h_segs, nseg);
  *passes_run = 0;
  *in_a = true;
  if (tiles == 0) return CHGPU_OK;
  const int mask_slot = take_ctr(ctx);
  TRY(upload(ctx, ctx->d_segs, ctx->h_segs, nseg * sizeof(SegDesc)));
  // reduce-then-scan passes take their digit bases from the column scan:
  // the global histogram only tells which passes a full-key sort may skip
  const bool scan_passes = lsd_scan_passes() && nseg <= 64;
  if (!(scan_passes && all_passes)) {
    CK(cudaMemsetAsync(ctx->d_hist, 0, (size_t)nseg * kPasses * kDigits * sizeof(u32), ctx->st));
    launch_hist(ksrc, vsrc, ctx->d_segs, nseg, tiles, mode, npasses, 1, ctx->d_hist, ctx->st);
    launch_hist_scan(ctx->d_hist, ctx->d_segs, nseg, npasses, ctx->d_digit_excl,
                     ctx->d_ctr + mask_slot, ctx->st);
    ctx->launches += 2;
  }
  if (timed) CK(cudaEventRecord(ctx->ev[3], ctx->st));
  // Bucket passes always move data; a full-key sort skips digit positions
  // that are constant in every segment (one host round trip).
  u32 mask = (1u << npasses) - 1;
  if (!all_passes) TRY(read_ctr(ctx, mask_slot, &mask));
  const u64* kin = ksrc;
  const u64* vin = vsrc;
  int use_src = 1, done = 0;
  if (timed) CK(cudaEventRecord(ctx->ev[4], ctx->st));
  for (int p = 0; p < npasses; ++p) {
    if (!(mask & (1u << p))) continue;
    u64* ko = (done % 2 == 0) ? kA : kB;
    u64* vo = (done % 2 == 0) ? vA : vB;
    if (scan_passes) {
      // reduce-then-scan: no inter-tile waiting (3 launches per pass)
      launch_lsd_pass(kin, vin, ko, vo, ctx->d_segs, nseg, tiles, use_src, mode,
                      ctx->d_digit_excl, p, ctx->d_raw, ctx->st);
      ctx->launches += 2;
    } else {
      launch_onesweep(kin, vin, ko, vo, ctx->d_segs, nseg, tiles, use_src, mode,
                      ctx->d_digit_excl, p, ctx->d_status, next_tag(ctx),
                      ctx->d_ctr + take_ctr(ctx), ctx->d_raw, ctx->st);
    }
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

struct Run {
  u64 start;
  u32 len;
  int seg;
};

// Groups left for the host to resolve after the in-place fix-up.
struct PendingLong {
  int slot = -1;      // device counter of pending groups
  int eqmode = 0;
  int depth = 0;
  std::vector<int> regions;
  u64 *kF = nullptr, *vF = nullptr, *kS = nullptr, *vS = nullptr;
};

int resolve_long(chgpu_ctx* ctx, const PendingLong& p, bool* had_long);

// Orders every group of the sorted layout (segments in ctx->h_segs, at
// dst_off of (kF, vF)) by (canon k, v), in place. eqmode kEqQ: groups of
// equal quantized primary; kEqPrim: groups of ==-equal primary. Small and
// medium groups are fixed on the device without a host round trip; groups
// longer than a shared-memory sort are recorded in *pend and sorted by
// resolve_long() (immediately unless `defer`).
int fix_groups(chgpu_ctx* ctx, int nseg, u64* kF, u64* vF, u64* kS, u64* vS, int eqmode,
               PendingLong* pend, bool defer, int depth = 0) {
  const u32 tiles = plan_tiles(ctx->h_segs, nseg);
  pend->slot = -1;
  if (tiles == 0) return CHGPU_OK;
  const int s_medium = take_ctr(ctx), s_long = take_ctr(ctx);
  TRY(upload(ctx, ctx->d_segs, ctx->h_segs, nseg * sizeof(SegDesc)));
  launch_group_scan(kF, vF, ctx->d_segs, nseg, tiles, eqmode, ctx->d_medium,
                    ctx->d_ctr + s_medium, ctx->d_u64 + 10, ctx->st);
  launch_group_fix_medium(kF, vF, ctx->d_segs, ctx->d_medium, ctx->d_ctr + s_medium, ctx->d_long,
                          ctx->d_ctr + s_long, ctx->st);
  ctx->launches += 2;
  CK(cudaGetLastError());
  pend->slot = s_long;
  pend->eqmode = eqmode;
  pend->depth = depth;
  pend->regions.resize(nseg);
  for (int s = 0; s < nseg; ++s) pend->regions[s] = ctx->h_segs[s].region;
  pend->kF = kF;
  pend->vF = vF;
  pend->kS = kS;
  pend->vS = vS;
  if (defer) return CHGPU_OK;
  bool had = false;
  return resolve_long(ctx, *pend, &had);
}

// Long groups: a full sort of each group with the onesweep engine (on k
// for quantizer groups, then their ==-primary runs on v; on v for
// ==-primary runs).
int resolve_long(chgpu_ctx* ctx, const PendingLong& p, bool* had_long) {
  *had_long = false;
  if (p.slot < 0) return CHGPU_OK;
  u32 nlong = 0;
  TRY(read_ctr(ctx, p.slot, &nlong));
  if (nlong == 0) return CHGPU_OK;
  *had_long = true;
  std::vector<Run> runs(nlong);
  CK(cudaMemcpyAsync(runs.data(), ctx->d_long, nlong * sizeof(Run), cudaMemcpyDeviceToHost,
                     ctx->st));
  TRY(sync(ctx));
  std::sort(runs.begin(), runs.end(), [](const Run& a, const Run& b) { return a.start < b.start; });
  TRY(ensure_segs(ctx, nlong));
  auto load_segs = [&]() {
    for (u32 i = 0; i < nlong; ++i)
      ctx->h_segs[i] = make_seg(runs[i].start, runs[i].start, runs[i].len, p.regions[runs[i].seg]);
  };
  load_segs();
  bool in_a = true;
  int passes = 0;
  // A = scratch, B = F: an even pass count ends back in F.
  const int mode = (p.eqmode == kEqQ) ? kDigitK : kDigitV;
  TRY(radix_sort(ctx, (int)nlong, p.kF, p.vF, p.kS, p.vS, p.kF, p.vF, mode, kPasses, &in_a,
                 &passes));
  if (passes % 2 == 1) {
    const u32 t2 = plan_tiles(ctx->h_segs, (int)nlong);
    launch_seg_copy(p.kS, p.vS, p.kF, p.vF, ctx->d_segs, (int)nlong, t2, 0, ctx->st);
    ++ctx->launches;
  }
  CK(cudaGetLastError());
  // After a full sort on k, ==-equal primaries still need their v order.
  if (p.eqmode == kEqQ && p.depth == 0) {
    load_segs();
    PendingLong inner;
    TRY(fix_groups(ctx, (int)nlong, p.kF, p.vF, p.kS, p.vS, kEqPrim, &inner, false, 1));
  }
  return CHGPU_OK;
}

// Sorts the nseg segments in ctx->h_segs (src layout in kbuf/vbuf) into
// region order. Bucket phase keyed on the quantized primary when qbits > 0,
// else a full LSD on k; then the in-place group fix-up.
struct Sorted {
  u64 *kF, *vF, *kS, *vS;
  int passes;
  PendingLong pend;  // long groups still to resolve (see fix_groups)
};

// Sorts the nseg segments in ctx->h_segs (src layout in kbuf/vbuf) into
// region order. Bucket phase keyed on the quantized primary when qbits > 0
// (all qbits/8 passes run: no histogram round trip), else a full LSD on k
// with trivial passes skipped; then the in-place group fix-up. With
// defer_long the caller must call resolve_long(out->pend) later.
int sort_segments(chgpu_ctx* ctx, int nseg, int qbits, bool timed, bool defer_long, Sorted* out) {
  std::vector<SegDesc> segs(ctx->h_segs, ctx->h_segs + nseg);
  bool in_a = true;
  int passes = 0;
  const int mode = qbits ? kDigitQ : kDigitK;
  const int npasses = qbits ? qbits / 8 : kPasses;
  TRY(radix_sort(ctx, nseg, ctx->d_kbuf, ctx->d_vbuf, ctx->d_ka, ctx->d_va, ctx->d_kbuf,
                 ctx->d_vbuf, mode, npasses, &in_a, &passes, timed, qbits != 0));
  out->kF = in_a ? ctx->d_ka : ctx->d_kbuf;
  out->vF = in_a ? ctx->d_va : ctx->d_vbuf;
  out->kS = in_a ? ctx->d_kbuf : ctx->d_ka;
  out->vS = in_a ? ctx->d_vbuf : ctx->d_va;
  out->passes = passes;
  for (int s = 0; s < nseg; ++s) {
    ctx->h_segs[s] = segs[s];
    ctx->h_segs[s].src_off = segs[s].dst_off;
  }
  TRY(fix_groups(ctx, nseg, out->kF, out->vF, out->kS, out->vS, qbits ? kEqQ : kEqPrim, &out->pend,
                 defer_long));
  return CHGPU_OK;
}

int plan_regions(chgpu_ctx* ctx, const u64 m[4], const double* quad, int* qbits);

// The four region streams of K2 (two-ended layout), sorted into region
// order LL | LR | UR | UL.
int sort_regions(chgpu_ctx* ctx, const u64 m[4], const double* quad, bool timed, bool defer,
                 Sorted* out) {
  int qbits = 0;
  TRY(plan_regions(ctx, m, quad, &qbits));
  return sort_segments(ctx, 4, qbits, timed, defer, out);
}

// Largest region (log2 records) sorted on a 24-bit quantized primary (3
// passes) instead of 32 bits (4): more equal-q groups for the fix-up.
int q24_log2() {
  static const int v = [] {
    const char* e = std::getenv("CHGPU_Q24_LOG2");  // tuning knob
    return e ? std::max(0, std::min(30, std::atoi(e))) : 22;
  }();
  return v;
}

// Region segments of the K2 two-ended layout, with quantizers.
int plan_regions(chgpu_ctx* ctx, const u64 m[4], const double* quad, int* qbits) {
  TRY(ensure_segs(ctx, 4));
  const u64 cap = ctx->cap;
  const u64 src_off[4] = {0, cap - m[1], cap, 2 * cap - m[3]};
  const u64 mmax = std::max(std::max(m[0], m[1]), std::max(m[2], m[3]));
  *qbits = mmax <= (u64(1) << q24_log2()) ? 24 : 32;
  u64 dst = 0;
  for (int s = 0; s < 4; ++s) {
    ctx->h_segs[s] = make_seg(src_off[s], dst, m[s], s + 1);
    double lo, hi;
    region_range(quad, s + 1, &lo, &hi);
    set_quantizer(ctx->h_segs[s], lo, hi, *qbits);
    dst += m[s];
  }
  return CHGPU_OK;
}

SpaPlan make_spa_plan(const u64 m[4], size_t chunk_count, const double* quad) {
  SpaPlan plan{};
  u32 chunks = 0;
  u64 off = 0;
  for (int r = 0; r < 4; ++r) {
    plan.off[r] = off;
    plan.m[r] = m[r];
    plan.chunk_begin[r] = chunks;
    const u64 cs = m[r] ? (m[r] + chunk_count - 1) / chunk_count : 1;  // spa.cpp:121
    plan.chunk_size[r] = cs;
    if (m[r]) chunks += (u32)((m[r] + cs - 1) / cs);                   // spa.cpp:122
    off += m[r];
    // guarded(region, anchors.first): LL left.y, LR bottom.x, UR right.y, UL top.x
    plan.seed[r] = (r == 0 || r == 2) ? quad[2 * r + 1] : quad[2 * r];
  }
  plan.total_chunks = chunks;
  return plan;
}

// Degenerate-branch survivors: one LEX segment, sorted, unique-compacted
// into d_kept; returns the unique count.
int sorted_unique_survivors(chgpu_ctx* ctx, u64 s1, const double* quad, size_t* nuniq, int* passes,
                            size_t* groups) {
  double lo, hi;
  region_range(quad, 0, &lo, &hi);
  Sorted so{};
  TRY(ensure_segs(ctx, 1));
  ctx->h_segs[0] = make_seg(0, 0, s1, 0);
  const int qbits = s1 <= (u64(1) << 22) ? 24 : 32;
  set_quantizer(ctx->h_segs[0], lo, hi, qbits);
  TRY(sort_segments(ctx, 1, qbits, false, false, &so));
  *passes = so.passes;
  *groups = 0;
  const int slot = take_ctr(ctx);
  launch_unique(so.kF, so.vF, s1, ctx->d_kept, ctx->d_status, next_tag(ctx), ctx->d_ctr + slot,
                ctx->d_u64 + 4, ctx->st);
  if (s1) ++ctx->launches;
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(&ctx->h->uniq, ctx->d_u64 + 4, sizeof(unsigned long long),
                     cudaMemcpyDeviceToHost, ctx->st));
  TRY(sync(ctx));
  *nuniq = (size_t)ctx->h->uniq;
  return CHGPU_OK;
}

// K4/K5 over the sorted regions in (kF, vF): kept chains, decoded, in
// d_kept (region order) and per-region counts in d_u64[0..3]. The input
// copy d_pts is dead by now and serves as the per-chunk scratch.
int run_spa(chgpu_ctx* ctx, const u64* kF, const u64* vF, const SpaPlan& plan) {
  const u64 total = plan.m[0] + plan.m[1] + plan.m[2] + plan.m[3];
  const int ticket = take_ctr(ctx);
  // (the kept counts are accumulated: + region end, - region start)
  CK(cudaMemsetAsync(ctx->d_u64, 0, 4 * sizeof(unsigned long long), ctx->st));
  launch_spa_tile(kF, vF, plan, total, ctx->d_status, next_tag(ctx),
                  reinterpret_cast<u64*>(ctx->d_raw), ctx->d_ctr + ticket, ctx->d_kept,
                  ctx->d_u64, ctx->st);
  if (total) ctx->launches += 1;
  CK(cudaGetLastError());
  return CHGPU_OK;
}

// Bins per region for the SPA pre-filter: about 256 per chunk (so a
// chunk's first bin, whose records are all candidates, is ~1/256 of it),
// at most 2^kMaxFilterBits, and not many more than there are points.
int filter_bits(size_t n, size_t chunk_count) {
  static const int per_chunk_log2 = [] {
    const char* e = std::getenv("CHGPU_FILTER_BINS_PER_CHUNK_LOG2");  // tuning knob
    return e ? std::max(0, std::min(12, std::atoi(e))) : 8;
  }();
  int b = 11;
  while (b < kMaxFilterBits && ((size_t(1) << b) >> per_chunk_log2) < chunk_count) ++b;
  while (b > 11 && (size_t(1) << b) > 2 * n) --b;
  return b;
}

// Records per bin whose w feeds the bin's max (1 in 2^k; tuning knob).
// Any subset gives a valid threshold (the max of a subset is a lower bound).
u32 filter_wmask() {
  static const u32 m = [] {
    const char* e = std::getenv("CHGPU_FILTER_WSAMPLE_LOG2");
    const int k = e ? std::max(0, std::min(8, std::atoi(e))) : 1;
    return (1u << k) - 1u;
  }();
  return m;
}

struct FilterTabs {
  u32* w;  // (in the first half of its 8-byte-per-bin slot range)
  u32* cnt;
  u32* cur;
  u32* bmap;  // one bit per bin: the bin holds a candidate
};
FilterTabs filter_tabs(chgpu_ctx* ctx, int log2nb) {
  const size_t nbt = size_t(4) << log2nb;
  FilterTabs t;
  t.w = reinterpret_cast<u32*>(ctx->d_ftab);
  t.cnt = t.w + 2 * nbt;
  t.cur = t.cnt + nbt;
  t.bmap = t.cur + nbt;
  return t;
}

// Enqueues the pre-filtered SPA (k_filter.cu) right behind K2, with no
// host round trip: the bin scan builds the plan on the device from the bin
// counts (and writes the region sizes to cnt_slot + 1 .. 4), then the
// filter, the big-bin sorts and the per-chunk SPA over the candidates;
// kept chains land in d_kept exactly as run_spa leaves them and the kept
// counts in d_u64[0..3].
// Bounds the host knows (n records, min(4 C, n) chunks) size the grids.
// *ovf_slot / *ncand land in the counters for the caller's read-back.
int enqueue_filter_spa(chgpu_ctx* ctx, const double2* pts, size_t n, size_t chunk_count,
                       int log2nb, int cnt_slot, int* ovf_slot, int nonfinite_slot = -1,
                       size_t host_chains = 0) {
  cudaStream_t st = ctx->st;
  const FilterPlan* P = ctx->d_plan;
  const u32 max_chunks = (u32)(chunk_count > n / 4 ? n : std::min<size_t>(4 * chunk_count, n));
  if ((size_t)max_chunks > ctx->ffirst_cap) {
    cudaFree(ctx->d_ffirst);
    cudaFree(ctx->d_fdefer);
    ctx->d_ffirst = ctx->d_fdefer = nullptr;
    const size_t want = std::max<size_t>((size_t)max_chunks, 8192);
    CK(cudaMalloc(&ctx->d_ffirst, want * sizeof(u32)));
    CK(cudaMalloc(&ctx->d_fdefer, want * sizeof(u32)));
    ctx->ffirst_cap = want;
  }
  u32* first_bin = ctx->d_ffirst;
  FilterAux aux;
  aux.tsum = reinterpret_cast<u32*>(ctx->d_faux);
  aux.agg_seg = aux.tsum + 512;
  aux.agg_val = reinterpret_cast<u64*>(ctx->d_faux + 8192);
  const FilterTabs t = filter_tabs(ctx, log2nb);
  const int nbig_slot = take_ctr(ctx), nbig2_slot = take_ctr(ctx);
  (void)nbig2_slot;  // nbig_slot + 1: the CTA-sort list count
  *ovf_slot = take_ctr(ctx);
  // plan + bin starts + thresholds: one cooperative launch
  // (the coarse threshold table lives in the upper half of d_fthr)
  u32* const tcoarse = reinterpret_cast<u32*>(ctx->d_fthr) + (size_t(4) << kMaxFilterBits);
  CK(launch_bin_scan(ctx->d_qinfo, ctx->d_ctr + cnt_slot + 1, chunk_count, log2nb, t.cnt, t.w,
                     ctx->d_plan, ctx->d_fstart, reinterpret_cast<u32*>(ctx->d_fthr), tcoarse,
                     first_bin, aux, ctx->d_ctr + take_ctr(ctx), ctx->d_ctr + *ovf_slot, st));
  if (ctx->stage_times) CK(cudaEventRecord(ctx->ev[3], st));
  // K2's survivor segments: filter keys in kbuf, input indices in the upper
  // half of vbuf, each segment's survivor count in its lower part
  launch_filter(ctx->d_kbuf, ctx->d_vbuf,
                (u32)((n + kSegPts - 1) / kSegPts), pts, P, ctx->d_qinfo, ctx->d_fstart,
                reinterpret_cast<const u32*>(ctx->d_fthr), tcoarse, log2nb,
                t.cur, t.bmap, ctx->d_ka, ctx->d_va, ctx->d_fbig, ctx->d_ctr + nbig_slot,
                ctx->d_u64 + 11, ctx->d_ctr + *ovf_slot, st);
  CK(cudaEventRecord(ctx->ev[4], st));
  // the chunk SPA over the sparse candidates, kept records via d_ck / d_cv
  // (raw scratch: per-chunk kept counts, then their sums per 256 chunks):
  // k_spa_small per chunk; chunks over its capacity are deferred to the
  // bin sorts + k_spa_chunks (both idle when none was)
  const int ndefer_slot = take_ctr(ctx);
  launch_spa_small(ctx->d_ka, ctx->d_va, t.cur, ctx->d_fstart, t.bmap, first_bin, P, max_chunks,
                   ctx->d_ck, ctx->d_cv, ctx->d_raw, ctx->d_raw + max_chunks, ctx->d_u64,
                   ctx->d_fdefer, ctx->d_ctr + ndefer_slot,
                   ctx->spa_mode == CHGPU_SPA_FILTER_SORTED ? 0u : kSpaSmallCap, st);
  if (ctx->stage_times) CK(cudaEventRecord(ctx->ev[5], st));
  // the finish kernel also hands the call's counters to the host and
  // clears them (what k_readback does on the other paths)
  ReadbackArgs rb;
  rb.qinfo = ctx->d_qinfo;
  rb.ctr = ctx->d_ctr;
  rb.nctr = kCtrSlots;
  rb.cnt_slot = cnt_slot;
  rb.ovf_slot = *ovf_slot;
  rb.nonfinite_slot = nonfinite_slot;
  rb.u64s = ctx->d_u64;
  rb.h_qi = reinterpret_cast<u32*>(&ctx->h->qi);
  rb.h_ctr = ctx->h->ctr;
  rb.h_kept = ctx->h->kept;
  rb.h_ncand = &ctx->h->ncand;
  // the first host_chains kept points also go to the pinned h_out (mapped)
  rb.h_chains = host_chains ? ctx->h_out : nullptr;
  rb.h_chains_cap = (u32)host_chains;
  // (process-wide sequence: pinned memory recycled from a destroyed context
  // may still hold that context's last flag value)
  static std::atomic<u32> g_seq{0};
  u32 seq = g_seq.fetch_add(1, std::memory_order_relaxed) + 1;
  if (seq == 0) seq = g_seq.fetch_add(1, std::memory_order_relaxed) + 1;
  ctx->h->done = 0;
  // (the flag and its system-scope fences only serve the mapped emit)
  rb.h_done = host_chains ? &ctx->h->done : nullptr;
  rb.seq = ctx->call_seq = seq;
  CK(launch_spa_finish(ctx->d_ka, ctx->d_va, t.cur, ctx->d_fstart, t.bmap, first_bin, P, ctx->d_fbig,
                       ctx->d_ctr + nbig_slot, ctx->d_ctr + *ovf_slot, ctx->d_fdefer,
                       ctx->d_ctr + ndefer_slot, ctx->d_ck, ctx->d_cv, ctx->d_raw,
                       ctx->d_raw + max_chunks, ctx->d_u64, ctx->d_kept, ctx->d_ctr + take_ctr(ctx),
                       max_chunks, rb, st));
  if (ctx->stage_times) CK(cudaEventRecord(ctx->ev[6], st));
  ctx->launches += 5;
  CK(cudaGetLastError());
  CK(cudaEventRecord(ctx->ev[8], st));
  return CHGPU_OK;
}

// Melkman's all-vertices-kept trajectory checked on the device
// (k_convex.cu). On success the canonical hull is in h_out (hull_ptr /
// hull_n set, event 9 after its copy) and *convex = true.
int convex_finish(chgpu_ctx* ctx, const size_t kept_counts[4], size_t kept, bool* convex) {
  cudaStream_t st = ctx->st;
  *convex = false;
  const int ok_slot = take_ctr(ctx);
  const u32 one = 1;
  TRY(upload(ctx, ctx->d_ctr + ok_slot, &one, sizeof one));
  const u64 k4[4] = {kept_counts[0], kept_counts[1], kept_counts[2], kept_counts[3]};
  u64* block_best = reinterpret_cast<u64*>(ctx->d_faux + 16384);
  launch_convex_check(ctx->d_kept, k4, ctx->d_qinfo, ctx->d_ctr + ok_slot, block_best, st);
  ++ctx->launches;
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(&ctx->h->ctr[ok_slot], ctx->d_ctr + ok_slot, sizeof(u32),
                     cudaMemcpyDeviceToHost, st));
  TRY(sync(ctx));
  if (!ctx->h->ctr[ok_slot]) return CHGPU_OK;
  const size_t N = kept + 4;
  launch_convex_emit(ctx->d_kept, k4, ctx->d_qinfo, block_best, ctx->d_pts, st);
  ++ctx->launches;
  CK(cudaGetLastError());
  TRY(ensure_host_out(ctx, N + 4));
  CK(cudaMemcpyAsync(ctx->h_out, ctx->d_pts, N * sizeof(double2), cudaMemcpyDeviceToHost, st));
  CK(cudaEventRecord(ctx->ev[9], st));
  TRY(sync(ctx));
  ctx->hull_ptr = reinterpret_cast<const Pt*>(ctx->h_out);
  ctx->hull_n = N;
  *convex = true;
  return CHGPU_OK;
}

void frame_of(const double* quad, Pt* fr, int* nf) {
  *nf = 0;
  for (int c = 0; c < 4; ++c) {
    const Pt p{quad[2 * c], quad[2 * c + 1]};
    if (*nf == 0 || !(fr[*nf - 1].x == p.x && fr[*nf - 1].y == p.y)) fr[(*nf)++] = p;
  }
  if (*nf > 1 && fr[0].x == fr[*nf - 1].x && fr[0].y == fr[*nf - 1].y) --*nf;
}

int begin_call(chgpu_ctx* ctx) {
  TRY(sync(ctx));  // nothing of an earlier call may still read the staging arena
  ctx->stage_used = 0;
  ctx->launches = 0;
  ctx->ctr_used = 0;
  if (!ctx->counters_clean) {  // (k_readback cleared them at the end of the last call)
    CK(cudaMemsetAsync(ctx->d_ctr, 0, kCtrSlots * sizeof(u32), ctx->st));
    CK(cudaMemsetAsync(ctx->d_u64, 0, 16 * sizeof(unsigned long long), ctx->st));
  }
  ctx->counters_clean = false;
  return CHGPU_OK;
}

// Core of chgpu_hull / chgpu_hull_device. h_src != nullptr: the input is on
// the host and is staged in chunks on a copy stream, overlapped with K1.
// memcpy into the pinned staging slot with non-temporal stores: the slot is
// read next by the copy engine, not by this core, so a cached store only
// adds a read-for-ownership of every destination line to the host memory
// traffic. dst is 16-byte aligned (slot offsets are multiples of 4 KB).
void copy_stream(unsigned char* dst, const unsigned char* src, size_t len) {
  static const bool nt = [] {
    const char* e = std::getenv("CHGPU_STAGE_NT");  // A/B knob
    return !e || std::atoi(e) != 0;
  }();
  if (!nt || (reinterpret_cast<uintptr_t>(dst) & 15)) {
    std::memcpy(dst, src, len);
    return;
  }
  size_t i = 0;
  for (; i + 64 <= len; i += 64) {
    const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i));
    const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 16));
    const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 32));
    const __m128i d = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 48));
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i), a);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 16), b);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 32), c);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 48), d);
  }
  _mm_sfence();
  if (i < len) std::memcpy(dst + i, src + i, len - i);
}

// Copies bytes [off, off + len) of the source into dst with up to
// `threads` parallel workers: pread from fd (>= 0), else memcpy from the
// pageable host array src (page-cache reads and pageable copies are
// memcpy-bound on one core). false on a read error.
// Host threads that stage pageable or file input into the pinned ring: one
// process-wide pool, started on first use (a chunk used to spawn its own
// threads: 15 thread creations per 32 MB chunk cost more than the copy).
// A job is cut into parts, taken from an atomic counter by the caller and
// the workers. Workers spin briefly after a job (the next chunk follows
// within a millisecond), then park. Serves one job at a time (a mutex).
class StagePool {
 public:
  // the staging threads besides the caller: CHGPU_STAGE_THREADS - 1
  // (default min(16, cores) - 1)
  static int max_threads() {
    static const int m = [] {
      const char* e = std::getenv("CHGPU_STAGE_THREADS");
      const int hw = (int)std::thread::hardware_concurrency();
      return std::max(0, (e ? std::atoi(e) : std::min(16, std::max(1, hw))) - 1);
    }();
    return m;
  }
  static StagePool& get() {
    static StagePool* p = new StagePool();  // (never destroyed: its threads live with the process)
    return *p;
  }
  // f(part) for every part in [0, parts), parts handed out through an
  // atomic counter to the caller and the workers; false if any part
  // returned false
  bool run(int parts, const std::function<bool(int)>& f) {
    std::lock_guard<std::mutex> busy(busy_);
    start(parts - 1);
    if (th_.empty() || parts <= 1) {
      bool ok = true;
      for (int i = 0; i < parts; ++i) ok = f(i) && ok;
      return ok;
    }
    {
      std::lock_guard<std::mutex> lk(m_);
      job_ = &f;
      nparts_ = parts;
      next_.store(0);
      ok_.store(true);
      active_.store((int)th_.size());
      gen_.fetch_add(1, std::memory_order_release);
    }
    cv_.notify_all();
    work();
    while (active_.load(std::memory_order_acquire) != 0) std::this_thread::yield();
    return ok_.load();
  }

 private:
  void work() {
    for (int i = next_.fetch_add(1); i < nparts_; i = next_.fetch_add(1))
      if (!(*job_)(i)) ok_.store(false);
  }
  void start(int want) {
    const pid_t me = getpid();
    if (pid_ != me) {
      // a forked child has none of these threads: it starts its own (the
      // parent's std::thread objects are moved out of the way, never
      // destroyed: destroying a joinable std::thread terminates)
      if (!th_.empty()) new std::vector<std::thread>(std::move(th_));
      th_.clear();
      pid_ = me;
      failed_ = false;
    }
    want = std::min(want, max_threads());
    while ((int)th_.size() < want && !failed_) {
      try {
        th_.emplace_back([this, g = gen_.load()] { loop(g); });
      } catch (...) {
        failed_ = true;  // run with the threads that did start
      }
    }
  }
  // seen = the generation when the thread was created: a thread that is
  // first scheduled after the job was posted still takes part in it
  void loop(unsigned seen) {
    for (;;) {
      // spin ~200 us for the next job, then park
      const auto until = std::chrono::steady_clock::now() + std::chrono::microseconds(200);
      while (gen_.load(std::memory_order_acquire) == seen && std::chrono::steady_clock::now() < until)
        std::this_thread::yield();
      if (gen_.load(std::memory_order_acquire) == seen) {
        std::unique_lock<std::mutex> lk(m_);
        cv_.wait(lk, [&] { return gen_.load() != seen; });
      }
      seen = gen_.load(std::memory_order_acquire);
      work();
      active_.fetch_sub(1, std::memory_order_acq_rel);
    }
  }
  std::mutex busy_, m_;
  std::condition_variable cv_;
  std::vector<std::thread> th_;
  pid_t pid_ = 0;
  bool failed_ = false;
  const std::function<bool(int)>* job_ = nullptr;
  int nparts_ = 0;
  std::atomic<unsigned> gen_{0};
  std::atomic<int> next_{0}, active_{0};
  std::atomic<bool> ok_{true};
};

// Copies bytes [off, off + len) of the source into dst with up to
// `threads` parallel workers: pread from fd (>= 0), else memcpy from the
// pageable host array src (page-cache reads and pageable copies are
// memcpy-bound on one core). false on a read error.
bool stage_bytes(int fd, const unsigned char* src, unsigned char* dst, size_t off, size_t len,
                 int threads) {
  auto part = [&](size_t a, size_t b) -> bool {
    if (fd < 0) {
      copy_stream(dst + (a - off), src + a, b - a);
      return true;
    }
    while (a < b) {
      const ssize_t r = pread(fd, dst + (a - off), b - a, (off_t)a);
      if (r <= 0) return false;
      a += (size_t)r;
    }
    return true;
  };
  if (threads <= 1 || len < (size_t(1) << 20)) return part(off, off + len);
  const size_t step = ((len + threads - 1) / threads + 4095) & ~size_t(4095);
  const int parts = (int)((len + step - 1) / step);
  return StagePool::get().run(parts, [&](int t) -> bool {
    const size_t a = off + (size_t)t * step, b = std::min(off + len, a + step);
    return a >= b ? true : part(a, b);
  });
}

// Core of chgpu_hull / chgpu_hull_device / chgpu_hull_xy_binary. h_src !=
// nullptr: the input is on the host and is staged in chunks on a copy
// stream, overlapped with K1; fd >= 0: the input is read from a file
// (xy_binary: the bytes of Point2[]) chunk by chunk into a pinned ring,
// each chunk's copy and K1 overlapping the next chunk's read, and K1 also
// checks finiteness (io.cpp:38-42).
int run_pipeline(chgpu_ctx* ctx, const double* h_src, const double2* pts_dev, size_t n,
                 size_t chunk_count, int fallback, const double** hull_xy, size_t* n_hull,
                 chgpu_stats* stats, chgpu_diag* diag, int fd = -1) {
  const auto t_wall0 = std::chrono::steady_clock::now();
  chgpu_stats S{};
  chgpu_diag D{};
  S.n_input = n;
  cudaStream_t st = ctx->st;
  TRY(begin_call(ctx));
  ctx->tap.clear();
  for (auto& c : ctx->tap_counts) c = 0;
  // Which SPA path (decided before K1: K2 follows K1 with no stream
  // operation in between, so it can launch programmatically)
  bool want_filter =
      chunk_count >= 1 &&
      (ctx->spa_mode == CHGPU_SPA_FILTER || ctx->spa_mode == CHGPU_SPA_FILTER_SORTED ||
       (ctx->spa_mode == CHGPU_SPA_AUTO && chunk_count <= n / 64));
  const bool hinted = want_filter && ctx->spa_mode == CHGPU_SPA_AUTO && ctx->sort_hint &&
                      n >= ctx->sort_hint_n / 2 && n / 2 <= ctx->sort_hint_n;
  if (hinted) want_filter = false;
  int log2nb = want_filter ? filter_bits(n, chunk_count) : 0;
  // the bin scan is one cooperative launch: every CTA must be resident
  if (want_filter && bin_scan_blocks(log2nb) > (u32)device_limits().binscan_coop) {
    want_filter = false;
    log2nb = 0;
  }
  if (want_filter) TRY(ftab_prepare(ctx, log2nb, st));
  CK(cudaEventRecord(ctx->ev[0], st));
  // a call like the last one will reach the split finisher in a few hundred
  // microseconds: its worker threads spin instead of parking
  chgpu::host::finisher_prewake(ctx->kept_hint);

  // ---- K1: extremes (extremes.cpp:28-47).
  int nparts = 0;
  const bool from_file = fd >= 0;
  int nonfinite_slot = -1;
  // Pageable host input goes through the pinned ring too (a copy engine
  // reads pageable memory at a fraction of PCIe speed).
  bool pageable = false;
  if (h_src) {
    cudaPointerAttributes attr{};
    pageable = cudaPointerGetAttributes(&attr, h_src) != cudaSuccess ||
               attr.type == cudaMemoryTypeUnregistered;
    cudaGetLastError();  // clear a non-sticky "invalid value" for unknown pointers
  }
  const bool staged = from_file || pageable;
  if (h_src || from_file) {
    // staged input moves in smaller chunks through more slots (the same
    // pinned ring): the first chunk's host copy is not overlapped
    static const int stage_split = [] {
      const char* e = std::getenv("CHGPU_STAGE_SPLIT");  // tuning knob (log2)
      return e ? std::max(0, std::min(4, std::atoi(e))) : 2;
    }();
    static const size_t pinned_chunk = [] {
      const char* e = std::getenv("CHGPU_H2D_CHUNK_LOG2");  // tuning knob (points, log2)
      return e ? size_t(1) << std::max(16, std::min(30, std::atoi(e))) : kH2DChunk;
    }();
    const size_t chunk = staged ? kH2DChunk >> stage_split : pinned_chunk;
    const size_t slots = staged ? kFileSlots << stage_split : kFileSlots;
    const size_t nchunks = (n + chunk - 1) / chunk;
    const int per = std::max(1, std::min(kPartialBlocks, kMaxPartials / (int)nchunks));
    if (ctx->ev_copy.size() < nchunks) {
      size_t old = ctx->ev_copy.size();
      ctx->ev_copy.resize(nchunks);
      for (size_t i = old; i < nchunks; ++i)
        CK(cudaEventCreateWithFlags(&ctx->ev_copy[i], cudaEventDisableTiming));
    }
    CK(cudaEventRecord(ctx->ev[11], st));
    CK(cudaStreamWaitEvent(ctx->st_copy, ctx->ev[11], 0));
    // the last partial block of the call merges the quad (no final launch)
    u32 total_parts = 0;
    for (size_t c = 0; c < nchunks; ++c) {
      const size_t cnt = std::min(chunk, n - c * chunk);
      total_parts += (u32)extremes_blocks((int)std::min<size_t>(per, (cnt + 255) / 256));
    }
    const int ticket = take_ctr(ctx);
    if (from_file) nonfinite_slot = take_ctr(ctx);
    if (staged && !ctx->h_fslots)
      CK(cudaMallocHost(&ctx->h_fslots, kFileSlots * kH2DChunk * sizeof(double2)));
    static const int readers = [] {
      const char* e = std::getenv("CHGPU_STAGE_THREADS");  // tuning knob
      const int hw = (int)std::thread::hardware_concurrency();
      return std::max(1, e ? std::atoi(e) : std::min(16, hw));
    }();
    for (size_t c = 0; c < nchunks; ++c) {
      const size_t off = c * chunk, cnt = std::min(chunk, n - off);
      const double* src = h_src ? h_src + 2 * off : nullptr;
      if (staged) {
        // the slot's previous chunk must have reached the device
        if (c >= slots) CK(cudaEventSynchronize(ctx->ev_copy[c - slots]));
        double2* slot = ctx->h_fslots + (c % slots) * chunk;
        if (!stage_bytes(fd, reinterpret_cast<const unsigned char*>(h_src),
                         reinterpret_cast<unsigned char*>(slot), off * sizeof(double2),
                         cnt * sizeof(double2), readers)) {
          sync(ctx);
          return fail(ctx, CHGPU_IO_ERROR, "cannot read the xy_binary input");
        }
        src = reinterpret_cast<const double*>(slot);
      }
      CK(cudaMemcpyAsync(ctx->d_pts + off, src, cnt * sizeof(double2),
                         cudaMemcpyHostToDevice, ctx->st_copy));
      CK(cudaEventRecord(ctx->ev_copy[c], ctx->st_copy));
      CK(cudaStreamWaitEvent(st, ctx->ev_copy[c], 0));
      const int blocks = (int)std::min<size_t>(per, (cnt + 255) / 256);
      nparts += launch_extremes_partial(ctx->d_pts + off, cnt, off, ctx->d_partials, blocks, st,
                                        (u32)nparts, ctx->d_ctr + ticket, total_parts,
                                        ctx->d_qinfo,
                                        from_file ? ctx->d_ctr + nonfinite_slot : nullptr, log2nb);
      ++ctx->launches;
    }
    if (ctx->stage_times) CK(cudaEventRecord(ctx->ev[10], ctx->st_copy));
  } else {
    const int blocks = (int)std::min<size_t>(kPartialBlocks, (n + 255) / 256);
    const int ticket = take_ctr(ctx);
    nparts = launch_extremes_partial(pts_dev, n, 0, ctx->d_partials, blocks, st, 0,
                                     ctx->d_ctr + ticket, (u32)extremes_blocks(blocks),
                                     ctx->d_qinfo, nullptr, log2nb);
    ++ctx->launches;
  }
  const double2* pts = (h_src || from_file) ? ctx->d_pts : pts_dev;
  // K2 on the filter path launches programmatically right behind K1 (its
  // CTAs load their points while K1's last block merges the quad): no
  // event between them, the two are timed together
  const bool pdl = want_filter && ctx->pdl;
  if (!pdl) CK(cudaEventRecord(ctx->ev[1], st));

  // ---- K2: classify + round-1 discard (classify.cpp:9-87), plus the SPA
  // pre-filter's per-bin statistics when that path is taken.
  const FilterTabs ftabs = filter_tabs(ctx, log2nb);
  const int cnt_slot = ctx->ctr_used;
  ctx->ctr_used += 5;
  if (want_filter) {
    // raw survivor points + bin statistics (a degenerate frame writes the
    // LEX records of stream 1 instead)
    launch_classify_survivors(pts, (u32)n, ctx->d_qinfo, ctx->d_kbuf, ctx->d_vbuf,
                              ctx->d_kbuf, ctx->d_vbuf,
                              ctx->d_ctr + cnt_slot, log2nb, ftabs.cnt, ftabs.w, filter_wmask(), pdl,
                              st);
  } else {
    launch_classify_compact(pts, (u32)n, ctx->d_qinfo, nullptr, 0, ctx->d_kbuf, ctx->d_vbuf,
                            ctx->cap, ctx->d_ctr + cnt_slot, st);
  }
  ctx->launches += 1;  // K2 (K1 counted at its launch)
  CK(cudaGetLastError());
  CK(cudaEventRecord(ctx->ev[2], st));
  // The filter path is enqueued before the host sees K2's results (it idles
  // itself on a degenerate frame), with a speculative read-back of the
  // chains sized by the previous call.
  int ovf_slot = -1;
  size_t spec = 0;
  if (want_filter) {
    // (small chains only: a survivor-heavy call reads its result back once
    // it knows the size, or not at all on the convex fast path). The emit
    // writes up to `spec` kept points straight into the pinned h_out.
    if (ctx->kept_hint + 4 < kConvexMin)
      spec = std::min<size_t>(ctx->cap, std::max<size_t>(4096, ctx->kept_hint + ctx->kept_hint / 16 + 256));
    TRY(ensure_host_out(ctx, spec + 4));
    TRY(enqueue_filter_spa(ctx, pts, n, chunk_count, log2nb, cnt_slot, &ovf_slot,
                           from_file ? nonfinite_slot : -1, emit_mapped() ? spec : 0));
    if (spec && !emit_mapped())
      CK(cudaMemcpyAsync(ctx->h_out, ctx->d_kept, spec * sizeof(double2), cudaMemcpyDeviceToHost,
                         st));
  }
  // every counter the host needs, in one launch straight into the pinned
  // (device-mapped) host block instead of one DMA per value (the filter
  // path's k_spa_finish did it already)
  if (!want_filter) {
    k_readback<<<1, 64, 0, st>>>(ctx->d_qinfo, ctx->d_ctr, cnt_slot, ovf_slot,
                                 from_file ? nonfinite_slot : -1, ctx->d_u64, ctx->h);
    ++ctx->launches;
    CK(cudaGetLastError());
  }
  if (want_filter && ctx->stage_times) CK(cudaEventRecord(ctx->ev[9], st));
  const auto t_enq = std::chrono::steady_clock::now();
  // (per-kernel events want a drained stream; a DMA read-back of the chains
  // comes after the flag)
  if (want_filter && !ctx->stage_times && emit_mapped() && spec)
    TRY(wait_filter_flag(ctx));
  else
    TRY(sync(ctx));
  D.t_host_enqueue_ms = std::chrono::duration<double, std::milli>(t_enq - t_wall0).count();
  D.t_host_wait_ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_enq).count();
  if (want_filter) TRY(ftab_clear_behind(ctx));  // K2 and the filter path are done with them
  // read_points rejects the file before convex_hull runs (io.cpp:38-42)
  if (from_file && ctx->h->ctr[nonfinite_slot])
    return fail(ctx, CHGPU_NONFINITE, "non-finite coordinate");

  const QuadInfo qi = ctx->h->qi;
  const bool overflow = want_filter && !qi.degenerate && ctx->h->ctr[ovf_slot] != 0;
  if (overflow) {
    // The full region sort needs K2's (k, v) streams, which the filter
    // path's K2 does not write: run the record-writing K2 (the input is
    // intact; the counts are the same classification).
    const int rec_slot = take_ctr(ctx);
    (void)take_ctr(ctx), (void)take_ctr(ctx), (void)take_ctr(ctx), (void)take_ctr(ctx);
    launch_classify_compact(pts, (u32)n, ctx->d_qinfo, nullptr, 0, ctx->d_kbuf, ctx->d_vbuf,
                            ctx->cap, ctx->d_ctr + rec_slot, st);
    ctx->launches += 1;
    CK(cudaGetLastError());
  }
  u64 m[4];
  for (int s = 0; s < 4; ++s) m[s] = ctx->h->ctr[cnt_slot + 1 + s];
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
    size_t nu = 0;
    TRY(sorted_unique_survivors(ctx, s1, qi.q, &nu, &D.sort_passes, &D.tie_runs));
    TRY(ensure_host_out(ctx, nu + 4));
    CK(cudaMemcpyAsync(ctx->h_out, ctx->d_kept, nu * sizeof(double2), cudaMemcpyDeviceToHost, st));
    TRY(sync(ctx));
    t_fin0 = std::chrono::steady_clock::now();
    const Pt* up = reinterpret_cast<const Pt*>(ctx->h_out);
    ctx->chains.assign(up, up + nu);
    // frame_vertices(quad) joins the survivors (pipeline.cpp:63-64).
    Pt fr[4];
    int nf = 0;
    frame_of(qi.q, fr, &nf);
    for (int f = 0; f < nf; ++f) chgpu::host::insert_sorted_unique(ctx->chains, fr[f]);
    chgpu::host::monotone_chain(ctx->chains.data(), ctx->chains.size(), ctx->hull);
    ctx->hull_ptr = ctx->hull.data();
    ctx->hull_n = ctx->hull.size();
  } else {
    for (int s = 0; s < 4; ++s) D.region_counts[s + 1] = m[s];
    D.region_counts[0] = n - s1;
    // chunk_count == 0 raises on the non-degenerate branch only, exactly
    // like the reference (spa.cpp:112-113).
    if (chunk_count == 0) return fail(ctx, CHGPU_INVALID_ARG, "spa_filter: chunk_count must be >= 1");
    const SpaPlan plan = make_spa_plan(m, chunk_count, qi.q);
    bool filtered = false;
    if (want_filter) {
      // ---- K3 + K4/K5 ran on the SPA candidates only (k_filter.cu).
      D.n_candidates = (size_t)ctx->h->ncand;
      D.filter_log2nb = log2nb;
      D.spa_path = overflow ? 2 : 1;
      filtered = !overflow;
      if (!filtered) {  // the attempt
        CK(cudaEventSynchronize(ctx->ev[8]));
        t_sort_ms = ms_between(ctx->ev[2], ctx->ev[8]);
      }
      // (a filtered call's stage times are read after the finisher: the
      // host may be here before the stream has drained, see wait_filter_flag)
    }
    if (!filtered) {
      // ---- K3: region sort (spa.cpp:59-81) of every survivor.
      CK(cudaEventRecord(ctx->ev[7], st));
      Sorted so{};
      TRY(sort_regions(ctx, m, qi.q, ctx->stage_times, true, &so));
      D.sort_passes = so.passes;
      const bool sort_timed = s1 > 0;
      CK(cudaEventRecord(ctx->ev[6], st));

      // ---- K4/K5: SPA (spa.cpp:109-163).
      auto spa_and_read = [&]() -> int {
        CK(cudaMemsetAsync(ctx->d_u64, 0, 4 * sizeof(unsigned long long), st));
        TRY(run_spa(ctx, so.kF, so.vF, plan));
        CK(cudaEventRecord(ctx->ev[8], st));
        // kept counts, the group count and the long-group count in one trip
        CK(cudaMemcpyAsync(ctx->h->kept, ctx->d_u64, 4 * sizeof(unsigned long long),
                           cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(&ctx->h->uniq, ctx->d_u64 + 10, sizeof(unsigned long long),
                           cudaMemcpyDeviceToHost, st));
        if (so.pend.slot >= 0)
          CK(cudaMemcpyAsync(&ctx->h->ctr[so.pend.slot], ctx->d_ctr + so.pend.slot, sizeof(u32),
                             cudaMemcpyDeviceToHost, st));
        return sync(ctx);
      };
      TRY(spa_and_read());
      D.tie_runs = (size_t)ctx->h->uniq;
      if (so.pend.slot >= 0 && ctx->h->ctr[so.pend.slot] > 0) {
        // Rare: groups too long for shared memory. Sort them, then redo the
        // SPA over the now fully ordered regions.
        bool had = false;
        TRY(resolve_long(ctx, so.pend, &had));
        TRY(spa_and_read());
      }
      t_sort_ms += ms_between(ctx->ev[7], ctx->ev[6]);
      t_spa_ms = ms_between(ctx->ev[6], ctx->ev[8]);
      D.t_spa_kernel_ms = t_spa_ms;
      if (sort_timed && ctx->stage_times) {
        D.t_hist_ms = ms_between(ctx->ev[7], ctx->ev[3]);
        D.t_passes_ms = ms_between(ctx->ev[4], ctx->ev[5]);
        D.t_ties_ms = ms_between(ctx->ev[5], ctx->ev[6]);
      }
    }
    size_t kept_counts[4], kept = 0;
    for (int r = 0; r < 4; ++r) {
      kept_counts[r] = (size_t)ctx->h->kept[r];
      D.kept_counts[r] = kept_counts[r];
      kept += kept_counts[r];
    }
    S.n_after_spa = kept + qi.frame_size;  // pipeline.cpp:96
    if (ctx->chains_tap) {  // parity tap: the chains as the device left them
      ctx->tap.resize(kept);
      CK(cudaMemcpyAsync(ctx->tap.data(), ctx->d_kept, kept * sizeof(double2),
                         cudaMemcpyDeviceToHost, st));
      TRY(sync(ctx));
      for (int r = 0; r < 4; ++r) ctx->tap_counts[r] = kept_counts[r];
    }

    // ---- D2H of the chains, then polygon.cpp + melkman.cpp on the host.
    t_fin0 = std::chrono::steady_clock::now();
    ctx->kept_hint = kept;
    // (a filter-path call that fit clears the sort hint; an overflow sets
    // it; a hinted sort keeps it while the chains stay dense)
    ctx->sort_hint = overflow || (hinted && kept > n / 64);
    ctx->sort_hint_n = n;
    if (kept + 4 >= kConvexMin) {
      // Survivor-heavy: try Melkman's convex-position trajectory on the
      // device (k_convex.cu); on success the hull comes back canonical.
      bool convex = false;
      TRY(convex_finish(ctx, kept_counts, kept, &convex));
      if (convex) {
        D.convex_fast_path = 1;
        if (ctx->stage_times) D.t_d2h_ms = ms_between(ctx->ev[8], ctx->ev[9]);
        goto finished;
      }
    }
    if (!(filtered && kept <= spec)) {  // else the speculative read-back holds them
      TRY(ensure_host_out(ctx, kept + 4));
      CK(cudaMemcpyAsync(ctx->h_out, ctx->d_kept, kept * sizeof(double2), cudaMemcpyDeviceToHost,
                         st));
      if (ctx->stage_times) CK(cudaEventRecord(ctx->ev[9], st));
      TRY(sync(ctx));
    }
    if (ctx->stage_times) D.t_d2h_ms = ms_between(ctx->ev[8], ctx->ev[9]);
    const auto t_host0 = std::chrono::steady_clock::now();
    // polygon.cpp:7-29 + melkman.cpp:17-86 in one streaming pass
    // (the four chains concurrently when they are long, verified: finisher.cpp)
    const int mk = chgpu::host::finish_chains_split(reinterpret_cast<const Pt*>(ctx->h_out),
                                                    kept_counts, corners, ctx->hull);
    if (mk) return fail(ctx, CHGPU_DEGENERATE, "assemble_polygon/melkman: degenerate polygon");
    // the filter path touched no counter after k_readback cleared them
    if (filtered) ctx->counters_clean = true;
    D.t_host_ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_host0).count();
    ctx->hull_ptr = ctx->hull.data();
    ctx->hull_n = ctx->hull.size();
  }
finished:
  const auto t_end = std::chrono::steady_clock::now();
  if (want_filter) {
    CK(cudaEventSynchronize(ctx->ev[8]));  // (drained long ago: the finisher ran since)
    if (D.spa_path == 1) {
      // sort = bin scan + filter (what replaces sort_region); spa = the
      // chunk SPA (k_spa_small, deferred bin sorts + k_spa_chunks, emit)
      t_sort_ms = ms_between(ctx->ev[2], ctx->ev[4]);
      t_spa_ms = ms_between(ctx->ev[4], ctx->ev[8]);
      D.t_spa_kernel_ms = t_spa_ms;
      if (ctx->stage_times) {
        D.t_binscan_ms = ms_between(ctx->ev[2], ctx->ev[3]);
        D.t_filter_ms = ms_between(ctx->ev[3], ctx->ev[4]);
        D.t_binsort_ms = ms_between(ctx->ev[5], ctx->ev[6]);
      }
    }
  }

  S.n_hull = ctx->hull_n;
  if (pdl) {
    // K1 and K2 overlap (programmatic launch): one interval for both, the
    // discard stage, reported as extremes + classify
    S.t_extremes_ms = ms_between(ctx->ev[0], ctx->ev[2]);
    S.t_classify_ms = 0.0;
  } else {
    S.t_extremes_ms = ms_between(ctx->ev[0], ctx->ev[1]);
    S.t_classify_ms = ms_between(ctx->ev[1], ctx->ev[2]);
  }
  D.k1k2_overlapped = pdl ? 1 : 0;
  S.t_partition_ms = 0.0;
  S.t_sort_ms = t_sort_ms;
  S.t_spa_ms = t_spa_ms;
  S.t_melkman_ms = std::chrono::duration<double, std::milli>(t_end - t_fin0).count();
  S.t_total_ms = std::chrono::duration<double, std::milli>(t_end - t_wall0).count();
  D.t_k1_ms = S.t_extremes_ms;  // (K1 + K2 when k1k2_overlapped)
  D.t_k2_ms = S.t_classify_ms;
  if ((h_src || from_file) && ctx->stage_times) D.t_h2d_ms = ms_between(ctx->ev[0], ctx->ev[10]);
  D.launches = ctx->launches;

  *hull_xy = reinterpret_cast<const double*>(ctx->hull_ptr);
  *n_hull = ctx->hull_n;
  if (stats) *stats = S;
  if (diag) *diag = D;
  return CHGPU_OK;
}

int upload_points(chgpu_ctx* ctx, const double* xy, size_t n) {
  TRY(ensure_cap(ctx, n));
  CK(cudaMemcpyAsync(ctx->d_pts, xy, n * sizeof(double2), cudaMemcpyHostToDevice, ctx->st));
  return CHGPU_OK;
}

int upload_quad(chgpu_ctx* ctx, const double* quad, int log2nb = 0) {
  QuadInfo qi{};
  std::memcpy(qi.q, quad, sizeof qi.q);
  Pt fr[4];
  int nf = 0;
  frame_of(quad, fr, &nf);
  qi.frame_size = (u32)nf;
  qi.degenerate = nf <= 2;
  quad_derive(qi, log2nb);
  ctx->h->qi = qi;
  TRY(upload(ctx, ctx->d_qinfo, &ctx->h->qi, sizeof(QuadInfo)));
  return CHGPU_OK;
}

}  // namespace

namespace chgpu {

const DeviceLimits& device_limits() {
  constexpr int kMaxDevices = 64;
  static std::once_flag once[kMaxDevices];
  static DeviceLimits lim[kMaxDevices];
  static DeviceLimits none = [] {
    DeviceLimits d;
    d.status = cudaErrorInvalidDevice;
    return d;
  }();
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return none;
  std::call_once(once[dev], [dev] {
    DeviceLimits& d = lim[dev];
    cudaError_t e = cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev);
    if (e == cudaSuccess) e = configure_sort_kernels();
    if (e == cudaSuccess) e = configure_spa_kernels();
    if (e == cudaSuccess) e = configure_k2_kernels();
    if (e == cudaSuccess) e = configure_filter_kernels(&d);
    if (e == cudaSuccess) d.k1_wave = extremes_wave(d.sms);
    d.status = e;
  });
  return lim[dev];
}

}  // namespace chgpu

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
  if (device_limits().status != cudaSuccess) {  // kernel attributes of this device
    delete ctx;
    return CHGPU_CUDA_ERR;
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
      bad(cudaMalloc(&ctx->d_ftab, filter_tab_bytes(kMaxFilterBits))) ||
      bad(cudaMalloc(&ctx->d_fstart, (size_t(4) << kMaxFilterBits) * sizeof(u32))) ||
      bad(cudaMalloc(&ctx->d_fthr, (size_t(4) << kMaxFilterBits) * sizeof(u64))) ||
      bad(cudaMalloc(&ctx->d_fbig, 2 * (size_t)kBigListB * sizeof(u32))) ||
      bad(cudaMalloc(&ctx->d_faux, 32768)) ||
      bad(cudaMalloc(&ctx->d_plan, sizeof(FilterPlan))) ||
      bad(cudaMallocHost(&ctx->h, sizeof(Pinned)))) {
    chgpu_ctx_destroy(ctx);
    return CHGPU_CUDA_ERR;
  }
  std::memset(ctx->h, 0, sizeof(Pinned));
  for (auto& e : ctx->ev) cudaEventCreate(&e);
  if (const char* e = std::getenv("CHGPU_PDL")) ctx->pdl = std::atoi(e) != 0;
  if (const char* e = std::getenv("CHGPU_STAGE_TIMES")) ctx->stage_times = std::atoi(e) != 0;
  if (const char* e = std::getenv("CHGPU_SPA")) {
    if (std::strcmp(e, "sort") == 0) ctx->spa_mode = CHGPU_SPA_SORT;
    if (std::strcmp(e, "filter") == 0) ctx->spa_mode = CHGPU_SPA_FILTER;
    if (std::strcmp(e, "filter_sorted") == 0) ctx->spa_mode = CHGPU_SPA_FILTER_SORTED;
  }
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
  cudaFree(ctx->d_ftab);
  cudaFree(ctx->d_fstart);
  cudaFree(ctx->d_fthr);
  cudaFree(ctx->d_fbig);
  cudaFree(ctx->d_faux);
  cudaFree(ctx->d_plan);
  cudaFree(ctx->d_ffirst);
  cudaFree(ctx->d_fdefer);
  cudaFree(ctx->d_store);
  cudaFree(ctx->d_union);
  cudaFree(ctx->d_digit_excl);
  cudaFreeHost(ctx->h);
  cudaFreeHost(ctx->h_segs);
  cudaFreeHost(ctx->h_out);
  cudaFreeHost(ctx->h_stage);
  cudaFreeHost(ctx->h_fslots);
  for (auto& e : ctx->ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : ctx->ev_copy) cudaEventDestroy(e);
  if (ctx->st) cudaStreamDestroy(ctx->st);
  if (ctx->st_copy) cudaStreamDestroy(ctx->st_copy);
  delete ctx;
}

const char* chgpu_last_error(const chgpu_ctx* ctx) { return ctx ? ctx->err.c_str() : "no context"; }

int chgpu_ctx_set_option(chgpu_ctx* ctx, int option, long long value) {
  if (!ctx) return CHGPU_INVALID_ARG;
  switch (option) {
    case CHGPU_OPT_SPA_PATH:
      if (value < CHGPU_SPA_AUTO || value > CHGPU_SPA_FILTER_SORTED) break;
      ctx->spa_mode = (int)value;
      ctx->sort_hint = false;
      return CHGPU_OK;
    case CHGPU_OPT_CHAINS_TAP:
      if (value != 0 && value != 1) break;
      ctx->chains_tap = value != 0;
      return CHGPU_OK;
    case CHGPU_OPT_PDL:
      if (value != 0 && value != 1) break;
      ctx->pdl = value != 0;
      return CHGPU_OK;
    case CHGPU_OPT_STAGE_TIMES:
      if (value != 0 && value != 1) break;
      ctx->stage_times = value != 0;
      return CHGPU_OK;
    default:
      break;
  }
  return fail(ctx, CHGPU_INVALID_ARG, "chgpu_ctx_set_option: unknown option or value");
}

void* chgpu_ctx_stream(chgpu_ctx* ctx) { return ctx ? (void*)ctx->st : nullptr; }

int chgpu_last_chains(chgpu_ctx* ctx, const double** chains_xy, size_t* kept_counts) {
  if (!ctx || !ctx->chains_tap)
    return ctx ? fail(ctx, CHGPU_INVALID_ARG, "chgpu_last_chains: CHGPU_OPT_CHAINS_TAP is off")
               : CHGPU_INVALID_ARG;
  *chains_xy = reinterpret_cast<const double*>(ctx->tap.data());
  for (int r = 0; r < 4; ++r) kept_counts[r] = ctx->tap_counts[r];
  return CHGPU_OK;
}

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
  TRY(ensure_cap(ctx, n));
  return run_pipeline(ctx, xy, nullptr, n, chunk_count, degenerate_fallback, hull_xy, n_hull, stats,
                      diag);
}

int chgpu_hull_xy_binary(chgpu_ctx* ctx, const char* path, size_t chunk_count,
                         int degenerate_fallback, const double** hull_xy, size_t* n_hull,
                         chgpu_stats* stats, chgpu_diag* diag) {
  *n_hull = 0;
  const int fd = open(path, O_RDONLY | O_CLOEXEC);
  if (fd < 0)
    return fail(ctx, CHGPU_IO_ERROR, (std::string("cannot open '") + path + "' for reading").c_str());
  struct stat sb;
  if (fstat(fd, &sb) != 0) {
    close(fd);
    return fail(ctx, CHGPU_IO_ERROR, "cannot stat the xy_binary input");
  }
  const size_t bytes = (size_t)sb.st_size;
  int st = CHGPU_OK;
  if (bytes % 16 != 0) {  // io.cpp:105-106
    st = fail(ctx, CHGPU_PARSE_ERROR,
              "parse error: binary payload is not a whole number of float64 pairs");
  } else if (bytes == 0) {
    st = fail(ctx, CHGPU_EMPTY, "convex_hull: no points");
  } else if (bytes / 16 >= (size_t(1) << 32)) {
    st = fail(ctx, CHGPU_TOO_LARGE, "more than 2^32-1 points per call");
  } else {
    cudaSetDevice(ctx->device);
    const size_t n = bytes / 16;
    st = ensure_cap(ctx, n);
    if (st == CHGPU_OK)
      st = run_pipeline(ctx, nullptr, nullptr, n, chunk_count, degenerate_fallback, hull_xy, n_hull,
                        stats, diag, fd);
  }
  close(fd);
  return st;
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
  TRY(ensure_cap(ctx, n));
  return run_pipeline(ctx, nullptr, reinterpret_cast<const double2*>(d_xy), n, chunk_count,
                      degenerate_fallback, hull_xy, n_hull, stats, diag);
}

// ---------------------------------------------------------------- stage taps

int chgpu_find_extremes(chgpu_ctx* ctx, const double* xy, size_t n, double* quad_out) {
  if (n == 0) return fail(ctx, CHGPU_EMPTY, "find_extremes: no points");
  if (n >= (size_t(1) << 32)) return fail(ctx, CHGPU_TOO_LARGE, "too many points");
  cudaSetDevice(ctx->device);
  TRY(upload_points(ctx, xy, n));
  const int blocks = launch_extremes_partial(
      ctx->d_pts, n, 0, ctx->d_partials, (int)std::min<size_t>(kPartialBlocks, (n + 255) / 256),
      ctx->st);
  launch_extremes_final(ctx->d_partials, blocks, ctx->d_qinfo, nullptr, ctx->st);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(&ctx->h->qi, ctx->d_qinfo, sizeof(QuadInfo), cudaMemcpyDeviceToHost, ctx->st));
  TRY(sync(ctx));
  std::memcpy(quad_out, ctx->h->qi.q, 8 * sizeof(double));
  return CHGPU_OK;
}

int chgpu_classify(chgpu_ctx* ctx, const double* xy, size_t n, const double* quad, uint8_t* labels,
                   size_t* counts) {
  for (int r = 0; r < 5; ++r) counts[r] = 0;
  if (n == 0) return CHGPU_OK;
  cudaSetDevice(ctx->device);
  TRY(upload_points(ctx, xy, n));
  TRY(upload_quad(ctx, quad));
  CK(cudaMemsetAsync(ctx->d_u64 + 5, 0, 5 * sizeof(unsigned long long), ctx->st));
  const int blocks = (int)std::min<size_t>(148 * 8, (n + 255) / 256);
  launch_classify_labels(ctx->d_pts, n, ctx->d_qinfo, ctx->d_flags, ctx->d_u64 + 5, blocks, ctx->st);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(labels, ctx->d_flags, n, cudaMemcpyDeviceToHost, ctx->st));
  CK(cudaMemcpyAsync(ctx->h->counts5, ctx->d_u64 + 5, 5 * sizeof(unsigned long long),
                     cudaMemcpyDeviceToHost, ctx->st));
  TRY(sync(ctx));
  for (int r = 0; r < 5; ++r) counts[r] = (size_t)ctx->h->counts5[r];
  return CHGPU_OK;
}

int chgpu_discard_round1(chgpu_ctx* ctx, const double* xy, const uint8_t* labels, size_t n,
                         double* out_xy, uint8_t* out_labels, size_t* counts) {
  for (int r = 0; r < 5; ++r) counts[r] = 0;
  if (n == 0) return CHGPU_OK;
  if (n >= (size_t(1) << 32)) return fail(ctx, CHGPU_TOO_LARGE, "too many points");
  cudaSetDevice(ctx->device);
  TRY(upload_points(ctx, xy, n));
  CK(cudaMemcpyAsync(ctx->d_flags, labels, n, cudaMemcpyHostToDevice, ctx->st));
  TRY(begin_call(ctx));
  const int cnt_slot = ctx->ctr_used;
  ctx->ctr_used += 5;
  launch_classify_compact(ctx->d_pts, (u32)n, ctx->d_qinfo, ctx->d_flags, 0, ctx->d_kbuf,
                          ctx->d_vbuf, ctx->cap, ctx->d_ctr + cnt_slot, ctx->st);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(&ctx->h->ctr[cnt_slot], ctx->d_ctr + cnt_slot, 5 * sizeof(u32),
                     cudaMemcpyDeviceToHost, ctx->st));
  TRY(sync(ctx));
  const u64 cap = ctx->cap;
  u64 m[4], s1 = 0;
  for (int s = 0; s < 4; ++s) {
    m[s] = ctx->h->ctr[cnt_slot + 1 + s];
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
  TRY(sync(ctx));
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
  TRY(upload_points(ctx, xy, m));
  TRY(begin_call(ctx));
  launch_encode(ctx->d_pts, m, region, ctx->d_kbuf, ctx->d_vbuf, ctx->st);
  // No quad here: a full 64-bit LSD on k, then the ==-primary fix-up.
  TRY(ensure_segs(ctx, 1));
  ctx->h_segs[0] = make_seg(0, 0, m, region);
  Sorted so{};
  TRY(sort_segments(ctx, 1, 0, false, false, &so));
  launch_decode(so.kF, so.vF, m, region, ctx->d_kept, ctx->st);
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
  TRY(upload_points(ctx, xy, m));
  TRY(begin_call(ctx));
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
  TRY(run_spa(ctx, ctx->d_ka, ctx->d_va, plan));
  CK(cudaMemcpyAsync(ctx->h->kept, ctx->d_u64, 4 * sizeof(unsigned long long),
                     cudaMemcpyDeviceToHost, ctx->st));
  TRY(sync(ctx));
  const size_t k = (size_t)ctx->h->kept[r];
  CK(cudaMemcpyAsync(out, ctx->d_kept, k * sizeof(double2), cudaMemcpyDeviceToHost, ctx->st));
  TRY(sync(ctx));
  *n_out = k;
  return CHGPU_OK;
}

// ---------------------------------------------------------------- sharded path

int chgpu_shard_extremes(chgpu_ctx* ctx, const double* d_xy, size_t n, uint64_t base_index,
                         double* quad_out, uint64_t* idx_out) {
  if (n == 0) return fail(ctx, CHGPU_EMPTY, "find_extremes: no points");
  cudaSetDevice(ctx->device);
  const int blocks =
      launch_extremes_partial(reinterpret_cast<const double2*>(d_xy), n, base_index,
                              ctx->d_partials,
                              (int)std::min<size_t>(kPartialBlocks, (n + 255) / 256), ctx->st);
  launch_extremes_final(ctx->d_partials, blocks, nullptr, ctx->d_rawquad, ctx->st);
  CK(cudaGetLastError());
  QuadCand qc;
  CK(cudaMemcpyAsync(&qc, ctx->d_rawquad, sizeof qc, cudaMemcpyDeviceToHost, ctx->st));
  TRY(sync(ctx));
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

namespace {
// Shard chains (see include/chgpu.h), delivered to the context's pinned host
// buffer (d_dst == nullptr) or to a caller's device buffer of d_cap points.
int shard_chains_impl(chgpu_ctx* ctx, const double* d_xy, size_t n, const double* quad,
                      size_t chunk_count, const double** chains_xy, double* d_dst, size_t d_cap,
                      size_t* kept_counts, bool keep_on_device = false) {
  // the chains: left in ctx->d_kept, D2D into the caller's buffer, or D2H
  // into the context's
  auto deliver = [&](size_t total) -> int {
    if (keep_on_device) return sync(ctx);
    if (d_dst) {
      if (total > d_cap) return fail(ctx, CHGPU_TOO_LARGE, "shard chains exceed the output buffer");
      CK(cudaMemcpyAsync(d_dst, ctx->d_kept, total * sizeof(double2), cudaMemcpyDeviceToDevice,
                         ctx->st));
      TRY(sync(ctx));
      return CHGPU_OK;
    }
    TRY(ensure_host_out(ctx, total + 4));
    CK(cudaMemcpyAsync(ctx->h_out, ctx->d_kept, total * sizeof(double2), cudaMemcpyDeviceToHost,
                       ctx->st));
    TRY(sync(ctx));
    *chains_xy = reinterpret_cast<const double*>(ctx->h_out);
    return CHGPU_OK;
  };
  for (int r = 0; r < 4; ++r) kept_counts[r] = 0;
  if (chains_xy) *chains_xy = nullptr;
  if (n == 0) return CHGPU_OK;
  if (n >= (size_t(1) << 32)) return fail(ctx, CHGPU_TOO_LARGE, "shard too large");
  cudaSetDevice(ctx->device);
  TRY(ensure_cap(ctx, n));
  cudaStream_t st = ctx->st;
  TRY(begin_call(ctx));
  const int log2nb = filter_bits(n, chunk_count);
  TRY(upload_quad(ctx, quad, log2nb));
  const bool degenerate = ctx->h->qi.degenerate != 0;
  const double2* pts = reinterpret_cast<const double2*>(d_xy);
  if (!degenerate && chunk_count >= 1 && ctx->spa_mode != CHGPU_SPA_SORT &&
      (ctx->spa_mode == CHGPU_SPA_FILTER || ctx->spa_mode == CHGPU_SPA_FILTER_SORTED || chunk_count <= n / 64)) {
    // The pre-filtered SPA against the global quad (the same kernels as
    // chgpu_hull), falling back to the full region sort on overflow.
    TRY(ftab_prepare(ctx, log2nb, st));
    const FilterTabs ftabs = filter_tabs(ctx, log2nb);
    const int cnt_slot = ctx->ctr_used;
    ctx->ctr_used += 5;
    launch_classify_survivors(pts, (u32)n, ctx->d_qinfo, ctx->d_kbuf, ctx->d_vbuf,
                              ctx->d_kbuf, ctx->d_vbuf,
                              ctx->d_ctr + cnt_slot, log2nb, ftabs.cnt, ftabs.w, filter_wmask(), false,
                              st);
    CK(cudaGetLastError());
    int ovf_slot = -1;
    // (k_spa_finish hands the kept counts and the overflow flag to ctx->h)
    TRY(enqueue_filter_spa(ctx, pts, n, chunk_count, log2nb, cnt_slot, &ovf_slot));
    TRY(sync(ctx));
    TRY(ftab_clear_behind(ctx));  // (for the next call, while the host exchanges)
    if (!ctx->h->ctr[ovf_slot]) {
      for (int r = 0; r < 4; ++r) kept_counts[r] = (size_t)ctx->h->kept[r];
      return deliver(kept_counts[0] + kept_counts[1] + kept_counts[2] + kept_counts[3]);
    }
  }
  const int cnt_slot = ctx->ctr_used;
  ctx->ctr_used += 5;
  launch_classify_compact(pts, (u32)n, ctx->d_qinfo, nullptr, degenerate ? 1 : 0, ctx->d_kbuf,
                          ctx->d_vbuf, ctx->cap, ctx->d_ctr + cnt_slot, st);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(&ctx->h->ctr[cnt_slot], ctx->d_ctr + cnt_slot, 5 * sizeof(u32),
                     cudaMemcpyDeviceToHost, st));
  TRY(sync(ctx));
  u64 m[4], s1 = 0;
  for (int s = 0; s < 4; ++s) {
    m[s] = ctx->h->ctr[cnt_slot + 1 + s];
    s1 += m[s];
  }
  if (degenerate) {
    // Survivors go back sorted and unique; the merge re-runs the
    // degenerate branch on their union.
    size_t nu = 0, groups = 0;
    int passes = 0;
    TRY(sorted_unique_survivors(ctx, s1, quad, &nu, &passes, &groups));
    kept_counts[0] = nu;
  } else {
    if (chunk_count == 0) return fail(ctx, CHGPU_INVALID_ARG, "spa_filter: chunk_count must be >= 1");
    Sorted so{};
    TRY(sort_regions(ctx, m, quad, false, false, &so));
    const SpaPlan plan = make_spa_plan(m, chunk_count, quad);
    TRY(run_spa(ctx, so.kF, so.vF, plan));
    CK(cudaMemcpyAsync(ctx->h->kept, ctx->d_u64, 4 * sizeof(unsigned long long),
                       cudaMemcpyDeviceToHost, st));
    TRY(sync(ctx));
    for (int r = 0; r < 4; ++r) kept_counts[r] = (size_t)ctx->h->kept[r];
  }
  return deliver(kept_counts[0] + kept_counts[1] + kept_counts[2] + kept_counts[3]);
}
}  // namespace

int chgpu_shard_chains(chgpu_ctx* ctx, const double* d_xy, size_t n, const double* quad,
                       size_t chunk_count, const double** chains_xy, size_t* kept_counts) {
  return shard_chains_impl(ctx, d_xy, n, quad, chunk_count, chains_xy, nullptr, 0, kept_counts);
}

int chgpu_shard_chains_device(chgpu_ctx* ctx, const double* d_xy, size_t n, const double* quad,
                              size_t chunk_count, double* d_chains, size_t cap_points,
                              size_t* kept_counts) {
  return shard_chains_impl(ctx, d_xy, n, quad, chunk_count, nullptr, d_chains, cap_points,
                           kept_counts);
}

}  // extern "C"

// ---------------------------------------------------------------- one process, several GPUs

namespace {

// Grows a device buffer of double2 (on the current device), keeping `keep`
// leading points.
int grow(chgpu_ctx* ctx, double2** buf, size_t* cap, size_t want, size_t keep) {
  if (want <= *cap) return CHGPU_OK;
  const size_t ncap = std::max(want, *cap * 2);
  double2* nb = nullptr;
  CK(cudaMalloc(&nb, ncap * sizeof(double2)));
  if (keep) CK(cudaMemcpyAsync(nb, *buf, keep * sizeof(double2), cudaMemcpyDeviceToDevice, ctx->st));
  TRY(sync(ctx));
  cudaFree(*buf);
  *buf = nb;
  *cap = ncap;
  return CHGPU_OK;
}

struct ShardSlice {
  const double* xy;  // host or device (on its context's device)
  size_t n;
  u64 base;          // global index of its first point
  int ctx;
  bool host;
};

// Runs fn(i) for every context index, one host thread per context (the
// contexts' devices work concurrently); the first failure wins.
template <typename F>
int for_each_ctx(int nctx, F fn) {
  if (nctx == 1) return fn(0);
  std::vector<int> st(nctx, CHGPU_OK);
  std::vector<std::thread> th;
  th.reserve(nctx);
  for (int i = 0; i < nctx; ++i) th.emplace_back([&, i] { st[i] = fn(i); });
  for (auto& t : th) t.join();
  for (int x : st)
    if (x != CHGPU_OK) return x;
  return CHGPU_OK;
}

// Largest slice of a host shard one context holds at a time (a span of
// 2^32 points or more is processed in slices; each slice's indices stay
// below 2^32). CHGPU_SLICE_MAX (points) lowers it (tests).
size_t slice_max() {
  const char* e = std::getenv("CHGPU_SLICE_MAX");
  const size_t v = e ? (size_t)std::strtoull(e, nullptr, 10) : 0;
  return v ? std::min(v, size_t(1) << 30) : size_t(1) << 30;
}

}  // namespace

extern "C" {

void chgpu_host_prefault(void* p, size_t bytes) {
  unsigned char* const b = static_cast<unsigned char*>(p);
  if (!b || bytes == 0) return;
  const size_t step = size_t(4) << 20;  // 4 MB per part
  const int parts = (int)((bytes + step - 1) / step);
  StagePool::get().run(parts, [&](int t) -> bool {
    const size_t a = (size_t)t * step, e = std::min(bytes, a + step);
    for (size_t o = a; o < e; o += 4096) b[o] = 0;
    b[e - 1] = 0;
    return true;
  });
}

int chgpu_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

int chgpu_hull_sharded(chgpu_ctx* const* ctxs, int nctx, const double* const* shards,
                       const size_t* counts, int nshards, int on_device, size_t chunk_count,
                       int degenerate_fallback, const double** hull_xy, size_t* n_hull,
                       chgpu_stats* stats) {
  *n_hull = 0;
  if (nctx < 1 || !ctxs || nshards < 1 || !shards || !counts) return CHGPU_INVALID_ARG;
  chgpu_ctx* const c0 = ctxs[0];
  if (on_device && nshards != nctx)
    return fail(c0, CHGPU_INVALID_ARG, "chgpu_hull_sharded: device shards need one context each");
  const auto t_wall0 = std::chrono::steady_clock::now();
  // slices in global index order
  std::vector<ShardSlice> slices;
  u64 total = 0;
  for (int s = 0; s < nshards; ++s) {
    const size_t per = on_device ? counts[s] : slice_max();
    if (on_device && counts[s] >= (size_t(1) << 32))
      return fail(c0, CHGPU_TOO_LARGE, "a device shard must hold fewer than 2^32 points");
    for (size_t off = 0; off < counts[s]; off += per) {
      const size_t n = std::min(per, counts[s] - off);
      slices.push_back({shards[s] + 2 * off, n, total + off, s % nctx, !on_device});
    }
    total += counts[s];
  }
  if (total == 0) return fail(c0, CHGPU_EMPTY, "convex_hull: no points");
  std::vector<std::vector<size_t>> mine(nctx);
  for (size_t i = 0; i < slices.size(); ++i) mine[slices[i].ctx].push_back(i);
  // a context with one host slice keeps it resident between the passes
  auto place = [&](chgpu_ctx* ctx, const ShardSlice& sl) -> int {
    if (!sl.host) return CHGPU_OK;
    TRY(ensure_cap(ctx, sl.n));
    CK(cudaMemcpyAsync(ctx->d_pts, sl.xy, sl.n * sizeof(double2), cudaMemcpyHostToDevice, ctx->st));
    return CHGPU_OK;
  };
  auto dev_ptr = [&](chgpu_ctx* ctx, const ShardSlice& sl) {
    return sl.host ? reinterpret_cast<const double*>(ctx->d_pts) : sl.xy;
  };

  // exchange 1: every slice's extreme candidates with global indices,
  // folded in index order (extremes.cpp:39-46, lowest index on ties)
  std::vector<double> quads(8 * slices.size());
  std::vector<uint64_t> idxs(4 * slices.size());
  TRY(for_each_ctx(nctx, [&](int i) -> int {
    chgpu_ctx* ctx = ctxs[i];
    cudaSetDevice(ctx->device);
    for (size_t j : mine[i]) {
      TRY(place(ctx, slices[j]));
      TRY(chgpu_shard_extremes(ctx, dev_ptr(ctx, slices[j]), slices[j].n, slices[j].base,
                               &quads[8 * j], &idxs[4 * j]));
    }
    return CHGPU_OK;
  }));
  double quad[8];
  chgpu_fold_extremes(quads.data(), idxs.data(), slices.size(), quad);

  // per slice: round-1 discard, region sort and SPA against the global quad
  // (every dropped point lies inside the global quad or inside a triangle
  // of kept points and global anchors, so no hull vertex is lost); each
  // context appends its slices' chains to its device store
  // (per slice: where its chains sit in its context's store, and its region counts)
  std::vector<size_t> run_off(slices.size(), 0), run_kc(4 * slices.size(), 0);
  TRY(for_each_ctx(nctx, [&](int i) -> int {
    chgpu_ctx* ctx = ctxs[i];
    cudaSetDevice(ctx->device);
    ctx->store_n = 0;
    const bool resident = mine[i].size() == 1;
    for (size_t j : mine[i]) {
      if (!resident) TRY(place(ctx, slices[j]));
      size_t kc[4];
      TRY(shard_chains_impl(ctx, dev_ptr(ctx, slices[j]), slices[j].n, quad, chunk_count, nullptr,
                            nullptr, 0, kc, /*keep_on_device=*/true));
      const size_t k = kc[0] + kc[1] + kc[2] + kc[3];
      TRY(grow(ctx, &ctx->d_store, &ctx->store_cap, ctx->store_n + k + 1, ctx->store_n));
      if (k)
        CK(cudaMemcpyAsync(ctx->d_store + ctx->store_n, ctx->d_kept, k * sizeof(double2),
                           cudaMemcpyDeviceToDevice, ctx->st));
      run_off[j] = ctx->store_n;
      for (int r = 0; r < 4; ++r) run_kc[4 * j + r] = kc[r];
      ctx->store_n += k;
    }
    return sync(ctx);
  }));

  Pt fr[4];
  int nf = 0;
  frame_of(quad, fr, &nf);
  if (nf > 2) {
    // a proper frame: every hull vertex of the whole set is in some slice's
    // chains. Each region's runs (one per slice, sorted in region order)
    // are merged on the host and the ring [L, chain 1, B, ..., chain 4] is
    // finished with Melkman (chgpu_merge_hull): no second device pipeline.
    std::vector<std::vector<Pt>> host(nctx);
    TRY(for_each_ctx(nctx, [&](int i) -> int {
      chgpu_ctx* ctx = ctxs[i];
      cudaSetDevice(ctx->device);
      host[i].resize(ctx->store_n);
      if (ctx->store_n)
        CK(cudaMemcpyAsync(host[i].data(), ctx->d_store, ctx->store_n * sizeof(double2),
                           cudaMemcpyDeviceToHost, ctx->st));
      return sync(ctx);
    }));
    std::vector<const Pt*> runs(slices.size());
    for (size_t j = 0; j < slices.size(); ++j) runs[j] = host[slices[j].ctx].data() + run_off[j];
    const auto t_m0 = std::chrono::steady_clock::now();
    const int mk = chgpu::host::merge_chains_hull(runs.data(), run_kc.data(), (int)slices.size(),
                                                  reinterpret_cast<const Pt*>(quad), c0->hull);
    if (mk) return fail(c0, CHGPU_DEGENERATE, "assemble_polygon/melkman: degenerate polygon");
    c0->hull_ptr = c0->hull.data();
    c0->hull_n = c0->hull.size();
    *hull_xy = reinterpret_cast<const double*>(c0->hull_ptr);
    *n_hull = c0->hull_n;
    if (stats) {
      // n_input and n_hull are the whole set's; n_after_spa counts the
      // shards' chains + frame (a sharded run's stage counters are not
      // comparable with a single-process run)
      chgpu_stats S{};
      S.n_input = total;
      size_t kept = 0;
      for (size_t x : run_kc) kept += x;
      S.n_after_spa = kept + (size_t)nf;
      S.n_hull = c0->hull_n;
      const auto t_end = std::chrono::steady_clock::now();
      S.t_melkman_ms = std::chrono::duration<double, std::milli>(t_end - t_m0).count();
      S.t_total_ms = std::chrono::duration<double, std::milli>(t_end - t_wall0).count();
      *stats = S;
    }
    return CHGPU_OK;
  }

  // A degenerate frame (pipeline.cpp:53-71): each slice left its sorted
  // unique survivors; they go to the first context's device (peer copies
  // over NVLink) with the frame, and the single-GPU pipeline's degenerate
  // branch runs over that union
  cudaSetDevice(c0->device);
  size_t nu = 0;
  for (int i = 0; i < nctx; ++i) nu += ctxs[i]->store_n;
  TRY(grow(c0, &c0->d_union, &c0->union_cap, nu + 4, 0));
  size_t off = 0;
  for (int i = 0; i < nctx; ++i) {
    chgpu_ctx* ctx = ctxs[i];
    if (ctx->store_n)
      CK(cudaMemcpyPeerAsync(c0->d_union + off, c0->device, ctx->d_store, ctx->device,
                             ctx->store_n * sizeof(double2), c0->st));
    off += ctx->store_n;
  }
  TRY(upload(c0, c0->d_union + off, fr, nf * sizeof(Pt)));
  off += nf;
  TRY(ensure_cap(c0, off));
  chgpu_stats S{};
  TRY(run_pipeline(c0, nullptr, c0->d_union, off, chunk_count, degenerate_fallback, hull_xy, n_hull,
                   &S, nullptr));
  if (stats) {
    // n_input and n_hull are the whole set's; the stage counters and times
    // are the merge's (a sharded run's intermediate counters are not
    // comparable with a single-process run)
    S.n_input = total;
    S.t_total_ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_wall0).count();
    *stats = S;
  }
  return CHGPU_OK;
}

}  // extern "C"
