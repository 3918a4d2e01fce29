// Host-callable launchers for the hull kernels (internal to libchgpu).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>

#include "chgpu_internal.cuh"

namespace chgpu {

struct SpaPlan {
  u64 off[4];         // region offset in the sorted array
  u64 m[4];           // region size
  u64 chunk_size[4];  // ceil(m / chunk_count)            (spa.cpp:121)
  u32 chunk_begin[4]; // prefix of per-region chunk counts (spa.cpp:122)
  u32 total_chunks;
  double seed[4];     // guarded(anchors.first)           (spa.cpp:130-132)
};

// SPA pre-filter (k_filter.cu + k_spa.cu k_spa_bins).
constexpr int kBinSortMax = 4096;   // candidates of one bin sorted in shared memory (a CTA)
constexpr int kWarpSortMax = 256;   // ... by one warp
constexpr int kMaxFilterLog2 = 18;
constexpr u32 kSpaSmallCap = 128;   // candidates of one chunk k_spa_small takes (else deferred)  // bins per region at most 2^18
constexpr u32 kBigListB = 4u << kMaxFilterLog2; // offset of the CTA-sort list in the big-bin lists
struct FilterPlan {
  SpaPlan spa;          // chunk geometry, region offsets of the sorted layout
  u64 seed_w[4];        // wkey of guarded(anchors.first)
  int log2nb;           // bins per region = 2^log2nb
};
// Small per-call scratch of the pre-filter (<= 512 bin tiles).
// The counters the host reads after the filter path, written straight into
// pinned, device-mapped host memory by the last kernel of the path, which
// then clears them for the next call (pipeline.cu k_readback does the same
// for the other paths).
struct ReadbackArgs {
  const QuadInfo* qinfo;
  u32* ctr;                      // device counters [nctr]
  int nctr, cnt_slot, ovf_slot, nonfinite_slot;
  unsigned long long* u64s;      // device 64-bit counters [16]: kept [0, 4), candidates [11]
  u32* h_qi;                     // host (mapped): QuadInfo words
  u32* h_ctr;                    // host (mapped): counters
  unsigned long long* h_kept;    // host (mapped): kept [4]
  unsigned long long* h_ncand;   // host (mapped): candidates
  double2* h_chains = nullptr;   // host (mapped): the emit also writes the first
  u32 h_chains_cap = 0;          // h_chains_cap kept points here (no D2H copy)
  u32* h_done = nullptr;         // host (mapped): set to `seq` once all of the above is
  u32 seq = 0;                   // visible (the host starts on it before the stream drains)
};
__device__ __forceinline__ void readback_block(const ReadbackArgs& a) {
  const int t = threadIdx.x;
  const u32* q = reinterpret_cast<const u32*>(a.qinfo);
  for (int i = t; i < (int)(sizeof(QuadInfo) / 4); i += blockDim.x) a.h_qi[i] = q[i];
  if (t < 5) a.h_ctr[a.cnt_slot + t] = a.ctr[a.cnt_slot + t];
  if (t == 5 && a.ovf_slot >= 0) a.h_ctr[a.ovf_slot] = a.ctr[a.ovf_slot];
  if (t == 6 && a.nonfinite_slot >= 0) a.h_ctr[a.nonfinite_slot] = a.ctr[a.nonfinite_slot];
  if (t >= 8 && t < 12) a.h_kept[t - 8] = a.u64s[t - 8];
  if (t == 12) *a.h_ncand = a.u64s[11];
  __syncthreads();
  for (int i = t; i < a.nctr; i += blockDim.x) a.ctr[i] = 0;
  if (t < 16) a.u64s[t] = 0;
}

struct FilterAux {
  u32* tsum;        // records per bin tile
  u32* agg_seg;     // tile aggregates of the segmented max
  u64* agg_val;
};
// The plan of the filter path on the device (from K2's counts).
cudaError_t launch_bin_scan(const QuadInfo* qinfo, u32* counts, u64 chunk_count, int log2nb,
                     const u32* bcnt, const u32* bw, FilterPlan* plan, u32* bstart, u32* bthr,
                     u32* tcoarse, u32* first_bin, FilterAux aux, u32* bar, u32* overflow,
                     cudaStream_t st);
// CTAs of the cooperative k_bin_scan launch for log2nb bins per region.
u32 bin_scan_blocks(int log2nb);
cudaError_t launch_spa_finish(u64* k, u64* v, const u32* bcur, const u32* bstart, const u32* bmap,
                              const u32* first_bin, const FilterPlan* P, const u32* big,
                              const u32* nbig, u32* overflow, const u32* defer, const u32* ndefer,
                              u64* sk, u64* sv, u32* chunk_kept, u32* group_kept,
                              unsigned long long* kept_counts, double2* out, u32* bar,
                              u32 max_chunks, const ReadbackArgs& rb, cudaStream_t st);
void launch_spa_small(const u64* k, const u64* v, const u32* bcur, const u32* bstart,
                      const u32* bmap, const u32* first_bin, const FilterPlan* P, u32 max_chunks,
                      u64* sk, u64* sv, u32* chunk_kept, u32* group_kept,
                      unsigned long long* kept_counts, u32* defer, u32* ndefer, u32 cap,
                      cudaStream_t st);
void launch_filter(const u64* seg, const u64* segcnt, u32 nseg,
                   const double2* pts, const FilterPlan* P, const QuadInfo* qinfo,
                   const u32* bstart, const u32* bthr, const u32* tcoarse, int log2nb, u32* bcur,
                   u32* bmap, u64* kout, u64* vout, u32* big, u32* nbig, unsigned long long* ncand,
                   const u32* overflow, cudaStream_t st);

// Melkman's convex-position trajectory on the device (k_convex.cu).
int convex_blocks();
void launch_convex_check(const double2* chains, const u64 kept[4], const QuadInfo* qinfo, u32* ok,
                         u64* block_best, cudaStream_t st);
void launch_convex_emit(const double2* chains, const u64 kept[4], const QuadInfo* qinfo,
                        const u64* block_best, double2* out, cudaStream_t st);

// Per-device launch limits. device_limits() configures the kernels'
// attributes (dynamic shared memory opt-ins are per device) and measures
// residency once per device, thread-safely; chgpu_ctx_create calls it after
// cudaSetDevice so a failure surfaces there. Launchers read it for the
// current device.
struct DeviceLimits {
  cudaError_t status = cudaSuccess;
  int sms = 0;              // multiprocessors
  int k1_wave = 0;          // K1 CTAs in one resident wave
  int filter_resident = 0;  // k_filter CTAs in one resident wave
  int binscan_coop = 0;     // k_bin_scan CTAs that can be co-resident (cooperative launch bound)
  int finish_coop = 0;      // k_spa_finish CTAs that can be co-resident
};
const DeviceLimits& device_limits();
cudaError_t configure_sort_kernels();
cudaError_t configure_spa_kernels();
cudaError_t configure_k2_kernels();
cudaError_t configure_filter_kernels(DeviceLimits* lim);

// K1
// Blocks launch_extremes_partial will use for a request of `requested`.
int extremes_blocks(int requested);
// K1 CTAs in one resident wave on a device with `sms` multiprocessors.
int extremes_wave(int sms);
// With a ticket counter (zeroed) and the call's total partial count, the
// last block merges every partial into *out: no launch_extremes_final.
int launch_extremes_partial(const double2* pts, u64 n, u64 base_index, QuadCand* partials,
                            int blocks, cudaStream_t st, u32 part_base = 0,
                            u32* ticket = nullptr, u32 total_parts = 0, QuadInfo* out = nullptr,
                            u32* nonfinite = nullptr, int log2nb = 0);
void launch_extremes_final(const QuadCand* partials, int nparts, QuadInfo* out, QuadCand* raw_out,
                           cudaStream_t st);
// K2
void launch_classify_compact(const double2* pts, u32 n, const QuadInfo* qinfo,
                             const unsigned char* given_labels, int force_lex, u64* kbuf, u64* vbuf,
                             u64 ncap, u32* counts_out, cudaStream_t st);
// K2 of the pre-filtered path: raw survivor points + bin statistics.
void launch_classify_survivors(const double2* pts, u32 n, const QuadInfo* qinfo, u64* seg,
                               u64* segcnt, u64* kbuf, u64* vbuf, u32* counts_out, int log2nb,
                               u32* bcnt, u32* bw, u32 wmask, bool programmatic, cudaStream_t st);
void launch_classify_labels(const double2* pts, u64 n, const QuadInfo* qinfo,
                            unsigned char* labels, unsigned long long* counts, int blocks,
                            cudaStream_t st);
// K3
void launch_hist(const u64* kin, const u64* vin, const SegDesc* segs, int nseg, u32 total_tiles,
                 int mode, int npasses, int use_src, u32* hist, cudaStream_t st);
void launch_hist_scan(const u32* hist, const SegDesc* segs, int nseg, int npasses, u32* digit_excl,
                      u32* needed_mask, cudaStream_t st);
// Reduce-then-scan LSD pass (upsweep, column scan, downsweep); counts needs
// total_tiles * 256 u32.
void launch_lsd_pass(const u64* kin, const u64* vin, u64* kout, u64* vout, const SegDesc* segs,
                     int nseg, u32 total_tiles, int use_src, int mode, const u32* digit_excl,
                     int pass, u32* counts, cudaStream_t st);
void launch_onesweep(const u64* kin, const u64* vin, u64* kout, u64* vout, const SegDesc* segs,
                     int nseg, u32 total_tiles, int use_src, int mode, const u32* digit_excl,
                     int pass, u64* status, u32 tag, u32* tile_ctr, u32* rows, cudaStream_t st);
void launch_seg_copy(const u64* kin, const u64* vin, u64* kout, u64* vout, const SegDesc* segs,
                     int nseg, u32 total_tiles, int use_src, cudaStream_t st);
void launch_group_scan(u64* k, u64* v, const SegDesc* segs, int nseg, u32 total_tiles, int eqmode,
                       void* medium, u32* nmedium, unsigned long long* ngroups, cudaStream_t st);
void launch_group_fix_medium(u64* k, u64* v, const SegDesc* segs, const void* medium,
                             const u32* nmedium, void* longr, u32* nlong, cudaStream_t st);
size_t group_run_bytes();
// K4/K5
void launch_spa_tile(const u64* k, const u64* v, const SpaPlan& plan, u64 total, u64* status,
                     u32 tag, u64* pay, u32* ticket, double2* out,
                     unsigned long long* kept_counts, cudaStream_t st);
void launch_unique(const u64* k, const u64* v, u64 n, double2* out, u64* status, u32 tag,
                   u32* tile_ctr, unsigned long long* total, cudaStream_t st);

}  // namespace chgpu

namespace chgpu {
void launch_encode(const double2* pts, u64 n, int region, u64* k, u64* v, cudaStream_t st);
void launch_decode(const u64* k, const u64* v, u64 n, int region, double2* out, cudaStream_t st);
}  // namespace chgpu
