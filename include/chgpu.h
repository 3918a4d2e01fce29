/* chgpu.h — C ABI of the B200-native CudaChain hull path.
 *
 * This is the drop-in boundary under the reference's C++ entry point
 * chainhull::convex_hull (reference: proj/core/include/chainhull/
 * pipeline.hpp:55, implemented in proj/core/src/pipeline.cpp:25-106).
 * The C++ shim in paper_1508_05488_b200/cpp/ re-exports the reference's
 * own API (the headers under include/chainhull/) on top of these entry points, and the
 * Python mirror (paper_1508_05488_b200/__init__.py) binds them with ctypes.
 * Signatures carry plain pointers and sizes only.
 *
 * Points are interleaved float64 pairs, byte-identical to
 * chainhull::Point2 (sizeof 16, alignof 8: geometry.hpp:8-15).
 *
 * Errors: every entry point returns a chgpu_status. The C++ shim maps
 * CHGPU_EMPTY -> chainhull::EmptyInput, CHGPU_DEGENERATE ->
 * chainhull::DegenerateInput, CHGPU_INVALID_ARG -> std::invalid_argument,
 * on exactly the branches where the reference throws them
 * (pipeline.cpp:27, :58-59, spa.cpp:112-113, polygon.cpp:26-27,
 * melkman.cpp:44-47). chgpu_last_error() gives the message.
 *
 * Threading: a context owns one CUDA stream, a device workspace and pinned
 * staging buffers. Calls on one context must be serialised by the caller;
 * distinct contexts may be used concurrently (the reference promises
 * reentrancy, pipeline.hpp:53).
 */
#ifndef CHGPU_H
#define CHGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  CHGPU_OK = 0,
  CHGPU_EMPTY = 1,       /* EmptyInput (pipeline.cpp:27, extremes.cpp:29) */
  CHGPU_DEGENERATE = 2,  /* DegenerateInput (pipeline.cpp:58, polygon.cpp:26, melkman.cpp:44) */
  CHGPU_INVALID_ARG = 3, /* std::invalid_argument (spa.cpp:112, region_less/sort_region) */
  CHGPU_CUDA_ERR = 4,    /* CUDA runtime failure; see chgpu_last_error */
  CHGPU_NO_DEVICE = 5,   /* no CUDA device: the product never falls back to the CPU */
  CHGPU_TOO_LARGE = 6,   /* n >= 2^32 points in one call (shard the input) */
  CHGPU_IO_ERROR = 7,    /* IoError (io.cpp open_input): unreadable file */
  CHGPU_PARSE_ERROR = 8, /* ParseError (io.cpp:105-106): not whole float64 pairs */
  CHGPU_NONFINITE = 9    /* NonFiniteCoordinate (io.cpp:38-42) */
} chgpu_status;

/* Layout-identical to chainhull::StageStats (pipeline.hpp:30-42). */
typedef struct {
  size_t n_input;
  size_t n_after_round1;
  size_t n_after_spa;
  size_t n_hull;
  double t_extremes_ms;
  double t_classify_ms;
  double t_partition_ms; /* 0: the partition is fused into the classify kernel */
  double t_sort_ms;
  double t_spa_ms;
  double t_melkman_ms;
  double t_total_ms;
} chgpu_stats;

/* Diagnostics of the last chgpu_hull* call (parity taps). */
typedef struct {
  double quad[8];           /* left, bottom, right, top (extremes.hpp:22-27) */
  size_t frame_size;        /* frame_vertices(quad).size() (extremes.cpp:49-57) */
  size_t region_counts[5];  /* Interior, LL, LR, UR, UL after classify */
  size_t kept_counts[4];    /* per-region SPA survivors (0 on the degenerate branch) */
  int degenerate_branch;    /* 1 when pipeline.cpp:53-71 was taken */
  int sort_passes;          /* radix passes actually executed */
  size_t tie_runs;          /* equal-primary runs fixed up after the radix sort */
  int launches;             /* kernels launched by this call */
  int pad_;
  /* Device time per stage from CUDA events on the context stream. */
  double t_h2d_ms;          /* host->device copy of the input (0 for device input) */
  double t_k1_ms;           /* extremes kernels (overlapping the copy for host input) */
  double t_k2_ms;           /* classify + compaction kernel */
  double t_hist_ms;         /* digit histogram + scan */
  double t_passes_ms;       /* all onesweep passes (sort_passes launches) */
  double t_ties_ms;         /* tie-run detect + fix */
  double t_spa_kernel_ms;   /* SPA scan + chain compaction */
  double t_d2h_ms;          /* chains device->host */
  double t_host_ms;         /* host assemble + Melkman */
  /* SPA path: 0 = full region sort, 1 = pre-filtered (k_filter.cu),
   * 2 = pre-filter overflowed (a bin too large) and the full sort ran. */
  int spa_path;
  int filter_log2nb;        /* pre-filter bins per region = 2^filter_log2nb */
  size_t n_candidates;      /* survivors left for the sort by the pre-filter */
  double t_binscan_ms;      /* pre-filter: bin ranks + thresholds */
  double t_filter_ms;       /* pre-filter: candidate selection */
  double t_binsort_ms;      /* pre-filter: sort of bins above 32 candidates */
  int convex_fast_path;     /* 1: Melkman's all-kept trajectory verified on the GPU (k_convex.cu) */
  int k1k2_overlapped;      /* 1: K2 launched programmatically behind K1; t_k1_ms covers both */
  double t_host_enqueue_ms; /* host: call entry until the device work is enqueued */
  double t_host_wait_ms;    /* host: blocked until the counters (and small chains) are back */
} chgpu_diag;

/* Options (chgpu_ctx_set_option). */
enum {
  CHGPU_OPT_SPA_PATH = 1,   /* value: one of the CHGPU_SPA_* below */
  CHGPU_OPT_CHAINS_TAP = 2, /* value 1: keep each hull call's SPA chains for
                               chgpu_last_chains (a parity tap; costs one D2H) */
  CHGPU_OPT_PDL = 3,        /* value 1 (default): K2 launched programmatically behind
                               K1 (overlapped; timed together); 0: separately timed */
  CHGPU_OPT_STAGE_TIMES = 4 /* value 1: per-kernel CUDA events for chgpu_diag's stage
                               times (default 0: only the StageStats intervals; each
                               event query costs ~3 us of host time per call) */
};
enum {
  CHGPU_SPA_AUTO = 0,     /* pre-filter when chunks average >= 16 records (default) */
  CHGPU_SPA_SORT = 1,     /* always sort every survivor (the reference's sort_region) */
  CHGPU_SPA_FILTER = 2,   /* always pre-filter (falls back to the sort on overflow) */
  CHGPU_SPA_FILTER_SORTED = 3  /* pre-filter, every chunk through the bin sorts and the
                                  sorted chunk SPA (the path k_spa_small defers to) */
};

typedef struct chgpu_ctx chgpu_ctx;

/* Context lifecycle. device < 0 selects the current device. */
int chgpu_ctx_create(int device, chgpu_ctx** out);
void chgpu_ctx_destroy(chgpu_ctx* ctx);
const char* chgpu_last_error(const chgpu_ctx* ctx);
/* The CUDA stream the context launches on (a cudaStream_t). */
void* chgpu_ctx_stream(chgpu_ctx* ctx);
/* Per-context option (CHGPU_OPT_*); CHGPU_INVALID_ARG for an unknown
 * option or value. The environment variable CHGPU_SPA=sort|filter sets
 * CHGPU_OPT_SPA_PATH for contexts created afterwards. Results never depend
 * on options: every path returns the reference's hull and counters. */
int chgpu_ctx_set_option(chgpu_ctx* ctx, int option, long long value);
/* Pre-size the workspace for n points (optional; grows on demand). */
int chgpu_reserve(chgpu_ctx* ctx, size_t n);

/* convex_hull (pipeline.hpp:55) over HOST points xy[2n]. On CHGPU_OK
 * *hull_xy points at 2*(*n_hull) doubles owned by ctx, valid until the next
 * call on ctx. Hull is canonical: CCW, starting at the lexicographic
 * minimum, strict (melkman.hpp:10-16). stats/diag may be NULL. */
int chgpu_hull(chgpu_ctx* ctx, const double* xy, size_t n, size_t chunk_count,
               int degenerate_fallback, const double** hull_xy, size_t* n_hull,
               chgpu_stats* stats, chgpu_diag* diag);

/* read_points(path, PointFormat::XyBinary) (io.hpp:29-36) followed by
 * convex_hull, fused: the file's bytes (little-endian float64 pairs, the
 * layout of Point2[]) are read in 32 MB chunks by parallel preads into a
 * pinned ring, each chunk's host->device copy and extremes pass overlapping
 * the next read. Errors in the reference's order: CHGPU_IO_ERROR,
 * CHGPU_PARSE_ERROR (size not a multiple of 16), CHGPU_NONFINITE, then the
 * convex_hull statuses (CHGPU_EMPTY for an empty file). */
int chgpu_hull_xy_binary(chgpu_ctx* ctx, const char* path, size_t chunk_count,
                         int degenerate_fallback, const double** hull_xy, size_t* n_hull,
                         chgpu_stats* stats, chgpu_diag* diag);

/* Same, with xy already resident in device memory (16-byte aligned). */
int chgpu_hull_device(chgpu_ctx* ctx, const double* d_xy, size_t n, size_t chunk_count,
                      int degenerate_fallback, const double** hull_xy, size_t* n_hull,
                      chgpu_stats* stats, chgpu_diag* diag);

/* The SPA chains of the last chgpu_hull* call on ctx (the kept points of
 * spa_filter per region, spa.cpp:109-163, concatenated LL|LR|UR|UL, as
 * the device pipeline produced them), when CHGPU_OPT_CHAINS_TAP is set:
 * *chains_xy (owned by ctx, valid until the next call) and kept_counts[4].
 * CHGPU_INVALID_ARG when the tap is off; all-zero counts on the degenerate
 * branch (it has no chains). */
int chgpu_last_chains(chgpu_ctx* ctx, const double** chains_xy, size_t* kept_counts);

/* ---- stage taps (the reference stage API, used by the C++ shim) -------- */

/* find_extremes (extremes.hpp:32): quad_out = left, bottom, right, top. */
int chgpu_find_extremes(chgpu_ctx* ctx, const double* xy, size_t n, double* quad_out);

/* classify (classify.hpp:55-58): labels[i] in {0..4}; counts[5]. */
int chgpu_classify(chgpu_ctx* ctx, const double* xy, size_t n, const double* quad,
                   uint8_t* labels, size_t* counts);

/* discard_round1 (classify.hpp:64): survivors grouped LL|LR|UR|UL into
 * out_xy (capacity n points), out_labels; counts[5] (Interior = 0). */
int chgpu_discard_round1(chgpu_ctx* ctx, const double* xy, const uint8_t* labels, size_t n,
                         double* out_xy, uint8_t* out_labels, size_t* counts);

/* sort_region (spa.hpp:43) in place on a host segment; region 1..4. */
int chgpu_sort_region(chgpu_ctx* ctx, int region, double* xy, size_t m);

/* spa_filter (spa.hpp:77) over a sorted host segment; anchors = first,
 * last; out capacity m points. */
int chgpu_spa_filter(chgpu_ctx* ctx, int region, const double* xy, size_t m,
                     const double* anchors, size_t chunk_count, double* out, size_t* n_out);

/* ---- host finisher (C++; identical semantics to the reference) --------- */

/* assemble_polygon (polygon.hpp:25): chains = the 4 kept chains
 * concatenated, kept_counts[4]; out capacity sum + 4. */
int chgpu_assemble_polygon(const double* chains, const size_t* kept_counts, const double* quad,
                           double* out, size_t* n_out);
/* melkman (melkman.hpp:29); out capacity n. */
int chgpu_melkman(const double* poly, size_t n, double* out, size_t* n_out);
/* assemble_polygon (polygon.hpp:25) followed by melkman (melkman.hpp:29)
 * in one streaming pass: the hull of the chains' polygon without
 * materialising it. out capacity sum + 4; CHGPU_DEGENERATE where either
 * reference stage throws DegenerateInput. */
int chgpu_finish_chains(const double* chains, const size_t* kept_counts, const double* quad,
                        double* out, size_t* n_out);

/* The hull of the union of several runs of SPA chains against one quad
 * (a run = one shard's 4 region chains concatenated, kept_counts[4 * k +
 * r]): each region's runs merged in region order (region_less, spa.cpp:38-52),
 * then assemble_polygon + melkman as chgpu_finish_chains. The multi-GPU
 * merge of a non-degenerate frame (every hull vertex of the whole set is in
 * some shard's chains). Host only. */
int chgpu_merge_hull(const double* const* runs, const size_t* kept_counts, int nruns,
                     const double* quad, double* out, size_t* n_out);

/* Counters of the split finisher (finisher.cpp finish_chains_split: chains
 * 1-4 run concurrently and are verified before use): calls that took it,
 * and calls whose checks fell back to the sequential pass. Diagnostics. */
void chgpu_finish_split_stats(unsigned long long* taken, unsigned long long* fallback);
/* The last split finisher call's timings in µs from the segments' submit:
 * segment A (calling thread), B, C, D done; all joined; result written.
 * Diagnostics. */
void chgpu_finish_split_times(double* out6);
/* canonicalize_ring (melkman.hpp:20), in place. */
void chgpu_canonicalize_ring(double* ring, size_t n);
/* hull_oracle (pipeline.hpp:62): host reference hull; out capacity n. */
int chgpu_hull_oracle(const double* xy, size_t n, double* out, size_t* n_out);

/* ---- data plumbing ------------------------------------------------------ */

/* generate (datasets.hpp:35): bit-identical to the reference's
 * mt19937_64-based generator. dist follows datasets.hpp:13-21. */
int chgpu_generate(int dist, size_t n, uint64_t seed, double* out_xy);
/* Points [begin, begin + count) of generate(dist, n, seed) into out_xy
 * (2*count doubles): the contiguous shard of one rank of the sharded run,
 * without materialising the whole set (draws before `begin` are discarded;
 * datasets.cpp:17-106 consumes a fixed number per point). */
int chgpu_generate_range(int dist, size_t n, uint64_t seed, size_t begin, size_t count,
                         double* out_xy);

/* Touches every page of [p, p + bytes) from the library's host staging
 * threads, so that a fresh allocation (the C++ API's result vector of a
 * survivor-heavy hull: 320 MB for 20M points) takes its first-touch page
 * faults in parallel instead of inside a single-threaded copy. The bytes'
 * contents are unspecified afterwards (the caller overwrites them). */
void chgpu_host_prefault(void* p, size_t bytes);

/* ---- sharded path (multi-GPU, one rank per GPU) ------------------------- */

/* Local extremes of a device-resident shard with global tie-break indices:
 * quad_out[8], idx_out[4] = base_index + local index of each corner. */
int chgpu_shard_extremes(chgpu_ctx* ctx, const double* d_xy, size_t n, uint64_t base_index,
                         double* quad_out, uint64_t* idx_out);
/* Fold of per-rank candidates in rank order (extremes.cpp:39-46 semantics
 * with lowest global index on ties): quads[8*k], idxs[4*k] -> quad_out. */
void chgpu_fold_extremes(const double* quads, const uint64_t* idxs, size_t k, double* quad_out);
/* Round-1 discard, region sort and SPA of a device-resident shard against
 * a GIVEN (global) quad. Chains (host, owned by ctx until the next call)
 * are the kept points of the 4 regions concatenated; kept_counts[4]. */
int chgpu_shard_chains(chgpu_ctx* ctx, const double* d_xy, size_t n, const double* quad,
                       size_t chunk_count, const double** chains_xy, size_t* kept_counts);
/* Same, with the chains copied into a caller's device buffer of cap_points
 * points (on the context's device; CHGPU_TOO_LARGE if they do not fit): the
 * multi-GPU merge gathers them over NCCL without a host round trip. A shard
 * of n points never has more than n chain points. */
int chgpu_shard_chains_device(chgpu_ctx* ctx, const double* d_xy, size_t n, const double* quad,
                              size_t chunk_count, double* d_chains, size_t cap_points,
                              size_t* kept_counts);

/* convex_hull (pipeline.hpp:55) of the concatenation shard[0], shard[1],
 * ... (global point index = position in that concatenation) with several
 * contexts, one per GPU, in one process: the multi-GPU drop-in for
 * chainhull::convex_hull, and its route for spans of 2^32 points or more.
 * on_device = 0: shards are host memory; shard s runs on ctxs[s % nctx],
 *   in slices of at most 2^30 points (any size: a span too large for one
 *   device is processed slice by slice).
 * on_device = 1: shard s is device memory on ctxs[s]'s device (nshards ==
 *   nctx, each under 2^32 points).
 * Steps: each slice's extreme candidates with global indices,
 * folded in index order into the quad find_extremes returns for the whole
 * set; per slice the round-1 discard, region sort and SPA against that
 * quad; the chains copied to ctxs[0]'s device (cudaMemcpyPeerAsync, NVLink
 * between GPUs) with the frame; the single-GPU pipeline over that union.
 * The hull equals the reference's for the whole set bit for bit; stats
 * n_input and n_hull are the whole set's, the other counters the merge's
 * (not comparable with a single-device run). The hull is owned by ctxs[0]
 * until its next call. Contexts on the same device are allowed. */
/* CUDA devices visible to this process (0 without a GPU). */
int chgpu_device_count(void);
int chgpu_hull_sharded(chgpu_ctx* const* ctxs, int nctx, const double* const* shards,
                       const size_t* counts, int nshards, int on_device, size_t chunk_count,
                       int degenerate_fallback, const double** hull_xy, size_t* n_hull,
                       chgpu_stats* stats);

#ifdef __cplusplus
}
#endif

#endif /* CHGPU_H */
