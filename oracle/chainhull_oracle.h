/* TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.
 *
 * Plain-C restatement of the reference chainhull CPU pipeline
 * (/root/reference/proj/core). Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load liboracle.so, and only as the
 * checker. Parity is pinned: tests/test_oracle.py checks every function
 * here against the reference's own known-answer tests (transcribed from
 * /root/reference/proj/tests/*_test.cpp) and against tests/golden/, which
 * oracle/make_golden.py produced by running the unmodified reference
 * (oracle/_ref/libchainhull_ref.so).
 *
 * Points are {double x, y} pairs, the same bytes as chainhull::Point2.
 * Status codes: 0 ok, 1 EmptyInput, 2 DegenerateInput, 3 invalid_argument.
 */
#ifndef CHAINHULL_ORACLE_H
#define CHAINHULL_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  double x, y;
} orc_pt;

/* datasets.hpp:13-21 order: 0 uniform_square, 1 uniform_disk, 2 circle,
 * 3 gaussian, 4 collinear, 5 duplicates_heavy. */
int orc_generate(int dist, size_t n, uint64_t seed, orc_pt* out);

int orc_find_extremes(const orc_pt* p, size_t n, orc_pt quad[4]);
size_t orc_frame_vertices(const orc_pt quad[4], orc_pt out[4]);
int orc_classify_point(orc_pt p, const orc_pt quad[4]);
void orc_classify_points(const orc_pt* p, size_t n, const orc_pt quad[4], uint8_t* labels);
int orc_sort_region(int region, orc_pt* seg, size_t m);
int orc_spa_filter(int region, const orc_pt* seg, size_t m, const orc_pt anchors[2],
                   size_t chunk_count, orc_pt* out, size_t* nout);
/* chains: kept points of the 4 regions concatenated, kept_counts[4]. */
int orc_assemble_polygon(const orc_pt* chains, const size_t kept_counts[4],
                         const orc_pt quad[4], orc_pt* out, size_t* nout);
int orc_melkman(const orc_pt* poly, size_t n, orc_pt* out, size_t* nout);
int orc_hull_oracle(const orc_pt* p, size_t n, orc_pt* out, size_t* nout);

/* pipeline.cpp:25-106. counts = {n_input, n_after_round1, n_after_spa,
 * n_hull}; region_counts[5] after classify; kept_counts[4] after SPA
 * (zeros on the degenerate branch). out_hull needs capacity n. */
int orc_convex_hull(const orc_pt* p, size_t n, size_t chunk_count, int degenerate_fallback,
                    orc_pt* out_hull, size_t* nhull, size_t counts[4],
                    size_t region_counts[5], size_t kept_counts[4]);

#ifdef __cplusplus
}
#endif

#endif
