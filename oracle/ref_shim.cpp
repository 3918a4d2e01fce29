// TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.
//
// extern "C" shim over the UNMODIFIED reference chainhull sources
// (/root/reference/proj/core/src/*.cpp, compiled in place by oracle/Makefile
// into oracle/_ref/libchainhull_ref.so). Only tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline / --impl reference legs may load it. It exists
// so that the restated oracle (oracle/chainhull_oracle.c) and the golden
// fixtures (tests/golden/) are pinned to the reference's own outputs.
//
// Status codes mirror include/chgpu.h: 0 ok, 1 EmptyInput, 2 DegenerateInput,
// 3 std::invalid_argument, 9 any other exception.

#include <cstddef>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <vector>

#include "chainhull/chainhull.hpp"

using namespace chainhull;

namespace {

int status_of_current_exception() {
  try {
    throw;
  } catch (const EmptyInput&) {
    return 1;
  } catch (const DegenerateInput&) {
    return 2;
  } catch (const std::invalid_argument&) {
    return 3;
  } catch (...) {
    return 9;
  }
}

std::span<const Point2> as_points(const double* xy, std::size_t n) {
  return {reinterpret_cast<const Point2*>(xy), n};
}

void put_points(const std::vector<Point2>& pts, double* out) {
  if (!pts.empty()) std::memcpy(out, pts.data(), pts.size() * sizeof(Point2));
}

}  // namespace

extern "C" {

// datasets.hpp:35 generate(); dist uses the Distribution enum order
// (datasets.hpp:13-21).
int ref_generate(int dist, std::size_t n, std::uint64_t seed, double* out_xy) {
  try {
    const auto pts = generate({static_cast<Distribution>(dist), n, seed});
    put_points(pts, out_xy);
    return 0;
  } catch (...) {
    return status_of_current_exception();
  }
}

// pipeline.hpp:55 convex_hull(). counts = {n_input, n_after_round1,
// n_after_spa, n_hull}; ms = the seven StageStats timers.
int ref_convex_hull(const double* xy, std::size_t n, std::size_t chunk_count,
                    std::size_t parallelism, int degenerate_fallback, double* out_hull,
                    std::size_t* out_nhull, std::size_t* counts, double* ms) {
  try {
    PipelineConfig cfg;
    cfg.chunk_count = chunk_count;
    cfg.parallelism = parallelism;
    cfg.degenerate_fallback = degenerate_fallback != 0;
    const HullResult r = convex_hull(as_points(xy, n), cfg);
    put_points(r.hull.vertices, out_hull);
    *out_nhull = r.hull.vertices.size();
    if (counts) {
      counts[0] = r.stats.n_input;
      counts[1] = r.stats.n_after_round1;
      counts[2] = r.stats.n_after_spa;
      counts[3] = r.stats.n_hull;
    }
    if (ms) {
      ms[0] = r.stats.t_extremes_ms;
      ms[1] = r.stats.t_classify_ms;
      ms[2] = r.stats.t_partition_ms;
      ms[3] = r.stats.t_sort_ms;
      ms[4] = r.stats.t_spa_ms;
      ms[5] = r.stats.t_melkman_ms;
      ms[6] = r.stats.t_total_ms;
    }
    return 0;
  } catch (...) {
    return status_of_current_exception();
  }
}

// pipeline.hpp:62 hull_oracle().
int ref_hull_oracle(const double* xy, std::size_t n, double* out_hull,
                    std::size_t* out_nhull) {
  try {
    const Hull h = hull_oracle(as_points(xy, n));
    put_points(h.vertices, out_hull);
    *out_nhull = h.vertices.size();
    return 0;
  } catch (...) {
    return status_of_current_exception();
  }
}

// extremes.hpp:32 find_extremes(); quad = {left, bottom, right, top}.
int ref_find_extremes(const double* xy, std::size_t n, std::size_t workers, double* quad) {
  try {
    const ExtremeQuad q = find_extremes(as_points(xy, n), workers);
    const Point2 c[4] = {q.left, q.bottom, q.right, q.top};
    std::memcpy(quad, c, sizeof c);
    return 0;
  } catch (...) {
    return status_of_current_exception();
  }
}

// classify.hpp:42 classify_point() over a batch (labels only).
int ref_classify_points(const double* xy, std::size_t n, const double* quad,
                        std::uint8_t* labels) {
  ExtremeQuad q;
  std::memcpy(&q, quad, sizeof q);
  const Point2* p = reinterpret_cast<const Point2*>(xy);
  for (std::size_t i = 0; i < n; ++i) labels[i] = static_cast<std::uint8_t>(classify_point(p[i], q));
  return 0;
}

// Stage dump of the non-degenerate pipeline branch (pipeline.cpp:36-96):
// find_extremes -> classify -> discard_round1 -> sort_region x4 ->
// spa_filter x4. Writes region_counts[5] (after classify), the sorted
// segments concatenated in block order into sorted_out (capacity n), and
// the kept chains concatenated into kept_out with kept_counts[4].
int ref_stage_dump(const double* xy, std::size_t n, std::size_t chunk_count, double* quad_out,
                   std::size_t* region_counts, double* sorted_out, double* kept_out,
                   std::size_t* kept_counts) {
  try {
    const auto pts = as_points(xy, n);
    const ExtremeQuad quad = find_extremes(pts);
    std::memcpy(quad_out, &quad, sizeof quad);
    LabeledPoints labeled = classify(pts, quad);
    for (std::size_t r = 0; r < kRegionCount; ++r) region_counts[r] = labeled.region_counts[r];
    labeled = discard_round1(std::move(labeled));
    auto segments = region_segments(labeled);
    for (auto& s : segments) sort_region(s);
    put_points(labeled.points, sorted_out);
    std::size_t off = 0;
    for (std::size_t s = 0; s < 4; ++s) {
      const RegionChain c =
          spa_filter(segments[s], region_anchors(quad, segments[s].region), SpaConfig{chunk_count});
      if (!c.kept.empty()) std::memcpy(kept_out + 2 * off, c.kept.data(), c.kept.size() * 16);
      kept_counts[s] = c.kept.size();
      off += c.kept.size();
    }
    return 0;
  } catch (...) {
    return status_of_current_exception();
  }
}

// spa.hpp:43 sort_region() on a caller-owned segment (region 1..4).
int ref_sort_region(int region, double* xy, std::size_t m) {
  try {
    sort_region(RegionSegment{static_cast<Region>(region),
                              std::span<Point2>(reinterpret_cast<Point2*>(xy), m)});
    return 0;
  } catch (...) {
    return status_of_current_exception();
  }
}

// spa.hpp:77 spa_filter(); anchors = {first, last}.
int ref_spa_filter(int region, const double* xy, std::size_t m, const double* anchors,
                   std::size_t chunk_count, double* out, std::size_t* nout) {
  try {
    RegionAnchors a;
    std::memcpy(&a, anchors, sizeof a);
    const RegionChain c =
        spa_filter(as_points(xy, m), static_cast<Region>(region), a, SpaConfig{chunk_count});
    put_points(c.kept, out);
    *nout = c.kept.size();
    return 0;
  } catch (...) {
    return status_of_current_exception();
  }
}

// melkman.hpp:29 melkman() of a simple polygon.
int ref_melkman(const double* xy, std::size_t n, double* out, std::size_t* nout) {
  try {
    const Hull h = melkman(SimplePolygon{std::vector<Point2>(
        reinterpret_cast<const Point2*>(xy), reinterpret_cast<const Point2*>(xy) + n)});
    put_points(h.vertices, out);
    *nout = h.vertices.size();
    return 0;
  } catch (...) {
    return status_of_current_exception();
  }
}

}  // extern "C"
