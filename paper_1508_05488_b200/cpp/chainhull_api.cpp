// libchainhull.so: the reference chainhull C++ API (include/chainhull/api.hpp)
// implemented over the C ABI in include/chgpu.h.
//
// convex_hull and the GPU-backed stage functions borrow a context from a
// process-wide pool (the reference API has no handles and promises
// reentrancy, pipeline.hpp:53): concurrent calls each get their own
// context, hence their own stream and workspace. If no CUDA device is
// present every GPU-backed call throws chainhull::Error — there is no CPU
// fallback for the preprocessing path. Status codes are mapped back to the
// reference's exception types on the same branches (include/chgpu.h).

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "chainhull/api.hpp"
#include "chgpu.h"
#include "chainhull_capi.h"

namespace chainhull {

ParseError::ParseError(std::size_t line_number, const std::string& reason)
    : Error(line_number > 0 ? "parse error at line " + std::to_string(line_number) + ": " + reason
                            : "parse error: " + reason),
      line(line_number) {}

namespace {

static_assert(sizeof(Point2) == 16, "Point2 must be two packed doubles");
static_assert(sizeof(StageStats) == sizeof(chgpu_stats), "StageStats layout");

// One pool per device (-1: the calling thread's current device).
class ContextPool {
 public:
  explicit ContextPool(int device = -1) : device_(device) {}
  ~ContextPool() {
    for (chgpu_ctx* c : free_) chgpu_ctx_destroy(c);
  }
  chgpu_ctx* acquire() {
    {
      std::lock_guard<std::mutex> lock(mu_);
      if (!free_.empty()) {
        chgpu_ctx* c = free_.back();
        free_.pop_back();
        return c;
      }
    }
    chgpu_ctx* c = nullptr;
    const int st = chgpu_ctx_create(device_, &c);
    if (st != CHGPU_OK || !c)
      throw Error(st == CHGPU_NO_DEVICE ? "chainhull: no CUDA device (the GPU path has no CPU fallback)"
                                        : "chainhull: CUDA context creation failed");
    return c;
  }
  void release(chgpu_ctx* c) {
    std::lock_guard<std::mutex> lock(mu_);
    free_.push_back(c);
  }

 private:
  int device_;
  std::mutex mu_;
  std::vector<chgpu_ctx*> free_;
};

ContextPool& pool(int device = -1) {
  static std::mutex mu;
  static std::vector<std::unique_ptr<ContextPool>> per_device;  // [device + 1]
  std::lock_guard<std::mutex> lock(mu);
  const size_t i = (size_t)(device + 1);
  if (per_device.size() <= i) per_device.resize(i + 1);
  if (!per_device[i]) per_device[i] = std::make_unique<ContextPool>(device);
  return *per_device[i];
}

struct Lease {
  int device;
  chgpu_ctx* ctx;
  explicit Lease(int dev = -1) : device(dev), ctx(pool(dev).acquire()) {}
  ~Lease() { pool(device).release(ctx); }
  Lease(const Lease&) = delete;
  Lease& operator=(const Lease&) = delete;
};

// Shards of convex_hull for a span of 2^32 points or more (beyond one call
// of the single-device path), or CHAINHULL_SHARDS=k (k > 1) to force k
// shards: one per visible device, round robin.
std::size_t forced_shards() {
  const char* e = std::getenv("CHAINHULL_SHARDS");
  return e ? (std::size_t)std::strtoull(e, nullptr, 10) : 0;
}

[[noreturn]] void raise(int status, const std::string& msg) {
  switch (status) {
    case CHGPU_EMPTY: throw EmptyInput(msg);
    case CHGPU_DEGENERATE: throw DegenerateInput(msg);
    case CHGPU_INVALID_ARG: throw std::invalid_argument(msg);
    default: throw Error("chainhull (GPU): " + msg);
  }
}

void check(int status, chgpu_ctx* ctx) {
  if (status != CHGPU_OK) raise(status, ctx ? chgpu_last_error(ctx) : "error");
}

const double* raw(std::span<const Point2> p) { return reinterpret_cast<const double*>(p.data()); }
double* raw(Point2* p) { return reinterpret_cast<double*>(p); }

std::array<double, 8> quad_array(const ExtremeQuad& q) {
  return {q.left.x, q.left.y, q.bottom.x, q.bottom.y, q.right.x, q.right.y, q.top.x, q.top.y};
}

}  // namespace

// ---------------------------------------------------------------- pipeline

HullResult convex_hull(std::span<const Point2> points, const PipelineConfig& config) {
  if (points.empty()) throw EmptyInput("convex_hull: no points");
  const double* hull_xy = nullptr;
  std::size_t n_hull = 0;
  chgpu_stats st{};
  const std::size_t n = points.size();
  const std::size_t forced = forced_shards();
  std::unique_ptr<Lease> lease;
  std::vector<std::unique_ptr<Lease>> leases;
  if (n >= (std::size_t(1) << 32) || forced > 1) {
    // several GPUs (or slices of one): chgpu_hull_sharded over contiguous
    // host shards, one context per device
    const int ndev = std::max(1, chgpu_device_count());
    const std::size_t k = std::max<std::size_t>(forced > 1 ? forced : (std::size_t)ndev, 1);
    std::vector<chgpu_ctx*> ctxs;
    for (int d = 0; d < (int)std::min<std::size_t>(k, (std::size_t)ndev); ++d) {
      leases.push_back(std::make_unique<Lease>(d));
      ctxs.push_back(leases.back()->ctx);
    }
    std::vector<const double*> shards;
    std::vector<std::size_t> counts;
    for (std::size_t s = 0; s < k; ++s) {
      const std::size_t b = n * s / k, e = n * (s + 1) / k;
      shards.push_back(raw(points) + 2 * b);
      counts.push_back(e - b);
    }
    check(chgpu_hull_sharded(ctxs.data(), (int)ctxs.size(), shards.data(), counts.data(), (int)k, 0,
                             config.chunk_count, config.degenerate_fallback ? 1 : 0, &hull_xy,
                             &n_hull, &st),
          ctxs[0]);
  } else {
    lease = std::make_unique<Lease>();
    check(chgpu_hull(lease->ctx, raw(points), n, config.chunk_count,
                     config.degenerate_fallback ? 1 : 0, &hull_xy, &n_hull, &st, nullptr),
          lease->ctx);
  }
  HullResult r;
  const Point2* h = reinterpret_cast<const Point2*>(hull_xy);
  if (n_hull >= (std::size_t(1) << 16)) {
    // a survivor-heavy hull: take the fresh vector's page faults on the
    // library's threads first (one thread faulting 320 MB in the copy
    // costs ~140 ms on the B200 host; prefaulted, the copy is ~25 ms)
    r.hull.vertices.reserve(n_hull);
    chgpu_host_prefault(r.hull.vertices.data(), n_hull * sizeof(Point2));
  }
  r.hull.vertices.assign(h, h + n_hull);
  r.stats = StageStats{st.n_input,       st.n_after_round1, st.n_after_spa,    st.n_hull,
                       st.t_extremes_ms, st.t_classify_ms,  st.t_partition_ms, st.t_sort_ms,
                       st.t_spa_ms,      st.t_melkman_ms,   st.t_total_ms};
  return r;
}

Hull hull_oracle(std::span<const Point2> points) {
  if (points.empty()) throw EmptyInput("hull_oracle: no points");
  Hull h;
  h.vertices.resize(points.size());
  std::size_t k = 0;
  const int st = chgpu_hull_oracle(raw(points), points.size(), raw(h.vertices.data()), &k);
  if (st) raise(st, "hull_oracle");
  h.vertices.resize(k);
  return h;
}

// ---------------------------------------------------------------- stages

ExtremeQuad find_extremes(std::span<const Point2> points, std::size_t /*workers*/) {
  if (points.empty()) throw EmptyInput("find_extremes: no points");
  Lease lease;
  double q[8];
  check(chgpu_find_extremes(lease.ctx, raw(points), points.size(), q), lease.ctx);
  return ExtremeQuad{{q[0], q[1]}, {q[2], q[3]}, {q[4], q[5]}, {q[6], q[7]}};
}

std::vector<Point2> frame_vertices(const ExtremeQuad& quad) {
  std::vector<Point2> ring;
  for (const Point2& p : {quad.left, quad.bottom, quad.right, quad.top})
    if (ring.empty() || !(ring.back() == p)) ring.push_back(p);
  if (ring.size() > 1 && ring.front() == ring.back()) ring.pop_back();
  return ring;
}

LabeledPoints classify(std::vector<Point2> points, const ExtremeQuad& quad, std::size_t) {
  LabeledPoints out;
  out.points = std::move(points);
  out.labels.resize(out.points.size());
  if (out.points.empty()) return out;
  Lease lease;
  const auto q = quad_array(quad);
  std::size_t counts[5];
  check(chgpu_classify(lease.ctx, raw(out.points.data()), out.points.size(), q.data(),
                       reinterpret_cast<std::uint8_t*>(out.labels.data()), counts),
        lease.ctx);
  for (std::size_t r = 0; r < kRegionCount; ++r) out.region_counts[r] = counts[r];
  return out;
}

LabeledPoints classify(std::span<const Point2> points, const ExtremeQuad& quad, std::size_t workers) {
  return classify(std::vector<Point2>(points.begin(), points.end()), quad, workers);
}

LabeledPoints discard_round1(LabeledPoints labeled) {
  LabeledPoints out;
  const std::size_t n = labeled.points.size();
  if (n == 0) return out;
  Lease lease;
  out.points.resize(n);
  out.labels.resize(n);
  std::size_t counts[5];
  check(chgpu_discard_round1(lease.ctx, raw(labeled.points.data()),
                             reinterpret_cast<const std::uint8_t*>(labeled.labels.data()), n,
                             raw(out.points.data()), reinterpret_cast<std::uint8_t*>(out.labels.data()),
                             counts),
        lease.ctx);
  const std::size_t s1 = counts[1] + counts[2] + counts[3] + counts[4];
  out.points.resize(s1);
  out.labels.resize(s1);
  for (std::size_t r = 0; r < kRegionCount; ++r) out.region_counts[r] = counts[r];
  return out;
}

RegionAnchors region_anchors(const ExtremeQuad& quad, Region region) {
  switch (region) {
    case Region::LowerLeft: return {quad.left, quad.bottom};
    case Region::LowerRight: return {quad.bottom, quad.right};
    case Region::UpperRight: return {quad.right, quad.top};
    case Region::UpperLeft: return {quad.top, quad.left};
    default: break;
  }
  throw std::invalid_argument("region_anchors: interior has no anchors");
}

std::array<RegionSegment, 4> region_segments(LabeledPoints& labeled) {
  std::array<RegionSegment, 4> segs;
  std::size_t off = 0;
  for (std::size_t r = 1; r <= 4; ++r) {
    const std::size_t m = labeled.region_counts[r];
    segs[r - 1] = RegionSegment{static_cast<Region>(r), std::span<Point2>(labeled.points).subspan(off, m)};
    off += m;
  }
  return segs;
}

bool region_less(Region region, Point2 a, Point2 b) {
  switch (region) {
    case Region::LowerLeft: return a.x < b.x || (a.x == b.x && a.y > b.y);
    case Region::LowerRight: return a.y < b.y || (a.y == b.y && a.x < b.x);
    case Region::UpperRight: return a.x > b.x || (a.x == b.x && a.y < b.y);
    case Region::UpperLeft: return a.y > b.y || (a.y == b.y && a.x > b.x);
    default: break;
  }
  throw std::invalid_argument("region_less: interior segments are never sorted");
}

void sort_region(RegionSegment segment) {
  if (segment.region == Region::Interior)
    throw std::invalid_argument("sort_region: interior segments are never sorted");
  if (segment.points.size() <= 1) return;
  Lease lease;
  check(chgpu_sort_region(lease.ctx, static_cast<int>(segment.region), raw(segment.points.data()),
                          segment.points.size()),
        lease.ctx);
}

RegionChain spa_filter(std::span<const Point2> segment, Region region, const RegionAnchors& anchors,
                       const SpaConfig& config, std::size_t) {
  if (config.chunk_count == 0) throw std::invalid_argument("spa_filter: chunk_count must be >= 1");
  RegionChain chain;
  chain.region = region;
  if (segment.empty()) return chain;
  Lease lease;
  const double a[4] = {anchors.first.x, anchors.first.y, anchors.last.x, anchors.last.y};
  chain.kept.resize(segment.size());
  std::size_t k = 0;
  check(chgpu_spa_filter(lease.ctx, static_cast<int>(region), raw(segment), segment.size(), a,
                         config.chunk_count, raw(chain.kept.data()), &k),
        lease.ctx);
  chain.kept.resize(k);
  return chain;
}

RegionChain spa_filter(const RegionSegment& segment, const RegionAnchors& anchors,
                       const SpaConfig& config, std::size_t workers) {
  return spa_filter(std::span<const Point2>(segment.points.data(), segment.points.size()),
                    segment.region, anchors, config, workers);
}

SimplePolygon assemble_polygon(const std::array<RegionChain, 4>& chains, const ExtremeQuad& quad) {
  std::vector<Point2> all;
  std::size_t counts[4];
  for (int r = 0; r < 4; ++r) {
    counts[r] = chains[r].kept.size();
    all.insert(all.end(), chains[r].kept.begin(), chains[r].kept.end());
  }
  SimplePolygon poly;
  poly.vertices.resize(all.size() + 4);
  std::size_t k = 0;
  const auto q = quad_array(quad);
  const int st = chgpu_assemble_polygon(raw(all.data()), counts, q.data(), raw(poly.vertices.data()), &k);
  if (st) raise(st, "assemble_polygon: fewer than 3 distinct vertices");
  poly.vertices.resize(k);
  return poly;
}

void canonicalize_ring(std::vector<Point2>& ring) { chgpu_canonicalize_ring(raw(ring.data()), ring.size()); }

Hull melkman(const SimplePolygon& polygon) {
  Hull h;
  h.vertices.resize(polygon.vertices.size());
  std::size_t k = 0;
  const int st = chgpu_melkman(reinterpret_cast<const double*>(polygon.vertices.data()),
                               polygon.vertices.size(), raw(h.vertices.data()), &k);
  if (st) raise(st, "melkman: fewer than 3 distinct vertices or all collinear");
  h.vertices.resize(k);
  return h;
}

// ---------------------------------------------------------------- datasets

std::vector<Point2> generate(const DatasetSpec& spec) {
  if (spec.n == 0) throw std::invalid_argument("generate: n must be positive");
  std::vector<Point2> pts(spec.n);
  if (chgpu_generate(static_cast<int>(spec.distribution), spec.n, spec.seed, raw(pts.data())))
    throw std::invalid_argument("generate: unknown distribution");
  return pts;
}

namespace {
constexpr const char* kDistNames[] = {"uniform_square", "uniform_disk", "circle",
                                      "gaussian",       "collinear",    "duplicates_heavy"};
}

const char* distribution_name(Distribution d) {
  const int i = static_cast<int>(d);
  if (i < 0 || i > 5) throw std::invalid_argument("distribution_name: unknown distribution");
  return kDistNames[i];
}

Distribution parse_distribution(const std::string& name) {
  for (int i = 0; i < 6; ++i)
    if (name == kDistNames[i]) return static_cast<Distribution>(i);
  throw std::invalid_argument("parse_distribution: unknown distribution '" + name + "'");
}

}  // namespace chainhull

// ---------------------------------------------------------------- C entry (include/chainhull_capi.h)

extern "C" int chainhull_capi_convex_hull(const double* xy, std::size_t n, std::size_t chunk_count,
                                          std::size_t parallelism, int degenerate_fallback,
                                          double* hull_out, std::size_t hull_cap,
                                          std::size_t* n_hull, std::size_t* counts) {
  try {
    chainhull::PipelineConfig cfg;
    cfg.chunk_count = chunk_count;
    cfg.parallelism = parallelism;
    cfg.degenerate_fallback = degenerate_fallback != 0;
    const chainhull::HullResult r = chainhull::convex_hull(
        std::span<const chainhull::Point2>(reinterpret_cast<const chainhull::Point2*>(xy), n), cfg);
    const std::size_t k = r.hull.vertices.size();
    *n_hull = k;
    if (hull_out) {
      if (k > hull_cap) return CHGPU_TOO_LARGE;
      std::memcpy(hull_out, r.hull.vertices.data(), k * sizeof(chainhull::Point2));
    }
    if (counts) {
      counts[0] = r.stats.n_input;
      counts[1] = r.stats.n_after_round1;
      counts[2] = r.stats.n_after_spa;
      counts[3] = r.stats.n_hull;
    }
    return CHGPU_OK;
  } catch (const chainhull::EmptyInput&) {
    return CHGPU_EMPTY;
  } catch (const chainhull::DegenerateInput&) {
    return CHGPU_DEGENERATE;
  } catch (const std::invalid_argument&) {
    return CHGPU_INVALID_ARG;
  } catch (...) {
    return CHGPU_CUDA_ERR;
  }
}
