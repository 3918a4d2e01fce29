// The chainhull public API, re-declared for the B200 drop-in library
// (libchainhull.so). Every name, type and signature matches the reference
// headers (/root/reference/proj/core/include/chainhull/*.hpp) so code
// written against the reference — including the reference's own
// tests/acceptance.cpp — compiles and links unchanged. The preprocessing
// stages run on the GPU through include/chgpu.h; the reference-named
// headers next to this one all include it.
#pragma once

#include <array>
#include <cstddef>
#include <cstdint>
#include <filesystem>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

namespace chainhull {

// ---- geometry (ref geometry.hpp:8-44) ------------------------------------

struct Point2 {
  double x = 0.0;
  double y = 0.0;
  friend constexpr bool operator==(Point2 a, Point2 b) { return a.x == b.x && a.y == b.y; }
};

enum class Orientation { Left, Right, Collinear };

// (b - a) x (p - a), each operation rounded separately.
constexpr double cross(Point2 a, Point2 b, Point2 p) {
  return (b.x - a.x) * (p.y - a.y) - (b.y - a.y) * (p.x - a.x);
}
constexpr Orientation orient(Point2 a, Point2 b, Point2 p) {
  const double c = cross(a, b, p);
  return c > 0.0 ? Orientation::Left : (c < 0.0 ? Orientation::Right : Orientation::Collinear);
}
constexpr bool less_xy(Point2 a, Point2 b) { return a.x < b.x || (a.x == b.x && a.y < b.y); }
constexpr bool less_yx(Point2 a, Point2 b) { return a.y < b.y || (a.y == b.y && a.x < b.x); }

// ---- errors (ref errors.hpp:10-44) ----------------------------------------

struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct EmptyInput : Error {
  using Error::Error;
};
struct DegenerateInput : Error {
  using Error::Error;
};
struct ParseError : Error {
  ParseError(std::size_t line_number, const std::string& reason);
  std::size_t line;
};
struct NonFiniteCoordinate : Error {
  using Error::Error;
};
struct IoError : Error {
  using Error::Error;
};

// ---- extreme quad (ref extremes.hpp:22-37) ----------------------------------

struct ExtremeQuad {
  Point2 left;
  Point2 bottom;
  Point2 right;
  Point2 top;
};

ExtremeQuad find_extremes(std::span<const Point2> points, std::size_t workers = 1);
std::vector<Point2> frame_vertices(const ExtremeQuad& quad);

// ---- classification and round-one discard (ref classify.hpp:18-64) --------

enum class Region : std::uint8_t {
  Interior = 0,
  LowerLeft = 1,
  LowerRight = 2,
  UpperRight = 3,
  UpperLeft = 4,
};
inline constexpr std::size_t kRegionCount = 5;

struct LabeledPoints {
  std::vector<Point2> points;
  std::vector<Region> labels;
  std::array<std::size_t, kRegionCount> region_counts{};
};

// First CCW quad edge the point lies strictly right of; else Interior.
inline Region classify_point(Point2 p, const ExtremeQuad& q) {
  const Point2 ring[5] = {q.left, q.bottom, q.right, q.top, q.left};
  for (int e = 0; e < 4; ++e)
    if (orient(ring[e], ring[e + 1], p) == Orientation::Right) return static_cast<Region>(e + 1);
  return Region::Interior;
}

LabeledPoints classify(std::vector<Point2> points, const ExtremeQuad& quad, std::size_t workers = 1);
LabeledPoints classify(std::span<const Point2> points, const ExtremeQuad& quad,
                       std::size_t workers = 1);
LabeledPoints discard_round1(LabeledPoints labeled);

// ---- sort and SPA (ref spa.hpp:14-81) ---------------------------------------

struct RegionSegment {
  Region region = Region::Interior;
  std::span<Point2> points;
};
struct RegionAnchors {
  Point2 first;
  Point2 last;
};
RegionAnchors region_anchors(const ExtremeQuad& quad, Region region);
std::array<RegionSegment, 4> region_segments(LabeledPoints& labeled);
void sort_region(RegionSegment segment);
bool region_less(Region region, Point2 a, Point2 b);

struct SpaConfig {
  std::size_t chunk_count = 1024;
};
struct RegionChain {
  Region region = Region::Interior;
  std::vector<Point2> kept;
};
RegionChain spa_filter(std::span<const Point2> segment, Region region, const RegionAnchors& anchors,
                       const SpaConfig& config = {}, std::size_t workers = 1);
RegionChain spa_filter(const RegionSegment& segment, const RegionAnchors& anchors,
                       const SpaConfig& config = {}, std::size_t workers = 1);

// ---- polygon and Melkman (ref polygon.hpp:13-26, melkman.hpp:10-29) -------

struct SimplePolygon {
  std::vector<Point2> vertices;
};
SimplePolygon assemble_polygon(const std::array<RegionChain, 4>& chains, const ExtremeQuad& quad);

struct Hull {
  std::vector<Point2> vertices;
};
void canonicalize_ring(std::vector<Point2>& ring);
Hull melkman(const SimplePolygon& polygon);

// ---- pipeline (ref pipeline.hpp:10-62) ----------------------------------------

struct PipelineConfig {
  std::size_t chunk_count = 1024;
  std::size_t parallelism = 0;  // accepted for compatibility; the GPU grid replaces it
  bool degenerate_fallback = true;
};

struct StageStats {
  std::size_t n_input = 0;
  std::size_t n_after_round1 = 0;
  std::size_t n_after_spa = 0;
  std::size_t n_hull = 0;
  double t_extremes_ms = 0.0;
  double t_classify_ms = 0.0;
  double t_partition_ms = 0.0;
  double t_sort_ms = 0.0;
  double t_spa_ms = 0.0;
  double t_melkman_ms = 0.0;
  double t_total_ms = 0.0;
};

struct HullResult {
  Hull hull;
  StageStats stats;
};

HullResult convex_hull(std::span<const Point2> points, const PipelineConfig& config = {});
Hull hull_oracle(std::span<const Point2> points);

// ---- datasets (ref datasets.hpp:13-40) ----------------------------------------

enum class Distribution { UniformSquare, UniformDisk, Circle, Gaussian, Collinear, DuplicatesHeavy };

struct DatasetSpec {
  Distribution distribution = Distribution::UniformSquare;
  std::size_t n = 0;
  std::uint64_t seed = 0;
};

std::vector<Point2> generate(const DatasetSpec& spec);
const char* distribution_name(Distribution distribution);
Distribution parse_distribution(const std::string& name);

// ---- point / stats files (ref io.hpp:14-52) --------------------------------------

enum class PointFormat { XyText, XyBinary, ObjVertices };
enum class StatsFormat { Csv, Json };

const char* point_format_name(PointFormat format);
PointFormat parse_point_format(const std::string& name);
StatsFormat parse_stats_format(const std::string& name);
std::vector<Point2> read_points(const std::filesystem::path& path, PointFormat format);
void write_points(std::span<const Point2> points, const std::filesystem::path& path,
                  PointFormat format);
void write_hull(const Hull& hull, const std::filesystem::path& path);
void write_stats(const StageStats& stats, const std::filesystem::path& path, StatsFormat format);

}  // namespace chainhull
