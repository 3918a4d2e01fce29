// Point and stats files for the drop-in API (reference io.hpp:14-52).
// xy_binary is exactly the device layout (16-byte little-endian double
// pairs), so a file read lands in memory ready for chgpu_hull.
// Text output uses 17 significant digits (exact double round trip).

#include <bit>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <fstream>
#include <sstream>
#include <string_view>

#include "chainhull/api.hpp"

namespace chainhull {

namespace {

std::string_view strip(std::string_view s) {
  while (!s.empty() && (s.front() == ' ' || s.front() == '\t')) s.remove_prefix(1);
  while (!s.empty() && (s.back() == ' ' || s.back() == '\t' || s.back() == '\r')) s.remove_suffix(1);
  return s;
}

bool next_number(std::string_view& s, double& v) {
  while (!s.empty() && (s.front() == ' ' || s.front() == '\t')) s.remove_prefix(1);
  const auto res = std::from_chars(s.data(), s.data() + s.size(), v);
  if (res.ec != std::errc{}) return false;
  s.remove_prefix(static_cast<std::size_t>(res.ptr - s.data()));
  return true;
}

void finite_or_throw(const Point2& p, std::size_t line) {
  if (std::isfinite(p.x) && std::isfinite(p.y)) return;
  throw NonFiniteCoordinate(line ? "non-finite coordinate at line " + std::to_string(line)
                                 : std::string("non-finite coordinate"));
}

std::string fmt17(double v) {
  char buf[64];
  auto r = std::to_chars(buf, buf + sizeof buf, v, std::chars_format::general, 17);
  return std::string(buf, r.ptr);
}

// Shortest round-trip form with a trailing ".0" on integral values (the
// JSON number style of the reference's stats writer).
std::string json_double(double v) {
  char buf[64];
  auto r = std::to_chars(buf, buf + sizeof buf, v);
  std::string s(buf, r.ptr);
  if (s.find_first_of(".eE") == std::string::npos && s.find("inf") == std::string::npos &&
      s.find("nan") == std::string::npos)
    s += ".0";
  return s;
}

std::ifstream open_in(const std::filesystem::path& p, bool bin) {
  std::ifstream in(p, bin ? std::ios::binary : std::ios::in);
  if (!in) throw IoError("cannot open '" + p.string() + "' for reading");
  return in;
}

std::ofstream open_out(const std::filesystem::path& p, bool bin) {
  std::ofstream out(p, bin ? std::ios::binary : std::ios::out);
  if (!out) throw IoError("cannot open '" + p.string() + "' for writing");
  return out;
}

void close_out(std::ofstream& out, const std::filesystem::path& p) {
  out.flush();
  if (!out) throw IoError("failed writing '" + p.string() + "'");
}

std::vector<Point2> read_text(std::istream& in, bool obj) {
  std::vector<Point2> pts;
  std::string line;
  std::size_t no = 0;
  while (std::getline(in, line)) {
    ++no;
    std::string_view s = strip(line);
    Point2 p{};
    if (obj) {
      if (s.size() < 2 || s[0] != 'v' || (s[1] != ' ' && s[1] != '\t')) continue;
      s.remove_prefix(2);
      if (!next_number(s, p.x) || !next_number(s, p.y))
        throw ParseError(no, "vertex line needs at least x and y");
      double z;
      next_number(s, z);
      if (!strip(s).empty()) throw ParseError(no, "trailing characters after vertex");
    } else {
      if (s.empty() || s.front() == '#') continue;
      if (!next_number(s, p.x) || !next_number(s, p.y))
        throw ParseError(no, "expected two decimal coordinates");
      if (!strip(s).empty()) throw ParseError(no, "trailing characters after coordinates");
    }
    finite_or_throw(p, no);
    pts.push_back(p);
  }
  return pts;
}

std::vector<Point2> read_binary(std::istream& in) {
  std::ostringstream ss;
  ss << in.rdbuf();
  const std::string bytes = std::move(ss).str();
  if (bytes.size() % 16) throw ParseError(0, "binary payload is not a whole number of float64 pairs");
  std::vector<Point2> pts(bytes.size() / 16);
  const auto* b = reinterpret_cast<const unsigned char*>(bytes.data());
  for (std::size_t i = 0; i < pts.size(); ++i) {
    std::uint64_t w[2] = {0, 0};
    for (int h = 0; h < 2; ++h)
      for (int j = 7; j >= 0; --j) w[h] = (w[h] << 8) | b[16 * i + 8 * h + j];
    pts[i] = {std::bit_cast<double>(w[0]), std::bit_cast<double>(w[1])};
    finite_or_throw(pts[i], 0);
  }
  return pts;
}

constexpr const char* kFmt[] = {"xy_text", "xy_binary", "obj_vertices"};

}  // namespace

const char* point_format_name(PointFormat f) {
  const int i = static_cast<int>(f);
  if (i < 0 || i > 2) throw std::invalid_argument("point_format_name: unknown format");
  return kFmt[i];
}

PointFormat parse_point_format(const std::string& name) {
  for (int i = 0; i < 3; ++i)
    if (name == kFmt[i]) return static_cast<PointFormat>(i);
  throw std::invalid_argument("parse_point_format: unknown format '" + name + "'");
}

StatsFormat parse_stats_format(const std::string& name) {
  if (name == "csv") return StatsFormat::Csv;
  if (name == "json") return StatsFormat::Json;
  throw std::invalid_argument("parse_stats_format: unknown format '" + name + "'");
}

std::vector<Point2> read_points(const std::filesystem::path& path, PointFormat format) {
  switch (format) {
    case PointFormat::XyText: {
      auto in = open_in(path, false);
      return read_text(in, false);
    }
    case PointFormat::XyBinary: {
      auto in = open_in(path, true);
      return read_binary(in);
    }
    case PointFormat::ObjVertices: {
      auto in = open_in(path, false);
      return read_text(in, true);
    }
  }
  throw std::invalid_argument("read_points: unknown format");
}

void write_points(std::span<const Point2> points, const std::filesystem::path& path,
                  PointFormat format) {
  if (format == PointFormat::ObjVertices)
    throw std::invalid_argument("write_points: obj_vertices is a read-only format");
  if (format == PointFormat::XyBinary) {
    auto out = open_out(path, true);
    unsigned char rec[16];
    for (const Point2& p : points) {
      const std::uint64_t w[2] = {std::bit_cast<std::uint64_t>(p.x), std::bit_cast<std::uint64_t>(p.y)};
      for (int h = 0; h < 2; ++h)
        for (int j = 0; j < 8; ++j) rec[8 * h + j] = static_cast<unsigned char>(w[h] >> (8 * j));
      out.write(reinterpret_cast<const char*>(rec), 16);
    }
    close_out(out, path);
    return;
  }
  if (format != PointFormat::XyText) throw std::invalid_argument("write_points: unknown format");
  auto out = open_out(path, false);
  std::string line;
  for (const Point2& p : points) {
    line = fmt17(p.x) + ' ' + fmt17(p.y) + '\n';
    out.write(line.data(), static_cast<std::streamsize>(line.size()));
  }
  close_out(out, path);
}

void write_hull(const Hull& hull, const std::filesystem::path& path) {
  write_points(hull.vertices, path, PointFormat::XyText);
}

void write_stats(const StageStats& s, const std::filesystem::path& path, StatsFormat format) {
  auto out = open_out(path, false);
  const char* keys[] = {"n_input",       "n_after_round1", "n_after_spa",    "n_hull",
                        "t_extremes_ms", "t_classify_ms",  "t_partition_ms", "t_sort_ms",
                        "t_spa_ms",      "t_melkman_ms",   "t_total_ms"};
  const std::size_t counts[] = {s.n_input, s.n_after_round1, s.n_after_spa, s.n_hull};
  const double times[] = {s.t_extremes_ms, s.t_classify_ms, s.t_partition_ms, s.t_sort_ms,
                          s.t_spa_ms,      s.t_melkman_ms,  s.t_total_ms};
  if (format == StatsFormat::Csv) {
    for (int i = 0; i < 11; ++i) out << keys[i] << (i < 10 ? "," : "\n");
    for (int i = 0; i < 4; ++i) out << counts[i] << ',';
    for (int i = 0; i < 7; ++i) out << fmt17(times[i]) << (i < 6 ? "," : "\n");
  } else {
    out << "{\n";
    for (int i = 0; i < 11; ++i) {
      out << "  \"" << keys[i] << "\": ";
      if (i < 4)
        out << counts[i];
      else
        out << json_double(times[i - 4]);
      out << (i < 10 ? ",\n" : "\n");
    }
    out << "}\n";
  }
  close_out(out, path);
}

}  // namespace chainhull
