// Point and stats files of the drop-in API (reference io.hpp:14-52; formats
// and error behaviour from SPEC.md "io-datasets": read_points, write_points,
// write_hull, write_stats).
//
// Files are read whole with one fread into memory and scanned in place:
// * xy_binary is the in-memory layout of Point2[] (16-byte little-endian
//   double pairs, the device layout chgpu_hull takes), so the payload is
//   copied straight into the result vector and then checked for finiteness;
// * the text formats are scanned line by line with memchr over the buffer,
//   numbers parsed with std::from_chars.
// Output goes through one stdio stream per file; text coordinates use 17
// significant digits ("%.17g", an exact double round trip).

#include <bit>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string_view>
#include <utility>

#include "chainhull/api.hpp"

namespace chainhull {

namespace {

static_assert(std::endian::native == std::endian::little,
              "xy_binary is little-endian: this reader copies it as Point2[]");
static_assert(sizeof(Point2) == 16, "Point2 must be two packed doubles");

struct FileCloser {
  void operator()(std::FILE* f) const {
    if (f) std::fclose(f);
  }
};
using File = std::unique_ptr<std::FILE, FileCloser>;

File open_file(const std::filesystem::path& path, const char* mode, const char* what) {
  File f(std::fopen(path.c_str(), mode));
  if (!f) throw IoError("cannot open '" + path.string() + "' for " + what);
  return f;
}

// The whole file as bytes.
std::string slurp(const std::filesystem::path& path, bool binary) {
  File f = open_file(path, binary ? "rb" : "r", "reading");
  std::string bytes;
  char block[1 << 16];
  for (;;) {
    const size_t got = std::fread(block, 1, sizeof block, f.get());
    bytes.append(block, got);
    if (got < sizeof block) break;
  }
  return bytes;
}

bool is_blank(char c) { return c == ' ' || c == '\t'; }

// Cursor over one line of text.
class LineCursor {
 public:
  explicit LineCursor(std::string_view line) : s_(line) {
    while (!s_.empty() && is_blank(s_.front())) s_.remove_prefix(1);
    while (!s_.empty() && (is_blank(s_.back()) || s_.back() == '\r')) s_.remove_suffix(1);
  }
  bool empty() const { return s_.empty(); }
  char first() const { return s_.front(); }
  // An OBJ vertex record: "v" then a blank.
  bool take_vertex_tag() {
    if (s_.size() < 2 || s_[0] != 'v' || !is_blank(s_[1])) return false;
    s_.remove_prefix(2);
    return true;
  }
  bool take_number(double& out) {
    while (!s_.empty() && is_blank(s_.front())) s_.remove_prefix(1);
    const auto [end, ec] = std::from_chars(s_.data(), s_.data() + s_.size(), out);
    if (ec != std::errc{}) return false;
    s_.remove_prefix(static_cast<size_t>(end - s_.data()));
    return true;
  }
  bool at_end() const {
    for (char c : s_)
      if (!is_blank(c)) return false;
    return true;
  }

 private:
  std::string_view s_;
};

void require_finite_point(const Point2& p, size_t line_no) {
  if (std::isfinite(p.x) && std::isfinite(p.y)) return;
  if (line_no == 0) throw NonFiniteCoordinate("non-finite coordinate");
  throw NonFiniteCoordinate("non-finite coordinate at line " + std::to_string(line_no));
}

// xy_text (obj = false) or obj_vertices (obj = true).
std::vector<Point2> scan_text(const std::string& text, bool obj) {
  std::vector<Point2> out;
  size_t line_no = 0;
  const char* p = text.data();
  const char* const end = p + text.size();
  while (p < end) {
    const char* nl = static_cast<const char*>(std::memchr(p, '\n', static_cast<size_t>(end - p)));
    const char* stop = nl ? nl : end;
    ++line_no;
    LineCursor cur(std::string_view(p, static_cast<size_t>(stop - p)));
    p = nl ? nl + 1 : end;
    Point2 pt{};
    if (obj) {
      if (!cur.take_vertex_tag()) continue;  // every other OBJ record is ignored
      if (!cur.take_number(pt.x) || !cur.take_number(pt.y))
        throw ParseError(line_no, "vertex line needs at least x and y");
      double z;
      (void)cur.take_number(z);  // z is dropped (optional)
      if (!cur.at_end()) throw ParseError(line_no, "trailing characters after vertex");
    } else {
      if (cur.empty() || cur.first() == '#') continue;
      if (!cur.take_number(pt.x) || !cur.take_number(pt.y))
        throw ParseError(line_no, "expected two decimal coordinates");
      if (!cur.at_end()) throw ParseError(line_no, "trailing characters after coordinates");
    }
    require_finite_point(pt, line_no);
    out.push_back(pt);
  }
  return out;
}

std::vector<Point2> decode_binary(const std::string& bytes) {
  if (bytes.size() % sizeof(Point2) != 0)
    throw ParseError(0, "binary payload is not a whole number of float64 pairs");
  std::vector<Point2> out(bytes.size() / sizeof(Point2));
  if (!out.empty()) std::memcpy(out.data(), bytes.data(), bytes.size());
  for (const Point2& pt : out) require_finite_point(pt, 0);
  return out;
}

void finish_file(File& f, const std::filesystem::path& path) {
  const bool bad = std::ferror(f.get()) != 0;
  const int rc = std::fclose(f.release());
  if (bad || rc != 0) throw IoError("failed writing '" + path.string() + "'");
}

void put_g17(std::FILE* f, double v) { std::fprintf(f, "%.17g", v); }

// Shortest round-trip form, ".0" appended to integral values (the JSON
// number style of the stats writer).
void put_json_number(std::FILE* f, double v) {
  char buf[64];
  const auto r = std::to_chars(buf, buf + sizeof buf, v);
  std::string_view s(buf, static_cast<size_t>(r.ptr - buf));
  std::fwrite(s.data(), 1, s.size(), f);
  if (s.find_first_of(".eE") == std::string_view::npos && s.find("inf") == std::string_view::npos &&
      s.find("nan") == std::string_view::npos)
    std::fputs(".0", f);
}

constexpr std::string_view kPointFormats[] = {"xy_text", "xy_binary", "obj_vertices"};

}  // namespace

const char* point_format_name(PointFormat format) {
  const auto i = static_cast<size_t>(format);
  if (i >= std::size(kPointFormats)) throw std::invalid_argument("point_format_name: unknown format");
  return kPointFormats[i].data();
}

PointFormat parse_point_format(const std::string& name) {
  for (size_t i = 0; i < std::size(kPointFormats); ++i)
    if (kPointFormats[i] == name) return static_cast<PointFormat>(i);
  throw std::invalid_argument("parse_point_format: unknown format '" + name + "'");
}

StatsFormat parse_stats_format(const std::string& name) {
  if (name == "csv") return StatsFormat::Csv;
  if (name == "json") return StatsFormat::Json;
  throw std::invalid_argument("parse_stats_format: unknown format '" + name + "'");
}

std::vector<Point2> read_points(const std::filesystem::path& path, PointFormat format) {
  if (format == PointFormat::XyBinary) return decode_binary(slurp(path, true));
  if (format == PointFormat::XyText) return scan_text(slurp(path, false), false);
  if (format == PointFormat::ObjVertices) return scan_text(slurp(path, false), true);
  throw std::invalid_argument("read_points: unknown format");
}

void write_points(std::span<const Point2> points, const std::filesystem::path& path,
                  PointFormat format) {
  if (format == PointFormat::ObjVertices)
    throw std::invalid_argument("write_points: obj_vertices is a read-only format");
  if (format != PointFormat::XyText && format != PointFormat::XyBinary)
    throw std::invalid_argument("write_points: unknown format");
  const bool binary = format == PointFormat::XyBinary;
  File f = open_file(path, binary ? "wb" : "w", "writing");
  if (binary) {
    if (!points.empty()) std::fwrite(points.data(), sizeof(Point2), points.size(), f.get());
  } else {
    for (const Point2& pt : points) {
      put_g17(f.get(), pt.x);
      std::fputc(' ', f.get());
      put_g17(f.get(), pt.y);
      std::fputc('\n', f.get());
    }
  }
  finish_file(f, path);
}

void write_hull(const Hull& hull, const std::filesystem::path& path) {
  write_points(hull.vertices, path, PointFormat::XyText);
}

void write_stats(const StageStats& s, const std::filesystem::path& path, StatsFormat format) {
  struct Field {
    const char* name;
    bool is_count;
    size_t count;
    double ms;
  };
  const Field fields[] = {
      {"n_input", true, s.n_input, 0},         {"n_after_round1", true, s.n_after_round1, 0},
      {"n_after_spa", true, s.n_after_spa, 0}, {"n_hull", true, s.n_hull, 0},
      {"t_extremes_ms", false, 0, s.t_extremes_ms}, {"t_classify_ms", false, 0, s.t_classify_ms},
      {"t_partition_ms", false, 0, s.t_partition_ms}, {"t_sort_ms", false, 0, s.t_sort_ms},
      {"t_spa_ms", false, 0, s.t_spa_ms},      {"t_melkman_ms", false, 0, s.t_melkman_ms},
      {"t_total_ms", false, 0, s.t_total_ms}};
  File f = open_file(path, "w", "writing");
  std::FILE* o = f.get();
  if (format == StatsFormat::Csv) {
    const char* sep = "";
    for (const Field& fd : fields) std::fprintf(o, "%s%s", std::exchange(sep, ","), fd.name);
    std::fputc('\n', o);
    sep = "";
    for (const Field& fd : fields) {
      std::fputs(std::exchange(sep, ","), o);
      if (fd.is_count)
        std::fprintf(o, "%zu", fd.count);
      else
        put_g17(o, fd.ms);
    }
    std::fputc('\n', o);
  } else {
    std::fputs("{\n", o);
    const size_t nf = std::size(fields);
    for (size_t i = 0; i < nf; ++i) {
      std::fprintf(o, "  \"%s\": ", fields[i].name);
      if (fields[i].is_count)
        std::fprintf(o, "%zu", fields[i].count);
      else
        put_json_number(o, fields[i].ms);
      std::fputs(i + 1 < nf ? ",\n" : "\n", o);
    }
    std::fputs("}\n", o);
  }
  finish_file(f, path);
}

}  // namespace chainhull
