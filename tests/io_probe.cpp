// I/O parity probe (test infrastructure): exercises the chainhull file API
// (io.hpp: read_points / write_points / write_hull / write_stats, and the
// format-name helpers) through the public headers only. Built twice: against
// the reference's own io.cpp (oracle/Makefile, oracle/_ref/io_probe_ref) and
// against the drop-in libchainhull (top-level Makefile, build/io_probe_b200);
// tests/test_io_parity.py runs both and compares every byte they write and
// every line they print.
//
// usage: io_probe <out_dir>
#include <cmath>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <limits>
#include <string>
#include <vector>

#include "chainhull/chainhull.hpp"

namespace fs = std::filesystem;
using namespace chainhull;

static void write_text(const fs::path& p, const std::string& s) {
  std::ofstream o(p, std::ios::binary);
  o << s;
}

static void report_read(const fs::path& p, PointFormat f) {
  try {
    const auto v = read_points(p, f);
    std::printf("read %s %s: %zu points", p.filename().c_str(), point_format_name(f), v.size());
    double sx = 0, sy = 0;
    for (const auto& q : v) sx += q.x, sy += q.y;
    std::printf(" sum %.17g %.17g\n", sx, sy);
  } catch (const ParseError& e) {
    std::printf("read %s: ParseError line %zu: %s\n", p.filename().c_str(), e.line, e.what());
  } catch (const NonFiniteCoordinate& e) {
    std::printf("read %s: NonFiniteCoordinate: %s\n", p.filename().c_str(), e.what());
  } catch (const IoError& e) {
    std::printf("read %s: IoError\n", p.filename().c_str());
  }
}

int main(int argc, char** argv) {
  if (argc < 2) return 2;
  const fs::path dir = argv[1];
  fs::create_directories(dir);
  // points with awkward decimal expansions, signed zeros, tiny and huge values
  std::vector<Point2> pts = generate({Distribution::Gaussian, 257, 5});
  pts.push_back({-0.0, 0.0});
  pts.push_back({1e-310, -5e-324});
  pts.push_back({1.7976931348623157e308, -2.2250738585072014e-308});
  pts.push_back({0.1, 1.0 / 3.0});
  pts.push_back({123456789.125, -0.5});
  write_points(pts, dir / "pts.txt", PointFormat::XyText);
  write_points(pts, dir / "pts.bin", PointFormat::XyBinary);
  report_read(dir / "pts.txt", PointFormat::XyText);
  report_read(dir / "pts.bin", PointFormat::XyBinary);

  const Hull h = hull_oracle(generate({Distribution::UniformDisk, 5000, 9}));
  write_hull(h, dir / "hull.txt");

  StageStats s{};
  s.n_input = 20000000;
  s.n_after_round1 = 8783071;
  s.n_after_spa = 33155;
  s.n_hull = 46;
  s.t_extremes_ms = 0.068;
  s.t_classify_ms = 1.0 / 3.0;
  s.t_partition_ms = 0.0;
  s.t_sort_ms = 1e-9;
  s.t_spa_ms = 12345.678;
  s.t_melkman_ms = 2.5e-5;
  s.t_total_ms = 100.0;
  write_stats(s, dir / "stats.csv", StatsFormat::Csv);
  write_stats(s, dir / "stats.json", StatsFormat::Json);

  // readers: comments, blank lines, OBJ, and each error the reference defines
  write_text(dir / "ok.txt", "# header\n\n1 2\n  3.5\t-4  \n# c\n5e-1 6\n");
  write_text(dir / "ok.obj", "o mesh\nv 1 2 3\nvn 0 0 1\nv -1.5 2.5 9\nf 1 2 3\nv 0 0 0\n");
  write_text(dir / "bad1.txt", "1 2\n3\n");
  write_text(dir / "bad2.txt", "1 2\n3 4 5\n");
  write_text(dir / "bad3.txt", "1 2\nx 4\n");
  write_text(dir / "nan.txt", "1 2\nnan 4\n");
  write_text(dir / "inf.obj", "v 1 2 0\nv inf 2 0\n");
  write_text(dir / "bad.bin", std::string(24, '\0'));
  for (const char* f : {"ok.txt", "bad1.txt", "bad2.txt", "bad3.txt", "nan.txt"})
    report_read(dir / f, PointFormat::XyText);
  report_read(dir / "ok.obj", PointFormat::ObjVertices);
  report_read(dir / "inf.obj", PointFormat::ObjVertices);
  report_read(dir / "bad.bin", PointFormat::XyBinary);
  report_read(dir / "missing.txt", PointFormat::XyText);

  for (auto f : {PointFormat::XyText, PointFormat::XyBinary, PointFormat::ObjVertices})
    std::printf("format %s -> %d\n", point_format_name(f),
                (int)parse_point_format(point_format_name(f)));
  std::printf("stats csv %d json %d\n", (int)parse_stats_format("csv"),
              (int)parse_stats_format("json"));
  return 0;
}
