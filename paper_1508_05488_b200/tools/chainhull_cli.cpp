// chainhull — the reference command line (proj/tools/src/main.cpp) over the
// B200 drop-in (libchainhull.so): `hull`, `gen`, `verify` and `bench` with
// the reference's flags, defaults, messages, exit codes (0 success, 1
// runtime error, including malformed input files; 2 usage error) and bench CSV schema
// (main.cpp:150-205: size,seed,repeat,n_input,...,frac_after_spa[,t_oracle_ms]).
//
// The reference parses its options with CLI11 (not vendored here); this tool
// parses the same options itself. Stage timings come from the drop-in's
// StageStats (CUDA events for the device stages, the host clock for the
// finisher and the total).
//
// usage: chainhull <hull|gen|verify|bench> [options]   (chainhull --help)

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <map>
#include <optional>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include "chainhull/chainhull.hpp"

namespace {

using chainhull::Point2;

// A usage error: exit code 2 with the message on stderr.
struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

const std::set<std::string> kDistributions = {"uniform_square", "uniform_disk", "circle",
                                              "gaussian",       "collinear",    "duplicates_heavy"};
const std::set<std::string> kReadFormats = {"xy_text", "xy_binary", "obj_vertices"};
const std::set<std::string> kWriteFormats = {"xy_text", "xy_binary"};

// --name value / --name=value options and --flag switches of one
// subcommand. List options (CLI11 vector options in the reference) take
// every following argument up to the next "--option", each of which may
// itself be a comma-separated list: "--sizes 1000 2000" == "--sizes 1000,2000".
class Args {
 public:
  Args(int argc, char** argv, int first, const std::set<std::string>& options,
       const std::set<std::string>& flags, const std::set<std::string>& lists = {}) {
    for (int i = first; i < argc; ++i) {
      std::string a = argv[i];
      if (a.rfind("--", 0) != 0) throw UsageError("unexpected argument '" + a + "'");
      std::string value;
      const auto eq = a.find('=');
      const bool inline_value = eq != std::string::npos;
      if (inline_value) {
        value = a.substr(eq + 1);
        a = a.substr(0, eq);
      }
      const std::string name = a.substr(2);
      if (flags.count(name)) {
        if (inline_value) throw UsageError("--" + name + " takes no value");
        flags_.insert(name);
        continue;
      }
      if (!options.count(name) && !lists.count(name)) throw UsageError("unknown option '" + a + "'");
      if (!inline_value) {
        if (i + 1 >= argc) throw UsageError(a + " needs a value");
        value = argv[++i];
      }
      std::string& v = values_[name];
      if (!lists.count(name)) {
        v = value;
        continue;
      }
      v += (v.empty() ? "" : ",") + value;
      while (i + 1 < argc && std::string(argv[i + 1]).rfind("--", 0) != 0) v += "," + std::string(argv[++i]);
    }
  }
  bool has(const std::string& n) const { return values_.count(n) != 0; }
  bool flag(const std::string& n) const { return flags_.count(n) != 0; }
  std::string str(const std::string& n, const std::string& def) const {
    const auto it = values_.find(n);
    return it == values_.end() ? def : it->second;
  }
  std::string required(const std::string& n) const {
    if (!has(n)) throw UsageError("--" + n + " is required");
    return values_.at(n);
  }

 private:
  std::map<std::string, std::string> values_;
  std::set<std::string> flags_;
};

std::uint64_t to_u64(const std::string& name, const std::string& s, bool positive) {
  std::size_t pos = 0;
  unsigned long long v = 0;
  try {
    if (s.empty() || s[0] == '-') throw std::invalid_argument(s);
    v = std::stoull(s, &pos, 10);
  } catch (const std::exception&) {
    throw UsageError("--" + name + ": '" + s + "' is not a non-negative integer");
  }
  if (pos != s.size()) throw UsageError("--" + name + ": '" + s + "' is not a non-negative integer");
  if (positive && v == 0) throw UsageError("--" + name + ": value must be positive");
  return v;
}

std::vector<std::uint64_t> to_u64_list(const std::string& name, const std::string& s, bool positive) {
  std::vector<std::uint64_t> out;
  std::size_t start = 0;
  while (true) {
    const auto comma = s.find(',', start);
    out.push_back(to_u64(name, s.substr(start, comma - start), positive));
    if (comma == std::string::npos) break;
    start = comma + 1;
  }
  return out;
}

std::string member(const std::string& name, const std::string& v, const std::set<std::string>& allowed) {
  if (!allowed.count(v)) throw UsageError("--" + name + ": '" + v + "' is not one of the allowed values");
  return v;
}

// --threads, else CHAINHULL_THREADS (main.cpp: envname), else 0 (auto).
std::size_t threads_opt(const Args& a) {
  if (a.has("threads")) return to_u64("threads", a.str("threads", "0"), false);
  if (const char* e = std::getenv("CHAINHULL_THREADS")) return to_u64("threads", e, false);
  return 0;
}

std::string fmt_ms(double value) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "%.6f", value);
  return buf;
}

chainhull::PipelineConfig config_of(std::size_t chunk_count, std::size_t threads) {
  chainhull::PipelineConfig c;
  c.chunk_count = chunk_count;
  c.parallelism = threads;
  return c;
}

std::vector<Point2> generated(const std::string& dist, std::size_t n, std::uint64_t seed) {
  chainhull::DatasetSpec spec;
  spec.distribution = chainhull::parse_distribution(dist);
  spec.n = n;
  spec.seed = seed;
  return chainhull::generate(spec);
}

// ---------------------------------------------------------------- hull (main.cpp:71-85)
int run_hull(const Args& a) {
  const std::string input = a.required("input");
  if (!std::filesystem::is_regular_file(input))
    throw UsageError("--input: File does not exist: " + input);
  const std::string format = member("format", a.str("format", "xy_text"), kReadFormats);
  const std::size_t chunks = to_u64("chunk-count", a.str("chunk-count", "1024"), true);
  const std::string output = a.required("output");
  const std::string stats_output = a.str("stats-output", "");
  const std::string stats_format = member("stats-format", a.str("stats-format", "csv"), {"csv", "json"});
  const std::size_t threads = threads_opt(a);

  const auto points = chainhull::read_points(input, chainhull::parse_point_format(format));
  const auto result = chainhull::convex_hull(points, config_of(chunks, threads));
  chainhull::write_hull(result.hull, output);
  if (!stats_output.empty())
    chainhull::write_stats(result.stats, stats_output, chainhull::parse_stats_format(stats_format));
  std::cout << "hull: " << result.stats.n_hull << " vertices from " << result.stats.n_input
            << " points -> " << output << '\n';
  return 0;
}

// ---------------------------------------------------------------- gen (main.cpp:87-98)
int run_gen(const Args& a) {
  const std::string dist = member("distribution", a.str("distribution", "uniform_square"), kDistributions);
  const std::size_t n = to_u64("n", a.required("n"), true);
  const std::uint64_t seed = to_u64("seed", a.str("seed", "0"), false);
  const std::string output = a.required("output");
  const std::string format = member("format", a.str("format", "xy_text"), kWriteFormats);
  const auto points = generated(dist, n, seed);
  chainhull::write_points(points, output, chainhull::parse_point_format(format));
  std::cout << "gen: " << points.size() << ' ' << dist << " points -> " << output << '\n';
  return 0;
}

// ---------------------------------------------------------------- verify (main.cpp:100-148)
int run_verify(const Args& a) {
  const std::string input = a.str("input", "");
  if (!input.empty()) {
    if (!std::filesystem::is_regular_file(input))
      throw UsageError("--input: File does not exist: " + input);
    for (const char* o : {"distribution", "n", "seed"})
      if (a.has(o)) throw UsageError(std::string("--") + o + " excludes --input");
  } else if (a.has("format")) {
    throw UsageError("--format requires --input");
  }
  const std::string format = member("format", a.str("format", "xy_text"), kReadFormats);
  const std::string dist = member("distribution", a.str("distribution", "uniform_square"), kDistributions);
  const std::size_t n = a.has("n") ? to_u64("n", a.str("n", "0"), true) : 0;
  const std::uint64_t seed0 = to_u64("seed", a.str("seed", "0"), false);
  const std::size_t trials = to_u64("trials", a.str("trials", "1"), true);
  const auto chunk_counts = to_u64_list("chunk-counts", a.str("chunk-counts", "1024"), true);
  const std::size_t threads = threads_opt(a);
  if (input.empty() && !a.has("n")) {
    std::cerr << "verify: needs either --input or --n\n";
    return 2;
  }

  std::vector<Point2> file_points;
  if (!input.empty()) file_points = chainhull::read_points(input, chainhull::parse_point_format(format));
  std::size_t failures = 0;
  std::optional<std::uint64_t> first_failing_seed;
  for (std::size_t trial = 0; trial < trials; ++trial) {
    const std::uint64_t seed = seed0 + trial;
    std::vector<Point2> gen;
    if (input.empty()) gen = generated(dist, n, seed);
    const auto& points = input.empty() ? gen : file_points;
    // the exact reference hull (sort everything + monotone chain) against
    // the pipeline at every chunk count
    const auto expected = chainhull::hull_oracle(points);
    bool ok = true;
    for (const std::size_t chunks : chunk_counts) {
      const auto result = chainhull::convex_hull(points, config_of(chunks, threads));
      if (result.hull.vertices != expected.vertices) {
        ok = false;
        break;
      }
    }
    if (!ok) {
      ++failures;
      if (!first_failing_seed) first_failing_seed = seed;
    }
    std::cout << "trial " << trial << " seed=" << seed << " n=" << points.size()
              << " n_hull=" << expected.vertices.size() << (ok ? " PASS" : " FAIL") << '\n';
  }
  if (failures > 0) {
    std::cout << "FAILED " << failures << '/' << trials << " trials; first failing seed "
              << *first_failing_seed << '\n';
    return 1;
  }
  std::cout << "verified " << trials << '/' << trials << " trials\n";
  return 0;
}

// ---------------------------------------------------------------- bench (main.cpp:150-205)
int run_bench(const Args& a) {
  const auto sizes = to_u64_list("sizes", a.required("sizes"), true);
  const std::string dist = member("distribution", a.str("distribution", "uniform_square"), kDistributions);
  const auto seeds = to_u64_list("seeds", a.str("seeds", "0"), false);
  const std::size_t repeats = to_u64("repeats", a.str("repeats", "1"), true);
  const std::string csv_output = a.str("csv-output", "");
  const std::size_t chunks = to_u64("chunk-count", a.str("chunk-count", "1024"), true);
  const std::size_t threads = threads_opt(a);
  const bool with_oracle = a.flag("with-oracle");

  std::ofstream file;
  if (!csv_output.empty()) {
    file.open(csv_output);
    if (!file) throw chainhull::IoError("cannot open '" + csv_output + "' for writing");
  }
  std::ostream& out = csv_output.empty() ? std::cout : file;
  out << "size,seed,repeat,n_input,n_after_round1,n_after_spa,n_hull,t_extremes_ms,"
         "t_classify_ms,t_partition_ms,t_sort_ms,t_spa_ms,t_melkman_ms,t_total_ms,"
         "frac_after_round1,frac_after_spa";
  if (with_oracle) out << ",t_oracle_ms";
  out << '\n';
  for (const std::size_t size : sizes) {
    for (const std::uint64_t seed : seeds) {
      const auto points = generated(dist, size, seed);
      for (std::size_t repeat = 0; repeat < repeats; ++repeat) {
        const auto result = chainhull::convex_hull(points, config_of(chunks, threads));
        const auto& s = result.stats;
        const double n = static_cast<double>(s.n_input);
        out << size << ',' << seed << ',' << repeat << ',' << s.n_input << ',' << s.n_after_round1
            << ',' << s.n_after_spa << ',' << s.n_hull << ',' << fmt_ms(s.t_extremes_ms) << ','
            << fmt_ms(s.t_classify_ms) << ',' << fmt_ms(s.t_partition_ms) << ','
            << fmt_ms(s.t_sort_ms) << ',' << fmt_ms(s.t_spa_ms) << ',' << fmt_ms(s.t_melkman_ms)
            << ',' << fmt_ms(s.t_total_ms) << ',' << fmt_ms(static_cast<double>(s.n_after_round1) / n)
            << ',' << fmt_ms(static_cast<double>(s.n_after_spa) / n);
        if (with_oracle) {
          const auto t0 = std::chrono::steady_clock::now();
          const auto oracle = chainhull::hull_oracle(points);
          const double oracle_ms =
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
          if (oracle.vertices.size() != s.n_hull)
            throw chainhull::Error("bench: pipeline and reference hull disagree");
          out << ',' << fmt_ms(oracle_ms);
        }
        out << '\n';
      }
    }
  }
  out.flush();
  if (!out) throw chainhull::IoError("failed writing benchmark rows");
  return 0;
}

const char* kUsage =
    "Data-parallel 2D convex hull pipeline (B200)\n"
    "usage: chainhull <subcommand> [options]\n"
    "  hull    --input FILE [--format xy_text|xy_binary|obj_vertices] [--chunk-count N]\n"
    "          [--threads N] --output FILE [--stats-output FILE] [--stats-format csv|json]\n"
    "  gen     [--distribution D] --n N [--seed S] --output FILE [--format xy_text|xy_binary]\n"
    "  verify  (--input FILE [--format F] | [--distribution D] --n N [--seed S])\n"
    "          [--trials T] [--chunk-counts C1,C2,...] [--threads N]\n"
    "  bench   --sizes N1,N2,... [--distribution D] [--seeds S1,...] [--repeats R]\n"
    "          [--csv-output FILE] [--chunk-count N] [--threads N] [--with-oracle]\n"
    "distributions: uniform_square uniform_disk circle gaussian collinear duplicates_heavy\n";

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::cerr << kUsage << "A subcommand is required\n";
    return 2;
  }
  const std::string sub = argv[1];
  if (sub == "--help" || sub == "-h") {
    std::cout << kUsage;
    return 0;
  }
  try {
    if (sub == "hull")
      return run_hull(Args(argc, argv, 2,
                           {"input", "format", "chunk-count", "threads", "output", "stats-output",
                            "stats-format"},
                           {}));
    if (sub == "gen")
      return run_gen(Args(argc, argv, 2, {"distribution", "n", "seed", "output", "format"}, {}));
    if (sub == "verify")
      return run_verify(Args(argc, argv, 2,
                             {"input", "format", "distribution", "n", "seed", "trials", "threads"}, {},
                             {"chunk-counts"}));
    if (sub == "bench")
      return run_bench(Args(argc, argv, 2,
                            {"distribution", "repeats", "csv-output", "chunk-count", "threads"},
                            {"with-oracle"}, {"sizes", "seeds"}));
    throw UsageError("unknown subcommand '" + sub + "'");
  } catch (const UsageError& e) {
    std::cerr << e.what() << '\n' << "Run with --help for more information.\n";
    return 2;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << '\n';
    return 1;
  }
}
