// Host finisher: chain assembly, Melkman, canonical rotation and the
// sort-based reference hull. These run on the CPU in the reference too
// (polygon.cpp, melkman.cpp, oracle.cpp) and operate on the few survivors
// the GPU stages leave (33 K points of 20 M uniform). Semantics are
// identical to the reference: same orient predicate and evaluation order
// (built with -ffp-contract=off), same collapse rules, same pop order.
// The deque is a flat array with head/tail cursors instead of std::deque.

#include "finisher.h"

#include <algorithm>
#include <cstring>
#include <memory>

namespace chgpu {
namespace host {

namespace {

inline bool same(const Pt& a, const Pt& b) { return a.x == b.x && a.y == b.y; }

// geometry.hpp:22-35
inline int turn(const Pt& a, const Pt& b, const Pt& p) {
  const double c = (b.x - a.x) * (p.y - a.y) - (b.y - a.y) * (p.x - a.x);
  return c > 0.0 ? +1 : (c < 0.0 ? -1 : 0);
}
constexpr int kLeft = +1;

inline bool lex_less(const Pt& a, const Pt& b) { return a.x < b.x || (a.x == b.x && a.y < b.y); }

// Appends p unless it repeats the ring's current last vertex.
inline void push_distinct(std::vector<Pt>& ring, const Pt& p) {
  if (ring.empty() || !same(ring.back(), p)) ring.push_back(p);
}

}  // namespace

int assemble_ring(const Pt* chains, const size_t kept_counts[4], const Pt corners[4],
                  std::vector<Pt>& ring) {
  // polygon.cpp:7-29: corner r, then region r's chain, for r = 0..3.
  size_t total = 4;
  for (int r = 0; r < 4; ++r) total += kept_counts[r];
  ring.clear();
  ring.reserve(total);
  const Pt* c = chains;
  for (int r = 0; r < 4; ++r) {
    push_distinct(ring, corners[r]);
    for (size_t j = 0; j < kept_counts[r]; ++j) push_distinct(ring, c[j]);
    c += kept_counts[r];
  }
  if (ring.size() > 1 && same(ring.front(), ring.back())) ring.pop_back();
  return ring.size() < 3 ? kDegenerate : kOk;
}

void canonicalize(Pt* ring, size_t n) {
  // melkman.cpp:10-15: rotate so the first lexicographic minimum leads.
  if (n < 2) return;
  size_t lo = 0;
  for (size_t i = 1; i < n; ++i)
    if (lex_less(ring[i], ring[lo])) lo = i;
  std::rotate(ring, ring + lo, ring + n);
}

namespace {

// Per-thread scratch that only ever grows: the finisher runs once per hull
// call, and re-allocating (and page-faulting) megabytes each time costs more
// than the scan itself.
struct Scratch {
  std::unique_ptr<Pt[]> buf;
  size_t cap = 0;
  Pt* get(size_t n) {
    if (n > cap) {
      cap = n + n / 2;
      buf.reset(new Pt[cap]);
    }
    return buf.get();
  }
};

}  // namespace

int melkman(const Pt* poly, size_t n_in, std::vector<Pt>& hull) {
  // melkman.cpp:20-25: consecutive duplicates (and a closing repeat) go.
  thread_local Scratch ring_s, deque_s;
  Pt* ring = ring_s.get(n_in + 1);
  size_t n = 0;
  for (size_t i = 0; i < n_in; ++i)
    if (n == 0 || !same(ring[n - 1], poly[i])) ring[n++] = poly[i];
  if (n > 1 && same(ring[0], ring[n - 1])) --n;

  // melkman.cpp:30-47: absorb the leading collinear run; remember its two
  // extreme endpoints (lo, hi) and the last vertex visited.
  Pt lo = n ? ring[0] : Pt{0.0, 0.0};
  Pt hi = lo, last = lo;
  size_t i = 1;
  while (i < n) {
    const Pt& p = ring[i];
    if (turn(lo, hi, p) != 0) break;
    if (lex_less(p, lo))
      lo = p;
    else if (lex_less(hi, p))
      hi = p;
    last = p;
    ++i;
  }
  if (i >= n) return kDegenerate;

  // melkman.cpp:52-60: seed triangle; the deque lives in buf[head, tail).
  Pt* buf = deque_s.get(2 * n + 8);
  size_t head = n + 4, tail = head;
  const Pt w = ring[i];
  const Pt second = last;
  const Pt first = same(last, lo) ? hi : lo;
  const bool ccw = turn(first, second, w) == kLeft;
  buf[tail++] = w;
  buf[tail++] = ccw ? first : second;
  buf[tail++] = ccw ? second : first;
  buf[tail++] = w;

  // melkman.cpp:62-80
  for (++i; i < n; ++i) {
    const Pt v = ring[i];
    if (turn(buf[head], buf[head + 1], v) == kLeft && turn(buf[tail - 2], buf[tail - 1], v) == kLeft)
      continue;
    while (tail - head >= 2 && turn(buf[tail - 2], buf[tail - 1], v) != kLeft) --tail;
    buf[tail++] = v;
    while (tail - head >= 2 && turn(v, buf[head], buf[head + 1]) != kLeft) ++head;
    buf[--head] = v;
  }
  hull.assign(buf + head, buf + (tail - 1));  // ends coincide (:83)
  canonicalize(hull.data(), hull.size());
  return kOk;
}

int monotone_chain(const Pt* pts, size_t n, std::vector<Pt>& hull) {
  // oracle.cpp:19-37 over lexicographically sorted, duplicate-free points.
  hull.clear();
  if (n == 0) return kEmpty;
  if (n == 1) {
    hull.push_back(pts[0]);
    return kOk;
  }
  std::vector<Pt> h(2 * n);
  size_t k = 0;
  for (size_t i = 0; i < n; ++i) {
    while (k >= 2 && turn(h[k - 2], h[k - 1], pts[i]) != kLeft) --k;
    h[k++] = pts[i];
  }
  const size_t lower_end = k + 1;
  for (size_t i = n - 1; i-- > 0;) {
    while (k >= lower_end && turn(h[k - 2], h[k - 1], pts[i]) != kLeft) --k;
    h[k++] = pts[i];
  }
  h.resize(k - 1);
  hull.swap(h);
  return kOk;
}

int sorted_hull(const Pt* pts, size_t n, std::vector<Pt>& hull) {
  // oracle.cpp:12-38: sort, unique, monotone chain.
  if (n == 0) return kEmpty;
  std::vector<Pt> s(pts, pts + n);
  std::sort(s.begin(), s.end(), lex_less);
  s.erase(std::unique(s.begin(), s.end(), same), s.end());
  return monotone_chain(s.data(), s.size(), hull);
}

void insert_sorted_unique(std::vector<Pt>& sorted, const Pt& p) {
  auto it = std::lower_bound(sorted.begin(), sorted.end(), p, lex_less);
  if (it != sorted.end() && same(*it, p)) return;
  sorted.insert(it, p);
}

}  // namespace host
}  // namespace chgpu

// ---------------------------------------------------------------- C ABI

using chgpu::host::Pt;

extern "C" int chgpu_assemble_polygon(const double* chains, const size_t* kept_counts,
                                      const double* quad, double* out, size_t* n_out) {
  std::vector<Pt> ring;
  const int st = chgpu::host::assemble_ring(reinterpret_cast<const Pt*>(chains), kept_counts,
                                            reinterpret_cast<const Pt*>(quad), ring);
  std::memcpy(out, ring.data(), ring.size() * sizeof(Pt));
  *n_out = ring.size();
  return st;
}

extern "C" int chgpu_melkman(const double* poly, size_t n, double* out, size_t* n_out) {
  std::vector<Pt> hull;
  const int st = chgpu::host::melkman(reinterpret_cast<const Pt*>(poly), n, hull);
  if (st) {
    *n_out = 0;
    return st;
  }
  std::memcpy(out, hull.data(), hull.size() * sizeof(Pt));
  *n_out = hull.size();
  return 0;
}

extern "C" void chgpu_canonicalize_ring(double* ring, size_t n) {
  chgpu::host::canonicalize(reinterpret_cast<Pt*>(ring), n);
}

extern "C" int chgpu_hull_oracle(const double* xy, size_t n, double* out, size_t* n_out) {
  std::vector<Pt> hull;
  const int st = chgpu::host::sorted_hull(reinterpret_cast<const Pt*>(xy), n, hull);
  if (st) {
    *n_out = 0;
    return st;
  }
  std::memcpy(out, hull.data(), hull.size() * sizeof(Pt));
  *n_out = hull.size();
  return 0;
}
