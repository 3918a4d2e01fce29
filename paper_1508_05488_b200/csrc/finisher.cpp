// Host finisher: chain assembly, Melkman, canonical rotation and the
// sort-based reference hull. These run on the CPU in the reference too
// (polygon.cpp, melkman.cpp, oracle.cpp) and operate on the few survivors
// the GPU stages leave (33 K points of 20 M uniform). Semantics are
// identical to the reference: same orient predicate and evaluation order
// (built with -ffp-contract=off), same collapse rules, same pop order.
// The deque is a flat array with head/tail cursors instead of std::deque.

#include "finisher.h"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <new>
#include <thread>

#include <unistd.h>

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

int melkman_ring(const Pt* ring, size_t n, std::vector<Pt>& hull) {
  thread_local Scratch deque_s;
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

  // melkman.cpp:52-60: seed triangle; the deque lives in [head, tail).
  Pt* buf = deque_s.get(2 * n + 8);
  Pt* head = buf + n + 4;
  Pt* tail = head;
  const Pt w = ring[i];
  const Pt second = last;
  const Pt first = same(last, lo) ? hi : lo;
  const bool ccw = turn(first, second, w) == kLeft;
  *tail++ = w;
  *tail++ = ccw ? first : second;
  *tail++ = ccw ? second : first;
  *tail++ = w;

  // melkman.cpp:62-80. The two end edges of the deque are cached as
  // (origin, edge vector): the edge vector is the same rounded difference
  // turn() computes, so every predicate is bit-identical; they change only
  // when a vertex is pushed.
  double hax = head[0].x, hay = head[0].y, hex = head[1].x - hax, hey = head[1].y - hay;
  double tax = tail[-2].x, tay = tail[-2].y, tex = tail[-1].x - tax, tey = tail[-1].y - tay;
  for (const Pt* rp = ring + i + 1; rp < ring + n; ++rp) {
    const double vx = rp->x, vy = rp->y;
    const bool left_head = hex * (vy - hay) - hey * (vx - hax) > 0.0;
    const bool left_tail = tex * (vy - tay) - tey * (vx - tax) > 0.0;
    if (left_head & left_tail) continue;  // inside the current hull
    // pop the back while v is not strictly left of its last edge (the first
    // test is left_tail)
    if (!left_tail && tail - head >= 2) {
      --tail;
      while (tail - head >= 2) {
        const Pt a = tail[-2], b = tail[-1];
        if ((b.x - a.x) * (vy - a.y) - (b.y - a.y) * (vx - a.x) > 0.0) break;
        --tail;
      }
    }
    *tail++ = *rp;
    // pop the front while turn(v, front, next) is not left
    while (tail - head >= 2) {
      const Pt a = head[0], b = head[1];
      if ((a.x - vx) * (b.y - vy) - (a.y - vy) * (b.x - vx) > 0.0) break;
      ++head;
    }
    *--head = *rp;
    hax = vx;
    hay = vy;
    hex = head[1].x - vx;
    hey = head[1].y - vy;
    tax = tail[-2].x;
    tay = tail[-2].y;
    tex = tail[-1].x - tax;
    tey = tail[-1].y - tay;
  }
  hull.assign(head, tail - 1);  // ends coincide (:83)
  canonicalize(hull.data(), hull.size());
  return kOk;
}

int melkman(const Pt* poly, size_t n_in, std::vector<Pt>& hull) {
  // melkman.cpp:20-25: consecutive duplicates (and a closing repeat) go.
  thread_local Scratch ring_s;
  Pt* ring = ring_s.get(n_in + 1);
  size_t n = 0;
  for (size_t i = 0; i < n_in; ++i)
    if (n == 0 || !same(ring[n - 1], poly[i])) ring[n++] = poly[i];
  if (n > 1 && same(ring[0], ring[n - 1])) --n;
  return melkman_ring(ring, n, hull);
}

// assemble_polygon + melkman in one streaming pass over the chains: the
// ring (corner r, then chain r, consecutive duplicates collapsed, the
// closing duplicate dropped: polygon.cpp:7-29) is fed to Melkman point by
// point instead of being materialised, and the canonical rotation
// (melkman.cpp:10-15) is written straight into `hull`. Same predicates,
// same pop order, same output as assemble_ring + melkman_ring; a ring of
// fewer than three distinct vertices (polygon.cpp:26) cannot seed the
// triangle either, so both report kDegenerate. For survivor-heavy inputs
// (20 M on-circle points) this removes three full passes over the polygon.
int finish_chains(const Pt* chains, const size_t kept_counts[4], const Pt corners[4],
                  std::vector<Pt>& hull) {
  size_t total = 4;
  for (int r = 0; r < 4; ++r) total += kept_counts[r];
  thread_local Scratch deque_s;
  Pt* buf = deque_s.get(2 * total + 8);
  Pt* head = buf + total + 4;
  Pt* tail = head;

  // Phase A (melkman.cpp:30-60): absorb the leading collinear run, then
  // seed the triangle. Phase B (:62-80): the deque loop with cached edges.
  int phase = 0;  // 0: no point yet, 1: collinear run, 2: deque
  Pt lo{0.0, 0.0}, hi{0.0, 0.0}, last{0.0, 0.0};
  double hax = 0, hay = 0, hex = 0, hey = 0, tax = 0, tay = 0, tex = 0, tey = 0;
  auto feed = [&](const Pt& v) {
    if (phase == 2) {
      const double vx = v.x, vy = v.y;
      const bool left_head = hex * (vy - hay) - hey * (vx - hax) > 0.0;
      const bool left_tail = tex * (vy - tay) - tey * (vx - tax) > 0.0;
      if (left_head & left_tail) return;
      if (!left_tail && tail - head >= 2) {
        --tail;
        while (tail - head >= 2) {
          const Pt a = tail[-2], b = tail[-1];
          if ((b.x - a.x) * (vy - a.y) - (b.y - a.y) * (vx - a.x) > 0.0) break;
          --tail;
        }
      }
      *tail++ = v;
      while (tail - head >= 2) {
        const Pt a = head[0], b = head[1];
        if ((a.x - vx) * (b.y - vy) - (a.y - vy) * (b.x - vx) > 0.0) break;
        ++head;
      }
      *--head = v;
      hax = vx;
      hay = vy;
      hex = head[1].x - vx;
      hey = head[1].y - vy;
      tax = tail[-2].x;
      tay = tail[-2].y;
      tex = tail[-1].x - tax;
      tey = tail[-1].y - tay;
      return;
    }
    if (phase == 0) {
      lo = hi = last = v;
      phase = 1;
      return;
    }
    if (turn(lo, hi, v) == 0) {  // still collinear
      if (lex_less(v, lo))
        lo = v;
      else if (lex_less(hi, v))
        hi = v;
      last = v;
      return;
    }
    const Pt second = last;
    const Pt first = same(last, lo) ? hi : lo;
    const bool ccw = turn(first, second, v) == kLeft;
    *tail++ = v;
    *tail++ = ccw ? first : second;
    *tail++ = ccw ? second : first;
    *tail++ = v;
    hax = head[0].x, hay = head[0].y, hex = head[1].x - hax, hey = head[1].y - hay;
    tax = tail[-2].x, tay = tail[-2].y, tex = tail[-1].x - tax, tey = tail[-1].y - tay;
    phase = 2;
  };

  // The virtual ring: 8 segments (corner r, chain r). The run of trailing
  // elements equal to the very last one emits at most one vertex, which
  // polygon.cpp:22-24 drops when it repeats the first vertex (corner 0).
  const Pt* seg_ptr[8];
  size_t seg_len[8];
  {
    const Pt* c = chains;
    for (int r = 0; r < 4; ++r) {
      seg_ptr[2 * r] = &corners[r];
      seg_len[2 * r] = 1;
      seg_ptr[2 * r + 1] = c;
      seg_len[2 * r + 1] = kept_counts[r];
      c += kept_counts[r];
    }
  }
  int last_seg = 7;
  while (seg_len[last_seg] == 0) --last_seg;  // segment 6 (corner 3) is never empty
  const Pt last_pt = seg_ptr[last_seg][seg_len[last_seg] - 1];
  const bool drop_last = same(last_pt, corners[0]);
  // cut the trailing run of last_pt off the segments
  int cut_seg = last_seg;
  size_t cut_idx = seg_len[last_seg] - 1;
  for (;;) {
    if (cut_idx > 0 && same(seg_ptr[cut_seg][cut_idx - 1], last_pt)) {
      --cut_idx;
      continue;
    }
    if (cut_idx == 0) {
      int s2 = cut_seg - 1;
      while (s2 >= 0 && seg_len[s2] == 0) --s2;
      if (s2 >= 0 && same(seg_ptr[s2][seg_len[s2] - 1], last_pt)) {
        cut_seg = s2;
        cut_idx = seg_len[s2] - 1;
        continue;
      }
    }
    break;
  }
  Pt prev{0.0, 0.0};
  bool have_prev = false;
  size_t ring_n = 0;
  for (int sgi = 0; sgi <= cut_seg; ++sgi) {
    const size_t end = sgi == cut_seg ? cut_idx : seg_len[sgi];
    const Pt* p = seg_ptr[sgi];
    size_t j = 0;
    for (; j < end && phase != 2; ++j) {
      if (have_prev && same(prev, p[j])) continue;
      prev = p[j];
      have_prev = true;
      ++ring_n;
      feed(p[j]);
    }
    if (j == end) continue;
    // The deque loop proper, with every piece of state in locals that no
    // store through the deque pointers can alias (the lambda's captures
    // would be reloaded after each deque store).
    Pt* h = head;
    Pt* t = tail;
    double h_ax = hax, h_ay = hay, h_ex = hex, h_ey = hey;
    double t_ax = tax, t_ay = tay, t_ex = tex, t_ey = tey;
    double qx = prev.x, qy = prev.y;  // have_prev holds in phase 2
    size_t fed = 0;
    for (; j < end; ++j) {
      const double vx = p[j].x, vy = p[j].y;
      if (vx == qx && vy == qy) continue;  // consecutive duplicate (polygon.cpp:16-18)
      qx = vx;
      qy = vy;
      ++fed;
      const bool left_head = h_ex * (vy - h_ay) - h_ey * (vx - h_ax) > 0.0;
      const bool left_tail = t_ex * (vy - t_ay) - t_ey * (vx - t_ax) > 0.0;
      if (left_head & left_tail) continue;  // inside the hull so far: ~70% of chain points
      if (!left_tail && t - h >= 2) {
        --t;
        while (t - h >= 2) {
          const Pt a = t[-2], b = t[-1];
          if ((b.x - a.x) * (vy - a.y) - (b.y - a.y) * (vx - a.x) > 0.0) break;
          --t;
        }
      }
      *t++ = Pt{vx, vy};
      while (t - h >= 2) {
        const Pt a = h[0], b = h[1];
        if ((a.x - vx) * (b.y - vy) - (a.y - vy) * (b.x - vx) > 0.0) break;
        ++h;
      }
      *--h = Pt{vx, vy};
      h_ax = vx;
      h_ay = vy;
      h_ex = h[1].x - vx;
      h_ey = h[1].y - vy;
      t_ax = t[-2].x;
      t_ay = t[-2].y;
      t_ex = t[-1].x - t_ax;
      t_ey = t[-1].y - t_ay;
    }
    head = h;
    tail = t;
    hax = h_ax, hay = h_ay, hex = h_ex, hey = h_ey;
    tax = t_ax, tay = t_ay, tex = t_ex, tey = t_ey;
    prev = Pt{qx, qy};
    ring_n += fed;
  }
  // the trailing run: one vertex unless it repeats the previous one or
  // closes the ring onto corner 0 (when the ring has more than one vertex)
  if (!(have_prev && same(prev, last_pt)) && !(drop_last && ring_n >= 1)) {
    ++ring_n;
    feed(last_pt);
  }
  if (phase != 2) return kDegenerate;

  // hull = deque [head, tail - 1) rotated to its first lexicographic
  // minimum (canonicalize_ring), written once.
  const size_t m = (size_t)(tail - 1 - head);
  size_t lo_i = 0;
  for (size_t i = 1; i < m; ++i)
    if (lex_less(head[i], head[lo_i])) lo_i = i;
  hull.resize(m);
  std::memcpy(hull.data(), head + lo_i, (m - lo_i) * sizeof(Pt));
  std::memcpy(hull.data() + (m - lo_i), head, lo_i * sizeof(Pt));
  return kOk;
}

// ------------------------------------------------------------------
// The split finisher: finish_chains with the four chain segments run
// concurrently, bit-identical by construction.
//
// Segment A is the ring up to and including corner B (L, chain 1, B),
// segment B is chain 2 and corner R, segment C is chain 3 and corner T,
// segment D is chain 4 with the closing logic. A runs exactly like
// finish_chains. B, C and D run Melkman's deque loop speculatively on a
// local model of the deque they will meet: their own corner K at the back
// (with an unknown vertex Y below it) and at the front (with the ring's first
// vertex L and an unknown vertex X beyond it). Every predicate they evaluate
// uses the same expression as finish_chains on the same values, except the
// ones touching X or Y: those take the outcome "strictly left" (no pop), and
// the point is recorded. Popping K or L aborts. Once A (and B, for C) are
// done, X and Y are known: the recorded predicates are evaluated for real,
// and the handover states are checked (A's deque is [B, L, X, …, Y, B]; B
// ends as [R, L, …, R]). Only if every check holds is the merged deque the one
// the sequential pass would hold after corner T; otherwise the sequential
// pass runs. The checks cost a few predicates per chain.

namespace {

inline double turn_v(const Pt& a, const Pt& b, double vx, double vy) {  // turn(a, b, v)
  return (b.x - a.x) * (vy - a.y) - (b.y - a.y) * (vx - a.x);
}
inline double turn_front(double vx, double vy, const Pt& a, const Pt& b) {  // turn(v, a, b)
  return (a.x - vx) * (b.y - vy) - (a.y - vy) * (b.x - vx);
}

// Melkman's deque loop (melkman.cpp:62-80) over p[0, len), consecutive
// duplicates of (qx, qy) dropped: the same steps as finish_chains' loop.
void deque_loop(Pt*& hp, Pt*& tp, const Pt* p, size_t len, double& qx, double& qy) {
  Pt* h = hp;
  Pt* t = tp;
  double h_ax = h[0].x, h_ay = h[0].y, h_ex = h[1].x - h_ax, h_ey = h[1].y - h_ay;
  double t_ax = t[-2].x, t_ay = t[-2].y, t_ex = t[-1].x - t_ax, t_ey = t[-1].y - t_ay;
  for (size_t j = 0; j < len; ++j) {
    const double vx = p[j].x, vy = p[j].y;
    if (vx == qx && vy == qy) continue;
    qx = vx;
    qy = vy;
    const bool left_head = h_ex * (vy - h_ay) - h_ey * (vx - h_ax) > 0.0;
    const bool left_tail = t_ex * (vy - t_ay) - t_ey * (vx - t_ax) > 0.0;
    if (left_head & left_tail) continue;
    if (!left_tail && t - h >= 2) {
      --t;
      while (t - h >= 2) {
        const Pt a = t[-2], b = t[-1];
        if ((b.x - a.x) * (vy - a.y) - (b.y - a.y) * (vx - a.x) > 0.0) break;
        --t;
      }
    }
    *t++ = Pt{vx, vy};
    while (t - h >= 2) {
      const Pt a = h[0], b = h[1];
      if ((a.x - vx) * (b.y - vy) - (a.y - vy) * (b.x - vx) > 0.0) break;
      ++h;
    }
    *--h = Pt{vx, vy};
    h_ax = vx;
    h_ay = vy;
    h_ex = h[1].x - vx;
    h_ey = h[1].y - vy;
    t_ax = t[-2].x;
    t_ay = t[-2].y;
    t_ex = t[-1].x - t_ax;
    t_ey = t[-1].y - t_ay;
  }
  hp = h;
  tp = t;
}

// Segment A: phase A (collinear run, seed) then the deque loop, over the
// ring points of `segs` (finish_chains' feed + loop). Returns false if the
// deque was never seeded.
bool run_prefix(const Pt* const* sp, const size_t* sl, int nseg, Pt*& head, Pt*& tail, double& qx,
                double& qy) {
  int phase = 0;
  Pt lo{0, 0}, hi{0, 0}, last{0, 0};
  bool have_prev = false;
  for (int s = 0; s < nseg; ++s) {
    const Pt* p = sp[s];
    size_t j = 0;
    for (; j < sl[s] && phase != 2; ++j) {
      const Pt v = p[j];
      if (have_prev && v.x == qx && v.y == qy) continue;
      qx = v.x;
      qy = v.y;
      have_prev = true;
      if (phase == 0) {
        lo = hi = last = v;
        phase = 1;
        continue;
      }
      if (turn(lo, hi, v) == 0) {
        if (lex_less(v, lo))
          lo = v;
        else if (lex_less(hi, v))
          hi = v;
        last = v;
        continue;
      }
      const Pt second = last;
      const Pt first = same(last, lo) ? hi : lo;
      const bool ccw = turn(first, second, v) == kLeft;
      *tail++ = v;
      *tail++ = ccw ? first : second;
      *tail++ = ccw ? second : first;
      *tail++ = v;
      phase = 2;
    }
    if (j < sl[s]) deque_loop(head, tail, p + j, sl[s] - j, qx, qy);
  }
  return phase == 2;
}

// Segments B / C: the deque loop on the local model (see above).
struct SpecRun {
  Pt K, L;                    // own corner (back base, first front element), ring start
  Scratch bks, frs;           // stack storage (grows only)
  Pt* bk = nullptr;           // back stack above K, bk[nb - 1] = tail[-1]
  Pt* fr = nullptr;           // front stack before L, fr[nf - 1] = head[0]
  size_t nb = 0, nf = 0;
  std::vector<Pt> xt;         // v with turn(v, L, X) taken as > 0
  std::vector<Pt> yt;         // v with turn(Y, K, v) taken as > 0
  bool ok = true;

  // chain p[0, len), then the next corner `end` (also a ring point) unless
  // !with_end (chain 4 closing onto corner 0). The end edges are cached as
  // in deque_loop (same rounded differences as turn()).
  void run(const Pt* p, size_t len, const Pt& end, bool with_end = true) {
    bk = bks.get(len + 2);
    fr = frs.get(len + 3);
    nb = 0;
    nf = 0;
    xt.clear();
    yt.clear();
    fr[nf++] = K;
    ok = true;
    double qx = K.x, qy = K.y;
    double h_ax = K.x, h_ay = K.y, h_ex = L.x - K.x, h_ey = L.y - K.y;
    double t_ax = 0, t_ay = 0, t_ex = 0, t_ey = 0;  // (unused while nb == 0: Y is unknown)
    const size_t n = len + (with_end ? 1 : 0);
    for (size_t j = 0; j < n; ++j) {
      const double vx = j < len ? p[j].x : end.x, vy = j < len ? p[j].y : end.y;
      if (vx == qx && vy == qy) continue;
      qx = vx;
      qy = vy;
      const bool left_head = h_ex * (vy - h_ay) - h_ey * (vx - h_ax) > 0.0;
      bool left_tail;
      if (nb == 0) {  // turn(Y, K, v)
        yt.push_back(Pt{vx, vy});
        left_tail = true;
      } else {
        left_tail = t_ex * (vy - t_ay) - t_ey * (vx - t_ax) > 0.0;
      }
      if (left_head & left_tail) continue;
      if (!left_tail) {
        --nb;  // (left_tail is false only with nb > 0)
        for (;;) {
          if (nb == 0) {
            yt.push_back(Pt{vx, vy});
            break;
          }
          const Pt& t1 = bk[nb - 1];
          const Pt& t0 = nb >= 2 ? bk[nb - 2] : K;
          if (turn_v(t0, t1, vx, vy) > 0.0) break;
          --nb;
        }
      }
      const Pt t0 = nb >= 1 ? bk[nb - 1] : K;  // the new tail edge: (t0, v)
      bk[nb++] = Pt{vx, vy};
      for (;;) {
        if (nf == 0) {  // turn(v, L, X)
          xt.push_back(Pt{vx, vy});
          break;
        }
        const Pt& a = fr[nf - 1];
        const Pt& b = nf >= 2 ? fr[nf - 2] : L;
        if (turn_front(vx, vy, a, b) > 0.0) break;
        --nf;
      }
      const Pt h1 = nf >= 1 ? fr[nf - 1] : L;  // the new front edge: (v, h1)
      fr[nf++] = Pt{vx, vy};
      h_ax = vx;
      h_ay = vy;
      h_ex = h1.x - vx;
      h_ey = h1.y - vy;
      t_ax = t0.x;
      t_ay = t0.y;
      t_ex = vx - t0.x;
      t_ey = vy - t0.y;
    }
  }
  // the recorded predicates with the real X and Y
  bool verify(const Pt& X, const Pt& Y) const {
    for (const Pt& v : xt)
      if (!(turn_front(v.x, v.y, L, X) > 0.0)) return false;
    for (const Pt& v : yt)
      if (!(turn_v(Y, K, v.x, v.y) > 0.0)) return false;
    return true;
  }
};

// One pause of a spin loop (x86 PAUSE, aarch64 YIELD).
inline void cpu_relax() {
#if defined(__x86_64__) || defined(__i386__)
  __builtin_ia32_pause();
#elif defined(__aarch64__) || defined(__arm__)
  asm volatile("yield" ::: "memory");
#endif
}

using Clock = std::chrono::steady_clock;

// How long a worker spins for a job before it parks: after a job, and after
// finisher_prewake() (a call on its way to the finisher). A wake-up from the
// parked state costs tens of microseconds; a spin costs a core.
Clock::duration spin_budget() {
  static const Clock::duration d = [] {
    const char* e = std::getenv("CHGPU_FINISH_SPIN_US");  // tuning knob
    return std::chrono::duration_cast<Clock::duration>(
        std::chrono::microseconds(e ? std::strtol(e, nullptr, 10) : 1000));
  }();
  return d;
}

// A worker thread for segment B, C or D: parked on a condition variable
// while idle; spins (bounded by a steady_clock deadline) only after a job
// or a pre-wake, so an idle library burns no host cores.
struct Worker {
  std::thread th;
  std::mutex m;
  std::condition_variable cv;
  std::function<void()> job;
  std::atomic<int> state{0};  // 0 idle, 1 job ready, 2 job done
  std::atomic<bool> parked{false};
  std::atomic<long long> spin_until{0};  // steady_clock ticks: spin (not park) until then
  void start() {
    th = std::thread([this] {
      for (;;) {
        for (unsigned i = 0; state.load(std::memory_order_acquire) != 1; ++i) {
          if ((i & 63) == 0 &&
              Clock::now().time_since_epoch().count() >= spin_until.load(std::memory_order_relaxed)) {
            std::unique_lock<std::mutex> lk(m);
            parked.store(true);
            cv.wait(lk, [this] {
              return state.load(std::memory_order_acquire) == 1 ||
                     Clock::now().time_since_epoch().count() <
                         spin_until.load(std::memory_order_relaxed);
            });
            parked.store(false);
            continue;
          }
          cpu_relax();
        }
        job();
        spin_until.store((Clock::now() + spin_budget()).time_since_epoch().count(),
                         std::memory_order_relaxed);
        state.store(2, std::memory_order_release);
      }
    });
  }
  // (never destroyed: see WorkerPool)
  void wake() {  // spin from now on for a while: a job is on its way
    spin_until.store((Clock::now() + spin_budget()).time_since_epoch().count(),
                     std::memory_order_relaxed);
    if (parked.load()) {
      std::lock_guard<std::mutex> lk(m);
      cv.notify_all();
    }
  }
  void submit(std::function<void()> j) {
    job = std::move(j);
    {
      std::lock_guard<std::mutex> lk(m);  // (orders the job before a parked wait re-checks)
      state.store(1, std::memory_order_release);
    }
    if (parked.load()) cv.notify_all();
  }
  void wait() {
    while (state.load(std::memory_order_acquire) != 2) cpu_relax();
    state.store(0, std::memory_order_relaxed);
  }
};

// The process's three workers. Created on first use and never destroyed (the
// threads end with the process); a forked child (whose copy has no threads)
// makes its own. If the threads cannot be started, the failure is
// remembered for this process and every call takes the sequential pass.
struct WorkerPool {
  Worker b, c, d;
  pid_t pid = getpid();
};
WorkerPool* worker_pool() {  // nullptr if threads cannot be made here
  static std::mutex mu;
  static WorkerPool* pool = nullptr;
  static pid_t failed_pid = 0;
  std::lock_guard<std::mutex> lk(mu);
  const pid_t me = getpid();
  if (pool && pool->pid == me) return pool;
  if (failed_pid == me) return nullptr;
  // (a pool whose threads could not all start is kept alive, unused: its
  // running threads still reference it)
  WorkerPool* p = new (std::nothrow) WorkerPool;
  try {
    if (!p) throw std::bad_alloc();
    p->b.start();
    p->c.start();
    p->d.start();
    pool = p;
  } catch (...) {
    failed_pid = me;
    pool = nullptr;
  }
  return pool;
}

std::atomic<unsigned long long> g_split_taken{0}, g_split_fallback{0};
// the last split call's segment times (µs from the submit: A, B, C, D, all
// joined) and its total (set after the merge)
double g_seg_us[6] = {0, 0, 0, 0, 0, 0};

size_t split_min() {
  static const size_t v = [] {
    const char* e = std::getenv("CHGPU_FINISH_SPLIT_MIN");
    return e ? (size_t)std::strtoull(e, nullptr, 10) : (size_t)2048;
  }();
  return v;
}

}  // namespace

void finisher_prewake(size_t expected_chain_points) {
  if (expected_chain_points < 4 * split_min()) return;
  if (WorkerPool* pool = worker_pool()) {
    pool->b.wake();
    pool->c.wake();
    pool->d.wake();
  }
}

int finish_chains_split(const Pt* chains, const size_t kept_counts[4], const Pt corners[4],
                        std::vector<Pt>& hull) {
  for (int r = 0; r < 4; ++r)
    if (kept_counts[r] < split_min() || kept_counts[r] < 8)
      return finish_chains(chains, kept_counts, corners, hull);
  const Pt* c[4];
  c[0] = chains;
  for (int r = 1; r < 4; ++r) c[r] = c[r - 1] + kept_counts[r - 1];
  // the closing logic of finish_chains stays simple when chain 4's trailing
  // run of its last point does not reach back to corner T
  const Pt last_pt = c[3][kept_counts[3] - 1];
  size_t cut = kept_counts[3] - 1;
  while (cut > 0 && same(c[3][cut - 1], last_pt)) --cut;
  if (cut == 0) return finish_chains(chains, kept_counts, corners, hull);

  size_t total = 4;
  for (int r = 0; r < 4; ++r) total += kept_counts[r];
  thread_local Scratch deque_s;
  Pt* buf = deque_s.get(2 * total + 8);
  Pt* head = buf + total + 4;
  Pt* tail = head;

  // the workers serve one call at a time (concurrent calls on other
  // contexts take the sequential pass)
  static std::mutex busy;
  std::unique_lock<std::mutex> own(busy, std::try_to_lock);
  if (!own.owns_lock()) return finish_chains(chains, kept_counts, corners, hull);
  WorkerPool* const pool = worker_pool();
  if (!pool) return finish_chains(chains, kept_counts, corners, hull);
  static SpecRun sb, sc, sd;
  sb.K = corners[1];
  sc.K = corners[2];
  sd.K = corners[3];
  sb.L = sc.L = sd.L = corners[0];
  // B: chain 2 then corner R; C: chain 3 then corner T; D: chain 4 up to
  // its trailing run, then the run's one vertex unless it closes the ring
  // onto corner 0 (finish_chains' closing logic; a repeat of the previous
  // ring point drops as a consecutive duplicate)
  const bool drop_last = same(last_pt, corners[0]);
  const auto t_sub = Clock::now();
  double seg_us[4] = {0, 0, 0, 0};
  auto us_since = [&](Clock::time_point a) {
    return std::chrono::duration<double, std::micro>(Clock::now() - a).count();
  };
  pool->b.submit([&] { sb.run(c[1], kept_counts[1], corners[2]); seg_us[1] = us_since(t_sub); });
  pool->c.submit([&] { sc.run(c[2], kept_counts[2], corners[3]); seg_us[2] = us_since(t_sub); });
  pool->d.submit([&] { sd.run(c[3], cut, last_pt, !drop_last); seg_us[3] = us_since(t_sub); });
  double qx = 0, qy = 0;
  const Pt* sp[3] = {&corners[0], c[0], &corners[1]};
  const size_t sl[3] = {1, kept_counts[0], 1};
  const bool seeded = run_prefix(sp, sl, 3, head, tail, qx, qy);
  seg_us[0] = us_since(t_sub);
  pool->b.wait();
  pool->c.wait();
  pool->d.wait();
  for (int q = 0; q < 4; ++q) g_seg_us[q] = seg_us[q];  // (diagnostics: chgpu_finish_split_times)
  g_seg_us[4] = us_since(t_sub);

  // handover checks: A ends as [B, L, X, ..., Y, B]; B as [R, L, ..., R]; C as [T, L, ..., T]
  bool ok = seeded && sb.ok && sc.ok && sd.ok && tail - head >= 5 && same(head[0], corners[1]) &&
            same(head[1], corners[0]) && same(tail[-1], corners[1]);
  ok = ok && sb.nf == 1 && same(sb.fr[0], corners[2]) && sb.nb > 0 &&
       same(sb.bk[sb.nb - 1], corners[2]);
  ok = ok && sc.nf == 1 && same(sc.fr[0], corners[3]) && sc.nb > 0 &&
       same(sc.bk[sc.nb - 1], corners[3]);
  if (ok) {
    const Pt X = head[2], Y = tail[-2];
    const Pt YC = sb.nb >= 2 ? sb.bk[sb.nb - 2] : corners[1];
    const Pt YD = sc.nb >= 2 ? sc.bk[sc.nb - 2] : corners[2];
    ok = sb.verify(X, Y) && sc.verify(X, YC) && sd.verify(X, YD);
  }
  if (!ok) {
    g_split_fallback.fetch_add(1, std::memory_order_relaxed);
    return finish_chains(chains, kept_counts, corners, hull);
  }
  g_split_taken.fetch_add(1, std::memory_order_relaxed);

  // the final deque: D's front stack, then A's [L, X, ..., Y, B] (its front
  // copy of B was popped by R's front pops), then the back stacks of B, C, D
  Pt* h = head + 1 - (ptrdiff_t)sd.nf;
  for (size_t i = 0; i < sd.nf; ++i) h[i] = sd.fr[sd.nf - 1 - i];
  head = h;
  for (const SpecRun* sr : {&sb, &sc, &sd}) {
    std::memcpy(tail, sr->bk, sr->nb * sizeof(Pt));
    tail += sr->nb;
  }
  const size_t m = (size_t)(tail - 1 - head);
  size_t lo_i = 0;
  for (size_t i = 1; i < m; ++i)
    if (lex_less(head[i], head[lo_i])) lo_i = i;
  hull.resize(m);
  std::memcpy(hull.data(), head + lo_i, (m - lo_i) * sizeof(Pt));
  std::memcpy(hull.data() + (m - lo_i), head, lo_i * sizeof(Pt));
  g_seg_us[5] = us_since(t_sub);
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

namespace chgpu {
namespace host {

// region_less (spa.cpp:38-52) on points, with == ties (the chains' order).
static inline bool region_before(int region, const Pt& a, const Pt& b) {
  switch (region) {
    case 1: return a.x < b.x || (a.x == b.x && a.y > b.y);  // LL: x asc, y desc
    case 2: return a.y < b.y || (a.y == b.y && a.x < b.x);  // LR: y asc, x asc
    case 3: return a.x > b.x || (a.x == b.x && a.y < b.y);  // UR: x desc, y asc
    default: return a.y > b.y || (a.y == b.y && a.x > b.x); // UL: y desc, x desc
  }
}

int merge_chains_hull(const Pt* const* runs, const size_t* counts4, int nruns, const Pt corners[4],
                      std::vector<Pt>& hull) {
  // per region, the runs' chains (each sorted in region order) merged into
  // one sorted chain, ties to the earlier run
  size_t total[4] = {0, 0, 0, 0};
  for (int k = 0; k < nruns; ++k)
    for (int r = 0; r < 4; ++r) total[r] += counts4[4 * k + r];
  finisher_prewake(total[0] + total[1] + total[2] + total[3]);  // (workers wake during the merge)
  if (nruns == 1) return finish_chains_split(runs[0], total, corners, hull);
  std::vector<Pt> merged(total[0] + total[1] + total[2] + total[3]);
  std::vector<size_t> pos(nruns);
  std::vector<const Pt*> start(nruns);
  for (int k = 0; k < nruns; ++k) start[k] = runs[k];
  Pt* out = merged.data();
  for (int r = 0; r < 4; ++r) {
    for (int k = 0; k < nruns; ++k) pos[k] = 0;
    for (size_t i = 0; i < total[r]; ++i) {
      int best = -1;
      for (int k = 0; k < nruns; ++k) {
        if (pos[k] == counts4[4 * k + r]) continue;
        if (best < 0 || region_before(r + 1, start[k][pos[k]], start[best][pos[best]])) best = k;
      }
      *out++ = start[best][pos[best]++];
    }
    for (int k = 0; k < nruns; ++k) start[k] += counts4[4 * k + r];
  }
  return finish_chains_split(merged.data(), total, corners, hull);
}

}  // namespace host
}  // namespace chgpu

extern "C" int chgpu_merge_hull(const double* const* runs, const size_t* kept_counts, int nruns,
                                const double* quad, double* out, size_t* n_out) {
  std::vector<Pt> hull;
  const int st = chgpu::host::merge_chains_hull(reinterpret_cast<const Pt* const*>(runs), kept_counts,
                                                nruns, reinterpret_cast<const Pt*>(quad), hull);
  if (st) {
    *n_out = 0;
    return st;
  }
  std::memcpy(out, hull.data(), hull.size() * sizeof(Pt));
  *n_out = hull.size();
  return 0;
}

extern "C" int chgpu_finish_chains(const double* chains, const size_t* kept_counts,
                                   const double* quad, double* out, size_t* n_out) {
  std::vector<Pt> hull;
  const int st = chgpu::host::finish_chains_split(reinterpret_cast<const Pt*>(chains), kept_counts,
                                                  reinterpret_cast<const Pt*>(quad), hull);
  if (st) {
    *n_out = 0;
    return st;
  }
  std::memcpy(out, hull.data(), hull.size() * sizeof(Pt));
  *n_out = hull.size();
  return 0;
}

// Split-finisher counters (tests): calls that took the concurrent path, and
// calls whose checks sent them to the sequential pass.
extern "C" void chgpu_finish_split_times(double* out6) {
  for (int q = 0; q < 6; ++q) out6[q] = chgpu::host::g_seg_us[q];
}

extern "C" void chgpu_finish_split_stats(unsigned long long* taken, unsigned long long* fallback) {
  *taken = chgpu::host::g_split_taken.load();
  *fallback = chgpu::host::g_split_fallback.load();
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
