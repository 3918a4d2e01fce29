/* TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT (see chainhull_oracle.h).
 *
 * A plain-C restatement of the reference CPU path, one function per
 * reference function, each citing the file:line it follows
 * (paths relative to /root/reference/proj/core). Built with
 * -ffp-contract=off so cross() is evaluated exactly as the reference's
 * Release build evaluates it (two roundings for the products, one for the
 * difference, no FMA).
 */
#include "chainhull_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---- geometry.hpp:8-44 ------------------------------------------------- */

static int pt_eq(orc_pt a, orc_pt b) { return a.x == b.x && a.y == b.y; } /* :12-14 */

static double cross(orc_pt a, orc_pt b, orc_pt p) { /* :22-24 */
  return (b.x - a.x) * (p.y - a.y) - (b.y - a.y) * (p.x - a.x);
}

enum { LEFT = 0, RIGHT = 1, COLLINEAR = 2 };

static int orient(orc_pt a, orc_pt b, orc_pt p) { /* :30-35 */
  const double c = cross(a, b, p);
  if (c > 0.0) return LEFT;
  if (c < 0.0) return RIGHT;
  return COLLINEAR;
}

static int less_xy(orc_pt a, orc_pt b) { return a.x < b.x || (a.x == b.x && a.y < b.y); } /* :39-41 */
static int less_yx(orc_pt a, orc_pt b) { return a.y < b.y || (a.y == b.y && a.x < b.x); } /* :42-44 */

/* ---- datasets.cpp:17-106 ----------------------------------------------- */

typedef struct {
  uint64_t mt[312];
  int i;
} mt64;

static void mt64_seed(mt64* g, uint64_t seed) { /* std::mt19937_64(seed) */
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->i = 312;
}

static uint64_t mt64_next(mt64* g) {
  if (g->i >= 312) {
    for (int k = 0; k < 312; ++k) {
      const uint64_t y = (g->mt[k] & 0xFFFFFFFF80000000ULL) | (g->mt[(k + 1) % 312] & 0x7FFFFFFFULL);
      g->mt[k] = g->mt[(k + 156) % 312] ^ (y >> 1) ^ ((y & 1ULL) ? 0xB5026F5AA96619E9ULL : 0ULL);
    }
    g->i = 0;
  }
  uint64_t x = g->mt[g->i++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}

static double unit_double(mt64* g) { return (double)(mt64_next(g) >> 11) * 0x1.0p-53; } /* :17-19 */

static const double kPi = 3.141592653589793; /* std::numbers::pi */

int orc_generate(int dist, size_t n, uint64_t seed, orc_pt* out) {
  if (n == 0) return 3; /* :95 */
  mt64* g = (mt64*)malloc(sizeof(mt64));
  mt64_seed(g, seed);
  switch (dist) {
    case 0: /* uniform_square :21-28 */
      for (size_t i = 0; i < n; ++i) {
        out[i].x = unit_double(g);
        out[i].y = unit_double(g);
      }
      break;
    case 1: /* uniform_disk :30-39 */
      for (size_t i = 0; i < n; ++i) {
        const double r = sqrt(unit_double(g));
        const double theta = 2.0 * kPi * unit_double(g);
        out[i].x = r * cos(theta);
        out[i].y = r * sin(theta);
      }
      break;
    case 2: { /* circle :41-52 */
      const double phase = 2.0 * kPi * unit_double(g);
      for (size_t i = 0; i < n; ++i) {
        const double theta = phase + 2.0 * kPi * (double)i / (double)n;
        out[i].x = cos(theta);
        out[i].y = sin(theta);
      }
      break;
    }
    case 3: /* gaussian :54-66 */
      for (size_t i = 0; i < n; ++i) {
        const double u1 = 1.0 - unit_double(g);
        const double u2 = unit_double(g);
        const double mag = sqrt(-2.0 * log(u1));
        out[i].x = mag * cos(2.0 * kPi * u2);
        out[i].y = mag * sin(2.0 * kPi * u2);
      }
      break;
    case 4: /* collinear :68-79 */
      for (size_t i = 0; i < n; ++i) {
        const double u = unit_double(g);
        out[i].x = u;
        out[i].y = u;
      }
      break;
    case 5: /* duplicates_heavy :81-90 */
      for (size_t i = 0; i < n; ++i) {
        out[i].x = (double)(mt64_next(g) % 9) / 8.0;
        out[i].y = (double)(mt64_next(g) % 9) / 8.0;
      }
      break;
    default:
      free(g);
      return 3;
  }
  free(g);
  return 0;
}

/* ---- extremes.cpp:12-57 ------------------------------------------------ */

int orc_find_extremes(const orc_pt* p, size_t n, orc_pt quad[4]) {
  if (n == 0) return 1; /* :29 */
  orc_pt l = p[0], b = p[0], r = p[0], t = p[0]; /* reduce_range :21 */
  for (size_t i = 1; i < n; ++i) { /* fold :12-17 */
    if (less_xy(p[i], l)) l = p[i];
    if (less_yx(p[i], b)) b = p[i];
    if (less_xy(r, p[i])) r = p[i];
    if (less_yx(t, p[i])) t = p[i];
  }
  quad[0] = l;
  quad[1] = b;
  quad[2] = r;
  quad[3] = t;
  return 0;
}

size_t orc_frame_vertices(const orc_pt quad[4], orc_pt out[4]) { /* :49-57 */
  size_t k = 0;
  for (int c = 0; c < 4; ++c)
    if (k == 0 || !pt_eq(out[k - 1], quad[c])) out[k++] = quad[c];
  if (k > 1 && pt_eq(out[0], out[k - 1])) --k;
  return k;
}

/* ---- classify.hpp:42-48 ------------------------------------------------ */

int orc_classify_point(orc_pt p, const orc_pt q[4]) {
  if (orient(q[0], q[1], p) == RIGHT) return 1;
  if (orient(q[1], q[2], p) == RIGHT) return 2;
  if (orient(q[2], q[3], p) == RIGHT) return 3;
  if (orient(q[3], q[0], p) == RIGHT) return 4;
  return 0;
}

void orc_classify_points(const orc_pt* p, size_t n, const orc_pt quad[4], uint8_t* labels) {
  for (size_t i = 0; i < n; ++i) labels[i] = (uint8_t)orc_classify_point(p[i], quad); /* classify.cpp:20-27 */
}

/* ---- spa.cpp:10-169 ---------------------------------------------------- */

static int region_less(int region, orc_pt a, orc_pt b) { /* :38-52 */
  switch (region) {
    case 1: return a.x < b.x || (a.x == b.x && a.y > b.y);
    case 2: return a.y < b.y || (a.y == b.y && a.x < b.x);
    case 3: return a.x > b.x || (a.x == b.x && a.y < b.y);
    case 4: return a.y > b.y || (a.y == b.y && a.x > b.x);
  }
  return 0;
}

#define DEFINE_CMP(R)                                                  \
  static int cmp_r##R(const void* pa, const void* pb) {                \
    const orc_pt a = *(const orc_pt*)pa, b = *(const orc_pt*)pb;       \
    return region_less(R, a, b) ? -1 : (region_less(R, b, a) ? 1 : 0); \
  }
DEFINE_CMP(1)
DEFINE_CMP(2)
DEFINE_CMP(3)
DEFINE_CMP(4)

int orc_sort_region(int region, orc_pt* seg, size_t m) { /* :59-81 */
  int (*cmp)(const void*, const void*) = NULL;
  switch (region) {
    case 1: cmp = cmp_r1; break;
    case 2: cmp = cmp_r2; break;
    case 3: cmp = cmp_r3; break;
    case 4: cmp = cmp_r4; break;
    default: return 3; /* :80 */
  }
  if (m > 1) qsort(seg, m, sizeof(orc_pt), cmp);
  return 0;
}

static double guarded(int region, orc_pt p) { return (region == 1 || region == 3) ? p.y : p.x; } /* :86-88 */

static int steps_back(int region, double g, double t) { /* :92-105 */
  switch (region) {
    case 1: return g > t;
    case 2: return g < t;
    case 3: return g < t;
    case 4: return g > t;
  }
  return 0;
}

int orc_spa_filter(int region, const orc_pt* seg, size_t m, const orc_pt anchors[2],
                   size_t chunk_count, orc_pt* out, size_t* nout) {
  if (chunk_count == 0) return 3; /* :112-113 */
  *nout = 0;
  if (m == 0) return 0;                                          /* :119 */
  const size_t chunk_size = (m + chunk_count - 1) / chunk_count; /* :121 */
  const size_t chunks = (m + chunk_size - 1) / chunk_size;       /* :122 */
  size_t k = 0;
  for (size_t c = 0; c < chunks; ++c) { /* scan_chunk :125-147 */
    const size_t begin = c * chunk_size;
    const size_t end = begin + chunk_size < m ? begin + chunk_size : m;
    size_t i = begin;
    double t;
    if (c == 0) {
      t = guarded(region, anchors[0]);
    } else {
      out[k++] = seg[i];
      t = guarded(region, seg[i]);
      ++i;
    }
    for (; i < end; ++i) {
      const double g = guarded(region, seg[i]);
      if (!steps_back(region, g, t)) {
        out[k++] = seg[i];
        t = g;
      }
    }
  }
  *nout = k;
  return 0;
}

/* ---- polygon.cpp:7-29 -------------------------------------------------- */

int orc_assemble_polygon(const orc_pt* chains, const size_t kept_counts[4],
                         const orc_pt quad[4], orc_pt* out, size_t* nout) {
  size_t k = 0, off = 0;
  for (int r = 0; r < 4; ++r) {
    if (k == 0 || !pt_eq(out[k - 1], quad[r])) out[k++] = quad[r];
    for (size_t j = 0; j < kept_counts[r]; ++j) {
      const orc_pt p = chains[off + j];
      if (k == 0 || !pt_eq(out[k - 1], p)) out[k++] = p;
    }
    off += kept_counts[r];
  }
  if (k > 1 && pt_eq(out[0], out[k - 1])) --k; /* :24 */
  *nout = k;
  return k < 3 ? 2 : 0; /* :26-27 */
}

/* ---- melkman.cpp:10-86 ------------------------------------------------- */

static void canonicalize_ring(orc_pt* ring, size_t n) { /* :10-15 */
  if (n < 2) return;
  size_t lo = 0;
  for (size_t i = 1; i < n; ++i)
    if (less_xy(ring[i], ring[lo])) lo = i; /* min_element: first minimum */
  if (lo == 0) return;
  orc_pt* tmp = (orc_pt*)malloc(n * sizeof(orc_pt));
  memcpy(tmp, ring + lo, (n - lo) * sizeof(orc_pt));
  memcpy(tmp + (n - lo), ring, lo * sizeof(orc_pt));
  memcpy(ring, tmp, n * sizeof(orc_pt));
  free(tmp);
}

int orc_melkman(const orc_pt* poly, size_t n_in, orc_pt* out, size_t* nout) {
  /* :20-25 consecutive-duplicate collapse */
  orc_pt* ring = (orc_pt*)malloc((n_in + 1) * sizeof(orc_pt));
  size_t n = 0;
  for (size_t i = 0; i < n_in; ++i)
    if (n == 0 || !pt_eq(ring[n - 1], poly[i])) ring[n++] = poly[i];
  if (n > 1 && pt_eq(ring[0], ring[n - 1])) --n;

  /* :30-47 leading collinear run */
  orc_pt zero = {0.0, 0.0};
  orc_pt lo = n ? ring[0] : zero, hi = lo, last = lo;
  size_t i = 1;
  for (; i < n; ++i) {
    const orc_pt p = ring[i];
    if (orient(lo, hi, p) != COLLINEAR) break;
    if (less_xy(p, lo))
      lo = p;
    else if (less_xy(hi, p))
      hi = p;
    last = p;
  }
  if (i >= n) {
    free(ring);
    return 2;
  }

  /* :52-60 seed; the deque lives in dq[head .. tail) of a 2n+8 array */
  const size_t cap = 2 * n + 8;
  orc_pt* dq = (orc_pt*)malloc(cap * sizeof(orc_pt));
  size_t head = n + 4, tail = head;
  const orc_pt w = ring[i];
  const orc_pt second = last;
  const orc_pt first = pt_eq(last, lo) ? hi : lo;
  dq[tail++] = w;
  if (orient(first, second, w) == LEFT) {
    dq[tail++] = first;
    dq[tail++] = second;
  } else {
    dq[tail++] = second;
    dq[tail++] = first;
  }
  dq[tail++] = w;

  for (++i; i < n; ++i) { /* :62-80 */
    const orc_pt v = ring[i];
    if (orient(dq[head], dq[head + 1], v) == LEFT && orient(dq[tail - 2], dq[tail - 1], v) == LEFT)
      continue;
    while (tail - head >= 2 && orient(dq[tail - 2], dq[tail - 1], v) != LEFT) --tail;
    dq[tail++] = v;
    while (tail - head >= 2 && orient(v, dq[head], dq[head + 1]) != LEFT) ++head;
    dq[--head] = v;
  }

  const size_t h = tail - head - 1; /* :83 */
  memcpy(out, dq + head, h * sizeof(orc_pt));
  canonicalize_ring(out, h);
  *nout = h;
  free(dq);
  free(ring);
  return 0;
}

/* ---- oracle.cpp:12-38 -------------------------------------------------- */

static int cmp_xy(const void* pa, const void* pb) {
  const orc_pt a = *(const orc_pt*)pa, b = *(const orc_pt*)pb;
  return less_xy(a, b) ? -1 : (less_xy(b, a) ? 1 : 0);
}

int orc_hull_oracle(const orc_pt* p, size_t n_in, orc_pt* out, size_t* nout) {
  if (n_in == 0) return 1; /* :13 */
  orc_pt* pts = (orc_pt*)malloc(n_in * sizeof(orc_pt));
  memcpy(pts, p, n_in * sizeof(orc_pt));
  qsort(pts, n_in, sizeof(orc_pt), cmp_xy); /* :16 */
  size_t n = 0;                             /* std::unique :17 */
  for (size_t i = 0; i < n_in; ++i)
    if (n == 0 || !pt_eq(pts[n - 1], pts[i])) pts[n++] = pts[i];
  if (n == 1) {
    out[0] = pts[0];
    *nout = 1;
    free(pts);
    return 0;
  }
  orc_pt* h = (orc_pt*)malloc(2 * n * sizeof(orc_pt));
  size_t k = 0;
  for (size_t i = 0; i < n; ++i) { /* :24-27 */
    while (k >= 2 && orient(h[k - 2], h[k - 1], pts[i]) != LEFT) --k;
    h[k++] = pts[i];
  }
  const size_t lower_end = k + 1;
  for (size_t i = n - 1; i-- > 0;) { /* :29-32 */
    while (k >= lower_end && orient(h[k - 2], h[k - 1], pts[i]) != LEFT) --k;
    h[k++] = pts[i];
  }
  memcpy(out, h, (k - 1) * sizeof(orc_pt)); /* :33 */
  *nout = k - 1;
  free(h);
  free(pts);
  return 0;
}

/* ---- pipeline.cpp:25-106 ----------------------------------------------- */

int orc_convex_hull(const orc_pt* p, size_t n, size_t chunk_count, int degenerate_fallback,
                    orc_pt* out_hull, size_t* nhull, size_t counts[4],
                    size_t region_counts[5], size_t kept_counts[4]) {
  if (n == 0) return 1; /* :27 */
  orc_pt quad[4], frame[4];
  orc_find_extremes(p, n, quad);                   /* :36 */
  const size_t nf = orc_frame_vertices(quad, frame); /* :42 */

  /* classify (:45) + discard_round1 (:49): survivors grouped in block
   * order LL, LR, UR, UL (the reference partition is unstable; the blocks
   * are fully re-sorted next, so a stable grouping is equivalent). */
  unsigned char* lab = (unsigned char*)malloc(n);
  size_t rc[5] = {0, 0, 0, 0, 0};
  for (size_t i = 0; i < n; ++i) {
    lab[i] = (unsigned char)orc_classify_point(p[i], quad);
    ++rc[lab[i]];
  }
  size_t off[5];
  off[1] = 0;
  off[2] = rc[1];
  off[3] = off[2] + rc[2];
  off[4] = off[3] + rc[3];
  const size_t s1 = off[4] + rc[4];
  orc_pt* surv = (orc_pt*)malloc((s1 + 4) * sizeof(orc_pt));
  size_t cur[5] = {0, off[1], off[2], off[3], off[4]};
  for (size_t i = 0; i < n; ++i)
    if (lab[i]) surv[cur[lab[i]]++] = p[i];
  free(lab);
  for (int r = 0; r < 5; ++r) region_counts[r] = rc[r];
  counts[0] = n;
  counts[1] = s1 + nf; /* :51 */
  for (int r = 0; r < 4; ++r) kept_counts[r] = 0;

  int st = 0;
  if (nf <= 2) { /* :53-71 */
    if (!degenerate_fallback) {
      free(surv);
      return 2;
    }
    counts[2] = counts[1];
    memcpy(surv + s1, frame, nf * sizeof(orc_pt));
    st = orc_hull_oracle(surv, s1 + nf, out_hull, nhull);
    counts[3] = *nhull;
    free(surv);
    return st;
  }

  for (int r = 1; r <= 4; ++r) orc_sort_region(r, surv + off[r], rc[r]); /* :73-84 */

  orc_pt* chains = (orc_pt*)malloc((s1 + 1) * sizeof(orc_pt));
  size_t kept = 0;
  for (int r = 1; r <= 4; ++r) { /* :86-96 */
    const orc_pt anchors[2] = {quad[r - 1], quad[r % 4]};
    size_t k = 0;
    st = orc_spa_filter(r, surv + off[r], rc[r], anchors, chunk_count, chains + kept, &k);
    if (st) {
      free(chains);
      free(surv);
      return st;
    }
    kept_counts[r - 1] = k;
    kept += k;
  }
  counts[2] = kept + nf;

  orc_pt* poly = (orc_pt*)malloc((kept + 4) * sizeof(orc_pt));
  size_t npoly = 0;
  st = orc_assemble_polygon(chains, kept_counts, quad, poly, &npoly); /* :99 */
  if (!st) st = orc_melkman(poly, npoly, out_hull, nhull);           /* :100 */
  if (!st) counts[3] = *nhull;
  free(poly);
  free(chains);
  free(surv);
  return st;
}
