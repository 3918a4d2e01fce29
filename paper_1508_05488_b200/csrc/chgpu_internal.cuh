// Device-side building blocks shared by the hull kernels.
//
// Arithmetic contract (reference geometry.hpp:22-35): the orientation
// predicate is evaluated as (b.x-a.x)*(p.y-a.y) - (b.y-a.y)*(p.x-a.x) with
// every operation individually rounded (no FMA). All .cu files are built
// with -fmad=false AND the predicate spells the roundings out with
// __dmul_rn/__dsub_rn, so contraction cannot creep back in.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace chgpu {

typedef unsigned long long u64;
typedef unsigned int u32;

// ---------------------------------------------------------------- geometry

// cross(a, b, p) with a precomputed edge (ex, ey) = (b.x - a.x, b.y - a.y).
// Precomputing the edge is exact: it is the same rounded subtraction the
// reference performs per call.
__device__ __forceinline__ double cross_edge(double ax, double ay, double ex, double ey,
                                             double px, double py) {
  return __dsub_rn(__dmul_rn(ex, __dsub_rn(py, ay)), __dmul_rn(ey, __dsub_rn(px, ax)));
}

// Lexicographic orders (geometry.hpp:39-44).
__device__ __forceinline__ bool less_xy(double ax, double ay, double bx, double by) {
  return ax < bx || (ax == bx && ay < by);
}
__device__ __forceinline__ bool less_yx(double ax, double ay, double bx, double by) {
  return ay < by || (ay == by && ax < bx);
}

// ---------------------------------------------------------------- key codec
//
// Sort records are (k, v) pairs of 64-bit words. k is the region's primary
// coordinate and v its secondary, each mapped by an order-preserving
// bijection of the double's bits (descending orders use the complement),
// so ascending unsigned order on (k, v) is exactly region_less
// (spa.cpp:38-52):
//   region 1 LL: k = ord(x),  v = ~ord(y)   x asc,  ties y desc
//   region 2 LR: k = ord(y),  v = ord(x)    y asc,  ties x asc
//   region 3 UR: k = ~ord(x), v = ord(y)    x desc, ties y asc
//   region 4 UL: k = ~ord(y), v = ~ord(x)   y desc, ties x desc
//   mode 0 LEX : k = ord(x),  v = ord(y)    less_xy (degenerate branch)
// Both maps are bijective, so the point is recovered bit-exactly
// (including the sign of zero). -0.0 and +0.0 are adjacent in k-order and
// are merged into one tie run by prim_eq() below, restoring the
// reference's `==` tie semantics.

__host__ __device__ __forceinline__ u64 dbits(double d) {
#ifdef __CUDA_ARCH__
  return (u64)__double_as_longlong(d);
#else
  u64 u;
  __builtin_memcpy(&u, &d, 8);
  return u;
#endif
}
__host__ __device__ __forceinline__ double bitsd(u64 u) {
#ifdef __CUDA_ARCH__
  return __longlong_as_double((long long)u);
#else
  double d;
  __builtin_memcpy(&d, &u, 8);
  return d;
#endif
}
__host__ __device__ __forceinline__ u64 ord_enc(double d) {
  const u64 b = dbits(d);
  return b ^ ((u64)((long long)b >> 63) | 0x8000000000000000ull);
}
// ord_enc with -0.0 folded onto +0.0 (== does not tell them apart), in
// integer ops only (the same bits as ord_enc(d + 0.0)).
__host__ __device__ __forceinline__ u64 ord_enc_z(double d) {
  const u64 e = ord_enc(d);
  return e == 0x7FFFFFFFFFFFFFFFull ? 0x8000000000000000ull : e;
}
__host__ __device__ __forceinline__ double ord_dec(u64 u) {
  return bitsd(u ^ ((u >> 63) ? 0x8000000000000000ull : 0xFFFFFFFFFFFFFFFFull));
}

// Region codes: 0 = LEX (degenerate branch), 1..4 = LL, LR, UR, UL.
__host__ __device__ __forceinline__ void encode_point(int region, double x, double y, u64& k,
                                                      u64& v) {
  switch (region) {
    case 1: k = ord_enc(x); v = ~ord_enc(y); break;
    case 2: k = ord_enc(y); v = ord_enc(x); break;
    case 3: k = ~ord_enc(x); v = ord_enc(y); break;
    case 4: k = ~ord_enc(y); v = ~ord_enc(x); break;
    default: k = ord_enc(x); v = ord_enc(y); break;
  }
}
__host__ __device__ __forceinline__ void decode_point(int region, u64 k, u64 v, double& x,
                                                      double& y) {
  switch (region) {
    case 1: x = ord_dec(k); y = ord_dec(~v); break;
    case 2: y = ord_dec(k); x = ord_dec(v); break;
    case 3: x = ord_dec(~k); y = ord_dec(v); break;
    case 4: y = ord_dec(~k); x = ord_dec(~v); break;
    default: x = ord_dec(k); y = ord_dec(v); break;
  }
}
// The primary coordinate as a double (for == tie tests).
__host__ __device__ __forceinline__ double primary_of(int region, u64 k) {
  return (region == 3 || region == 4) ? ord_dec(~k) : ord_dec(k);
}
// The SPA guarded coordinate (spa.cpp:86-88) is always the secondary.
__host__ __device__ __forceinline__ double guarded_of(int region, u64 v) {
  return (region == 1 || region == 4) ? ord_dec(~v) : ord_dec(v);
}
// Primary equality under IEEE == (merges -0.0 and +0.0).
__host__ __device__ __forceinline__ bool prim_eq(int region, u64 a, u64 b) {
  return a == b || primary_of(region, a) == primary_of(region, b);
}

// -0.0 as primary compares like +0.0: map its code onto +0.0's.
__host__ __device__ __forceinline__ u64 canon_k(int region, u64 k) {
  const bool desc = (region == 3 || region == 4);
  const u64 neg0 = desc ? ~0x7FFFFFFFFFFFFFFFull : 0x7FFFFFFFFFFFFFFFull;
  const u64 pos0 = desc ? ~0x8000000000000000ull : 0x8000000000000000ull;
  return k == neg0 ? pos0 : k;
}

// region_less (spa.cpp:38-52) on (canonical k, v); ties (==-equal points)
// fall back to the raw k so the order is total on bits and every sort in
// this library produces the same sequence whatever order records arrive in.
__host__ __device__ __forceinline__ bool rec_less(int region, u64 ka, u64 va, u64 kb, u64 vb) {
  const u64 ca = canon_k(region, ka), cb = canon_k(region, kb);
  return ca < cb || (ca == cb && (va < vb || (va == vb && ka < kb)));
}

// ---------------------------------------------------------------- SPA bins
//
// The SPA pre-filter (k_filter.cu) groups each region's records into bins
// of its primary coordinate. The bin is a monotone map onto [0, nb) in the
// region's sort direction (subtract, multiply by positive constants, one of
// them a power of two, clamp, truncate: all monotone in round-to-nearest),
// so a region's sorted sequence visits its bins in increasing order and
// every bin is one contiguous run of it. The map's constants live in
// QuadInfo (quad_derive, computed once per call), so the classify kernel
// (which counts records per bin) and the filter kernel (which re-derives
// each record's bin from its primary) agree bit for bit.

// Primary range of region r (1..4) between its anchors: LL x in
// [left.x, bottom.x], LR y in [bottom.y, right.y], UR x in [top.x, right.x],
// UL y in [left.y, top.y] (quad = left, bottom, right, top).
__host__ __device__ __forceinline__ void bin_range(const double* q, int r, double* lo, double* hi) {
  switch (r) {
    case 1: *lo = q[0]; *hi = q[2]; break;
    case 2: *lo = q[3]; *hi = q[5]; break;
    case 3: *lo = q[6]; *hi = q[4]; break;
    default: *lo = q[1]; *hi = q[7]; break;
  }
}

// The record word v of region r (1..4) for point (x, y) (key codec above).
__device__ __forceinline__ u64 v_of(int r, double x, double y) {
  switch (r) {
    case 1: return ~ord_enc(y);
    case 2: return ord_enc(x);
    case 3: return ord_enc(y);
    default: return ~ord_enc(x);
  }
}
// ... and its word k.
__device__ __forceinline__ u64 k_of(int r, double x, double y) {
  switch (r) {
    case 1: return ord_enc(x);
    case 2: return ord_enc(y);
    case 3: return ~ord_enc(x);
    default: return ~ord_enc(y);
  }
}

// The guarded coordinate as a key w on which every region's SPA is a
// running MAX: steps_back(g, t) <=> w(g) < w(t) (spa.cpp:92-105). w is the
// record's v word (chgpu_internal codec: LL ~ord(y), LR ord(x), UR ord(y),
// UL ~ord(x)) with -0.0 mapped onto +0.0, since == does not tell them apart.
__host__ __device__ __forceinline__ u64 wkey(int r, u64 v) {
  if (r == 1 || r == 4) return v == 0x8000000000000000ull ? 0x7FFFFFFFFFFFFFFFull : v;
  return v == 0x7FFFFFFFFFFFFFFFull ? 0x8000000000000000ull : v;
}

// ---------------------------------------------------------------- look-back
//
// Decoupled look-back status words: [tag:30 | flag:2 | value:32]. The tag
// identifies the launch that wrote the word, so status arrays never need
// clearing between launches (a stale word from any earlier launch carries
// a different tag and reads as "not ready").
enum : u32 { kFlagNone = 0, kFlagAgg = 1, kFlagPrefix = 2 };

__device__ __forceinline__ u64 make_status(u32 tag, u32 flag, u32 value) {
  return ((u64)(tag & 0x3FFFFFFFu) << 34) | ((u64)flag << 32) | (u64)value;
}
__device__ __forceinline__ u32 status_flag(u64 w, u32 tag) {
  return ((u32)(w >> 34) == (tag & 0x3FFFFFFFu)) ? (u32)((w >> 32) & 3u) : 0u;
}
__device__ __forceinline__ void store_status(u64* p, u64 w) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(w) : "memory");
}
__device__ __forceinline__ u64 load_status_acquire(const u64* p) {
  u64 w;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(w) : "l"(p) : "memory");
  return w;
}
__device__ __forceinline__ void fence_acq_rel_gpu() {
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}
__device__ __forceinline__ u64 load_status(const u64* p) {
  u64 w;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(w) : "l"(p) : "memory");
  return w;
}

// Warp-cooperative look-back over a status column (stride between
// consecutive tiles). Returns the exclusive prefix for `tile`, given that
// tile `first` (the chain's first tile) publishes a prefix directly.
// Every lane returns the same value.
__device__ __forceinline__ u32 warp_lookback(const u64* col, size_t stride, int tile, int first,
                                             u32 tag) {
  const int lane = threadIdx.x & 31;
  u32 excl = 0;
  int base = tile - 1;
  while (true) {
    const int j = base - lane;
    u32 flag = kFlagPrefix, val = 0;
    if (j >= first) {
      u64 w;
      do {
        w = load_status(col + (size_t)j * stride);
        flag = status_flag(w, tag);
      } while (flag == kFlagNone);
      val = (u32)w;
    }
    const unsigned pmask = __ballot_sync(0xffffffffu, flag == kFlagPrefix);
    const int stop = pmask ? (__ffs(pmask) - 1) : 32;  // nearest predecessor holding a prefix
    u32 contrib = (lane <= stop) ? val : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) contrib += __shfl_xor_sync(0xffffffffu, contrib, o);
    excl += contrib;
    if (pmask) break;
    base -= 32;
  }
  return excl;
}

// ---------------------------------------------------------------- loads

// Loads of data the previous kernel of a programmatic launch produced, after
// griddepcontrol.wait: the default cached path (ld.global.ca), as asm
// volatile so that it stays below the wait. Not ld.global.nc: ptxas hoists
// those above the wait (the data counts as read-only for the kernel), which
// reads a stale quad.
__device__ __forceinline__ double ld_after_wait_f64(const double* p) {
  double v;
  asm volatile("ld.global.ca.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ u32 ld_after_wait_u32(const u32* p) {
  u32 v;
  asm volatile("ld.global.ca.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

__device__ __forceinline__ double2 ldg_stream(const double2* p) {
  double2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];"
               : "=d"(r.x), "=d"(r.y)
               : "l"(p));
  return r;
}

// SPA extremum and step-back test on guarded coordinates (spa.cpp:92-105):
// LL / UL keep running minima, LR / UR maxima.
__device__ __forceinline__ double op_ext(bool is_min, double a, double b) {
  return is_min ? (b < a ? b : a) : (b > a ? b : a);
}
__device__ __forceinline__ bool steps_back(bool is_min, double g, double t) {
  return is_min ? (g > t) : (g < t);
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ---------------------------------------------------------------- shared structs

// Device-resident result of the extremes reduction, consumed by the
// classify kernel without a host round trip. Doubles first, 16-byte
// aligned: K2 reads its constants with 16-byte uniform loads.
struct __align__(16) QuadInfo {
  double q[8];       // left.x, left.y, bottom.x, bottom.y, right.x, right.y, top.x, top.y
  // derived once per call (quad_derive)
  double ex[4], ey[4];     // edge c = corner (c + 1) & 3 - corner c (classify's cross products)
  double blo[4], bspan[4]; // SPA bin map of region r + 1: origin and span of its primary
  double bscale[4];        // ... and its scale (bin_scale of bspan at the call's bin count)
  u64 idx[4];        // index of each corner (earliest among == ties)
  u32 frame_size;    // frame_vertices(quad).size()
  u32 degenerate;    // frame_size <= 2
};

// The bin scale nb / span of a region (0 for a null, negative or denormal
// span: every record then falls in one bin). IEEE division on both sides,
// so host and device derive the same bits.
__host__ __device__ __forceinline__ double bin_scale(double span, int log2nb) {
#ifdef __CUDA_ARCH__
  double s = span > 0.0 ? __ddiv_rn((double)(1u << log2nb), span) : 0.0;
#else
  double s = span > 0.0 ? (double)(1u << log2nb) / span : 0.0;
#endif
  if (!(s < 1e300)) s = 0.0;  // inf / nan
  return s;
}

// Fills QuadInfo's derived fields from q (host and device: IEEE subtracts
// and divides, so both sides derive the same bits); log2nb = SPA bins per
// region of the call (0 when no bins are used).
__host__ __device__ inline void quad_derive(QuadInfo& qi, int log2nb) {
  for (int c = 0; c < 4; ++c) {
    const int d = (c + 1) & 3;
    qi.ex[c] = qi.q[2 * d] - qi.q[2 * c];
    qi.ey[c] = qi.q[2 * d + 1] - qi.q[2 * c + 1];
    double lo, hi;
    bin_range(qi.q, c + 1, &lo, &hi);
    qi.blo[c] = lo;
    qi.bspan[c] = hi - lo;
    qi.bscale[c] = bin_scale(qi.bspan[c], log2nb);
  }
}

// Bin of a record of region ri + 1 with primary coordinate p:
// min(trunc((p - lo) * scale), top), 0 below the range (rounding
// stragglers), in the region's sort direction. One dependent multiply: this
// sits on K2's per-survivor path.
//
// The truncation runs on the FP64 pipe, not the (narrow) XU pipe: adding 2^52
// rounding toward zero leaves trunc(t) in the low mantissa bits for t in
// [0, 2^51), and below 2^52's bit pattern for t < 0; the clamp is then two
// integer compares on the bits (a double fmin/fmax pair cost 8% of K2's
// instructions). Monotone in t, so in the primary coordinate.
__device__ __forceinline__ u32 bin_of(double lo, double scale, u32 top, u32 ri, double p) {
  const double t = __dmul_rn(__dsub_rn(p, lo), scale);
  const long long u = __double_as_longlong(__dadd_rz(t, 4503599627370496.0)) - 0x4330000000000000ll;
  const u32 b = u < 0 ? 0u : (u > (long long)top ? top : (u32)u);
  return ri >= 2 ? top - b : b;  // UR / UL sort descending
}

// One extremes candidate per corner: the point and its index.
struct Cand {
  double x, y;
  u64 i;
};
struct QuadCand {
  Cand c[4];
};

// Sort segment descriptor (one region, or one long group of a region).
struct SegDesc {
  u64 src_off;     // element offset of the segment in the pass's source array
  u64 dst_off;     // element offset in the destination array
  u32 len;         // elements
  u32 tile_begin;  // first global tile of the segment
  int region;      // key codec region (0 = LEX)
  int qbits;       // quantizer width (digit mode kDigitQ)
  double qlo;      // quantizer: q = clamp((primary - qlo) * qscale, 0, qmax)
  double qscale;
  double qmax;     // 2^qbits - 1
};

// Digit sources of a radix pass.
enum : int { kDigitK = 0, kDigitV = 1, kDigitQ = 2 };
// Group equality of the in-place fix-up.
enum : int { kEqQ = 0, kEqPrim = 1 };

constexpr int kSortThreads = 256;
#ifndef CHGPU_SORT_ITEMS
#define CHGPU_SORT_ITEMS 12
#endif
constexpr int kSortItems = CHGPU_SORT_ITEMS;
constexpr int kSortTile = kSortThreads * kSortItems;  // 3072
constexpr int kDigits = 256;
constexpr int kPasses = 8;

constexpr int kK2Threads = 256;
#ifndef CHGPU_K2C_ITEMS
#define CHGPU_K2C_ITEMS 6
#endif
constexpr int kK2Items = CHGPU_K2C_ITEMS;
constexpr int kK2Tile = kK2Threads * kK2Items;  // 1536
#ifndef CHGPU_SEG_ITEMS
#define CHGPU_SEG_ITEMS 8
#endif
constexpr int kSegItems = CHGPU_SEG_ITEMS;        // points per lane of the filter path's K2
constexpr int kSegPts = 32 * kSegItems;           // one K2 warp's survivor segment
// A survivor's filter key: its global SPA bin (< 4 * 2^18) in bits 40-63,
// its point's position inside its K2 segment in bits 32-39 (the filter
// recovers the input index from it: no index array), w >> 32 (sign,
// exponent and 20 mantissa bits of the guarded coordinate) in the low
// word. w >> 32 is monotone in w, so maxima and threshold tests on it are
// valid lower bounds / drops (k_filter.cu), and the bin tables of maxima
// and thresholds are 32-bit.
constexpr int kWShift = 32;
constexpr u64 kWMask = 0xFFFFFFFFull;
constexpr int kKeyBinShift = 40;
static_assert(kSegPts <= 256, "a survivor's segment position is 8 bits of its key");
__host__ __device__ __forceinline__ u64 filter_key(u32 gbin, u32 pos, u64 w) {
  return ((u64)gbin << kKeyBinShift) | ((u64)pos << 32) | (w >> kWShift);
}
__host__ __device__ __forceinline__ u32 key_bin(u64 key) { return (u32)(key >> kKeyBinShift); }
__host__ __device__ __forceinline__ u32 key_pos(u64 key) { return (u32)(key >> 32) & 255u; }

}  // namespace chgpu
