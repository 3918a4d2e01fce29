// Melkman on the GPU for polygons in convex position (all vertices kept).
//
// For survivor-heavy inputs (20 M points on a circle: every point is a hull
// vertex) the host finisher is a 20 M-step sequential loop. Melkman's
// behaviour on such a ring is fully determined, so it can be verified in
// parallel and the loop skipped, with the output it would produce.
//
// Let r_0 .. r_{N-1} be the ring assemble_polygon builds (polygon.cpp:7-29:
// corner r, then chain r, r = 0..3; here only when it has no consecutive or
// wrap duplicates, so melkman.cpp:20-25 leaves it unchanged). melkman
// (melkman.cpp:17-86) then runs this trajectory exactly when every
// predicate below evaluates as stated (turn = the reference's rounded cross
// product, geometry.hpp:22-35):
//   seed  (:30-60)  turn(lo, hi, r_2) != 0 with {lo, hi} = lex-sorted
//                   {r_0, r_1} (r_1 is absorbed: turn(r_0, r_0, r_1) is an
//                   exact 0), and turn(r_0, r_1, r_2) == Left, giving the
//                   deque [r_2, r_0, r_1, r_2];
//   step k >= 3 (:62-80), deque [r_{k-1}, r_0, .., r_{k-1}]:
//     A_k = turn(r_{k-2}, r_{k-1}, r_k) == Left   (no skip with B_k false,
//                                                  and no back pop)
//     B_k = turn(r_{k-1}, r_0, r_k)    != Left    (not skipped)
//     C_k = turn(r_k, r_{k-1}, r_0)    != Left    (front pop of r_{k-1})
//     D_k = turn(r_k, r_0, r_1)        == Left    (front pops stop)
//   leaving [r_k, r_0, .., r_k].
// By induction the final deque is [r_{N-1}, r_0, .., r_{N-1}], the hull
// before canonicalize_ring is (r_{N-1}, r_0, .., r_{N-2}), and the output is
// that sequence rotated to its first lexicographic minimum. If any
// predicate deviates, the host runs the reference loop instead.

#include "chgpu_internal.cuh"
#include "kernels.h"

namespace chgpu {

namespace {

__device__ __forceinline__ double turn_val(double ax, double ay, double bx, double by, double px,
                                           double py) {
  return __dsub_rn(__dmul_rn(__dsub_rn(bx, ax), __dsub_rn(py, ay)),
                   __dmul_rn(__dsub_rn(by, ay), __dsub_rn(px, ax)));
}

// Element i of the virtual ring sequence: corner r at seg_begin[r], then
// the r-th chain.
struct RingMap {
  u64 seg_begin[5];  // start of corner r's position (seg_begin[4] = N)
  u64 chain_off[4];  // chain r's offset in the chains array
};

// (constant indices only: a dynamically indexed parameter or QuadInfo copy
// would live in local memory)
__device__ __forceinline__ double2 ring_at(const RingMap& M, const double2* __restrict__ chains,
                                           const QuadInfo& qi, u64 i) {
  u64 sb = M.seg_begin[0], co = M.chain_off[0];
  double cx = qi.q[0], cy = qi.q[1];
  if (i >= M.seg_begin[1]) sb = M.seg_begin[1], co = M.chain_off[1], cx = qi.q[2], cy = qi.q[3];
  if (i >= M.seg_begin[2]) sb = M.seg_begin[2], co = M.chain_off[2], cx = qi.q[4], cy = qi.q[5];
  if (i >= M.seg_begin[3]) sb = M.seg_begin[3], co = M.chain_off[3], cx = qi.q[6], cy = qi.q[7];
  const u64 j = i - sb;
  if (j == 0) return make_double2(cx, cy);
  return chains[co + j - 1];
}

__device__ __forceinline__ bool same2(double2 a, double2 b) { return a.x == b.x && a.y == b.y; }

__device__ __forceinline__ bool lex_lt(double2 a, double2 b) {
  return a.x < b.x || (a.x == b.x && a.y < b.y);
}

}  // namespace

// Checks every predicate of the trajectory above (and the absence of
// duplicates); clears *ok on the first deviation. Also reduces the
// canonical start: the first lexicographic minimum in hull order
// (hull position of ring index i: (i + 1) mod N) into per-block winners.
__global__ __launch_bounds__(256) void k_convex_check(const double2* __restrict__ chains,
                                                      RingMap M, const QuadInfo* __restrict__ qinfo,
                                                      u32* __restrict__ ok,
                                                      u64* __restrict__ block_best) {
  const QuadInfo qi = *qinfo;
  const u64 N = M.seg_begin[4];
  const double2 r0 = ring_at(M, chains, qi, 0), r1 = ring_at(M, chains, qi, 1);
  bool good = true;
  u64 best = ~0ull;  // hull position of this thread's best candidate
  double2 bestp = make_double2(0.0, 0.0);
  // A warp covers 32 consecutive ring indices. Inside a chain (no corner in
  // [base - 2, base + 32)) ring index i of segment r is chains[i - r - 1]:
  // three plain loads, the two shifted ones L1 hits.
  const int lane = threadIdx.x & 31;
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 base = (u64)blockIdx.x * blockDim.x + (threadIdx.x & ~31u); base < N; base += stride) {
    const u64 k = base + lane;
    const bool valid = k < N;
    u64 sb = M.seg_begin[0], nx = M.seg_begin[1];
    int r = 0;
    if (base >= M.seg_begin[1]) r = 1, sb = M.seg_begin[1], nx = M.seg_begin[2];
    if (base >= M.seg_begin[2]) r = 2, sb = M.seg_begin[2], nx = M.seg_begin[3];
    if (base >= M.seg_begin[3]) r = 3, sb = M.seg_begin[3], nx = N;
    double2 rk, rp, rpp;
    if (base >= sb + 3 && base + 32 <= nx) {
      const double2* p = chains + (base - (u64)r - 1) + lane;
      rk = p[0];
      rp = p[-1];
      rpp = p[-2];
    } else {
      rk = ring_at(M, chains, qi, valid ? k : N - 1);
      rp = ring_at(M, chains, qi, !valid || k == 0 ? N - 1 : k - 1);
      rpp = valid && k >= 2 ? ring_at(M, chains, qi, k - 2) : rk;
    }
    if (!valid) continue;
    if (same2(rk, rp)) good = false;  // consecutive or wrap duplicate
    if (k == 2) {
      const double2 lo = lex_lt(r1, r0) ? r1 : r0, hi = lex_lt(r1, r0) ? r0 : r1;
      if (!(turn_val(lo.x, lo.y, hi.x, hi.y, rk.x, rk.y) != 0.0)) good = false;
      if (!(turn_val(r0.x, r0.y, r1.x, r1.y, rk.x, rk.y) > 0.0)) good = false;
    } else if (k >= 3) {
      if (!(turn_val(rpp.x, rpp.y, rp.x, rp.y, rk.x, rk.y) > 0.0)) good = false;   // A_k
      if (turn_val(rp.x, rp.y, r0.x, r0.y, rk.x, rk.y) > 0.0) good = false;        // B_k
      if (turn_val(rk.x, rk.y, rp.x, rp.y, r0.x, r0.y) > 0.0) good = false;        // C_k
      if (!(turn_val(rk.x, rk.y, r0.x, r0.y, r1.x, r1.y) > 0.0)) good = false;    // D_k
    }
    // a thread visits increasing k, so its hull positions k + 1 increase
    // except the last ring index (hull position 0), which wins ties
    if (best == ~0ull || lex_lt(rk, bestp) || (k + 1 == N && same2(rk, bestp))) {
      best = k + 1 == N ? 0 : k + 1;
      bestp = rk;
    }
  }
  if (!__all_sync(0xffffffffu, good) && (threadIdx.x & 31) == 0) atomicAnd(ok, 0u);
  // block-wide (value, hull position) minimum
  __shared__ double sx[256], sy[256];
  __shared__ u64 sp[256];
  sx[threadIdx.x] = bestp.x;
  sy[threadIdx.x] = bestp.y;
  sp[threadIdx.x] = best;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) {
      const int o = threadIdx.x + s;
      const double2 a = make_double2(sx[threadIdx.x], sy[threadIdx.x]);
      const double2 b = make_double2(sx[o], sy[o]);
      const bool take = sp[o] != ~0ull &&
                        (sp[threadIdx.x] == ~0ull || lex_lt(b, a) ||
                         (same2(a, b) && sp[o] < sp[threadIdx.x]));
      if (take) {
        sx[threadIdx.x] = b.x;
        sy[threadIdx.x] = b.y;
        sp[threadIdx.x] = sp[o];
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) block_best[blockIdx.x] = sp[0];
}

// Picks the start among the block winners (their points are re-read) and
// writes the hull: out[j] = hull[(start + j) mod N], hull[h] = r_{h-1 mod N}.
__global__ __launch_bounds__(256) void k_convex_emit(const double2* __restrict__ chains, RingMap M,
                                                     const QuadInfo* __restrict__ qinfo,
                                                     const u64* __restrict__ block_best,
                                                     int nblocks, double2* __restrict__ out) {
  const QuadInfo qi = *qinfo;
  const u64 N = M.seg_begin[4];
  // block-wide (point, hull position) minimum over the block winners
  __shared__ double sx[256], sy[256];
  __shared__ u64 sp[256];
  __shared__ u64 s_start;
  u64 best = ~0ull;
  double2 bp = make_double2(0.0, 0.0);
  for (int b = threadIdx.x; b < nblocks; b += blockDim.x) {
    const u64 hp = block_best[b];
    if (hp == ~0ull) continue;
    const double2 p = ring_at(M, chains, qi, hp == 0 ? N - 1 : hp - 1);
    if (best == ~0ull || lex_lt(p, bp) || (same2(p, bp) && hp < best)) {
      best = hp;
      bp = p;
    }
  }
  sx[threadIdx.x] = bp.x;
  sy[threadIdx.x] = bp.y;
  sp[threadIdx.x] = best;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) {
      const int o = threadIdx.x + s;
      const double2 a = make_double2(sx[threadIdx.x], sy[threadIdx.x]);
      const double2 b = make_double2(sx[o], sy[o]);
      const bool take = sp[o] != ~0ull &&
                        (sp[threadIdx.x] == ~0ull || lex_lt(b, a) ||
                         (same2(a, b) && sp[o] < sp[threadIdx.x]));
      if (take) {
        sx[threadIdx.x] = b.x;
        sy[threadIdx.x] = b.y;
        sp[threadIdx.x] = sp[o];
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) s_start = sp[0];
  __syncthreads();
  const u64 start = s_start;
  for (u64 j = (u64)blockIdx.x * blockDim.x + threadIdx.x; j < N; j += (u64)gridDim.x * blockDim.x) {
    u64 h = start + j;
    if (h >= N) h -= N;
    out[j] = ring_at(M, chains, qi, h == 0 ? N - 1 : h - 1);
  }
}

int convex_blocks() { return device_limits().sms * 8; }

void launch_convex_check(const double2* chains, const u64 kept[4], const QuadInfo* qinfo, u32* ok,
                         u64* block_best, cudaStream_t st) {
  RingMap M;
  u64 pos = 0, off = 0;
  for (int r = 0; r < 4; ++r) {
    M.seg_begin[r] = pos;
    M.chain_off[r] = off;
    pos += 1 + kept[r];
    off += kept[r];
  }
  M.seg_begin[4] = pos;
  k_convex_check<<<convex_blocks(), 256, 0, st>>>(chains, M, qinfo, ok, block_best);
}

void launch_convex_emit(const double2* chains, const u64 kept[4], const QuadInfo* qinfo,
                        const u64* block_best, double2* out, cudaStream_t st) {
  RingMap M;
  u64 pos = 0, off = 0;
  for (int r = 0; r < 4; ++r) {
    M.seg_begin[r] = pos;
    M.chain_off[r] = off;
    pos += 1 + kept[r];
    off += kept[r];
  }
  M.seg_begin[4] = pos;
  k_convex_emit<<<convex_blocks(), 256, 0, st>>>(chains, M, qinfo, block_best, convex_blocks(), out);
}

}  // namespace chgpu
