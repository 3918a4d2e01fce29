/* chainhull_capi.h — a C entry into the C++ drop-in (libchainhull.so).
 *
 * chainhull::convex_hull (reference pipeline.hpp:55) takes a
 * std::span<const Point2> and returns a HullResult by value; FFI callers
 * (ctypes, cgo) cannot build either, so this wrapper runs exactly that C++
 * call on xy[2n] (any host memory: pageable, as a std::vector's) and copies
 * the result out. It is how bench.py times the drop-in end to end.
 *
 * Returns a chgpu_status (include/chgpu.h): the reference's exceptions map
 * to CHGPU_EMPTY / CHGPU_DEGENERATE / CHGPU_INVALID_ARG on their branches,
 * anything else to CHGPU_CUDA_ERR; CHGPU_TOO_LARGE if the hull does not fit
 * hull_cap points (hull_out may be NULL to ask for the size only).
 * counts (may be NULL) = {n_input, n_after_round1, n_after_spa, n_hull}. */
#ifndef CHAINHULL_CAPI_H
#define CHAINHULL_CAPI_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

int chainhull_capi_convex_hull(const double* xy, size_t n, size_t chunk_count, size_t parallelism,
                               int degenerate_fallback, double* hull_out, size_t hull_cap,
                               size_t* n_hull, size_t* counts);

#ifdef __cplusplus
}
#endif

#endif /* CHAINHULL_CAPI_H */
