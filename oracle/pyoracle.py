"""TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.

ctypes bindings for the two CPU checkers:

* ``Oracle``   — oracle/liboracle.so, the plain-C restatement of the
  reference path (oracle/chainhull_oracle.c), always buildable.
* ``RefLib``   — oracle/_ref/libchainhull_ref.so, the unmodified reference
  sources compiled in place plus oracle/ref_shim.cpp (only present where
  /root/reference existed at build time, or shipped prebuilt).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libchainhull_ref.so")

DISTRIBUTIONS = ["uniform_square", "uniform_disk", "circle", "gaussian", "collinear",
                 "duplicates_heavy"]

_dp = C.POINTER(C.c_double)
_szp = C.POINTER(C.c_size_t)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _szptr(a: np.ndarray):
    return a.ctypes.data_as(_szp)


def as_points(xy) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(xy, dtype=np.float64)).reshape(-1, 2)
    return a


@dataclass
class HullOut:
    status: int
    hull: np.ndarray
    counts: np.ndarray        # n_input, n_after_round1, n_after_spa, n_hull
    region_counts: np.ndarray | None = None
    kept_counts: np.ndarray | None = None


class Oracle:
    """Plain-C restatement (oracle/chainhull_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        self.lib = C.CDLL(path)
        L = self.lib
        L.orc_generate.argtypes = [C.c_int, C.c_size_t, C.c_uint64, _dp]
        L.orc_find_extremes.argtypes = [_dp, C.c_size_t, _dp]
        L.orc_classify_points.argtypes = [_dp, C.c_size_t, _dp, C.POINTER(C.c_uint8)]
        L.orc_frame_vertices.argtypes = [_dp, _dp]
        L.orc_frame_vertices.restype = C.c_size_t
        L.orc_sort_region.argtypes = [C.c_int, _dp, C.c_size_t]
        L.orc_spa_filter.argtypes = [C.c_int, _dp, C.c_size_t, _dp, C.c_size_t, _dp, _szp]
        L.orc_assemble_polygon.argtypes = [_dp, _szp, _dp, _dp, _szp]
        L.orc_melkman.argtypes = [_dp, C.c_size_t, _dp, _szp]
        L.orc_hull_oracle.argtypes = [_dp, C.c_size_t, _dp, _szp]
        L.orc_convex_hull.argtypes = [_dp, C.c_size_t, C.c_size_t, C.c_int, _dp, _szp, _szp,
                                      _szp, _szp]

    def generate(self, dist: str | int, n: int, seed: int) -> np.ndarray:
        d = DISTRIBUTIONS.index(dist) if isinstance(dist, str) else dist
        out = np.empty((n, 2), np.float64)
        st = self.lib.orc_generate(d, n, seed, _ptr(out))
        if st:
            raise ValueError("generate: n must be positive")
        return out

    def classify(self, xy, quad) -> np.ndarray:
        xy = as_points(xy)
        q = as_points(quad)
        out = np.empty(len(xy), np.uint8)
        self.lib.orc_classify_points(_ptr(xy), len(xy), _ptr(q),
                                     out.ctypes.data_as(C.POINTER(C.c_uint8)))
        return out

    def find_extremes(self, xy) -> np.ndarray:
        xy = as_points(xy)
        q = np.empty((4, 2), np.float64)
        st = self.lib.orc_find_extremes(_ptr(xy), len(xy), _ptr(q))
        if st:
            raise ValueError("EmptyInput")
        return q

    def frame_vertices(self, quad) -> np.ndarray:
        q = as_points(quad)
        out = np.empty((4, 2), np.float64)
        k = self.lib.orc_frame_vertices(_ptr(q), _ptr(out))
        return out[:k]

    def sort_region(self, region: int, seg) -> np.ndarray:
        s = as_points(seg).copy()
        st = self.lib.orc_sort_region(region, _ptr(s), len(s))
        if st:
            raise ValueError("invalid region")
        return s

    def spa_filter(self, region: int, seg, anchors, chunk_count: int) -> np.ndarray:
        s = as_points(seg)
        a = as_points(anchors)
        out = np.empty((max(len(s), 1), 2), np.float64)
        k = np.zeros(1, np.uintp)
        st = self.lib.orc_spa_filter(region, _ptr(s), len(s), _ptr(a), chunk_count, _ptr(out),
                                     _szptr(k))
        if st == 3:
            raise ValueError("chunk_count must be >= 1")
        return out[: int(k[0])]

    def melkman(self, poly):
        p = as_points(poly)
        out = np.empty((max(len(p), 1), 2), np.float64)
        k = np.zeros(1, np.uintp)
        st = self.lib.orc_melkman(_ptr(p), len(p), _ptr(out), _szptr(k))
        return st, out[: int(k[0])]

    def hull_oracle(self, xy):
        p = as_points(xy)
        out = np.empty((max(len(p), 1), 2), np.float64)
        k = np.zeros(1, np.uintp)
        st = self.lib.orc_hull_oracle(_ptr(p), len(p), _ptr(out), _szptr(k))
        return st, out[: int(k[0])] if st == 0 else out[:0]

    def convex_hull(self, xy, chunk_count: int = 1024, degenerate_fallback: bool = True) -> HullOut:
        p = as_points(xy)
        out = np.empty((max(len(p), 1), 2), np.float64)
        k = np.zeros(1, np.uintp)
        counts = np.zeros(4, np.uintp)
        rc = np.zeros(5, np.uintp)
        kc = np.zeros(4, np.uintp)
        st = self.lib.orc_convex_hull(_ptr(p), len(p), chunk_count, int(degenerate_fallback),
                                      _ptr(out), _szptr(k), _szptr(counts), _szptr(rc), _szptr(kc))
        hull = out[: int(k[0])] if st == 0 else out[:0]
        return HullOut(st, hull, counts.astype(np.int64), rc.astype(np.int64), kc.astype(np.int64))


class RefLib:
    """The unmodified reference compiled in place (oracle/_ref)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = C.CDLL(path)
        L = self.lib
        L.ref_generate.argtypes = [C.c_int, C.c_size_t, C.c_uint64, _dp]
        L.ref_convex_hull.argtypes = [_dp, C.c_size_t, C.c_size_t, C.c_size_t, C.c_int, _dp, _szp,
                                      _szp, _dp]
        L.ref_hull_oracle.argtypes = [_dp, C.c_size_t, _dp, _szp]
        L.ref_find_extremes.argtypes = [_dp, C.c_size_t, C.c_size_t, _dp]
        L.ref_stage_dump.argtypes = [_dp, C.c_size_t, C.c_size_t, _dp, _szp, _dp, _dp, _szp]
        L.ref_sort_region.argtypes = [C.c_int, _dp, C.c_size_t]
        L.ref_spa_filter.argtypes = [C.c_int, _dp, C.c_size_t, _dp, C.c_size_t, _dp, _szp]
        L.ref_melkman.argtypes = [_dp, C.c_size_t, _dp, _szp]

    @staticmethod
    def available(path: str = REF_SO) -> bool:
        return os.path.exists(path)

    def generate(self, dist: str | int, n: int, seed: int) -> np.ndarray:
        d = DISTRIBUTIONS.index(dist) if isinstance(dist, str) else dist
        out = np.empty((n, 2), np.float64)
        if self.lib.ref_generate(d, n, seed, _ptr(out)):
            raise ValueError("generate failed")
        return out

    def convex_hull(self, xy, chunk_count: int = 1024, parallelism: int = 1,
                    degenerate_fallback: bool = True):
        p = as_points(xy)
        out = np.empty((max(len(p), 1), 2), np.float64)
        k = np.zeros(1, np.uintp)
        counts = np.zeros(4, np.uintp)
        ms = np.zeros(7, np.float64)
        st = self.lib.ref_convex_hull(_ptr(p), len(p), chunk_count, parallelism,
                                      int(degenerate_fallback), _ptr(out), _szptr(k),
                                      _szptr(counts), _ptr(ms))
        hull = out[: int(k[0])] if st == 0 else out[:0]
        return HullOut(st, hull, counts.astype(np.int64)), ms

    def find_extremes(self, xy, workers: int = 1) -> np.ndarray:
        p = as_points(xy)
        q = np.empty((4, 2), np.float64)
        if self.lib.ref_find_extremes(_ptr(p), len(p), workers, _ptr(q)):
            raise ValueError("EmptyInput")
        return q

    def stage_dump(self, xy, chunk_count: int = 1024):
        p = as_points(xy)
        quad = np.empty((4, 2), np.float64)
        rc = np.zeros(5, np.uintp)
        srt = np.empty((max(len(p), 1), 2), np.float64)
        kept = np.empty((max(len(p), 1), 2), np.float64)
        kc = np.zeros(4, np.uintp)
        st = self.lib.ref_stage_dump(_ptr(p), len(p), chunk_count, _ptr(quad), _szptr(rc),
                                     _ptr(srt), _ptr(kept), _szptr(kc))
        if st:
            raise ValueError(f"stage_dump status {st}")
        s1 = int(rc[1:].sum())
        return quad, rc.astype(np.int64), srt[:s1], kept[: int(kc.sum())], kc.astype(np.int64)

    def sort_region(self, region: int, seg) -> np.ndarray:
        s = as_points(seg).copy()
        self.lib.ref_sort_region(region, _ptr(s), len(s))
        return s

    def spa_filter(self, region: int, seg, anchors, chunk_count: int) -> np.ndarray:
        s = as_points(seg)
        a = as_points(anchors)
        out = np.empty((max(len(s), 1), 2), np.float64)
        k = np.zeros(1, np.uintp)
        st = self.lib.ref_spa_filter(region, _ptr(s), len(s), _ptr(a), chunk_count, _ptr(out),
                                     _szptr(k))
        if st == 3:
            raise ValueError("chunk_count must be >= 1")
        return out[: int(k[0])]

    def melkman(self, poly):
        p = as_points(poly)
        out = np.empty((max(len(p), 1), 2), np.float64)
        k = np.zeros(1, np.uintp)
        st = self.lib.ref_melkman(_ptr(p), len(p), _ptr(out), _szptr(k))
        return st, out[: int(k[0])]
