"""B200-native CudaChain convex hull (arXiv 1508.05488), Python host mirror.

This module mirrors the reference's public interface for the hull path
(reference proj/core/include/chainhull/pipeline.hpp:10-62):

    convex_hull(points, PipelineConfig()) -> HullResult(hull=Hull, stats=StageStats)

with the same argument meaning and the same error behaviour
(EmptyInput, DegenerateInput, ValueError for std::invalid_argument), on top
of the C ABI in include/chgpu.h (libchgpu.so, built in-tree by `make`).
Every call runs the sm_100a kernels; there is no CPU fallback: if the
library or a CUDA device is missing the call raises.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "PipelineConfig", "StageStats", "Hull", "HullResult", "Diag", "Error", "EmptyInput",
    "DegenerateInput", "Context", "convex_hull", "hull_oracle", "generate", "melkman",
    "find_extremes", "classify", "discard_round1", "sort_region", "spa_filter",
    "assemble_polygon", "canonicalize_ring", "DISTRIBUTIONS", "LIB_PATH", "load_library",
]

HERE = os.path.dirname(os.path.abspath(__file__))
# (CHGPU_LIB: an alternative in-tree build of the same library, for A/B timing)
LIB_PATH = os.environ.get("CHGPU_LIB") or os.path.join(HERE, "libchgpu.so")
DISTRIBUTIONS = ["uniform_square", "uniform_disk", "circle", "gaussian", "collinear",
                 "duplicates_heavy"]

CHGPU_OK, CHGPU_EMPTY, CHGPU_DEGENERATE, CHGPU_INVALID_ARG = 0, 1, 2, 3
CHGPU_CUDA_ERR, CHGPU_NO_DEVICE, CHGPU_TOO_LARGE = 4, 5, 6
CHGPU_IO_ERROR, CHGPU_PARSE_ERROR, CHGPU_NONFINITE = 7, 8, 9


class Error(RuntimeError):
    """chainhull::Error (errors.hpp:10)."""


class EmptyInput(Error):
    """chainhull::EmptyInput (errors.hpp:15)."""


class IoError(Error):
    """errors.hpp:42-44."""


class ParseError(Error):
    """errors.hpp:27-35 (binary payload errors carry line 0)."""
    line = 0


class NonFiniteCoordinate(Error):
    """errors.hpp:37-40."""


class DegenerateInput(Error):
    """chainhull::DegenerateInput (errors.hpp:21)."""


@dataclass
class PipelineConfig:
    """pipeline.hpp:10-22. `parallelism` is accepted and ignored: results are
    worker-independent by contract and the GPU grid replaces the threads."""
    chunk_count: int = 1024
    parallelism: int = 0
    degenerate_fallback: bool = True


_DEFAULT_CONFIG = PipelineConfig()


class _Stats(C.Structure):
    _fields_ = [("n_input", C.c_size_t), ("n_after_round1", C.c_size_t),
                ("n_after_spa", C.c_size_t), ("n_hull", C.c_size_t),
                ("t_extremes_ms", C.c_double), ("t_classify_ms", C.c_double),
                ("t_partition_ms", C.c_double), ("t_sort_ms", C.c_double),
                ("t_spa_ms", C.c_double), ("t_melkman_ms", C.c_double),
                ("t_total_ms", C.c_double)]


class _Diag(C.Structure):
    _fields_ = [("quad", C.c_double * 8), ("frame_size", C.c_size_t),
                ("region_counts", C.c_size_t * 5), ("kept_counts", C.c_size_t * 4),
                ("degenerate_branch", C.c_int), ("sort_passes", C.c_int),
                ("tie_runs", C.c_size_t), ("launches", C.c_int), ("pad_", C.c_int),
                ("t_h2d_ms", C.c_double), ("t_k1_ms", C.c_double), ("t_k2_ms", C.c_double),
                ("t_hist_ms", C.c_double), ("t_passes_ms", C.c_double),
                ("t_ties_ms", C.c_double), ("t_spa_kernel_ms", C.c_double),
                ("t_d2h_ms", C.c_double), ("t_host_ms", C.c_double),
                ("spa_path", C.c_int), ("filter_log2nb", C.c_int), ("n_candidates", C.c_size_t),
                ("t_binscan_ms", C.c_double), ("t_filter_ms", C.c_double),
                ("t_binsort_ms", C.c_double), ("convex_fast_path", C.c_int),
                ("k1k2_overlapped", C.c_int), ("t_host_enqueue_ms", C.c_double),
                ("t_host_wait_ms", C.c_double)]

# chgpu_ctx_set_option (include/chgpu.h)
OPT_SPA_PATH = 1
OPT_CHAINS_TAP = 2
OPT_PDL = 3
OPT_STAGE_TIMES = 4
SPA_AUTO, SPA_SORT, SPA_FILTER, SPA_FILTER_SORTED = 0, 1, 2, 3


@dataclass
class StageStats:
    """pipeline.hpp:30-42."""
    n_input: int = 0
    n_after_round1: int = 0
    n_after_spa: int = 0
    n_hull: int = 0
    t_extremes_ms: float = 0.0
    t_classify_ms: float = 0.0
    t_partition_ms: float = 0.0
    t_sort_ms: float = 0.0
    t_spa_ms: float = 0.0
    t_melkman_ms: float = 0.0
    t_total_ms: float = 0.0

    @classmethod
    def _from(cls, s: _Stats) -> "StageStats":
        return cls(**{f: getattr(s, f) for f, _ in _Stats._fields_})


@dataclass
class Diag:
    quad: np.ndarray
    frame_size: int
    region_counts: list
    kept_counts: list
    degenerate_branch: bool
    sort_passes: int
    tie_runs: int
    launches: int
    times_ms: dict
    spa_path: int = 0        # 0 full sort, 1 pre-filtered, 2 pre-filter overflowed -> sort
    n_candidates: int = 0
    filter_log2nb: int = 0
    convex_fast_path: bool = False
    k1k2_overlapped: bool = False  # K2 launched programmatically behind K1: t_k1_ms covers both

    @classmethod
    def _from(cls, d: _Diag) -> "Diag":
        times = {f: float(getattr(d, f)) for f, _ in _Diag._fields_ if f.startswith("t_")}
        return cls(np.array(d.quad[:], np.float64).reshape(4, 2), int(d.frame_size),
                   [int(c) for c in d.region_counts], [int(c) for c in d.kept_counts],
                   bool(d.degenerate_branch), int(d.sort_passes), int(d.tie_runs),
                   int(d.launches), times, int(d.spa_path), int(d.n_candidates),
                   int(d.filter_log2nb), bool(d.convex_fast_path), bool(d.k1k2_overlapped))


@dataclass
class Hull:
    """melkman.hpp:14-16: canonical CCW ring from the lexicographic minimum."""
    vertices: np.ndarray = field(default_factory=lambda: np.empty((0, 2)))


class HullResult:
    """pipeline.hpp:44-47 (+ GPU diagnostics). `stats` and `diag` are
    converted from the C structs on first access (neither is needed on the
    hot path)."""

    __slots__ = ("hull", "_stats", "_rstats", "_diag", "_raw")

    def __init__(self, hull: Hull, stats: "StageStats | None" = None, diag: "Diag | None" = None,
                 raw=None, raw_stats=None):
        self.hull, self._stats, self._rstats, self._diag, self._raw = hull, stats, raw_stats, diag, raw

    @property
    def stats(self) -> StageStats:
        if self._stats is None and self._rstats is not None:
            self._stats = StageStats._from(self._rstats)
        return self._stats

    @property
    def diag(self) -> "Diag | None":
        if self._diag is None and self._raw is not None:
            self._diag = Diag._from(self._raw)
        return self._diag

    def __repr__(self) -> str:
        return f"HullResult(hull={self.hull!r}, stats={self.stats!r})"


_dp = C.POINTER(C.c_double)
_sz = C.POINTER(C.c_size_t)
_lib = None
_lib_lock = threading.Lock()


def load_library(path: str = LIB_PATH) -> C.CDLL:
    """Loads libchgpu.so (raises if it was not built: no fallback)."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise ImportError(f"{path} is missing: run `make` (or __graft_entry__.build()) first")
        L = C.CDLL(path)
        vp = C.c_void_p
        L.chgpu_ctx_create.argtypes = [C.c_int, C.POINTER(vp)]
        L.chgpu_ctx_destroy.argtypes = [vp]
        L.chgpu_ctx_destroy.restype = None
        L.chgpu_last_error.argtypes = [vp]
        L.chgpu_last_error.restype = C.c_char_p
        L.chgpu_ctx_stream.argtypes = [vp]
        L.chgpu_ctx_stream.restype = vp
        L.chgpu_reserve.argtypes = [vp, C.c_size_t]
        L.chgpu_ctx_set_option.argtypes = [vp, C.c_int, C.c_longlong]
        L.chgpu_last_chains.argtypes = [vp, C.POINTER(_dp), _sz]
        hull_args = [vp, C.c_void_p, C.c_size_t, C.c_size_t, C.c_int, C.POINTER(_dp), _sz,
                     C.POINTER(_Stats), C.POINTER(_Diag)]
        L.chgpu_hull.argtypes = hull_args
        L.chgpu_hull_device.argtypes = hull_args
        L.chgpu_device_count.argtypes = []
        L.chgpu_merge_hull.argtypes = [C.POINTER(_dp), _sz, C.c_int, _dp, _dp, _sz]
        L.chgpu_hull_sharded.argtypes = [C.POINTER(vp), C.c_int, C.POINTER(_dp), _sz, C.c_int,
                                         C.c_int, C.c_size_t, C.c_int, C.POINTER(_dp), _sz,
                                         C.POINTER(_Stats)]
        L.chgpu_hull_xy_binary.argtypes = [vp, C.c_char_p, C.c_size_t, C.c_int, C.POINTER(_dp), _sz,
                                           C.POINTER(_Stats), C.POINTER(_Diag)]
        L.chgpu_find_extremes.argtypes = [vp, _dp, C.c_size_t, _dp]
        L.chgpu_classify.argtypes = [vp, _dp, C.c_size_t, _dp, C.POINTER(C.c_uint8), _sz]
        L.chgpu_discard_round1.argtypes = [vp, _dp, C.POINTER(C.c_uint8), C.c_size_t, _dp,
                                           C.POINTER(C.c_uint8), _sz]
        L.chgpu_sort_region.argtypes = [vp, C.c_int, _dp, C.c_size_t]
        L.chgpu_spa_filter.argtypes = [vp, C.c_int, _dp, C.c_size_t, _dp, C.c_size_t, _dp, _sz]
        L.chgpu_assemble_polygon.argtypes = [_dp, _sz, _dp, _dp, _sz]
        L.chgpu_finish_chains.argtypes = [_dp, _sz, _dp, _dp, _sz]
        L.chgpu_melkman.argtypes = [_dp, C.c_size_t, _dp, _sz]
        L.chgpu_canonicalize_ring.argtypes = [_dp, C.c_size_t]
        L.chgpu_canonicalize_ring.restype = None
        L.chgpu_hull_oracle.argtypes = [_dp, C.c_size_t, _dp, _sz]
        L.chgpu_generate.argtypes = [C.c_int, C.c_size_t, C.c_uint64, _dp]
        L.chgpu_generate_range.argtypes = [C.c_int, C.c_size_t, C.c_uint64, C.c_size_t,
                                           C.c_size_t, _dp]
        L.chgpu_shard_extremes.argtypes = [vp, C.c_void_p, C.c_size_t, C.c_uint64, _dp,
                                           C.POINTER(C.c_uint64)]
        L.chgpu_fold_extremes.argtypes = [_dp, C.POINTER(C.c_uint64), C.c_size_t, _dp]
        L.chgpu_fold_extremes.restype = None
        L.chgpu_shard_chains.argtypes = [vp, C.c_void_p, C.c_size_t, _dp, C.c_size_t,
                                         C.POINTER(_dp), _sz]
        L.chgpu_shard_chains_device.argtypes = [vp, C.c_void_p, C.c_size_t, _dp, C.c_size_t,
                                                C.c_void_p, C.c_size_t, _sz]
        _lib = L
        return L


def _pts(xy) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(xy, dtype=np.float64))
    if a.size == 0:
        return a.reshape(0, 2)
    return a.reshape(-1, 2)


def _p(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _raise(status: int, msg: str):
    if status == CHGPU_EMPTY:
        raise EmptyInput(msg)
    if status == CHGPU_DEGENERATE:
        raise DegenerateInput(msg)
    if status == CHGPU_INVALID_ARG:
        raise ValueError(msg)
    if status == CHGPU_IO_ERROR:
        raise IoError(msg)
    if status == CHGPU_PARSE_ERROR:
        raise ParseError(msg)
    if status == CHGPU_NONFINITE:
        raise NonFiniteCoordinate(msg)
    raise Error(f"chgpu status {status}: {msg}")


class Context:
    """One chgpu_ctx: a CUDA stream plus a device workspace (include/chgpu.h)."""

    def __init__(self, device: int = -1):
        self.lib = load_library()
        h = C.c_void_p()
        st = self.lib.chgpu_ctx_create(device, C.byref(h))
        if st != CHGPU_OK:
            raise Error("no CUDA device: the hull path has no CPU fallback"
                        if st == CHGPU_NO_DEVICE else f"context creation failed ({st})")
        self.h = h

    def close(self):
        if self.h:
            self.lib.chgpu_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st: int):
        if st != CHGPU_OK:
            _raise(st, self.lib.chgpu_last_error(self.h).decode())

    @property
    def stream(self) -> int:
        return int(self.lib.chgpu_ctx_stream(self.h) or 0)

    def reserve(self, n: int):
        self._check(self.lib.chgpu_reserve(self.h, n))

    def set_spa_path(self, mode: int):
        """SPA_AUTO (default), SPA_SORT (sort every survivor), SPA_FILTER, or
        SPA_FILTER_SORTED (pre-filter with every chunk through the bin sorts and
        the sorted chunk SPA, the path large chunks take)."""
        self._check(self.lib.chgpu_ctx_set_option(self.h, OPT_SPA_PATH, mode))

    def set_pdl(self, on: bool = True):
        """CHGPU_OPT_PDL: K2 launched programmatically behind K1 (default)."""
        self._check(self.lib.chgpu_ctx_set_option(self.h, OPT_PDL, int(bool(on))))

    def set_stage_times(self, on: bool = True):
        """CHGPU_OPT_STAGE_TIMES: per-kernel events for Diag.times_ms (off by
        default: each event query costs host time on every call)."""
        self._check(self.lib.chgpu_ctx_set_option(self.h, OPT_STAGE_TIMES, int(bool(on))))

    def set_chains_tap(self, on: bool = True):
        """Keep each hull call's SPA chains for last_chains() (parity tap)."""
        self._check(self.lib.chgpu_ctx_set_option(self.h, OPT_CHAINS_TAP, int(bool(on))))

    def last_chains(self):
        """(chains (k, 2) float64 copy, kept_counts[4]) of the last hull call:
        the kept points of spa_filter per region (spa.cpp:109-163), LL|LR|UR|UL."""
        out = _dp()
        kc = (C.c_size_t * 4)()
        self._check(self.lib.chgpu_last_chains(self.h, C.byref(out), kc))
        counts = [int(c) for c in kc]
        k = sum(counts)
        a = (np.ctypeslib.as_array(out, shape=(2 * k,)).reshape(-1, 2).copy() if k
             else np.empty((0, 2)))
        return a, counts

    def _hull(self, fn, ptr, n, config, copy=True):
        config = config or _DEFAULT_CONFIG
        out = _dp()
        k = C.c_size_t()
        s = _Stats()
        d = _Diag()
        st = fn(self.h, ptr, n, config.chunk_count, 1 if config.degenerate_fallback else 0,
                C.byref(out), C.byref(k), C.byref(s), C.byref(d))
        if st:
            self._check(st)
        kv = k.value
        if kv:
            # (a view of the C ABI's result buffer: frombuffer over a sized
            # ctypes array is several times cheaper than np.ctypeslib.as_array)
            addr = C.cast(out, C.c_void_p).value
            verts = np.frombuffer((C.c_double * (2 * kv)).from_address(addr), np.float64).reshape(kv, 2)
            if copy:
                verts = verts.copy()
        else:
            verts = np.empty((0, 2))
        return HullResult(Hull(verts), raw=d, raw_stats=s)

    def convex_hull(self, points, config: PipelineConfig | None = None,
                    copy: bool = True) -> HullResult:
        """pipeline.hpp:55 over host points (any (n, 2) float64 array);
        copy as in convex_hull_device."""
        a = _pts(points)
        if len(a) == 0:
            raise EmptyInput("convex_hull: no points")
        return self._hull(self.lib.chgpu_hull, a.ctypes.data, len(a), config, copy)

    def convex_hull_device(self, ptr: int, n: int, config: PipelineConfig | None = None,
                           copy: bool = True) -> HullResult:
        """Same, over n points already in device memory at `ptr` (e.g. a
        torch.float64 CUDA tensor's data_ptr(); synchronise its producer
        stream first). copy=False returns the hull as a view of the
        context's host buffer (the C ABI's result), valid until the next
        call on this context."""
        if n == 0:
            raise EmptyInput("convex_hull: no points")
        return self._hull(self.lib.chgpu_hull_device, C.c_void_p(ptr), n, config, copy)

    def hull_xy_binary(self, path, config: PipelineConfig | None = None,
                       copy: bool = True) -> HullResult:
        """read_points(path, xy_binary) + convex_hull (io.hpp:29-36,
        pipeline.hpp:55) fused: the file streams through pinned staging
        into the device pipeline."""
        config = config or PipelineConfig()
        out = _dp()
        k = C.c_size_t()
        s = _Stats()
        d = _Diag()
        st = self.lib.chgpu_hull_xy_binary(self.h, os.fsencode(path), config.chunk_count,
                                           int(bool(config.degenerate_fallback)), C.byref(out),
                                           C.byref(k), C.byref(s), C.byref(d))
        self._check(st)
        verts = np.ctypeslib.as_array(out, shape=(k.value * 2,)).reshape(-1, 2) \
            if k.value else np.empty((0, 2))
        if copy:
            verts = verts.copy()
        return HullResult(Hull(verts), raw=d, raw_stats=s)

    # ---- stage taps -----------------------------------------------------
    def find_extremes(self, points) -> np.ndarray:
        a = _pts(points)
        if len(a) == 0:
            raise EmptyInput("find_extremes: no points")
        q = np.empty(8, np.float64)
        self._check(self.lib.chgpu_find_extremes(self.h, _p(a), len(a), _p(q)))
        return q.reshape(4, 2)

    def classify(self, points, quad):
        a = _pts(points)
        q = np.ascontiguousarray(np.asarray(quad, np.float64).reshape(8))
        lab = np.zeros(len(a), np.uint8)
        counts = (C.c_size_t * 5)()
        if len(a):
            self._check(self.lib.chgpu_classify(self.h, _p(a), len(a), _p(q),
                                                lab.ctypes.data_as(C.POINTER(C.c_uint8)),
                                                counts))
        return lab, [int(c) for c in counts]

    def discard_round1(self, points, labels):
        a = _pts(points)
        lab = np.ascontiguousarray(np.asarray(labels, np.uint8))
        out = np.empty_like(a)
        olab = np.empty(len(a), np.uint8)
        counts = (C.c_size_t * 5)()
        if len(a):
            self._check(self.lib.chgpu_discard_round1(
                self.h, _p(a), lab.ctypes.data_as(C.POINTER(C.c_uint8)), len(a), _p(out),
                olab.ctypes.data_as(C.POINTER(C.c_uint8)), counts))
        s1 = sum(int(c) for c in counts[1:])
        return out[:s1], olab[:s1], [int(c) for c in counts]

    def sort_region(self, region: int, segment) -> np.ndarray:
        a = _pts(segment).copy()
        self._check(self.lib.chgpu_sort_region(self.h, int(region), _p(a), len(a)))
        return a

    def spa_filter(self, region: int, segment, anchors, chunk_count: int = 1024) -> np.ndarray:
        a = _pts(segment)
        an = np.ascontiguousarray(np.asarray(anchors, np.float64).reshape(4))
        out = np.empty((max(len(a), 1), 2), np.float64)
        k = C.c_size_t()
        self._check(self.lib.chgpu_spa_filter(self.h, int(region), _p(a), len(a), _p(an),
                                              chunk_count, _p(out), C.byref(k)))
        return out[:k.value]

    # ---- sharded path ---------------------------------------------------
    def shard_extremes(self, ptr: int, n: int, base_index: int):
        q = np.empty(8, np.float64)
        idx = np.empty(4, np.uint64)
        self._check(self.lib.chgpu_shard_extremes(self.h, C.c_void_p(ptr), n, base_index, _p(q),
                                                  idx.ctypes.data_as(C.POINTER(C.c_uint64))))
        return q, idx

    def shard_chains(self, ptr: int, n: int, quad, chunk_count: int = 1024):
        q = np.ascontiguousarray(np.asarray(quad, np.float64).reshape(8))
        out = _dp()
        kc = (C.c_size_t * 4)()
        self._check(self.lib.chgpu_shard_chains(self.h, C.c_void_p(ptr), n, _p(q), chunk_count,
                                                C.byref(out), kc))
        total = sum(int(c) for c in kc)
        chains = np.ctypeslib.as_array(out, shape=(total * 2,)).reshape(-1, 2).copy() \
            if total else np.empty((0, 2))
        return chains, [int(c) for c in kc]

    def shard_chains_device(self, ptr: int, n: int, quad, chunk_count: int, out_ptr: int,
                            cap_points: int):
        """shard_chains with the chains written to the device buffer at
        out_ptr (cap_points points); returns the kept counts."""
        q = np.ascontiguousarray(np.asarray(quad, np.float64).reshape(8))
        kc = (C.c_size_t * 4)()
        self._check(self.lib.chgpu_shard_chains_device(self.h, C.c_void_p(ptr), n, _p(q),
                                                       chunk_count, C.c_void_p(out_ptr),
                                                       cap_points, kc))
        return [int(c) for c in kc]


_tls = threading.local()


def _ctx() -> Context:
    c = getattr(_tls, "ctx", None)
    if c is None:
        c = Context()
        _tls.ctx = c
    return c


def convex_hull(points, config: PipelineConfig | None = None) -> HullResult:
    """chainhull::convex_hull (pipeline.hpp:55) on the GPU."""
    return _ctx().convex_hull(points, config)


def hull_sharded(contexts, shards, config: PipelineConfig | None = None,
                 on_device: bool = False) -> HullResult:
    """convex_hull of the concatenation of `shards` with several contexts
    (one per GPU) in one process: chgpu_hull_sharded (include/chgpu.h).
    Host shards: (n, 2) float64 arrays, shard s on contexts[s % len]; device
    shards (on_device=True): (ptr, n) pairs, shard s on contexts[s]'s device.
    stats: n_input and n_hull of the whole set, the rest the merge's."""
    config = config or PipelineConfig()
    L = load_library()
    keep = []
    ptrs, counts = [], []
    for sh in shards:
        if on_device:
            p, n = sh
        else:
            a = _pts(sh)
            keep.append(a)
            p, n = a.ctypes.data, len(a)
        ptrs.append(p)
        counts.append(n)
    ctxs = (C.c_void_p * len(contexts))(*[c.h for c in contexts])
    parr = (_dp * len(ptrs))(*[C.cast(C.c_void_p(p), _dp) for p in ptrs])
    carr = (C.c_size_t * len(counts))(*counts)
    out = _dp()
    k = C.c_size_t()
    s = _Stats()
    st = L.chgpu_hull_sharded(ctxs, len(contexts), parr, carr, len(ptrs), int(bool(on_device)),
                              config.chunk_count, int(bool(config.degenerate_fallback)),
                              C.byref(out), C.byref(k), C.byref(s))
    contexts[0]._check(st)
    verts = np.ctypeslib.as_array(out, shape=(k.value * 2,)).reshape(-1, 2).copy() \
        if k.value else np.empty((0, 2))
    return HullResult(Hull(verts), raw_stats=s)


def find_extremes(points) -> np.ndarray:
    return _ctx().find_extremes(points)


def classify(points, quad):
    return _ctx().classify(points, quad)


def discard_round1(points, labels):
    return _ctx().discard_round1(points, labels)


def sort_region(region: int, segment) -> np.ndarray:
    return _ctx().sort_region(region, segment)


def spa_filter(region: int, segment, anchors, chunk_count: int = 1024) -> np.ndarray:
    return _ctx().spa_filter(region, segment, anchors, chunk_count)


# ---- host finisher (no context needed) -----------------------------------

def melkman(polygon) -> np.ndarray:
    """melkman.hpp:29 (host C++ finisher)."""
    L = load_library()
    a = _pts(polygon)
    out = np.empty((max(len(a), 1), 2), np.float64)
    k = C.c_size_t()
    st = L.chgpu_melkman(_p(a), len(a), _p(out), C.byref(k))
    if st:
        _raise(st, "melkman: fewer than 3 distinct vertices or all collinear")
    return out[:k.value]


def _kept_counts(kept_counts, n_chain_points):
    """The four chain lengths as a C array, checked against the chains."""
    kc = [int(c) for c in kept_counts]
    if len(kc) != 4 or any(c < 0 for c in kc) or sum(kc) != n_chain_points:
        raise ValueError(f"kept_counts must be 4 non-negative counts summing to the "
                         f"{n_chain_points} chain points, got {list(kept_counts)}")
    return (C.c_size_t * 4)(*kc)


def assemble_polygon(chains, kept_counts, quad) -> np.ndarray:
    """polygon.hpp:25: chains = the 4 kept chains concatenated."""
    L = load_library()
    a = _pts(chains)
    kc = _kept_counts(kept_counts, len(a))
    q = np.ascontiguousarray(np.asarray(quad, np.float64).reshape(8))
    out = np.empty((len(a) + 4, 2), np.float64)
    k = C.c_size_t()
    st = L.chgpu_assemble_polygon(_p(a), kc, _p(q), _p(out), C.byref(k))
    if st:
        _raise(st, "assemble_polygon: fewer than 3 distinct vertices")
    return out[:k.value]


def merge_hull(runs, quad) -> np.ndarray:
    """chgpu_merge_hull: the hull of the union of several runs of SPA chains
    against one (non-degenerate) quad; runs = [(chains (k, 2), kept_counts[4])]."""
    L = load_library()
    arrs = [_pts(c) for c, _ in runs]
    kcs = []
    for a, (_, kc) in zip(arrs, runs):
        kcs.extend(list(_kept_counts(kc, len(a))))
    total = sum(len(a) for a in arrs)
    parr = (_dp * len(arrs))(*[_p(a) for a in arrs])
    carr = (C.c_size_t * len(kcs))(*kcs)
    q = np.ascontiguousarray(np.asarray(quad, np.float64).reshape(8))
    out = np.empty((total + 4, 2), np.float64)
    k = C.c_size_t()
    st = L.chgpu_merge_hull(parr, carr, len(arrs), _p(q), _p(out), C.byref(k))
    if st:
        _raise(st, "merge_hull: degenerate polygon")
    return out[:k.value]


def finish_chains(chains, kept_counts, quad) -> np.ndarray:
    """assemble_polygon (polygon.hpp:25) + melkman (melkman.hpp:29) in one
    streaming pass (the hull path's finisher)."""
    L = load_library()
    a = _pts(chains)
    kc = _kept_counts(kept_counts, len(a))
    q = np.ascontiguousarray(np.asarray(quad, np.float64).reshape(8))
    out = np.empty((len(a) + 4, 2), np.float64)
    k = C.c_size_t()
    st = L.chgpu_finish_chains(_p(a), kc, _p(q), _p(out), C.byref(k))
    if st:
        _raise(st, "finish_chains: degenerate polygon")
    return out[:k.value]


def canonicalize_ring(ring) -> np.ndarray:
    L = load_library()
    a = _pts(ring).copy()
    L.chgpu_canonicalize_ring(_p(a), len(a))
    return a


def hull_oracle(points) -> np.ndarray:
    """pipeline.hpp:62 reference hull (host sort + monotone chain)."""
    L = load_library()
    a = _pts(points)
    if len(a) == 0:
        raise EmptyInput("hull_oracle: no points")
    out = np.empty((len(a), 2), np.float64)
    k = C.c_size_t()
    st = L.chgpu_hull_oracle(_p(a), len(a), _p(out), C.byref(k))
    if st:
        _raise(st, "hull_oracle")
    return out[:k.value]


def generate(distribution: str | int, n: int, seed: int, begin: int = 0,
             count: int | None = None, out: np.ndarray | None = None) -> np.ndarray:
    """datasets.hpp:35, bit-identical to the reference generator; with
    begin/count, only points [begin, begin + count) of the n-point set (a
    contiguous shard), written into `out` when given (e.g. pinned memory)."""
    L = load_library()
    d = DISTRIBUTIONS.index(distribution) if isinstance(distribution, str) else int(distribution)
    if n <= 0:
        raise ValueError("generate: n must be positive")
    count = n - begin if count is None else count
    if begin < 0 or count < 0 or begin + count > n:
        raise ValueError("generate: slice outside the set")
    if out is None:
        out = np.empty((count, 2), np.float64)
    elif out.shape != (count, 2) or out.dtype != np.float64 or not out.flags.c_contiguous:
        raise ValueError("generate: out must be a contiguous (count, 2) float64 array")
    if count and L.chgpu_generate_range(d, n, seed, begin, count, _p(out)):
        raise ValueError("generate: unknown distribution")
    return out
