"""Multi-GPU behind the C ABI: chgpu_hull_sharded (include/chgpu.h), one
process driving one context per GPU, and the C++ drop-in's route through it
(chainhull::convex_hull for spans of 2^32 points or more; CHAINHULL_SHARDS
forces it here). The box has one GPU, so several contexts share it: the
exchange (extreme candidates folded in global index order, chains copied to
the first context's device with cudaMemcpyPeerAsync) is the same code.

The hull must equal the reference's convex_hull of the whole concatenated
set (pipeline.cpp:25-106) bit for bit; n_input and n_hull are the whole
set's (the other counters of a sharded run are the merge's)."""
import ctypes
import os

import numpy as np
import pytest

from conftest import sha

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctxs():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1508_05488_b200 as P
    cs = [P.Context(0) for _ in range(3)]
    yield cs
    for c in cs:
        c.close()


def _ref(dist, n, seed, chunk_count=1024):
    from pyoracle import RefLib
    ref = RefLib()
    pts = ref.generate(dist, n, seed)
    h, _ = ref.convex_hull(pts, chunk_count)
    return pts, h


CASES = [("uniform_square", 1_000_000, 3), ("uniform_disk", 600_000, 4), ("gaussian", 500_000, 5),
         ("circle", 200_000, 6), ("duplicates_heavy", 300_000, 7), ("collinear", 50_000, 8)]


@pytest.mark.parametrize("dist,n,seed", CASES)
@pytest.mark.parametrize("nshards,nctx", [(1, 1), (2, 2), (3, 3), (5, 2)])
def test_host_shards_match_reference(product, ctxs, dist, n, seed, nshards, nctx):
    pts, h = _ref(dist, n, seed)
    bounds = [n * s // nshards for s in range(nshards + 1)]
    shards = [pts[bounds[s]:bounds[s + 1]] for s in range(nshards)]
    r = product.hull_sharded(ctxs[:nctx], shards)
    assert r.hull.vertices.tobytes() == h.hull.tobytes(), (dist, nshards, nctx)
    assert r.stats.n_input == n and r.stats.n_hull == len(h.hull)


@pytest.mark.parametrize("dist,n,seed", CASES[:4])
def test_device_shards_match_reference(product, ctxs, dist, n, seed):
    import torch
    pts, h = _ref(dist, n, seed)
    parts = [torch.from_numpy(np.ascontiguousarray(p)).cuda()
             for p in np.array_split(pts, 3)]
    torch.cuda.synchronize()
    r = product.hull_sharded(ctxs, [(t.data_ptr(), t.shape[0]) for t in parts], on_device=True)
    assert r.hull.vertices.tobytes() == h.hull.tobytes()


def test_slices_of_a_large_span(product, ctxs, monkeypatch):
    """A host shard beyond the slice size (2^30 points; lowered here) is
    processed slice by slice: each slice's extremes with its global indices,
    its chains appended to the context's store."""
    monkeypatch.setenv("CHGPU_SLICE_MAX", "70000")
    for dist, n, seed in [("uniform_square", 1_000_000, 11), ("duplicates_heavy", 400_000, 12),
                          ("circle", 300_000, 13)]:
        pts, h = _ref(dist, n, seed)
        for nctx in (1, 2):
            r = product.hull_sharded(ctxs[:nctx], [pts[: n // 3], pts[n // 3:]])
            assert r.hull.vertices.tobytes() == h.hull.tobytes(), (dist, nctx)


def test_ties_across_shards(product, ctxs):
    """Equal extreme points in different shards: the fold keeps the lowest
    global index (the earliest point, as the reference's sequential fold)."""
    rng = np.random.default_rng(5)
    base = rng.random((40_000, 2))
    pts = np.concatenate([base, base[::-1], base]).copy()
    from pyoracle import RefLib
    h, _ = RefLib().convex_hull(pts, 64)
    for k in (2, 3, 4):
        r = product.hull_sharded(ctxs[:2], np.array_split(pts, k), product.PipelineConfig(chunk_count=64))
        assert r.hull.vertices.tobytes() == h.hull.tobytes()


def test_errors(product, ctxs):
    with pytest.raises(product.EmptyInput):
        product.hull_sharded(ctxs[:1], [np.empty((0, 2))])
    pts = product.generate("uniform_square", 10_000, 1)
    with pytest.raises(ValueError):  # chunk_count == 0 on the non-degenerate branch
        product.hull_sharded(ctxs[:2], [pts[:5000], pts[5000:]], product.PipelineConfig(chunk_count=0))


def test_cpp_drop_in_routes_through_shards(product, monkeypatch):
    """chainhull::convex_hull (libchainhull.so, through its C entry) with
    CHAINHULL_SHARDS: the same hull as the single-device call."""
    from conftest import ROOT
    L = ctypes.CDLL(os.path.join(ROOT, "paper_1508_05488_b200", "libchainhull.so"))
    L.chainhull_capi_convex_hull.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_size_t,
                                            ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p,
                                            ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t),
                                            ctypes.POINTER(ctypes.c_size_t)]
    pts, h = _ref("uniform_disk", 2_000_000, 21)
    out = np.empty((len(h.hull) + 16, 2))
    nh = ctypes.c_size_t()
    cnt = (ctypes.c_size_t * 4)()
    for k in ("0", "4"):
        monkeypatch.setenv("CHAINHULL_SHARDS", k)
        st = L.chainhull_capi_convex_hull(pts.ctypes.data, len(pts), 1024, 0, 1, out.ctypes.data,
                                          len(out), ctypes.byref(nh), cnt)
        assert st == 0
        assert out[: nh.value].tobytes() == h.hull.tobytes(), k
        assert cnt[0] == len(pts) and cnt[3] == len(h.hull)
        if k == "0":
            assert list(cnt) == [int(c) for c in h.counts]


def test_cpp_drop_in_large_hull(product, oracle):
    """chainhull::convex_hull returning a hull of 2^16 vertices or more (its
    result vector is prefaulted from the library's staging threads before
    the copy): the reference's hull, from pageable input."""
    from conftest import ROOT
    L = ctypes.CDLL(os.path.join(ROOT, "paper_1508_05488_b200", "libchainhull.so"))
    L.chainhull_capi_convex_hull.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_size_t,
                                            ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p,
                                            ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t),
                                            ctypes.POINTER(ctypes.c_size_t)]
    for dist, n, seed in (("circle", 300_000, 31), ("circle", 70_000, 32)):
        pts = oracle.generate(dist, n, seed)
        want = oracle.convex_hull(pts, 1024)
        out = np.empty((len(want.hull) + 16, 2))
        nh = ctypes.c_size_t()
        cnt = (ctypes.c_size_t * 4)()
        for _ in range(2):
            st = L.chainhull_capi_convex_hull(pts.ctypes.data, len(pts), 1024, 0, 1, out.ctypes.data,
                                              len(out), ctypes.byref(nh), cnt)
            assert st == 0
            assert nh.value == len(want.hull) >= (1 << 16)
            assert out[: nh.value].tobytes() == want.hull.tobytes()
            assert list(cnt) == [int(c) for c in want.counts]


def test_cpp_drop_in_concurrent_callers(product, oracle):
    """chainhull::convex_hull from several host threads at once (the C++ API
    pools contexts per device): every call returns the reference's hull."""
    import threading
    from conftest import ROOT
    L = ctypes.CDLL(os.path.join(ROOT, "paper_1508_05488_b200", "libchainhull.so"))
    L.chainhull_capi_convex_hull.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_size_t,
                                            ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p,
                                            ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t),
                                            ctypes.POINTER(ctypes.c_size_t)]
    cases = [("uniform_square", 1_500_000, 51), ("gaussian", 1_000_000, 52), ("uniform_disk", 800_000, 53),
             ("circle", 100_000, 54)]
    data = []
    for dist, n, seed in cases:
        pts = oracle.generate(dist, n, seed)
        want = oracle.convex_hull(pts, 1024)
        data.append((pts, want))
    errors = []

    def worker(t):
        for rep in range(3):
            pts, want = data[(t + rep) % len(data)]
            out = np.empty((len(want.hull) + 16, 2))
            nh = ctypes.c_size_t()
            cnt = (ctypes.c_size_t * 4)()
            st = L.chainhull_capi_convex_hull(pts.ctypes.data, len(pts), 1024, 0, 1, out.ctypes.data,
                                              len(out), ctypes.byref(nh), cnt)
            if st or out[: nh.value].tobytes() != want.hull.tobytes():
                errors.append((t, rep, st))

    ths = [threading.Thread(target=worker, args=(t,)) for t in range(4)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    assert not errors, errors
