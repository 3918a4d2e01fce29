"""GPU parity of the SPA pre-filter path (k_filter.cu + k_spa_bins) and of
the full-sort path it replaces, forced per context, against the reference's
golden outputs and the C oracle. Both paths must give the reference's hull
and every stage counter (n_after_spa counts the kept chains, so the kept set
itself is pinned)."""
import os

import numpy as np
import pytest

from conftest import load_golden, sha

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", params=["sort", "filter", "filter_sorted"])
def path_ctx(request):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1508_05488_b200 as P
    ctx = P.Context(0)
    ctx.set_spa_path({"sort": P.SPA_SORT, "filter": P.SPA_FILTER,
                      "filter_sorted": P.SPA_FILTER_SORTED}[request.param])
    ctx.path = request.param
    yield ctx
    ctx.close()


def _counts(r):
    s = r.stats
    return [s.n_input, s.n_after_round1, s.n_after_spa, s.n_hull]


def test_sweep_both_paths(path_ctx, product):
    """acceptance.cpp:57-94 sweep (n = 1 .. 100000, chunk counts 1, 4, 1024)."""
    n = 0
    for case in load_golden("pipeline_sweep.json"):
        pts = product.generate(case["dist"], case["n"], case["seed"])
        for run in case["runs"]:
            r = path_ctx.convex_hull(pts, product.PipelineConfig(chunk_count=run["chunk_count"]))
            assert _counts(r) == run["counts"], (path_ctx.path, case["dist"], case["n"], run)
            assert sha(r.hull.vertices) == run["hull_sha"]
            if not r.diag.degenerate_branch:
                assert r.diag.spa_path == (0 if path_ctx.path == "sort" else 1)
            n += 1
    assert n >= 700


@pytest.mark.parametrize("idx", range(10))
def test_big_configs_both_paths(path_ctx, product, idx):
    case = load_golden("big.json")[idx]
    pts = product.generate(case["dist"], case["n"], case["seed"])
    r = path_ctx.convex_hull(pts)
    assert _counts(r) == case["counts"]
    assert sha(r.hull.vertices) == case["hull_sha"]
    if path_ctx.path == "filter" and case["dist"] in ("uniform_square", "uniform_disk"):
        assert r.diag.spa_path == 1
        s1 = r.stats.n_after_round1
        assert r.diag.n_candidates < 0.1 * s1, (r.diag.n_candidates, s1)


def _clustered(n, seed):
    """Dense clusters (bins far above 32 candidates), exact duplicates and
    a ring of coincident extremes."""
    rng = np.random.default_rng(seed)
    c = rng.random((40, 2))
    pts = c[rng.integers(0, 40, n)] + 1e-4 * rng.standard_normal((n, 2))
    dup = pts[rng.integers(0, n, n // 10)]
    return np.vstack([pts, dup, [[-1, 0.5], [0.5, -1], [2, 0.5], [0.5, 2]] * 3])


@pytest.mark.parametrize("n,seed", [(1000, 1), (100_000, 2), (3_000_000, 3)])
def test_clustered_and_duplicates(path_ctx, product, oracle, n, seed):
    pts = _clustered(n, seed)
    for cc in (1, 5, 1024, 20_000):
        want = oracle.convex_hull(pts, cc)
        r = path_ctx.convex_hull(pts, product.PipelineConfig(chunk_count=cc))
        assert _counts(r) == want.counts.tolist(), (path_ctx.path, n, cc)
        assert np.array_equal(r.hull.vertices, want.hull)
        assert r.diag.kept_counts == want.kept_counts.tolist()


def test_grid_ties_and_signed_zeros(path_ctx, product, oracle):
    rng = np.random.default_rng(17)
    for trial in range(6):
        n = 50_000 * (trial + 1)
        x = rng.integers(0, 33, n) / 32.0 - 0.5
        y = rng.integers(0, 17, n) / 16.0 - 0.5
        pts = np.stack([x, y], 1)
        flip = rng.random(n) < 0.2
        pts[flip] = -pts[flip]
        pts = np.vstack([pts, [[-0.7, 0.0], [0.0, -0.7], [0.7, 0.0], [0.0, 0.7]]])
        for cc in (1, 16, 1024):
            want = oracle.convex_hull(pts, cc)
            r = path_ctx.convex_hull(pts, product.PipelineConfig(chunk_count=cc))
            assert _counts(r) == want.counts.tolist(), (trial, cc)
            assert (r.hull.vertices == want.hull).all()


def test_overflow_falls_back(product, oracle):
    """A bin with more than kBinSortMax candidates (all points on a circle
    arc, every one kept) makes the filter hand over to the full sort."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = product.Context(0)
    ctx.set_spa_path(product.SPA_FILTER)
    pts = product.generate("circle", 2_000_000, 3)
    want = oracle.convex_hull(pts, 1024)
    r = ctx.convex_hull(pts)
    assert _counts(r) == want.counts.tolist()
    assert np.array_equal(r.hull.vertices, want.hull)
    assert r.diag.spa_path in (1, 2)
    ctx.close()


def _ring_points(n, seed, r=1.0):
    rng = np.random.default_rng(seed)
    t = np.sort(rng.random(n)) * 2 * np.pi
    return np.stack([r * np.cos(t), r * np.sin(t)], 1)


def test_auto_sort_hint(product):
    """AUTO mode: after a call that overflowed the pre-filter (20M on a
    circle), a call of about the same size goes straight to the full sort
    (one K2); the hint holds while the chains stay dense and clears after a
    sparse one. Every call gives the reference's hull and counters."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    big = load_golden("big.json")
    circ_case, uni_case = big[4], big[1]
    assert circ_case["dist"] == "circle" and uni_case["dist"] == "uniform_square"
    circ = product.generate("circle", circ_case["n"], circ_case["seed"])
    uni = product.generate("uniform_square", uni_case["n"], uni_case["seed"])
    ctx = product.Context(0)
    paths = []
    for pts, case in ((circ, circ_case), (circ, circ_case), (circ, circ_case), (uni, uni_case),
                      (uni, uni_case)):
        r = ctx.convex_hull(pts)
        assert _counts(r) == case["counts"]
        assert sha(r.hull.vertices) == case["hull_sha"]
        paths.append(r.diag.spa_path)
    # overflow, hinted sort twice, hinted sort (sparse chains: clears), filter
    assert paths == [2, 0, 0, 0, 1], paths
    r = ctx.convex_hull(circ)  # overflows again, sets the hint
    assert r.diag.spa_path == 2
    small = product.generate("circle", 2_000_000, 3)  # outside 2x of the hinted size
    assert ctx.convex_hull(small).diag.spa_path != 0
    r = ctx.convex_hull(circ)
    assert r.diag.spa_path == 2  # (the hint, if any, now describes the small call)
    ctx.set_spa_path(product.SPA_AUTO)  # setting the mode clears the hint
    assert ctx.convex_hull(circ).diag.spa_path == 2
    ctx.close()


@pytest.mark.parametrize("case", ["circle", "circle_noisy", "square_edges", "duplicates",
                                  "near_flat_arc"])
def test_convex_fast_path(gpu_ctx, product, oracle, case):
    """Melkman's all-vertices-kept trajectory verified on the GPU
    (k_convex.cu) must give the reference hull, and must hand over to the
    host loop whenever any predicate deviates (inner survivors, collinear
    edge runs, duplicates, near-collinear arcs)."""
    rng = np.random.default_rng(7)
    if case == "circle":
        pts = product.generate("circle", 300_000, 11)
    elif case == "circle_noisy":
        pts = _ring_points(300_000, 1)
        pts[::97] *= 1.0 - 1e-9 * rng.random((len(pts[::97]), 1))  # a few just inside
    elif case == "square_edges":
        s = rng.random(200_000)
        side = rng.integers(0, 4, len(s))
        pts = np.stack([np.where(side == 0, s, np.where(side == 1, 1.0, np.where(side == 2, 1 - s, 0.0))),
                        np.where(side == 0, 0.0, np.where(side == 1, s, np.where(side == 2, 1.0, 1 - s)))], 1)
        pts = np.vstack([pts, [[0.5, -0.5], [1.5, 0.5], [0.5, 1.5], [-0.5, 0.5]]])
    elif case == "duplicates":
        pts = _ring_points(200_000, 2)
        pts = np.vstack([pts, pts[::1000]])
    else:  # points on a very flat arc: consecutive triples round to collinear
        x = np.sort(rng.random(300_000)) * 1e-3
        pts = np.stack([x, 1e-12 * x * x], 1)
        pts = np.vstack([pts, [[0.0005, -1.0], [0.0005, 1.0]]])
    for cc in (1024, 100_000):
        want = oracle.convex_hull(pts, cc)
        r = gpu_ctx.convex_hull(pts, product.PipelineConfig(chunk_count=cc))
        s = r.stats
        assert [s.n_input, s.n_after_round1, s.n_after_spa, s.n_hull] == want.counts.tolist(), \
            (case, cc)
        assert np.array_equal(r.hull.vertices, want.hull), (case, cc)
        if case == "circle":
            assert r.diag.convex_fast_path
        if case in ("duplicates", "square_edges"):
            assert not r.diag.convex_fast_path


def test_paths_interleaved_on_one_context(product):
    """One context alternating the full-sort and the pre-filtered paths (and
    the degenerate branch) over the acceptance sweep: every look-back of one
    path must ignore whatever the other left in the context's scratch."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = product.Context(0)
    modes = [product.SPA_SORT, product.SPA_FILTER]
    i = 0
    for case in load_golden("pipeline_sweep.json"):
        pts = product.generate(case["dist"], case["n"], case["seed"])
        for run in case["runs"]:
            ctx.set_spa_path(modes[i % 2])
            i += 1
            r = ctx.convex_hull(pts, product.PipelineConfig(chunk_count=run["chunk_count"]))
            assert _counts(r) == run["counts"], (case["dist"], case["n"], run)
            assert sha(r.hull.vertices) == run["hull_sha"]
    ctx.close()


def test_filter_tables_across_sizes(product, oracle):
    """One context, filter path, calls whose bin-table sizes (log2nb) and
    chunk counts change every time: the tables are cleared behind each call
    for the next one, and a call after a certain overflow (circle) or a
    degenerate frame must still start on clean tables."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = product.Context(0)
    ctx.set_spa_path(product.SPA_FILTER)
    cases = [("uniform_square", 3_000_000, 1, 1024), ("uniform_disk", 200_000, 2, 7),
             ("circle", 1_000_000, 3, 1024), ("uniform_square", 5_000_000, 4, 64),
             ("collinear", 100_000, 5, 1024), ("gaussian", 2_000_000, 6, 1024),
             ("uniform_square", 300_000, 7, 2048), ("uniform_disk", 4_000_000, 8, 1024)]
    for dist, n, seed, cc in cases + cases[::-1]:
        pts = product.generate(dist, n, seed)
        want = oracle.convex_hull(pts, cc)
        r = ctx.convex_hull(pts, product.PipelineConfig(chunk_count=cc))
        assert _counts(r) == want.counts.tolist(), (dist, n, cc)
        assert np.array_equal(r.hull.vertices, want.hull), (dist, n, cc)
    ctx.close()


def test_fresh_contexts_after_destroyed_ones(product, oracle):
    """The filter path's completion flag lives in pinned memory that a new
    context may recycle from a destroyed one: a stale flag value must never
    end the new call's wait (each call draws a process-wide sequence number)."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    inputs = [product.generate(d, n, s) for d, n, s in
              (("circle", 300_000, 1), ("uniform_square", 400_000, 2), ("uniform_disk", 300_000, 3),
               ("gaussian", 300_000, 4))]
    wants = [oracle.convex_hull(p, 1024) for p in inputs]
    for rep in range(3):
        for p, want in zip(inputs, wants):
            ctx = product.Context(0)
            r = ctx.convex_hull(p)
            assert _counts(r) == want.counts.tolist(), rep
            assert np.array_equal(r.hull.vertices, want.hull)
            ctx.close()


def test_mapped_emit_and_flag_wait(product):
    """CHGPU_EMIT_MAPPED=1 (chains written into pinned host memory by the
    emit, the host waiting on k_spa_finish's flag): the same hulls and
    counters as the default DMA read-back, across fresh contexts that may
    recycle a destroyed one's pinned memory (a separate process: the knob is
    read once per process)."""
    import json
    import subprocess
    import sys
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from conftest import ROOT
    cases = [("uniform_square", 2_000_000, 1), ("uniform_disk", 1_000_000, 2), ("gaussian", 800_000, 3),
             ("circle", 300_000, 4), ("uniform_square", 20_000, 5)]
    code = r'''
import hashlib, json, sys
sys.path.insert(0, sys.argv[1])
import paper_1508_05488_b200 as P
out = []
for rep in range(2):
    for d, n, s in json.loads(sys.argv[2]):
        ctx = P.Context(0)
        for _ in range(2):  # the second call reads back through the mapped buffer
            r = ctx.convex_hull(P.generate(d, n, s))
        st = r.stats
        out.append([hashlib.sha256(r.hull.vertices.tobytes()).hexdigest(),
                    [st.n_input, st.n_after_round1, st.n_after_spa, st.n_hull]])
        ctx.close()
print(json.dumps(out))
'''
    env = dict(os.environ, CHGPU_EMIT_MAPPED="1")
    res = subprocess.run([sys.executable, "-c", code, ROOT, json.dumps(cases)], env=env,
                         capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    got = json.loads(res.stdout.strip().splitlines()[-1])
    ctx = product.Context(0)
    want = []
    for d, n, s in cases:
        r = ctx.convex_hull(product.generate(d, n, s))
        want.append([sha(r.hull.vertices), _counts(r)])
    ctx.close()
    assert got == want + want


@pytest.mark.parametrize("mode", ["sort", "filter", "auto"])
def test_tile_and_chunk_boundaries(product, oracle, mode):
    """Sizes around the sort path's SPA tile (4096 records) and the sort
    tiles, odd chunk counts (1 record per chunk, chunks straddling tiles and
    region ends): counters and hull equal the oracle's on every path."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = product.Context(0)
    ctx.set_spa_path({"sort": product.SPA_SORT, "filter": product.SPA_FILTER,
                      "auto": product.SPA_AUTO}[mode])
    sizes = [3, 17, 257, 4095, 4096, 4097, 8193, 12289, 30001]
    dists = ["uniform_square", "uniform_disk", "circle", "gaussian", "duplicates_heavy"]
    for i, n in enumerate(sizes):
        d = dists[i % len(dists)]
        pts = product.generate(d, n, 100 + i)
        for cc in (1, 3, 64, 1024, n // 2 + 1, n + 5):
            want = oracle.convex_hull(pts, cc)
            r = ctx.convex_hull(pts, product.PipelineConfig(chunk_count=cc))
            assert _counts(r) == want.counts.tolist(), (mode, d, n, cc)
            assert np.array_equal(r.hull.vertices, want.hull), (mode, d, n, cc)
        # a circle of the same size: every point kept (the convex fast path
        # from 2^16 ring points, the host loop below)
        pts = product.generate("circle", n, 200 + i)
        want = oracle.convex_hull(pts, 7)
        r = ctx.convex_hull(pts, product.PipelineConfig(chunk_count=7))
        assert _counts(r) == want.counts.tolist(), (mode, "circle", n)
        assert np.array_equal(r.hull.vertices, want.hull)
    ctx.close()


def test_concurrent_contexts_in_threads(product):
    """Reentrancy (pipeline.hpp:53: concurrent calls on independent inputs):
    three host threads, one context each, hulls from pageable memory (the
    shared staging pool), device memory and the sort path, interleaved; each
    result equals the same call made alone."""
    import threading
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    inputs = [product.generate("uniform_square", 3_000_000, 41), product.generate("uniform_disk", 2_000_000, 42),
              product.generate("circle", 400_000, 43)]
    solo = []
    ctx = product.Context(0)
    for p in inputs:
        r = ctx.convex_hull(p)
        solo.append((sha(r.hull.vertices), _counts(r)))
    ctx.close()
    errors = []

    def worker(t):
        try:
            c = product.Context(0)
            if t == 2:
                c.set_spa_path(product.SPA_SORT)
            for rep in range(4):
                i = (t + rep) % len(inputs)
                r = c.convex_hull(inputs[i])
                if (sha(r.hull.vertices), _counts(r)) != solo[i]:
                    errors.append((t, rep, i))
            c.close()
        except Exception as e:  # surfaced below
            errors.append((t, repr(e)))

    ths = [threading.Thread(target=worker, args=(t,)) for t in range(3)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    assert not errors, errors
