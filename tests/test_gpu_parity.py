"""GPU parity: the sm_100a path through the C ABI (libchgpu.so) against the
reference's golden outputs (tests/golden, made by the unmodified reference)
and the C oracle. Bit-exact: hull vertex bytes and every stage counter."""
import threading

import numpy as np
import pytest

import kats
from conftest import load_golden, sha, unhex

pytestmark = pytest.mark.gpu


def test_kat_extremes_frames_classify(gpu_ctx):
    for pts, quad in kats.EXTREMES:
        assert gpu_ctx.find_extremes(pts).tolist() == quad
    pts = [p for p, _ in kats.CLASSIFY]
    lab, counts = gpu_ctx.classify(pts, kats.UNIT_QUAD)
    assert lab.tolist() == [r for _, r in kats.CLASSIFY]
    assert sum(counts) == len(pts)


def test_kat_sort_spa(gpu_ctx, product):
    for region, seg, want in kats.SORTS:
        assert gpu_ctx.sort_region(region, seg).tolist() == want
    for region, anchors, seg, cc, kept in kats.SPAS:
        assert gpu_ctx.spa_filter(region, seg, anchors, cc).tolist() == kept
    with pytest.raises(ValueError):
        gpu_ctx.spa_filter(1, [[1, 5]], [[0, 8], [4, 0]], 0)
    with pytest.raises(ValueError):
        gpu_ctx.sort_region(0, [[1, 2], [3, 4]])
    assert gpu_ctx.spa_filter(1, np.empty((0, 2)), [[0, 8], [4, 0]], 4).shape == (0, 2)


def test_kat_pipeline(gpu_ctx, product):
    pts, want = kats.SQUARE
    assert gpu_ctx.convex_hull(pts).hull.vertices.tolist() == want
    for pts, want in kats.PIPELINE_DEGENERATE:
        r = gpu_ctx.convex_hull(pts)
        assert r.hull.vertices.tolist() == want
        assert r.stats.n_after_spa == r.stats.n_after_round1
    with pytest.raises(product.EmptyInput):
        gpu_ctx.convex_hull(np.empty((0, 2)))
    col = product.generate("collinear", 50, 7)
    with pytest.raises(product.DegenerateInput):
        gpu_ctx.convex_hull(col, product.PipelineConfig(degenerate_fallback=False))
    # chunk_count == 0 raises only on the non-degenerate branch (spa.cpp:112)
    with pytest.raises(ValueError):
        gpu_ctx.convex_hull(product.generate("uniform_square", 1000, 1),
                            product.PipelineConfig(chunk_count=0))
    r = gpu_ctx.convex_hull(col, product.PipelineConfig(chunk_count=0))
    assert len(r.hull.vertices) == 2


def test_interior_points_ignored(gpu_ctx):
    # pipeline_test.cpp:27-38
    rng = np.random.default_rng(79)
    pts = np.vstack([[[0, 0], [1, 0], [1, 1], [0, 1]], 0.1 + 0.8 * rng.random((100, 2))])
    r = gpu_ctx.convex_hull(pts)
    assert r.hull.vertices.tolist() == [[0, 0], [1, 0], [1, 1], [0, 1]]
    assert r.stats.n_hull == 4


def test_pipeline_sweep_bit_exact(gpu_ctx, product):
    """acceptance.cpp:57-94 (criterion 1) against the reference's own outputs."""
    cases = 0
    for case in load_golden("pipeline_sweep.json"):
        pts = product.generate(case["dist"], case["n"], case["seed"])
        for run in case["runs"]:
            r = gpu_ctx.convex_hull(pts, product.PipelineConfig(chunk_count=run["chunk_count"]))
            s = r.stats
            got = [s.n_input, s.n_after_round1, s.n_after_spa, s.n_hull]
            assert got == run["counts"], (case["dist"], case["n"], case["seed"], run["chunk_count"])
            assert sha(r.hull.vertices) == run["hull_sha"], (case["dist"], case["n"], case["seed"])
            cases += 1
    assert cases >= 700


def test_stage_fixtures(gpu_ctx, product):
    for case in load_golden("stages.json"):
        pts = product.generate(case["dist"], case["n"], case["seed"])
        quad = gpu_ctx.find_extremes(pts)
        assert np.array_equal(quad, unhex(case["quad"]))
        lab, counts = gpu_ctx.classify(pts, quad)
        assert counts == case["region_counts"]
        for r in range(1, 5):
            seg = gpu_ctx.sort_region(r, pts[lab == r])
            g = case["segments"][r - 1]
            assert sha(seg) == g["sha"], (case["dist"], case["n"], r)
            anchors = np.array([quad[r - 1], quad[r % 4]])
            kept = gpu_ctx.spa_filter(r, seg, anchors, case["chunk_count"])
            assert sha(kept) == case["kept"][r - 1]["sha"], (case["dist"], r, case["chunk_count"])
        res = gpu_ctx.convex_hull(pts, product.PipelineConfig(chunk_count=case["chunk_count"]))
        if not res.diag.degenerate_branch:
            assert res.diag.region_counts == case["region_counts"]
            assert res.diag.kept_counts == [k["k"] for k in case["kept"]]


def test_discard_round1_groups_regions(gpu_ctx, product, oracle):
    pts = product.generate("uniform_disk", 50000, 3)
    quad = gpu_ctx.find_extremes(pts)
    lab, counts = gpu_ctx.classify(pts, quad)
    out, olab, c2 = gpu_ctx.discard_round1(pts, lab)
    assert c2[1:] == counts[1:] and c2[0] == 0
    off = 0
    for r in range(1, 5):
        blk = out[off:off + counts[r]]
        assert (olab[off:off + counts[r]] == r).all()
        want = pts[lab == r]
        assert np.array_equal(oracle.sort_region(r, blk), oracle.sort_region(r, want))
        off += counts[r]


@pytest.mark.parametrize("idx", range(10))
def test_big_configs_bit_exact(gpu_ctx, product, idx):
    """BASELINE.json configs at full size vs the reference's outputs."""
    case = load_golden("big.json")[idx]
    pts = product.generate(case["dist"], case["n"], case["seed"])
    assert sha(pts) == case["input_sha"]
    r = gpu_ctx.convex_hull(pts)
    s = r.stats
    assert [s.n_input, s.n_after_round1, s.n_after_spa, s.n_hull] == case["counts"]
    assert sha(r.hull.vertices) == case["hull_sha"]
    assert np.array_equal(r.diag.quad, unhex(case["quad"]))


def test_device_resident_input(gpu_ctx, product):
    import torch
    case = load_golden("big.json")[1]  # 20M uniform seed 42
    pts = product.generate(case["dist"], case["n"], case["seed"])
    t = torch.from_numpy(pts).cuda()
    torch.cuda.synchronize()
    r = gpu_ctx.convex_hull_device(t.data_ptr(), len(pts))
    s = r.stats
    assert [s.n_input, s.n_after_round1, s.n_after_spa, s.n_hull] == case["counts"]
    assert sha(r.hull.vertices) == case["hull_sha"]
    # properties at full size: repeat is idempotent; chunk_count only changes counters
    r2 = gpu_ctx.convex_hull_device(t.data_ptr(), len(pts), product.PipelineConfig(chunk_count=1))
    assert np.array_equal(r2.hull.vertices, r.hull.vertices)
    assert r2.stats.n_after_spa <= r.stats.n_after_spa


def _tie_heavy(n, seed, levels=101):
    rng = np.random.default_rng(seed)
    x = rng.integers(0, levels, n) / (levels - 1)
    y = rng.random(n)
    pts = np.stack([x, y], axis=1)
    diamond = np.array([[-0.01, 0.5], [0.5, -0.01], [1.01, 0.5], [0.5, 1.01]])
    return np.vstack([pts, diamond])


@pytest.mark.parametrize("n,levels", [(3000, 11), (200_000, 101), (2_000_000, 101),
                                      (1_000_000, 5)])
def test_tie_runs_match_oracle(gpu_ctx, product, oracle, n, levels):
    """Equal-primary runs (short ones in shared memory, long ones through the
    onesweep engine keyed on the secondary) reproduce region_less order."""
    pts = _tie_heavy(n, n + levels, levels)
    for cc in (1, 7, 1024):
        want = oracle.convex_hull(pts, cc)
        r = gpu_ctx.convex_hull(pts, product.PipelineConfig(chunk_count=cc))
        s = r.stats
        assert [s.n_input, s.n_after_round1, s.n_after_spa, s.n_hull] == want.counts.tolist()
        assert np.array_equal(r.hull.vertices, want.hull)
        assert r.diag.kept_counts == want.kept_counts.tolist()
    quad = gpu_ctx.find_extremes(pts)
    lab, _ = gpu_ctx.classify(pts, quad)
    for reg in range(1, 5):
        seg = pts[lab == reg]
        assert np.array_equal(gpu_ctx.sort_region(reg, seg), oracle.sort_region(reg, seg))


def test_signed_zero_ties(gpu_ctx, oracle):
    """-0.0 and +0.0 are == in the reference; they must form one tie run."""
    rng = np.random.default_rng(11)
    base = np.array([[0.0, 0.3], [-0.0, 0.7], [0.0, -0.2], [-0.0, 0.1], [-0.0, -0.6]])
    ring = np.array([[-1.0, 0.0], [0.0, -1.0], [1.0, 0.0], [0.0, 1.0]])
    for trial in range(20):
        pts = np.vstack([ring, base[rng.permutation(len(base))], rng.random((50, 2)) - 0.5])
        for reg in range(1, 5):
            seg = np.vstack([base, -base])[rng.permutation(10)]
            got = gpu_ctx.sort_region(reg, seg)
            want = oracle.sort_region(reg, seg)
            assert (got == want).all()   # == : the reference leaves +-0 order unspecified
        r = gpu_ctx.convex_hull(pts)
        w = oracle.convex_hull(pts)
        assert (r.hull.vertices == w.hull).all() and r.stats.n_after_spa == w.counts[2]


@pytest.mark.parametrize("dist", ["uniform_square", "uniform_disk", "gaussian", "circle",
                                  "duplicates_heavy", "collinear"])
def test_medium_sizes_all_chunk_counts(gpu_ctx, product, oracle, dist):
    for n, seed in ((4097, 1), (65_537, 2), (1_000_003, 3)):
        pts = product.generate(dist, n, seed)
        for cc in (1, 2, 64, 1024, 100_000):
            want = oracle.convex_hull(pts, cc)
            r = gpu_ctx.convex_hull(pts, product.PipelineConfig(chunk_count=cc))
            s = r.stats
            assert [s.n_input, s.n_after_round1, s.n_after_spa, s.n_hull] == want.counts.tolist(), \
                (dist, n, cc)
            assert np.array_equal(r.hull.vertices, want.hull)


def test_concurrent_contexts(product):
    """Reentrancy (pipeline.hpp:53): independent contexts on threads."""
    pts = [product.generate("uniform_disk", 300_000, s) for s in range(4)]
    want = [product.Context(0).convex_hull(p).hull.vertices for p in pts]
    out = [None] * 4

    def work(i):
        ctx = product.Context(0)
        for _ in range(3):
            out[i] = ctx.convex_hull(pts[i]).hull.vertices

    th = [threading.Thread(target=work, args=(i,)) for i in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for i in range(4):
        assert np.array_equal(out[i], want[i])
