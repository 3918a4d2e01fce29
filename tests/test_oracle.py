"""CPU: pin the plain-C oracle (oracle/chainhull_oracle.c) to the reference.

* against the known answers of the reference's own unit tests (tests/kats.py);
* against tests/golden/*.json, produced by the UNMODIFIED reference compiled
  in place (oracle/make_golden.py -> oracle/_ref/libchainhull_ref.so);
* against the live reference library when it is present (here, where
  /root/reference exists).
"""
import numpy as np
import pytest

import kats
from conftest import load_golden, sha, unhex


def test_kat_extremes(oracle):
    for pts, quad in kats.EXTREMES:
        assert oracle.find_extremes(pts).tolist() == quad


def test_kat_frames(oracle):
    for quad, frame in kats.FRAMES:
        assert oracle.frame_vertices(quad).tolist() == frame


def test_kat_classify(oracle):
    pts = [p for p, _ in kats.CLASSIFY]
    assert oracle.classify(pts, kats.UNIT_QUAD).tolist() == [r for _, r in kats.CLASSIFY]


def test_kat_sort_spa(oracle):
    for region, seg, want in kats.SORTS:
        assert oracle.sort_region(region, seg).tolist() == want
    for region, anchors, seg, cc, kept in kats.SPAS:
        assert oracle.spa_filter(region, seg, anchors, cc).tolist() == kept
    with pytest.raises(ValueError):
        oracle.spa_filter(1, [[1, 5]], [[0, 8], [4, 0]], 0)   # spa_test.cpp:109-115


def test_kat_melkman_oracle(oracle):
    for poly, want in kats.MELKMAN:
        st, hull = oracle.melkman(poly)
        if want is None:
            assert st == 2
        else:
            assert st == 0 and hull.tolist() == want
    for pts, want in kats.ORACLE:
        st, hull = oracle.hull_oracle(pts)
        assert st == 0 and hull.tolist() == want
    assert oracle.hull_oracle(np.empty((0, 2)))[0] == 1


def test_kat_pipeline_degenerate(oracle):
    for pts, want in kats.PIPELINE_DEGENERATE:
        h = oracle.convex_hull(pts)
        assert h.status == 0 and h.hull.tolist() == want
    pts = oracle.generate("collinear", 50, 7)
    assert oracle.convex_hull(pts, 1024, degenerate_fallback=False).status == 2


def test_generator_matches_reference_hashes(oracle):
    for case in load_golden("pipeline_sweep.json")[::7]:
        pts = oracle.generate(case["dist"], case["n"], case["seed"])
        assert sha(pts) == case["input_sha"], case


def test_oracle_pipeline_sweep_matches_golden(oracle):
    """acceptance.cpp:57-94 sweep: hull bytes and all four counters."""
    for case in load_golden("pipeline_sweep.json"):
        if case["n"] > 1000:
            continue
        pts = oracle.generate(case["dist"], case["n"], case["seed"])
        for run in case["runs"]:
            h = oracle.convex_hull(pts, run["chunk_count"])
            assert h.status == run["status"]
            assert h.counts.tolist() == run["counts"], (case["dist"], case["n"], run)
            assert sha(h.hull) == run["hull_sha"]
            if run["hull"] is not None:
                assert np.array_equal(h.hull, unhex(run["hull"]))


def test_oracle_stages_match_golden(oracle):
    for case in load_golden("stages.json"):
        pts = oracle.generate(case["dist"], case["n"], case["seed"])
        quad = oracle.find_extremes(pts)
        assert np.array_equal(quad, unhex(case["quad"]))
        h = oracle.convex_hull(pts, case["chunk_count"])
        assert h.region_counts.tolist() == case["region_counts"]
        # region by region: sort then SPA from the reference's own sorted data
        lab = oracle.classify(pts, quad)
        for r in range(1, 5):
            seg = oracle.sort_region(r, pts[lab == r])
            g = case["segments"][r - 1]
            assert len(seg) == g["m"] and sha(seg) == g["sha"], (case["dist"], r)
            anchors = np.array([quad[r - 1], quad[r % 4]])
            kept = oracle.spa_filter(r, seg, anchors, case["chunk_count"])
            assert sha(kept) == case["kept"][r - 1]["sha"], (case["dist"], r, case["chunk_count"])


@pytest.mark.parametrize("idx", range(10))
def test_oracle_big_configs(oracle, idx):
    case = load_golden("big.json")[idx]
    if case["n"] > 4_000_000:
        pytest.skip("20M configs are checked on the GPU (tests/test_gpu_parity.py)")
    pts = oracle.generate(case["dist"], case["n"], case["seed"])
    assert sha(pts) == case["input_sha"]
    h = oracle.convex_hull(pts, case["chunk_count"])
    assert h.counts.tolist() == case["counts"]
    assert sha(h.hull) == case["hull_sha"]


def test_oracle_against_live_reference(oracle):
    from pyoracle import RefLib
    if not RefLib.available():
        pytest.skip("oracle/_ref not built here")
    ref = RefLib()
    rng = np.random.default_rng(5)
    for trial in range(40):
        n = int(rng.integers(1, 3000))
        # small-integer lattices force ties, collinear runs and duplicates
        pts = rng.integers(-4, 5, size=(n, 2)).astype(np.float64) * rng.choice([1.0, 0.5, 0.125])
        for cc in (1, 3, 1024):
            a = oracle.convex_hull(pts, cc)
            b, _ = ref.convex_hull(pts, cc, 1)
            assert a.status == b.status and a.counts.tolist() == b.counts.tolist()
            assert np.array_equal(a.hull, b.hull)
