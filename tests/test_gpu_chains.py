"""GPU: the SPA chains of the default (pre-filtered) path pinned element by
element against the reference's own spa_filter output (spa.cpp:109-163, via
its stage dump, pipeline.cpp:36-96): tests/golden/chains.json was written by
oracle/make_golden_chains.py from the unmodified reference. A substituted or
misordered chain point that leaves the hull unchanged fails here.

Also: the sort path's chains equal the same goldens, and the small
stages.json inputs at every recorded chunk count on both paths."""
import numpy as np
import pytest

from conftest import load_golden, sha, unhex

pytestmark = pytest.mark.gpu

CHAINS = load_golden("chains.json")
STAGES = load_golden("stages.json")


@pytest.fixture(scope="module")
def tap_ctx(product):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = product.Context(0)
    ctx.set_chains_tap(True)
    yield ctx
    ctx.close()


_inputs = {}


def _points(product, dist, n, seed):
    key = (dist, n, seed)
    if key not in _inputs:
        _inputs.clear()
        _inputs[key] = product.generate(dist, n, seed)
    return _inputs[key]


def _check(chains, counts, want_regions, label):
    assert counts == [r["k"] for r in want_regions], (label, counts)
    o = 0
    for r, want in enumerate(want_regions):
        seg = chains[o:o + counts[r]]
        if sha(seg) != want["sha"]:
            # locate the first differing point for the message
            head = unhex(want["head"])
            raise AssertionError(f"{label}: region {r + 1} chain differs from the reference "
                                 f"(head ours {seg[:2].tolist()} ref {head[:2].tolist()})")
        o += counts[r]


@pytest.mark.parametrize("case", CHAINS, ids=lambda c: f"{c['dist']}-{c['n']}-cc{c['chunk_count']}")
@pytest.mark.parametrize("path", ["auto", "filter", "filter_sorted", "sort"])
def test_chains_match_reference(product, tap_ctx, case, path):
    if path == "sort" and case["n"] >= 20_000_000 and case["chunk_count"] == 1024 \
            and case["dist"] == "circle":
        pytest.skip("same kernels as the other circle cases")
    pts = _points(product, case["dist"], case["n"], case["seed"])
    assert sha(pts) == case["input_sha"]
    mode = {"auto": product.SPA_AUTO, "filter": product.SPA_FILTER, "sort": product.SPA_SORT,
            "filter_sorted": product.SPA_FILTER_SORTED}[path]
    tap_ctx.set_spa_path(mode)
    try:
        r = tap_ctx.convex_hull(pts, product.PipelineConfig(chunk_count=case["chunk_count"]))
    finally:
        tap_ctx.set_spa_path(product.SPA_AUTO)
    assert list(r.diag.region_counts) == case["region_counts"]
    chains, counts = tap_ctx.last_chains()
    if path in ("filter", "filter_sorted") or (path == "auto" and case["chunk_count"] <= case["n"] // 64):
        # the pre-filtered path really ran (no overflow fallback) where it applies
        assert r.diag.spa_path in (1, 2)
    _check(chains, counts, case["kept"], f"{case['dist']} cc={case['chunk_count']} {path}")


@pytest.mark.parametrize("path", ["filter", "filter_sorted", "sort"])
def test_stage_chains_small_inputs(product, tap_ctx, path):
    """Every stages.json case (8 inputs x up to 8 chunk counts): the chains
    point by point against the reference's kept arrays."""
    mode = {"filter": product.SPA_FILTER, "sort": product.SPA_SORT,
            "filter_sorted": product.SPA_FILTER_SORTED}[path]
    tap_ctx.set_spa_path(mode)
    checked = 0
    try:
        for c in STAGES:
            pts = product.generate(c["dist"], c["n"], c["seed"])
            assert sha(pts) == c["input_sha"]
            r = tap_ctx.convex_hull(pts, product.PipelineConfig(chunk_count=c["chunk_count"]))
            if r.diag.degenerate_branch:
                continue
            chains, counts = tap_ctx.last_chains()
            want = [k["k"] for k in c["kept"]]
            assert counts == want, (c["dist"], c["n"], c["chunk_count"], counts, want)
            o = 0
            for reg, k in enumerate(c["kept"]):
                assert sha(chains[o:o + k["k"]]) == k["sha"], (c["dist"], c["n"], c["chunk_count"], reg)
                o += k["k"]
            checked += 1
    finally:
        tap_ctx.set_spa_path(product.SPA_AUTO)
    assert checked >= 30


def test_tap_off_raises(product, gpu_ctx):
    with pytest.raises(ValueError):
        gpu_ctx.last_chains()
