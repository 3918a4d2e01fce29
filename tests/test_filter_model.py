"""CPU model of the SPA pre-filter (paper_1508_05488_b200/csrc/k_filter.cu)
checked against the oracle's spa_filter (reference spa.cpp:109-163).

The model follows the kernels step for step on a region the oracle sorted
(region_less order, reference spa.cpp:38-81): bins of the primary coordinate
(bin_of in chgpu_internal.cuh, same IEEE double arithmetic), exact per-bin
counts and guarded extremes, per-bin thresholds T_b from whole bins of the
same chunk, candidates = straddling bins + records that do not step back
from T_b, then the chunked SPA over the candidates only. The kept sequence
must equal spa_filter over the full region, bit for bit."""
import numpy as np
import pytest

import kats


def bin_geom(lo, hi, log2nb):
    nb = float(1 << log2nb)
    span = hi - lo
    s = nb / span if span > 0.0 else 0.0
    if not (s < 1e300):
        s = 0.0
    return lo, s, nb - 1.0


def bin_of(region, prim, geom):
    lo, scale, top = geom
    with np.errstate(invalid="ignore", over="ignore"):
        t = (prim - lo) * scale
    t = np.nan_to_num(t, nan=0.0)
    t = np.minimum(np.maximum(t, 0.0), top)
    b = np.trunc(t).astype(np.int64)
    return (int(top) - b) if region >= 3 else b


def region_range(quad, region):
    q = np.asarray(quad, np.float64).reshape(-1)
    return {1: (q[0], q[2]), 2: (q[3], q[5]), 3: (q[6], q[4]), 4: (q[1], q[7])}[region]


def model_filter_spa(region, srt, seed, chunk_count, quad, log2nb):
    """Kept chain of one sorted region via the pre-filter; also returns the
    candidate count."""
    m = len(srt)
    if m == 0:
        return srt[:0], 0
    is_min = region in (1, 4)
    prim = srt[:, 0] if region in (1, 3) else srt[:, 1]
    g = srt[:, 1] if region in (1, 3) else srt[:, 0]
    geom = bin_geom(*region_range(quad, region), log2nb)
    b = bin_of(region, prim, geom)
    assert (np.diff(b) >= 0).all(), "bins must be monotone in region_less order"
    nb = 1 << log2nb
    cnt = np.bincount(b, minlength=nb)
    start = np.concatenate([[0], np.cumsum(cnt)[:-1]])
    ident = np.inf if is_min else -np.inf
    ext = np.full(nb, ident)
    (np.minimum if is_min else np.maximum).at(ext, b, g)
    cs = -(-m // chunk_count)
    # thresholds: seed of the chunk, then whole bins of the chunk before b
    thr = np.full(nb, ident)
    straddle = np.zeros(nb, bool)
    run_chunk, run_val = -1, ident
    for i in range(nb):
        if cnt[i] == 0:
            continue
        clo, chi = start[i] // cs, (start[i] + cnt[i] - 1) // cs
        if clo != chi:
            straddle[i] = True
            run_chunk, run_val = chi, ident
            continue
        t = seed if clo == 0 else ident
        if run_chunk == clo:
            t = min(t, run_val) if is_min else max(t, run_val)
        thr[i] = t
        if run_chunk != clo:
            run_chunk, run_val = clo, ident
        run_val = min(run_val, ext[i]) if is_min else max(run_val, ext[i])
    steps_back = (g > thr[b]) if is_min else (g < thr[b])
    cand = straddle[b] | ~steps_back
    # chunked SPA over the candidates (spa.cpp:121-147)
    idx = np.nonzero(cand)[0]
    kept = []
    cur_chunk, t = -1, None
    for i in idx:
        c = i // cs
        if c != cur_chunk:
            cur_chunk = c
            t = seed if c == 0 else ident
        gi = g[i]
        if not (gi > t if is_min else gi < t):
            kept.append(i)
        t = min(t, gi) if is_min else max(t, gi)
    return srt[kept], int(cand.sum())


def _regions(oracle, pts):
    quad = oracle.find_extremes(pts)
    lab = oracle.classify(pts, quad)
    return quad, lab


def _check(oracle, pts, chunk_counts, log2nbs=(10, 12, 16)):
    quad, lab = _regions(oracle, pts)
    qv = np.asarray(quad).reshape(4, 2)
    total = cands = 0
    for region in range(1, 5):
        seg = pts[lab == region]
        srt = oracle.sort_region(region, seg)
        anchors = np.array([qv[region - 1], qv[region % 4]])
        seed = anchors[0][1] if region in (1, 3) else anchors[0][0]
        for cc in chunk_counts:
            want = oracle.spa_filter(region, srt, anchors, cc)
            for lb in log2nbs:
                got, nc = model_filter_spa(region, srt, seed, cc, qv, lb)
                assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), \
                    (region, cc, lb, len(got), len(want))
                total += len(srt)
                cands += nc
    return total, cands


@pytest.mark.parametrize("dist,n,seed", [("uniform_square", 200_000, 42), ("uniform_disk", 100_000, 7),
                                         ("gaussian", 100_000, 3), ("circle", 20_000, 5),
                                         ("duplicates_heavy", 50_000, 9), ("uniform_square", 1000, 1)])
def test_filter_model_equals_spa(oracle, dist, n, seed):
    pts = oracle.generate(dist, n, seed)
    quad, _ = _regions(oracle, pts)
    frame = oracle.frame_vertices(quad)
    if len(frame) <= 2:
        pytest.skip("degenerate frame: no SPA on this input")
    total, cands = _check(oracle, pts, (1, 2, 7, 64, 1024, 5000))
    if dist == "uniform_square" and n >= 100_000:
        assert cands < 0.35 * total  # the filter removes most records on spread inputs


def test_filter_model_ties_and_zeros(oracle):
    rng = np.random.default_rng(5)
    x = rng.integers(0, 9, 20_000) / 8.0 - 0.5
    y = rng.integers(0, 7, 20_000) / 6.0 - 0.5
    pts = np.stack([x, y], 1)
    pts[rng.random(len(pts)) < 0.1] *= -1.0  # sprinkle -0.0 in place of +0.0
    pts = np.vstack([pts, [[-0.6, 0.0], [0.0, -0.6], [0.6, 0.0], [0.0, 0.6]]])
    _check(oracle, pts, (1, 3, 100, 1024))


def test_filter_model_kats(oracle):
    """The SPA known answers (spa_test.cpp) through the model."""
    for region, anchors, seg, cc, kept in kats.SPAS:
        srt = oracle.sort_region(region, np.asarray(seg, np.float64).reshape(-1, 2))
        anchors = np.asarray(anchors, np.float64)
        seed = anchors[0][1] if region in (1, 3) else anchors[0][0]
        # a quad whose region range spans the anchors
        quad = np.zeros((4, 2))
        quad[region - 1] = anchors[0]
        quad[region % 4] = anchors[1]
        for lb in (10, 16):
            got, _ = model_filter_spa(region, srt, seed, cc, quad, lb)
            assert got.tolist() == kept
