"""GPU: xy_binary ingestion (chgpu_hull_xy_binary) = the reference's
read_points(path, XyBinary) (io.cpp:101-116) followed by convex_hull, with
the reference's errors in its order: IoError, ParseError (payload not whole
float64 pairs), NonFiniteCoordinate, then the hull's own (EmptyInput ...)."""
import os

import numpy as np
import pytest

from conftest import load_golden, sha

pytestmark = pytest.mark.gpu


def _write(path, pts):
    np.ascontiguousarray(pts, dtype="<f8").tofile(path)  # the xy_binary layout


@pytest.mark.parametrize("dist,n,seed", [("uniform_square", 1_000_000, 42), ("uniform_disk", 300_000, 7),
                                         ("circle", 100_000, 3), ("duplicates_heavy", 50_000, 5),
                                         ("collinear", 3_000, 9), ("gaussian", 5_000_003, 11)])
def test_file_hull_equals_reference(gpu_ctx, product, oracle, tmp_path, dist, n, seed):
    pts = product.generate(dist, n, seed)
    f = tmp_path / "pts.xyb"
    _write(f, pts)
    back = np.fromfile(f, dtype="<f8").reshape(-1, 2)  # read_xy_binary: LE decode
    for cc in (1024, 7):
        want = oracle.convex_hull(back, cc)
        r = gpu_ctx.hull_xy_binary(f, product.PipelineConfig(chunk_count=cc))
        s = r.stats
        assert [s.n_input, s.n_after_round1, s.n_after_spa, s.n_hull] == want.counts.tolist()
        assert np.array_equal(r.hull.vertices, want.hull)


def test_file_20m_headline(gpu_ctx, product, tmp_path):
    case = load_golden("big.json")[1]  # 20M uniform seed 42
    pts = product.generate(case["dist"], case["n"], case["seed"])
    f = tmp_path / "u20m.xyb"
    _write(f, pts)
    r = gpu_ctx.hull_xy_binary(f)
    s = r.stats
    assert [s.n_input, s.n_after_round1, s.n_after_spa, s.n_hull] == case["counts"]
    assert sha(r.hull.vertices) == case["hull_sha"]
    os.remove(f)


def test_file_errors(gpu_ctx, product, tmp_path):
    with pytest.raises(product.IoError):
        gpu_ctx.hull_xy_binary(tmp_path / "missing.xyb")
    f = tmp_path / "odd.xyb"
    f.write_bytes(b"\0" * 24)  # 1.5 pairs
    with pytest.raises(product.ParseError):
        gpu_ctx.hull_xy_binary(f)
    f.write_bytes(b"")
    with pytest.raises(product.EmptyInput):
        gpu_ctx.hull_xy_binary(f)
    pts = product.generate("uniform_square", 3_000_000, 1)
    for pos, bad in ((0, np.nan), (2_500_000, np.inf), (2_999_999, -np.inf)):
        q = pts.copy()
        q[pos, pos % 2] = bad
        _write(f, q)
        with pytest.raises(product.NonFiniteCoordinate):
            gpu_ctx.hull_xy_binary(f)
    # a payload that is both ragged and non-finite: the size check comes first
    q = pts[:10].copy()
    q[3, 0] = np.nan
    f.write_bytes(np.ascontiguousarray(q, dtype="<f8").tobytes() + b"\0" * 8)
    with pytest.raises(product.ParseError):
        gpu_ctx.hull_xy_binary(f)
    # the context stays usable after every error
    _write(f, pts)
    assert gpu_ctx.hull_xy_binary(f).stats.n_input == len(pts)
