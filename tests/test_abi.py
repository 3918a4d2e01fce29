"""CPU: the C-ABI library loads, exports every symbol include/chgpu.h
declares, and its host-side parts (finisher, generator, error mapping) agree
with the reference's known answers. No GPU compute is called here."""
import ctypes as C
import os
import re
import sys

import numpy as np
import pytest

import kats
from conftest import ROOT, load_golden, sha


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "chgpu.h")).read()
    return sorted(set(re.findall(r"\b(chgpu_[a-z_0-9]+)\s*\(", src)))


def test_header_symbols_exported(product):
    lib = product.load_library()
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in include/chgpu.h but not exported"


def test_capi_header_symbols_exported(product):
    product.load_library()
    lib = C.CDLL(os.path.join(ROOT, "paper_1508_05488_b200", "libchainhull.so"))
    src = open(os.path.join(ROOT, "include", "chainhull_capi.h")).read()
    syms = sorted(set(re.findall(r"\b(chainhull_capi_[a-z_0-9]+)\s*\(", src)))
    assert syms
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in include/chainhull_capi.h but not exported"


def test_no_device_fails_loudly(product):
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    with pytest.raises(product.Error):
        product.Context()


def test_host_melkman_kats(product):
    for poly, want in kats.MELKMAN:
        if want is None:
            with pytest.raises(product.DegenerateInput):
                product.melkman(poly)
        else:
            assert product.melkman(poly).tolist() == want


def test_host_assemble_kats(product):
    for quad, chains, want in kats.ASSEMBLE:
        flat = [p for c in chains for p in c]
        counts = [len(c) for c in chains]
        if want is None:
            with pytest.raises(product.DegenerateInput):
                product.assemble_polygon(np.array(flat).reshape(-1, 2), counts, quad)
        else:
            got = product.assemble_polygon(np.array(flat, np.float64).reshape(-1, 2), counts, quad)
            assert got.tolist() == want


def test_host_hull_oracle_and_canonicalize(product):
    for pts, want in kats.ORACLE:
        assert product.hull_oracle(pts).tolist() == want
    with pytest.raises(product.EmptyInput):
        product.hull_oracle(np.empty((0, 2)))
    ring = product.canonicalize_ring([[4, 4], [0, 4], [0, 0], [4, 0]])   # melkman_test.cpp:66-71
    assert ring.tolist() == [[0, 0], [4, 0], [4, 4], [0, 4]]


def test_product_generator_bit_identical(product):
    """chgpu_generate == the reference generate() (hashes from the reference)."""
    for case in load_golden("pipeline_sweep.json"):
        pts = product.generate(case["dist"], case["n"], case["seed"])
        assert sha(pts) == case["input_sha"], (case["dist"], case["n"], case["seed"])
    for case in load_golden("big.json"):
        if case["n"] <= 4_000_000:
            assert sha(product.generate(case["dist"], case["n"], case["seed"])) == case["input_sha"]
    with pytest.raises(ValueError):
        product.generate("uniform_square", 0, 1)


def test_host_finisher_matches_oracle_random_polygons(product, oracle):
    """acceptance.cpp:281-300 (criterion 7) style: melkman on radial polygons."""
    rng = np.random.default_rng(777)
    for _ in range(100):
        k = int(rng.integers(3, 400))
        pts = rng.random((k, 2))
        c = pts.mean(axis=0)
        ring = pts[np.argsort(np.arctan2(pts[:, 1] - c[1], pts[:, 0] - c[0]))]
        st, want = oracle.melkman(ring)
        assert st == 0
        assert np.array_equal(product.melkman(ring), want)
        assert np.array_equal(product.hull_oracle(ring), oracle.hull_oracle(ring)[1])


def test_stats_struct_layout(product):
    assert C.sizeof(product._Stats) == 4 * 8 + 7 * 8


def test_host_melkman_on_pipeline_polygons(product, oracle):
    """The finisher on the polygons the pipeline actually builds (SPA chains
    + corners, reference stage dumps) and on collinear-heavy grid rings:
    bit-identical hulls and the same degenerate verdicts as the reference's
    melkman (melkman.cpp:17-86)."""
    from pyoracle import RefLib
    if not RefLib.available():
        pytest.skip("oracle/_ref not built")
    ref = RefLib()
    for dist, n, seed in (("uniform_square", 200_000, 42), ("uniform_disk", 200_000, 3),
                          ("gaussian", 100_000, 5), ("circle", 5_000, 9)):
        pts = ref.generate(dist, n, seed)
        for cc in (1, 7, 1024):
            quad, rc, srt, kept, kc = ref.stage_dump(pts, cc)
            poly = product.assemble_polygon(kept, kc, quad)
            st, want = ref.melkman(poly)
            assert st == 0
            assert np.array_equal(product.melkman(poly), want), (dist, cc)
    rng = np.random.default_rng(4242)
    for trial in range(300):
        k = int(rng.integers(3, 60))
        g = rng.integers(0, 5, (k, 2)).astype(np.float64)
        c = g.mean(axis=0) + 1e-3
        ring = g[np.argsort(np.arctan2(g[:, 1] - c[1], g[:, 0] - c[0]), kind="stable")]
        st, want = ref.melkman(ring)
        if st != 0:
            with pytest.raises(product.DegenerateInput):
                product.melkman(ring)
        else:
            assert np.array_equal(product.melkman(ring), want), trial


def _finish_reference(ref, chains, kc, quad):
    """assemble_polygon + melkman of the reference (None when degenerate)."""
    try:
        poly = np.asarray(quad).reshape(4, 2)
        ring = []
        off = 0
        for r in range(4):
            for p in [poly[r]] + list(chains[off:off + kc[r]]):
                if not ring or not (ring[-1][0] == p[0] and ring[-1][1] == p[1]):
                    ring.append(p)
            off += kc[r]
        if len(ring) > 1 and ring[0][0] == ring[-1][0] and ring[0][1] == ring[-1][1]:
            ring.pop()
        if len(ring) < 3:
            return None
        st, hull = ref.melkman(np.array(ring))
        return None if st else hull
    except Exception:
        return None


def test_finish_chains_equals_assemble_then_melkman(product, oracle):
    """The fused streaming finisher == assemble_polygon + melkman (reference
    polygon.cpp:7-29, melkman.cpp:17-86) on pipeline chains and on
    adversarial rings: duplicates across segment joints, empty chains, a
    closing vertex equal to corner 0, collinear and tiny inputs."""
    from pyoracle import RefLib
    if not RefLib.available():
        pytest.skip("oracle/_ref not built")
    ref = RefLib()
    for dist, n, seed in (("uniform_square", 100_000, 42), ("circle", 3_000, 9),
                          ("gaussian", 50_000, 5), ("uniform_disk", 30_000, 1)):
        pts = ref.generate(dist, n, seed)
        for cc in (1, 3, 1024):
            quad, rc, srt, kept, kc = ref.stage_dump(pts, cc)
            want = _finish_reference(ref, kept, kc, quad)
            got = product.finish_chains(kept, kc, quad)
            assert np.array_equal(got, want), (dist, cc)
    rng = np.random.default_rng(99)
    for trial in range(2000):
        quad = rng.integers(0, 4, (4, 2)).astype(np.float64)
        kc = [int(x) for x in rng.integers(0, 4, 4)]
        chains = rng.integers(0, 4, (sum(kc), 2)).astype(np.float64)
        if rng.random() < 0.3 and sum(kc):  # close onto corner 0
            chains[-1] = quad[0]
        want = _finish_reference(ref, chains, kc, quad)
        if want is None:
            with pytest.raises(product.DegenerateInput):
                product.finish_chains(chains, kc, quad)
        else:
            assert np.array_equal(product.finish_chains(chains, kc, quad), want), trial
    # long chains (the finisher tests blocks of 8 points at once): runs of
    # duplicates, collinear grids and points inside the hull so far
    for trial in range(1500):
        span = (3, 7, 50)[trial % 3]
        quad = rng.integers(0, span, (4, 2)).astype(np.float64)
        kc = [int(x) for x in rng.integers(0, 40, 4)]
        chains = rng.integers(0, span, (sum(kc), 2)).astype(np.float64)
        if sum(kc) > 2 and rng.random() < 0.5:  # runs of repeats
            rep = rng.integers(0, sum(kc), sum(kc) // 3)
            chains[rep] = chains[np.maximum(rep - 1, 0)]
        want = _finish_reference(ref, chains, kc, quad)
        if want is None:
            with pytest.raises(product.DegenerateInput):
                product.finish_chains(chains, kc, quad)
        else:
            assert np.array_equal(product.finish_chains(chains, kc, quad), want), ("long", trial)


def test_split_finisher(product):
    """finish_chains_split (the four chains concurrently, verified) is bit-identical
    to the reference's assemble_polygon + melkman, takes the split path on
    pipeline chains, and survives fork (tests/split_finisher_check.py runs
    in its own process with the split threshold lowered to 8)."""
    import subprocess
    from pyoracle import RefLib
    if not RefLib.available():
        pytest.skip("oracle/_ref not built")
    env = dict(os.environ, CHGPU_FINISH_SPLIT_MIN="8")
    out = subprocess.run([sys.executable, os.path.join(os.path.dirname(__file__), "split_finisher_check.py")],
                         env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    taken = int(out.stdout.split("taken=")[1].split()[0])
    assert taken > 0, out.stdout


def test_host_prefault_pool_and_fork(product):
    """chgpu_host_prefault (the C++ API's result-vector prefault) runs on the
    library's staging threads: every page of the range is touched, a range
    far larger than the pool is split among its threads, and a forked child
    (which has none of the parent's threads) starts its own pool."""
    L = product.load_library()
    L.chgpu_host_prefault.argtypes = [C.c_void_p, C.c_size_t]
    L.chgpu_host_prefault.restype = None
    a = np.full(64 << 20, 7, np.uint8)  # 64 MB: 16 parts of 4 MB
    L.chgpu_host_prefault(a.ctypes.data, a.nbytes)
    assert a[::4096].max() == 0 and a[-1] == 0  # (the touched bytes are zeroed)
    pid = os.fork()
    if pid == 0:  # child: the pool must start fresh, not inherit dead threads
        try:
            b = np.full(32 << 20, 7, np.uint8)
            L.chgpu_host_prefault(b.ctypes.data, b.nbytes)
            os._exit(0 if b[::4096].max() == 0 else 3)
        except BaseException:
            os._exit(4)
    _, status = os.waitpid(pid, 0)
    assert os.WIFEXITED(status) and os.WEXITSTATUS(status) == 0, status
