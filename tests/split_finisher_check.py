"""Split finisher (finisher.cpp finish_chains_split) against the reference's
assemble_polygon + melkman: pipeline chains of several distributions and
adversarial rings (duplicate runs, collinear grids, tiny spans). Run in its
own process with CHGPU_FINISH_SPLIT_MIN=8 so small chains take the split
path too (tests/test_abi.py::test_split_finisher). Prints taken/fallback."""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import paper_1508_05488_b200 as P  # noqa: E402
from pyoracle import RefLib  # noqa: E402


def ring_of(quad, kept, kc):
    parts, off = [], 0
    for r in range(4):
        parts.append(quad[r:r + 1])
        parts.append(kept[off:off + kc[r]])
        off += kc[r]
    return np.concatenate(parts)


def reference(ref, quad, kept, kc):
    ring = []
    for p in ring_of(quad, kept, kc):
        p = (float(p[0]), float(p[1]))
        if not ring or ring[-1] != p:
            ring.append(p)
    if len(ring) > 1 and ring[0] == ring[-1]:
        ring.pop()
    if len(ring) < 3:
        return None
    try:
        st, hull = ref.melkman(np.array(ring))
    except Exception:
        return None
    return None if st else hull


def main():
    ref = RefLib()
    L = P.load_library()
    bad = 0
    for dist, n, seed in (("uniform_square", 400_000, 42), ("uniform_disk", 300_000, 7),
                          ("gaussian", 500_000, 5), ("circle", 20_000, 9)):
        pts = ref.generate(dist, n, seed)
        for cc in (64, 1024, 4096):
            quad, rc, srt, kept, kc = ref.stage_dump(pts, cc)
            want = reference(ref, quad, kept, kc)
            got = P.finish_chains(kept, kc, quad)
            bad += not np.array_equal(got, want)
    # lattice inputs: collinear runs and exact ties everywhere near the hull
    rng = np.random.default_rng(5)
    for grid, n in ((16, 200_000), (64, 300_000), (1024, 300_000), (1 << 20, 300_000)):
        pts = np.round(rng.random((n, 2)) * grid) / grid
        for cc in (64, 1024):
            quad, rc, srt, kept, kc = ref.stage_dump(pts, cc)
            if min(kc) == 0:
                continue
            want = reference(ref, quad, kept, kc)
            try:
                got = P.finish_chains(kept, kc, quad)
            except P.DegenerateInput:
                got = None
            bad += not ((want is None and got is None) or
                        (want is not None and got is not None and np.array_equal(got, want)))
    for trial in range(3000):
        span = (3, 5, 9, 60)[trial % 4]
        quad = rng.integers(0, span, (4, 2)).astype(np.float64)
        kc = [int(x) for x in rng.integers(8, 48, 4)]
        chains = rng.integers(0, span, (sum(kc), 2)).astype(np.float64)
        if rng.random() < 0.5:
            rep = rng.integers(1, sum(kc), sum(kc) // 3)
            chains[rep] = chains[rep - 1]
        if rng.random() < 0.2:
            chains[-1] = quad[0]
        want = reference(ref, quad, chains, kc)
        try:
            got = P.finish_chains(chains, kc, quad)
        except P.DegenerateInput:
            got = None
        if want is None or got is None:
            bad += (want is None) != (got is None)
        else:
            bad += not np.array_equal(got, want)
    # a forked child (the workers' threads do not survive fork) still finishes
    pts = ref.generate("uniform_square", 200_000, 11)
    quad, rc, srt, kept, kc = ref.stage_dump(pts, 1024)
    want = reference(ref, quad, kept, kc)
    pid = os.fork()
    if pid == 0:
        os._exit(0 if np.array_equal(P.finish_chains(kept, kc, quad), want) else 3)
    _, status = os.waitpid(pid, 0)
    bad += os.waitstatus_to_exitcode(status) != 0
    a, b = C.c_ulonglong(), C.c_ulonglong()
    L.chgpu_finish_split_stats(C.byref(a), C.byref(b))
    print(f"mismatches={bad} taken={a.value} fallback={b.value}")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
