"""TEST INFRASTRUCTURE — generates tests/golden/chains.json and
tests/golden/big_1b.json from the UNMODIFIED reference
(oracle/_ref/libchainhull_ref.so, built by `make -C oracle` from
/root/reference/proj/core/src). Run here, where /root/reference exists:

    python oracle/make_golden_chains.py [--no-1b]

chains.json: the reference's kept SPA chains (spa_filter output per region,
reference spa.cpp:109-163, via the stage dump of pipeline.cpp:36-96) for the
four 20M BASELINE configs at chunk counts {1, 7, 1024}, pinned by count and
sha256 of the float64 bytes, so the GPU's default (pre-filtered) path is
checked element by element, not only through the hull.

big_1b.json: BASELINE configs[4] (1B uniform_square, seed 42): counts and
hull of the reference's convex_hull on the whole set (all host threads), the
parity target of the sharded multi-GPU run.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from pyoracle import RefLib  # noqa: E402

OUT = os.path.join(os.path.dirname(HERE), "tests", "golden")


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()


def hexpts(a: np.ndarray):
    return [[float(x).hex(), float(y).hex()] for x, y in a]


def chain_cases(ref: RefLib):
    specs = [("uniform_square", 20_000_000, 42), ("uniform_disk", 20_000_000, 42),
             ("gaussian", 20_000_000, 42), ("circle", 20_000_000, 42),
             ("uniform_square", 1_000_000, 42)]
    out = []
    for d, n, seed in specs:
        pts = ref.generate(d, n, seed)
        for cc in (1, 7, 1024):
            t = time.time()
            q, rc, _srt, kept, kc = ref.stage_dump(pts, cc)
            ko = 0
            regions = []
            for r in range(4):
                k = int(kc[r])
                seg = kept[ko:ko + k]
                regions.append({"k": k, "sha": sha(seg),
                                "head": hexpts(seg[:4]), "tail": hexpts(seg[-4:])})
                ko += k
            out.append({"dist": d, "n": n, "seed": seed, "chunk_count": cc,
                        "input_sha": sha(pts), "region_counts": [int(c) for c in rc],
                        "kept": regions})
            print(d, n, seed, cc, [r["k"] for r in regions], f"{time.time() - t:.1f}s", flush=True)
    return out


def big_1b(ref: RefLib):
    n, seed = 1_000_000_000, 42
    t = time.time()
    pts = ref.generate("uniform_square", n, seed)
    tg = time.time() - t
    t = time.time()
    h, ms = ref.convex_hull(pts, 1024, 0)
    th = time.time() - t
    assert h.status == 0
    # prefixes of the 1B set (uniform_square draws two values per point in
    # index order, so the first m points of the 1B set are generate(m))
    return {"dist": "uniform_square", "n": n, "seed": seed, "chunk_count": 1024,
            "status": h.status, "counts": [int(c) for c in h.counts],
            "hull_sha": sha(h.hull), "hull_n": len(h.hull), "hull": hexpts(h.hull),
            "ref_s_generate": round(tg, 2), "ref_s_convex_hull_all_threads": round(th, 2),
            "host_threads": os.cpu_count()}


def main():
    ref = RefLib()
    with open(os.path.join(OUT, "chains.json"), "w") as f:
        json.dump(chain_cases(ref), f, indent=1)
    if "--no-1b" not in sys.argv:
        b = big_1b(ref)
        print(b["counts"], b["hull_sha"], flush=True)
        with open(os.path.join(OUT, "big_1b.json"), "w") as f:
            json.dump(b, f, indent=1)


if __name__ == "__main__":
    main()
