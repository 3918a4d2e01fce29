"""TEST INFRASTRUCTURE — generates tests/golden/*.json from the UNMODIFIED
reference (oracle/_ref/libchainhull_ref.so, built by `make -C oracle` from
/root/reference/proj/core/src). Run here, where /root/reference exists:

    python oracle/make_golden.py

The fixtures travel with the repo; nothing at test time needs
/root/reference. Every array is pinned by the sha256 of its float64 bytes
(little-endian, row-major (k, 2)), and small arrays are stored in full as
float.hex() pairs so failures are readable.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from pyoracle import DISTRIBUTIONS, RefLib  # noqa: E402

OUT = os.path.join(os.path.dirname(HERE), "tests", "golden")


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()


def hexpts(a: np.ndarray, limit: int = 64):
    if len(a) > limit:
        return None
    return [[float(x).hex(), float(y).hex()] for x, y in a]


def pipeline_sweep(ref: RefLib):
    """acceptance.cpp:57-94 (criterion 1) sweep + the pipeline_test.cpp cases."""
    sizes = [1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 100, 1000, 100000]
    seeds = [101, 202, 303]
    cases = []
    for d in DISTRIBUTIONS:
        for n in sizes:
            for seed in seeds:
                pts = ref.generate(d, n, seed)
                entry = {"dist": d, "n": n, "seed": seed, "input_sha": sha(pts), "runs": []}
                for cc in (1, 4, 1024):
                    h, _ = ref.convex_hull(pts, cc, 1)
                    entry["runs"].append({
                        "chunk_count": cc, "status": h.status,
                        "counts": [int(c) for c in h.counts],
                        "hull_sha": sha(h.hull), "hull_n": len(h.hull),
                        "hull": hexpts(h.hull)})
                cases.append(entry)
    return cases


def stage_cases(ref: RefLib):
    """Per-stage dumps (pipeline.cpp:36-96) for region-level parity."""
    out = []
    specs = [("uniform_square", 2000, 53), ("uniform_disk", 3000, 59), ("gaussian", 5000, 43),
             ("circle", 500, 5), ("uniform_square", 60000, 61), ("duplicates_heavy", 100, 101),
             ("duplicates_heavy", 1500, 67), ("uniform_disk", 100000, 7)]
    for d, n, seed in specs:
        pts = ref.generate(d, n, seed)
        quad = ref.find_extremes(pts)
        for cc in (1, 2, 4, 7, 16, 32, 64, 1024):
            try:
                q, rc, srt, kept, kc = ref.stage_dump(pts, cc)
            except ValueError:
                continue
            segs, kseg = [], []
            o = ko = 0
            for r in range(4):
                m = int(rc[r + 1])
                segs.append({"m": m, "sha": sha(srt[o:o + m]), "pts": hexpts(srt[o:o + m], 32)})
                kseg.append({"k": int(kc[r]), "sha": sha(kept[ko:ko + int(kc[r])]),
                             "pts": hexpts(kept[ko:ko + int(kc[r])], 32)})
                o += m
                ko += int(kc[r])
            out.append({"dist": d, "n": n, "seed": seed, "chunk_count": cc,
                        "input_sha": sha(pts), "quad": hexpts(quad),
                        "region_counts": [int(c) for c in rc], "segments": segs, "kept": kseg})
    return out


def big_cases(ref: RefLib):
    """BASELINE.json configs 1-4 at full size, seed 42 (and uniform seeds 1-3)."""
    specs = [("uniform_square", 1_000_000, 42), ("uniform_square", 20_000_000, 42),
             ("uniform_disk", 20_000_000, 42), ("gaussian", 20_000_000, 42),
             ("circle", 20_000_000, 42), ("uniform_square", 20_000_000, 1),
             ("uniform_square", 20_000_000, 2), ("duplicates_heavy", 20_000_000, 42),
             ("collinear", 4_000_000, 42), ("uniform_square", 4_000_000, 42)]
    out = []
    for d, n, seed in specs:
        pts = ref.generate(d, n, seed)
        quad = ref.find_extremes(pts)
        h, ms = ref.convex_hull(pts, 1024, 1)
        out.append({"dist": d, "n": n, "seed": seed, "input_sha": sha(pts), "quad": hexpts(quad),
                    "chunk_count": 1024, "status": h.status,
                    "counts": [int(c) for c in h.counts], "hull_sha": sha(h.hull),
                    "hull_n": len(h.hull), "hull": hexpts(h.hull, 64),
                    "ref_ms_1thread": [float(m) for m in ms]})
        print(d, n, seed, h.counts, f"{ms[6]:.1f} ms", flush=True)
    return out


def main():
    os.makedirs(OUT, exist_ok=True)
    ref = RefLib()
    with open(os.path.join(OUT, "pipeline_sweep.json"), "w") as f:
        json.dump(pipeline_sweep(ref), f, separators=(",", ":"))
    with open(os.path.join(OUT, "stages.json"), "w") as f:
        json.dump(stage_cases(ref), f, separators=(",", ":"))
    if "--no-big" not in sys.argv:
        with open(os.path.join(OUT, "big.json"), "w") as f:
            json.dump(big_cases(ref), f, indent=1)


if __name__ == "__main__":
    main()
