"""Hammer circle n=100000 (acceptance c1 case) through the Python API and
report any mismatch with the reference."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import paper_1508_05488_b200 as P
from pyoracle import RefLib
ref = RefLib()
ctx = P.Context(0)
bad = 0
cases = [("circle", 100000, s) for s in (101, 202, 303)] + [("uniform_square", 100000, 101), ("uniform_disk", 100000, 202)]
wants = {}
for d, n, seed in cases:
    pts = ref.generate(d, n, seed)
    ho, _ = ref.convex_hull(pts, 1024, 1)
    hull, counts = ho.hull, ho.counts
    wants[(d, n, seed)] = (pts, hull, counts)
for rep in range(40):
    for key, (pts, hull, counts) in wants.items():
        r = ctx.convex_hull(pts, P.PipelineConfig(chunk_count=1024))
        if not np.array_equal(r.hull.vertices, hull):
            bad += 1
            a = r.hull.vertices
            print("MISMATCH", key, rep, len(a), len(hull), "fast", r.diag.convex_fast_path, "path", r.diag.spa_path,
                  [r.stats.n_after_round1, r.stats.n_after_spa, r.stats.n_hull], list(counts), flush=True)
print("bad", bad)
