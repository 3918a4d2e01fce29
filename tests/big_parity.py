"""Parity at shard and full scale: our hull of N uniform points (1 GPU)
against the reference's own convex_hull (oracle/_ref, all host threads) on
the same input. usage: python tests/big_parity.py N [dist] [seed]"""
import json, os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import paper_1508_05488_b200 as P
from pyoracle import RefLib

n = int(float(sys.argv[1])); dist = sys.argv[2] if len(sys.argv) > 2 else "uniform_square"
seed = int(sys.argv[3]) if len(sys.argv) > 3 else 42
pts = P.generate(dist, n, seed)
ctx = P.Context(0)
t = time.perf_counter(); r = ctx.convex_hull(pts); t_ours = time.perf_counter() - t
ref = RefLib()
t = time.perf_counter(); w, _ = ref.convex_hull(pts, 1024, parallelism=0); t_ref = time.perf_counter() - t
ours = [r.stats.n_input, r.stats.n_after_round1, r.stats.n_after_spa, r.stats.n_hull]
out = {"n": n, "dist": dist, "seed": seed, "counts_ours": ours, "counts_ref": w.counts.tolist(),
       "hull_equal": bool(np.array_equal(r.hull.vertices, w.hull)),
       "s_ours_first_call": round(t_ours, 3), "s_ref_all_threads": round(t_ref, 3),
       "host_threads": os.cpu_count()}
print(json.dumps(out))
sys.exit(0 if out["hull_equal"] and ours == w.counts.tolist() else 1)
