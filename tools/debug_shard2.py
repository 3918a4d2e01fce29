"""Debug: the sharded test's call sequence on one context per 'rank' in
one process; reports the first mismatching stage."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle")); sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch
import paper_1508_05488_b200 as P
from paper_1508_05488_b200.sharded import GpuShardOps, fold_extremes, frame_vertices
from pyoracle import Oracle
from test_sharded import OracleShardOps, DATASETS
o = Oracle()
world = 2
ctxs = [P.Context(0), P.Context(0)]
for (dist_name, n, seed) in DATASETS:
    pts = o.generate(dist_name, n, seed)
    bounds = np.linspace(0, n, world + 1).astype(int)
    for cc in (1, 1024):
        qs, ids = [], []
        gops = []
        for r in range(world):
            sh = pts[bounds[r]:bounds[r + 1]]
            g = GpuShardOps(ctxs[r], torch.from_numpy(np.ascontiguousarray(sh)).cuda(), int(bounds[r]))
            gops.append((g, OracleShardOps(o, sh, int(bounds[r]))))
            a = g.extremes(); qs.append(a[0]); ids.append(a[1])
        quad = fold_extremes(np.stack(qs), np.stack(ids))
        parts = []
        for r, (g, c) in enumerate(gops):
            a, b = g.chains(quad, cc), c.chains(quad, cc)
            if not np.array_equal(a, b):
                print("MISMATCH chains", dist_name, n, cc, "rank", r, len(a), len(b))
            parts.append(a)
        fr = frame_vertices(quad)
        U = np.vstack(parts + [fr])
        hg = ctxs[0].convex_hull(U, P.PipelineConfig(chunk_count=cc))
        ho = o.convex_hull(U, cc)
        ok = np.array_equal(hg.hull.vertices, ho.hull)
        want = o.convex_hull(pts, 1024)
        print(dist_name, n, cc, "finish ok", ok, "path", hg.diag.spa_path, "global ok", np.array_equal(hg.hull.vertices, want.hull),
              [hg.stats.n_after_round1, hg.stats.n_after_spa, hg.stats.n_hull], ho.counts.tolist()[1:])
