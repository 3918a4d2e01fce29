"""Debug: the sharded flow for one dataset in one process (no
torch.distributed), every stage compared with the oracle stand-in."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle")); sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch
import paper_1508_05488_b200 as P
from paper_1508_05488_b200.sharded import GpuShardOps, fold_extremes, frame_vertices
from pyoracle import Oracle
from test_sharded import OracleShardOps

o = Oracle()
dist_name, n, seed, cc, world = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), 2
pts = o.generate(dist_name, n, seed)
bounds = np.linspace(0, n, world + 1).astype(int)
ctx = P.Context(0)
qs, ids, qo, io = [], [], [], []
for r in range(world):
    sh = pts[bounds[r]:bounds[r + 1]]
    g = GpuShardOps(ctx, torch.from_numpy(np.ascontiguousarray(sh)).cuda(), int(bounds[r]))
    c = OracleShardOps(o, sh, int(bounds[r]))
    a, b = g.extremes(), c.extremes()
    print("rank", r, "extremes equal", np.array_equal(a[0], b[0]), np.array_equal(a[1], b[1]))
    qs.append(a[0]); ids.append(a[1])
quad = fold_extremes(np.stack(qs), np.stack(ids))
print("quad", quad.tolist(), "oracle", o.find_extremes(pts).tolist())
parts_g, parts_o = [], []
for r in range(world):
    sh = pts[bounds[r]:bounds[r + 1]]
    g = GpuShardOps(ctx, torch.from_numpy(np.ascontiguousarray(sh)).cuda(), int(bounds[r]))
    c = OracleShardOps(o, sh, int(bounds[r]))
    a, b = g.chains(quad, cc), c.chains(quad, cc)
    print("rank", r, "chains", len(a), len(b), "equal", np.array_equal(a, b))
    parts_g.append(a); parts_o.append(b)
fr = frame_vertices(quad)
U = np.vstack(parts_o + [fr])
hg = ctx.convex_hull(U, P.PipelineConfig(chunk_count=cc))
ho = o.convex_hull(U, cc)
print("finish n", len(U), "counts gpu", [hg.stats.n_input, hg.stats.n_after_round1, hg.stats.n_after_spa, hg.stats.n_hull],
      "oracle", ho.counts.tolist(), "hull equal", np.array_equal(hg.hull.vertices, ho.hull), "spa_path", hg.diag.spa_path)
want = o.convex_hull(pts, 1024)
print("final equal to global", np.array_equal(ho.hull, want.hull))
