"""Median C-side wall time and per-stage times for env knob settings
(one process per setting), 20M uniform device-resident."""
import json, os, subprocess, sys
code = r'''
import os, sys, time, json
import numpy as np
sys.path.insert(0, os.getcwd())
import torch
import paper_1508_05488_b200 as P
ctx = P.Context(0)
pts = P.generate(os.environ.get("DIST", "uniform_square"), 20_000_000, 42)
d = torch.from_numpy(pts).cuda(); torch.cuda.synchronize()
cfg = P.PipelineConfig()
for _ in range(5): ctx.convex_hull_device(d.data_ptr(), len(pts), cfg, copy=False)
tw, ts = [], {}
for _ in range(15):
    r = ctx.convex_hull_device(d.data_ptr(), len(pts), cfg, copy=False)
    tw.append(r.stats.t_total_ms)
    for k, v in r.diag.times_ms.items(): ts.setdefault(k, []).append(v)
print(json.dumps({"wall": float(np.median(tw)), "cand": r.diag.n_candidates,
                  **{k: round(float(np.median(v)), 4) for k, v in ts.items() if np.median(v) > 0}}))
'''
for cfg in sys.argv[1:]:
    env = dict(os.environ)
    for kv in cfg.split():
        k, v = kv.split("=")
        env[k] = v
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print(cfg, out.stdout.strip() or out.stderr[-500:])
