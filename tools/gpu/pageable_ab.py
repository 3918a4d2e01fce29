"""e2e from pageable host memory (the staged path) for env settings."""
import os, subprocess, sys
code = r'''
import sys, time, numpy as np
sys.path.insert(0, ".")
import paper_1508_05488_b200 as P
n = 20_000_000
ctx = P.Context(0)
a = P.generate("uniform_square", n, 42)   # pageable numpy
ctx.reserve(n)
cfg = P.PipelineConfig()
for _ in range(3): ctx.convex_hull(a, cfg, copy=False)
ts = []
for _ in range(8):
    t0 = time.perf_counter(); r = ctx.convex_hull(a, cfg, copy=False); ts.append(time.perf_counter() - t0)
print(f"pageable e2e {np.median(ts)*1e3:.2f} ms (min {min(ts)*1e3:.2f})")
'''
for cfg in sys.argv[1:]:
    env = dict(os.environ)
    for kv in cfg.split():
        if "=" in kv:
            k, v = kv.split("=", 1); env[k] = v
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print(f"{cfg:28s}", out.stdout.strip() or out.stderr[-400:])
