"""Step and stage times for env knob settings (one process each):
python tools/gpu/knob_ab.py "VAR=a VAR2=b" "VAR=c" ..."""
import os, subprocess, sys
code = r'''
import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_1508_05488_b200 as P
n = int(__import__("os").environ.get("KN", "20000000"))
dist = __import__("os").environ.get("KDIST", "uniform_square")
ctx = P.Context(0)
h = torch.empty((n, 2), dtype=torch.float64, pin_memory=True)
P.generate(dist, n, 42, out=h.numpy())
d = h.cuda(); ctx.reserve(n); torch.cuda.synchronize()
cfg = P.PipelineConfig()
for _ in range(5): ctx.convex_hull_device(d.data_ptr(), n, cfg, copy=False)
s = torch.cuda.ExternalStream(ctx.stream)
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(s)
for _ in range(40): r = ctx.convex_hull_device(d.data_ptr(), n, cfg, copy=False)
e1.record(s); e1.synchronize()
step = e0.elapsed_time(e1) / 40 * 1e3
ctx.set_stage_times(True)
ts = []
for _ in range(15):
    r = ctx.convex_hull_device(d.data_ptr(), n, cfg, copy=False); ts.append(dict(r.diag.times_ms))
med = {k: float(np.median([t[k] for t in ts])) * 1e3 for k in ts[0]}
keys = ["t_k1_ms", "t_binscan_ms", "t_filter_ms", "t_spa_kernel_ms", "t_d2h_ms", "t_host_ms"]
print(f"step {step:.1f} us | " + " ".join(f"{k[2:-3]}={med[k]:.1f}" for k in keys) + f" | cand {r.diag.n_candidates} spa {r.stats.n_after_spa} hull {r.stats.n_hull}")
'''
for cfg in sys.argv[1:]:
    env = dict(os.environ)
    for kv in cfg.split():
        if "=" in kv:
            k, v = kv.split("=", 1); env[k] = v
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print(f"{cfg:40s}", out.stdout.strip() or out.stderr[-400:])
