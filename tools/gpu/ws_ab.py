"""Whole-step timing for bin-max sampling settings (env knob read at load)."""
import json, os, subprocess, sys
code = r'''
import sys, time, numpy as np, torch
sys.path.insert(0, ".")
import paper_1508_05488_b200 as P
n = 20_000_000
ctx = P.Context(0)
h = torch.empty((n, 2), dtype=torch.float64, pin_memory=True)
P.generate("uniform_square", n, 42, out=h.numpy())
d = h.cuda(); ctx.reserve(n); torch.cuda.synchronize()
cfg = P.PipelineConfig()
for _ in range(5): ctx.convex_hull_device(d.data_ptr(), n, cfg, copy=False)
s = torch.cuda.ExternalStream(ctx.stream)
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
k12 = []; f = []; sp = []
e0.record(s)
for _ in range(40):
    r = ctx.convex_hull_device(d.data_ptr(), n, cfg, copy=False)
    t = r.diag.times_ms; k12.append(t["t_k1_ms"] + t["t_k2_ms"]); f.append(t["t_filter_ms"]); sp.append(t["t_spa_kernel_ms"])
e1.record(s); e1.synchronize()
print(f"step {e0.elapsed_time(e1)/40*1e3:.1f} us k1k2 {np.median(k12)*1e3:.1f} filter {np.median(f)*1e3:.1f} spa {np.median(sp)*1e3:.1f} cand {r.diag.n_candidates}")
'''
for ws in sys.argv[1:]:
    env = dict(os.environ, CHGPU_FILTER_WSAMPLE_LOG2=ws)
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print("ws", ws, out.stdout.strip() or out.stderr[-400:])
