"""K1+K2 in-step (programmatic) for the library variants given (CHGPU_LIB)."""
import os, subprocess, sys
code = r'''
import sys, numpy as np, torch
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
k12 = []
e0.record(s)
for _ in range(40):
    r = ctx.convex_hull_device(d.data_ptr(), n, cfg, copy=False)
    t = r.diag.times_ms; k12.append(t["t_k1_ms"] + t["t_k2_ms"])
e1.record(s); e1.synchronize()
print(f"step {e0.elapsed_time(e1)/40*1e3:.1f} us k1k2 {np.median(k12)*1e3:.1f} us hull {r.stats.n_hull} spa {r.stats.n_after_spa}")
'''
for v in sys.argv[1:]:
    env = dict(os.environ)
    if v != "default":
        env["CHGPU_LIB"] = f"build/variants/libchgpu_{v}.so"
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print(f"{v:10s}", out.stdout.strip() or out.stderr[-400:])
