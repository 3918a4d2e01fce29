"""Device-resident 20M step (C-side t_total, host wall, finisher) for env
settings, interleaved: python tools/gpu/step_ab.py "A=1" "A=0" [rounds]."""
import os, subprocess, sys
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
for _ in range(10): ctx.convex_hull_device(d.data_ptr(), n, cfg, copy=False)
tot, host, wall = [], [], []
for _ in range(60):
    t0 = time.perf_counter(); r = ctx.convex_hull_device(d.data_ptr(), n, cfg, copy=False)
    wall.append(time.perf_counter() - t0); tot.append(r.stats.t_total_ms); host.append(r.diag.times_ms["t_host_ms"])
print(f"wall {np.median(wall)*1e3:.3f} ms  t_total {np.median(tot):.3f} ms  finisher {np.median(host)*1e3:.1f} us")
'''
cfgs = [a for a in sys.argv[1:] if "=" in a]
rounds = int(next((a for a in sys.argv[1:] if a.isdigit()), "2"))
for _ in range(rounds):
    for cfg in cfgs:
        env = dict(os.environ)
        for kv in cfg.split():
            k, v = kv.split("=", 1); env[k] = v
        out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
        print(f"{cfg:28s}", out.stdout.strip() or out.stderr[-300:])
