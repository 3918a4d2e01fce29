"""e2e (pinned host input through chgpu_hull) for env settings."""
import os, subprocess, sys
code = r'''
import sys, numpy as np, torch, time
sys.path.insert(0, ".")
import paper_1508_05488_b200 as P
n = 20_000_000
ctx = P.Context(0)
h = torch.empty((n, 2), dtype=torch.float64, pin_memory=True)
P.generate("uniform_square", n, 42, out=h.numpy())
ctx.reserve(n)
cfg = P.PipelineConfig()
a = h.numpy()
for _ in range(3): ctx.convex_hull(a, cfg, copy=False)
s = torch.cuda.ExternalStream(ctx.stream)
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(s)
for _ in range(10): r = ctx.convex_hull(a, cfg, copy=False)
e1.record(s); e1.synchronize()
print(f"e2e {e0.elapsed_time(e1)/10:.3f} ms total {r.stats.t_total_ms:.3f} host {r.diag.times_ms['t_host_ms']*1e3:.0f}us enq {r.diag.times_ms['t_host_enqueue_ms']:.3f} wait {r.diag.times_ms['t_host_wait_ms']:.3f}")
'''
for cfg in sys.argv[1:]:
    env = dict(os.environ)
    for kv in cfg.split():
        if "=" in kv:
            k, v = kv.split("="); env[k] = v
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print(cfg, out.stdout.strip() or out.stderr[-400:])
