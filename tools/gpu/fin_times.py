"""Per-segment times of the split finisher on the headline input."""
import ctypes as C, sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_1508_05488_b200 as P
dist = sys.argv[1] if len(sys.argv) > 1 else "uniform_square"
n = 20_000_000
ctx = P.Context(0)
h = torch.empty((n, 2), dtype=torch.float64, pin_memory=True)
P.generate(dist, n, 42, out=h.numpy())
d = h.cuda(); ctx.reserve(n); torch.cuda.synchronize()
L = P.load_library(); L.chgpu_finish_split_times.argtypes = [C.POINTER(C.c_double)]
cfg = P.PipelineConfig()
rows = []
for i in range(40):
    r = ctx.convex_hull_device(d.data_ptr(), n, cfg, copy=False)
    t = (C.c_double * 6)(); L.chgpu_finish_split_times(t)
    if i >= 5: rows.append(list(t) + [r.diag.times_ms["t_host_ms"] * 1e3])
a = np.median(np.array(rows), axis=0)
print(dist, "kept", r.diag.kept_counts, "| A %.1f B %.1f C %.1f D %.1f joined %.1f done %.1f | host %.1f us" % tuple(a))
