"""Split-finisher segment times and the CPU each process thread last ran on
(per-process variance diagnostic), 20M uniform device-resident."""
import ctypes as C, os, sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_1508_05488_b200 as P
n = 20_000_000
ctx = P.Context(0)
h = torch.empty((n, 2), dtype=torch.float64, pin_memory=True)
P.generate("uniform_square", n, 42, out=h.numpy())
d = h.cuda(); ctx.reserve(n); torch.cuda.synchronize()
L = P.load_library(); L.chgpu_finish_split_times.argtypes = [C.POINTER(C.c_double)]
cfg = P.PipelineConfig()
rows = []
for i in range(40):
    r = ctx.convex_hull_device(d.data_ptr(), n, cfg, copy=False)
    t = (C.c_double * 6)(); L.chgpu_finish_split_times(t)
    if i >= 5: rows.append(list(t))
a = np.median(np.array(rows), axis=0)
cpus = []
for tid in sorted(os.listdir("/proc/self/task"), key=int):
    f = open(f"/proc/self/task/{tid}/stat").read().rsplit(")", 1)[1].split()
    cpus.append((int(tid), int(f[36]), int(f[11]) + int(f[12])))  # processor, utime+stime
busy = [c for c in cpus if c[2] > 50]
print("A %.1f B %.1f C %.1f D %.1f joined %.1f | me cpu %d | busy threads (tid, cpu, ticks): %s" % (
    a[0], a[1], a[2], a[3], a[4], os.sched_getaffinity(0) and C.CDLL(None).sched_getcpu(), busy))
