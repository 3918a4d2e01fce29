"""Where the sharded path's time goes at one rank (host clock per phase)."""
import os, sys, time
import numpy as np, torch, torch.distributed as dist
sys.path.insert(0, ".")
import paper_1508_05488_b200 as P
from paper_1508_05488_b200 import sharded as S
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29534", RANK="0", WORLD_SIZE="1")
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
n = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000_000
ctx = P.Context(0)
h = torch.empty((n, 2), dtype=torch.float64, pin_memory=True)
P.generate("uniform_square", n, 42, out=h.numpy())
d = h.cuda(); ctx.reserve(n); torch.cuda.synchronize()
ops = S.GpuShardOps(ctx, d, 0)
T = {}
class Timed(S.GpuShardOps):
    def extremes(self):
        t0 = time.perf_counter(); r = super().extremes(); T["extremes"] = T.get("extremes", 0) + time.perf_counter() - t0; return r
    def chains(self, q, c):
        t0 = time.perf_counter(); r = super().chains(q, c); T["chains"] = T.get("chains", 0) + time.perf_counter() - t0; return r
    def merge(self, runs, q):
        t0 = time.perf_counter(); r = super().merge(runs, q); T["merge"] = T.get("merge", 0) + time.perf_counter() - t0; return r
ops = Timed(ctx, d, 0)
for _ in range(3): S.sharded_convex_hull(ops, 1024)
T.clear(); K = 10
t0 = time.perf_counter()
for _ in range(K): S.sharded_convex_hull(ops, 1024)
tot = time.perf_counter() - t0
print({k: round(v / K * 1e3, 3) for k, v in T.items()}, "total", round(tot / K * 1e3, 3), "glue", round((tot - sum(T.values())) / K * 1e3, 3))
dist.destroy_process_group()
