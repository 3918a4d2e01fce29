"""Phase timing of the sharded (N > 1) code path at one rank, 1B uniform."""
import os, sys, time
import numpy as np, torch, torch.distributed as dist
sys.path.insert(0, ".")
import paper_1508_05488_b200 as P
from paper_1508_05488_b200 import sharded as S
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29533")
os.environ.setdefault("RANK", "0"); os.environ.setdefault("WORLD_SIZE", "1")
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000_000
ctx = P.Context(0)
h = torch.empty((n, 2), dtype=torch.float64, pin_memory=True)
P.generate("uniform_square", n, 42, out=h.numpy())
d = h.cuda(); ctx.reserve(n); torch.cuda.synchronize()
ops = S.GpuShardOps(ctx, d, 0)
cfg = P.PipelineConfig()
def timed(f, k=5):
    for _ in range(2): f()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(k): out = f()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / k * 1e3, out
print("single  ms", timed(lambda: ctx.convex_hull_device(d.data_ptr(), n, cfg, copy=False))[0])
print("sharded ms", timed(lambda: S.sharded_convex_hull(ops, 1024))[0])
print("extremes ms", timed(lambda: ops.extremes())[0])
q, idx = ops.extremes()
quad = S.fold_extremes(q.reshape(1, 8), idx.reshape(1, 4))
print("chains ms", timed(lambda: ops.chains(quad, 1024))[0])
ch, kc = ops.chains(quad, 1024)
runs = [(ch.cpu().numpy(), kc)]
print("chain pts", ch.shape[0], "merge ms", timed(lambda: ops.merge(runs, quad))[0])
dist.destroy_process_group()
