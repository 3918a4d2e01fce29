"""Cost of the sharded path's collectives at one rank (host clock)."""
import os, sys, time
import torch, torch.distributed as dist
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29535", RANK="0", WORLD_SIZE="1")
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
g = dist.new_group(backend="gloo")
def t(f, k=50):
    for _ in range(5): f()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(k): f()
    torch.cuda.synchronize(); return round((time.perf_counter() - t0) / k * 1e6, 1)
h = torch.zeros(12, dtype=torch.float64)
print("gloo all_gather 12 doubles us", t(lambda: dist.all_gather([torch.empty_like(h)], h, group=g)))
d = torch.zeros((48840, 2), dtype=torch.float64, device="cuda")
print("nccl all_gather 780KB us", t(lambda: dist.all_gather([torch.empty_like(d)], d)))
print("nccl all_gather_into_tensor us", t(lambda: dist.all_gather_into_tensor(torch.empty((48840, 2), dtype=torch.float64, device="cuda"), d)))
print("d.cpu() us", t(lambda: d.cpu()))
dist.destroy_process_group()
