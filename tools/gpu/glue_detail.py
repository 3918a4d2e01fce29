"""Host-clock timestamps inside sharded_convex_hull at one rank (a traced
copy of its body), 1B uniform by default."""
import os, sys, time
import numpy as np, torch, torch.distributed as dist
sys.path.insert(0, ".")
import paper_1508_05488_b200 as P
from paper_1508_05488_b200 import sharded as S
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29536", RANK="0", WORLD_SIZE="1")
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000_000
ctx = P.Context(0)
h = torch.empty((n, 2), dtype=torch.float64, pin_memory=True)
P.generate("uniform_square", n, 42, out=h.numpy())
d = h.cuda(); ctx.reserve(n); torch.cuda.synchronize()
ops = S.GpuShardOps(ctx, d, 0)
group = None
acc = {}
def run():
    ts = [("start", time.perf_counter())]
    mark = lambda k: ts.append((k, time.perf_counter()))
    world = 1; dev = S._device_for(group); ctrl = S._ctrl_group(group); mark("groups")
    q, idx = ops.extremes(); mark("extremes")
    mine = torch.from_numpy(np.concatenate([np.asarray(q, np.float64).reshape(8), np.asarray(idx, np.float64)]))
    if os.environ.get("AG1_NCCL"):
        md = mine.cuda(non_blocking=True); od = torch.empty((1, 12), dtype=torch.float64, device="cuda")
        dist.all_gather_into_tensor(od, md); allq = list(od.cpu())
    else:
        allq = [torch.empty_like(mine)]; dist.all_gather(allq, mine, group=ctrl)
    mark("ag1")
    arr = torch.stack(allq).numpy(); quad = S.fold_extremes(arr[:, :8], arr[:, 8:].astype(np.int64)); mark("fold")
    ch, kc = ops.chains(quad, 1024); mark("chains")
    early = os.environ.get("EARLY")
    if early:
        pin = S._PINNED.get("own")
        if pin is None or pin.shape[0] < ch.shape[0]:
            pin = torch.empty((max(ch.shape[0], 1 << 16), 2), dtype=torch.float64, pin_memory=True); S._PINNED["own"] = pin
        own = pin[: ch.shape[0]]; own.copy_(ch, non_blocking=True)
        mark("own_d2h")
    cnt = torch.tensor([ch.shape[0]] + list(kc), dtype=torch.int64)
    counts = [torch.empty_like(cnt)]; dist.all_gather(counts, cnt, group=ctrl); mark("ag2")
    counts = [[int(x) for x in c.tolist()] for c in counts]; width = max(max(c[0] for c in counts), 1)
    buf = ch if (ch.shape[0] == width and ch.device == dev and ch.is_contiguous()) else None; mark("buf")
    flat = torch.empty((world * width, 2), dtype=torch.float64, device=dev)
    dist.all_gather_into_tensor(flat, buf, group=group); gathered = list(flat.view(world, width, 2)); mark("ag3")
    fv = len(S.frame_vertices(quad)); mark("frame")
    if early:
        torch.cuda.current_stream().synchronize()
        runs = [(own.numpy(), counts[0][1:])]
    else:
        runs = [(g[: c[0]].numpy(), c[1:]) for g, c in zip(S._to_host(gathered, counts), counts)]
    mark("to_host")
    out = ops.merge(runs, quad); mark("merge")
    for (k0, t0), (k1, t1) in zip(ts, ts[1:]):
        acc[k1] = acc.get(k1, 0) + (t1 - t0)
for _ in range(3): run()
acc.clear()
for _ in range(10): run()
print({k: round(v / 10 * 1e3, 3) for k, v in acc.items()})
dist.destroy_process_group()
