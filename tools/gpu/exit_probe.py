import os, sys, torch, torch.distributed as dist
sys.path.insert(0, ".")
import paper_1508_05488_b200 as P
rank = int(os.environ["RANK"]); local = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(0)
dist.init_process_group("gloo")
ctx = P.Context(0)
h = torch.empty((1000000, 2), dtype=torch.float64, pin_memory=True)
P.generate("uniform_square", 1000000, 1, out=h.numpy())
d = h.cuda(); torch.cuda.synchronize()
stream = torch.cuda.ExternalStream(ctx.stream)
mode = sys.argv[1]
r = ctx.convex_hull_device(d.data_ptr(), 1000000, P.PipelineConfig())
print(rank, "hull", r.stats.n_hull, flush=True)
dist.barrier(); dist.destroy_process_group()
if mode == "closefirst":
    ctx.close(); print(rank, "closed", flush=True)
elif mode == "delfirst":
    del stream; del d; del h; torch.cuda.synchronize(); ctx.close(); print(rank, "closed", flush=True)
elif mode == "noclose":
    pass
print(rank, "exit", flush=True)
