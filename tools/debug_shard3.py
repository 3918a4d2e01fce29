"""Debug: the sharded GPU test as written (mp.spawn + gloo), rank 0 dumps
every stage of the failing case."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle")); sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch.multiprocessing as mp

def worker(rank, world, port):
    sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle")); sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch, torch.distributed as dist
    import paper_1508_05488_b200 as P
    from paper_1508_05488_b200 import sharded as S
    from pyoracle import Oracle
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    ctx = P.Context(0)
    o = Oracle()
    from test_sharded import DATASETS
    for (dist_name, n, seed) in DATASETS:
        pts = P.generate(dist_name, n, seed)
        bounds = np.linspace(0, n, world + 1).astype(int)
        shard = torch.from_numpy(np.ascontiguousarray(pts[bounds[rank]:bounds[rank + 1]])).cuda()
        torch.cuda.synchronize()
        ops = S.GpuShardOps(ctx, shard, int(bounds[rank]))
        class Spy(S.GpuShardOps):
            def finish(self, points, cc):
                res = self.ctx.convex_hull(points, P.PipelineConfig(chunk_count=cc))
                want = o.convex_hull(points, cc)
                print(dist_name, cc, "finish n", len(points), "gpu", [res.stats.n_after_round1, res.stats.n_after_spa, res.stats.n_hull],
                      "oracle", want.counts.tolist()[1:], "eq", np.array_equal(res.hull.vertices, want.hull), "path", res.diag.spa_path, flush=True)
                if not np.array_equal(res.hull.vertices, want.hull):
                    d = res.diag
                    print("  degenerate", d.degenerate_branch, "frame", d.frame_size, "regions", d.region_counts, "kept", d.kept_counts, "want kept", want.kept_counts.tolist(), flush=True)
                    print("  quad", d.quad.tolist(), "oracle quad", o.find_extremes(points).tolist(), flush=True)
                    print("  hull", res.hull.vertices[:5].tolist(), flush=True)
                    r2 = self.ctx.convex_hull(points, P.PipelineConfig(chunk_count=cc))
                    print("  retry eq", np.array_equal(r2.hull.vertices, want.hull), r2.stats.n_hull, flush=True)
                    r3 = P.Context(0).convex_hull(points, P.PipelineConfig(chunk_count=cc))
                    print("  fresh ctx eq", np.array_equal(r3.hull.vertices, want.hull), r3.stats.n_hull, flush=True)
                    np.save("gpurun_out/fail_points.npy", points)
                return res.hull.vertices
        ops = Spy(ctx, shard, int(bounds[rank]))
        for cc in (1, 1024):
            hull = S.sharded_convex_hull(ops, cc)
            if rank == 0:
                want = o.convex_hull(o.generate(dist_name, n, seed), 1024)
                print(dist_name, cc, "final eq", np.array_equal(hull, want.hull), len(hull), len(want.hull), flush=True)
    dist.barrier(); dist.destroy_process_group()

if __name__ == "__main__":
    import socket
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    mp.spawn(worker, args=(2, port), nprocs=2, join=True)
