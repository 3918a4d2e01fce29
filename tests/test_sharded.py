"""CPU: the multi-GPU sharded hull (paper_1508_05488_b200/sharded.py) with
the gloo backend, world_size 2 (and 3), each rank's compute done by the C
oracle. The exchange logic (rank-ordered extremes fold with global-index
ties, chain gather, hull of the union + frame) must reproduce the
reference hull of the whole set bit-exactly."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT

DATASETS = [("uniform_square", 20000, 3), ("uniform_disk", 20000, 4), ("gaussian", 30000, 5),
            ("circle", 3000, 6), ("duplicates_heavy", 5000, 7), ("collinear", 2000, 8),
            ("uniform_square", 7, 9)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class OracleShardOps:
    """Per-rank compute on the CPU with the C oracle (test stand-in for
    GpuShardOps)."""

    def __init__(self, oracle, pts, base):
        self.o, self.p, self.base = oracle, pts, base

    def extremes(self):
        q = self.o.find_extremes(self.p)
        idx = []
        for c in q:  # earliest ==-equal point, as the sequential fold keeps
            hit = np.nonzero((self.p[:, 0] == c[0]) & (self.p[:, 1] == c[1]))[0]
            idx.append(self.base + int(hit[0]))
        return q, np.array(idx, np.int64)

    def chains(self, quad, chunk_count):
        from paper_1508_05488_b200.sharded import frame_vertices
        lab = self.o.classify(self.p, quad)
        if len(frame_vertices(quad)) <= 2:
            surv = self.p[lab != 0]
            if len(surv) == 0:
                return surv, [0, 0, 0, 0]
            order = np.lexsort((surv[:, 1], surv[:, 0]))
            return surv[order], [len(surv), 0, 0, 0]
        out = []
        for r in range(1, 5):
            seg = self.o.sort_region(r, self.p[lab == r])
            anchors = np.array([quad[r - 1], quad[r % 4]])
            out.append(self.o.spa_filter(r, seg, anchors, chunk_count))
        return (np.concatenate(out) if out else np.empty((0, 2))), [len(o) for o in out]

    def finish(self, points, chunk_count):
        res = self.o.convex_hull(points, chunk_count)
        assert res.status == 0
        return res.hull

    def merge(self, runs, quad):
        # the product's host merge (chgpu_merge_hull: no device involved)
        from paper_1508_05488_b200 import merge_hull
        return merge_hull(runs, quad)


def _worker(rank, world, port, results):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import torch.distributed as dist
    from pyoracle import Oracle
    from paper_1508_05488_b200.sharded import sharded_convex_hull
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    o = Oracle()
    for i, (dist_name, n, seed) in enumerate(DATASETS):
        pts = o.generate(dist_name, n, seed)
        bounds = np.linspace(0, n, world + 1).astype(int)
        shard = pts[bounds[rank]:bounds[rank + 1]]
        if len(shard) == 0:
            shard = pts[:0]
        ops = OracleShardOps(o, shard, int(bounds[rank]))
        for cc in (1, 1024):
            hull = sharded_convex_hull(ops, cc)
            if rank == 0:
                results[(i, cc)] = hull.tobytes()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_hull_matches_reference_gloo(world, oracle):
    # every shard must be non-empty for the extremes exchange
    assert min(n for _, n, _ in DATASETS) >= world
    mgr = mp.Manager()
    results = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(world, port, results), nprocs=world, join=True)
    for i, (dist_name, n, seed) in enumerate(DATASETS):
        pts = oracle.generate(dist_name, n, seed)
        want = oracle.convex_hull(pts, 1024)
        assert want.status == 0
        for cc in (1, 1024):
            got = np.frombuffer(results[(i, cc)], np.float64).reshape(-1, 2)
            assert np.array_equal(got, want.hull), (dist_name, n, cc)


def test_fold_extremes_python_and_c_agree(product):
    """chgpu_fold_extremes (C) == sharded.fold_extremes (Python) with ties."""
    import ctypes as C
    from paper_1508_05488_b200.sharded import fold_extremes
    rng = np.random.default_rng(3)
    lib = product.load_library()
    for _ in range(200):
        k = int(rng.integers(1, 6))
        quads = rng.integers(0, 3, size=(k, 4, 2)).astype(np.float64)
        idxs = rng.permutation(100)[: 4 * k].reshape(k, 4).astype(np.uint64)
        want = fold_extremes(quads, idxs.astype(np.int64))
        out = np.empty(8, np.float64)
        q = np.ascontiguousarray(quads.reshape(-1))
        ix = np.ascontiguousarray(idxs.reshape(-1))
        lib.chgpu_fold_extremes(q.ctypes.data_as(C.POINTER(C.c_double)),
                                ix.ctypes.data_as(C.POINTER(C.c_uint64)), k,
                                out.ctypes.data_as(C.POINTER(C.c_double)))
        assert np.array_equal(out.reshape(4, 2), want)
        # (the GPU ranks' fold goes through it)
        from paper_1508_05488_b200.sharded import GpuShardOps
        assert np.array_equal(GpuShardOps.fold(None, quads, idxs.astype(np.int64)), want)


def _gpu_worker(rank, world, port, results, mode=0, backend="gloo"):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    import paper_1508_05488_b200 as P
    from paper_1508_05488_b200.sharded import GpuShardOps, sharded_convex_hull
    kw = {"device_id": torch.device("cuda", 0)} if backend == "nccl" else {}
    dist.init_process_group(backend, init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world, **kw)
    ctx = P.Context(0)
    ctx.set_spa_path(mode)
    for i, (dist_name, n, seed) in enumerate(DATASETS):
        pts = P.generate(dist_name, n, seed)
        bounds = np.linspace(0, n, world + 1).astype(int)
        shard = torch.from_numpy(np.ascontiguousarray(pts[bounds[rank]:bounds[rank + 1]])).cuda()
        torch.cuda.synchronize()
        ops = GpuShardOps(ctx, shard, int(bounds[rank]))
        for cc in (1, 1024):
            hull = sharded_convex_hull(ops, cc)
            if rank == 0:
                results[(i, cc)] = np.ascontiguousarray(hull).tobytes()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("mode", [0, 1, 2])  # SPA_AUTO, SPA_SORT, SPA_FILTER
def test_sharded_hull_gpu_ranks(oracle, mode):
    """Two ranks sharing cuda:0 (gloo carries the exchange): the GPU shard
    entry points (chgpu_shard_extremes / chgpu_shard_chains) + merge."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    mgr = mp.Manager()
    results = mgr.dict()
    port = _free_port()
    mp.spawn(_gpu_worker, args=(2, port, results, mode), nprocs=2, join=True)
    for i, (dist_name, n, seed) in enumerate(DATASETS):
        pts = oracle.generate(dist_name, n, seed)
        want = oracle.convex_hull(pts, 1024)
        for cc in (1, 1024):
            got = np.frombuffer(results[(i, cc)], np.float64).reshape(-1, 2)
            assert np.array_equal(got, want.hull), (dist_name, n, cc)


@pytest.mark.gpu
def test_sharded_hull_nccl_one_rank(oracle):
    """The NCCL branch of sharded_convex_hull (device-resident exchange
    buffers, all_gather of the chains) at world size 1 on the one GPU: the
    hull equals the reference's."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    mgr = mp.Manager()
    results = mgr.dict()
    port = _free_port()
    mp.spawn(_gpu_worker, args=(1, port, results, 0, "nccl"), nprocs=1, join=True)
    for i, (dist_name, n, seed) in enumerate(DATASETS):
        pts = oracle.generate(dist_name, n, seed)
        want = oracle.convex_hull(pts, 1024)
        for cc in (1, 1024):
            got = np.frombuffer(results[(i, cc)], np.float64).reshape(-1, 2)
            assert np.array_equal(got, want.hull), (dist_name, n, cc)


@pytest.mark.parametrize("dist,n", [("uniform_square", 60_000), ("uniform_disk", 50_000),
                                    ("gaussian", 40_000), ("circle", 3_000)])
def test_merge_hull_of_shard_chains(oracle, product, dist, n):
    """chgpu_merge_hull (the rank-0 merge of a non-degenerate frame): each
    region's runs from 1..8 contiguous shards, SPA'd against the global quad
    by the reference's stage functions, merged in region order and finished
    with Melkman = the reference's convex_hull of the whole set."""
    pts = oracle.generate(dist, n, 3)
    quad = oracle.find_extremes(pts)
    for cc in (1, 7, 1024):
        want = oracle.convex_hull(pts, cc)
        for k in (1, 2, 5, 8):
            bounds = np.linspace(0, n, k + 1).astype(int)
            runs = [OracleShardOps(oracle, pts[bounds[s]:bounds[s + 1]], int(bounds[s])).chains(quad, cc)
                    for s in range(k)]
            got = product.merge_hull(runs, quad)
            assert np.array_equal(got, want.hull), (dist, cc, k)
