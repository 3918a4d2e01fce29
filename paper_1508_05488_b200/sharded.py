"""Multi-GPU hull: one rank per GPU, the point set sharded by contiguous
index ranges. Scaling is by sharding, with two tiny
exchanges over torch.distributed (NCCL on GPUs, gloo in the CPU tests):

1. all-gather of each rank's 4 extreme candidates (point + global index),
   folded in rank order with the lexicographic rules and lowest-global-index
   ties (reference extremes.cpp:39-46 semantics), so every rank holds the
   quad find_extremes would return on the whole set;
2. each rank runs round-1 discard, region sort and SPA of its shard against
   that global quad (every dropped point lies inside the global quad or
   inside a triangle of kept points and global anchors, so no hull vertex is
   lost), then the chains are gathered on rank 0: each region's chains from
   all ranks merged in region order (they are sorted runs), the ring
   assembled with the global frame and Melkman run on it on the host
   (chgpu_merge_hull) — the hull of the union is the hull of the whole set.
   A degenerate frame (the reference's sort-based branch) finishes with the
   single-GPU pipeline over (union of the ranks' unique survivors) + frame.

The per-rank compute is behind `ShardOps` so the exchange logic is tested
with the gloo backend on CPU (tests/test_sharded.py) and runs the sm_100a
kernels through the C ABI on GPUs (GpuShardOps).
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def frame_vertices(quad: np.ndarray) -> np.ndarray:
    """extremes.cpp:49-57."""
    ring = []
    for p in np.asarray(quad, np.float64).reshape(4, 2):
        if not ring or not (ring[-1][0] == p[0] and ring[-1][1] == p[1]):
            ring.append(p)
    if len(ring) > 1 and ring[0][0] == ring[-1][0] and ring[0][1] == ring[-1][1]:
        ring.pop()
    return np.array(ring, np.float64).reshape(-1, 2)


def _less_xy(a, b):
    return a[0] < b[0] or (a[0] == b[0] and a[1] < b[1])


def _less_yx(a, b):
    return a[1] < b[1] or (a[1] == b[1] and a[0] < b[0])


def fold_extremes(quads: np.ndarray, idxs: np.ndarray) -> np.ndarray:
    """Rank-ordered fold of per-rank corner candidates; ties -> lowest global
    index (the earliest point, as the reference's sequential fold keeps)."""
    quads = np.asarray(quads, np.float64).reshape(-1, 4, 2)
    idxs = np.asarray(idxs, np.int64).reshape(-1, 4)
    best = [None] * 4
    for r in range(len(quads)):
        for c in range(4):
            cand = (quads[r, c], int(idxs[r, c]))
            if best[c] is None:
                best[c] = cand
                continue
            a, b = cand[0], best[c][0]
            if c == 0:
                win, lose = _less_xy(a, b), _less_xy(b, a)
            elif c == 1:
                win, lose = _less_yx(a, b), _less_yx(b, a)
            elif c == 2:
                win, lose = _less_xy(b, a), _less_xy(a, b)
            else:
                win, lose = _less_yx(b, a), _less_yx(a, b)
            if win or (not lose and cand[1] < best[c][1]):
                best[c] = cand
    return np.array([b[0] for b in best], np.float64)


class ShardOps:
    """Per-rank compute used by sharded_convex_hull."""

    def extremes(self):  # -> (quad (4, 2), global indices (4,))
        raise NotImplementedError

    def chains(self, quad: np.ndarray, chunk_count: int):
        """-> ((k, 2) kept points: the 4 region chains concatenated, or on a
        degenerate frame the sorted unique survivors; kept counts[4])."""
        raise NotImplementedError

    def fold(self, quads: np.ndarray, idxs: np.ndarray) -> np.ndarray:  # -> quad (4, 2)
        """The global quad from every rank's corner candidates (rank order,
        lowest global index on ties)."""
        return fold_extremes(quads, idxs)

    def merge(self, runs, quad: np.ndarray) -> np.ndarray:  # -> hull vertices
        """Hull of the union of the ranks' chain runs ((chains, counts[4]) on
        the host), non-degenerate frame."""
        from . import merge_hull
        return merge_hull(runs, quad)

    def finish(self, points: np.ndarray, chunk_count: int) -> np.ndarray:  # -> hull vertices
        raise NotImplementedError


class GpuShardOps(ShardOps):
    """sm_100a kernels through the C ABI; `points` is a CUDA float64 (n, 2)
    tensor holding this rank's shard, `base_index` its global offset."""

    def __init__(self, ctx, points: torch.Tensor, base_index: int):
        self.ctx, self.t, self.base = ctx, points, int(base_index)
        self.out = None  # chain buffer (device), reused across calls

    def extremes(self):
        q, idx = self.ctx.shard_extremes(self.t.data_ptr(), self.t.shape[0], self.base)
        return q.reshape(4, 2), idx.astype(np.int64)

    def fold(self, quads, idxs):
        # chgpu_fold_extremes: the same fold in C (tests/test_sharded.py pins
        # it to fold_extremes)
        import ctypes as C
        from . import load_library
        q = np.ascontiguousarray(np.asarray(quads, np.float64).reshape(-1))
        ix = np.ascontiguousarray(np.asarray(idxs, np.uint64).reshape(-1))
        out = np.empty(8, np.float64)
        load_library().chgpu_fold_extremes(q.ctypes.data_as(C.POINTER(C.c_double)),
                                           ix.ctypes.data_as(C.POINTER(C.c_uint64)), len(q) // 8,
                                           out.ctypes.data_as(C.POINTER(C.c_double)))
        return out.reshape(4, 2)

    def chains(self, quad, chunk_count):
        # device-resident chains (a shard never keeps more than its points):
        # the gather and the merge read them without a host round trip
        n = self.t.shape[0]
        if self.out is None or self.out.shape[0] < n:
            self.out = torch.empty((max(n, 1), 2), dtype=torch.float64, device=self.t.device)
        kc = self.ctx.shard_chains_device(self.t.data_ptr(), n, quad, chunk_count,
                                          self.out.data_ptr(), self.out.shape[0])
        return self.out[: sum(kc)], [int(c) for c in kc]

    def finish(self, points, chunk_count):
        from . import PipelineConfig
        cfg = PipelineConfig(chunk_count=chunk_count)
        if isinstance(points, torch.Tensor) and points.is_cuda:
            p = points.contiguous()
            torch.cuda.current_stream(p.device).synchronize()  # the merge reads it on ctx's stream
            return self.ctx.convex_hull_device(p.data_ptr(), p.shape[0], cfg).hull.vertices
        if isinstance(points, torch.Tensor):
            points = points.numpy()
        return self.ctx.convex_hull(points, cfg).hull.vertices


_CTRL_GROUPS = {}


def _ctrl_group(group):
    """A gloo group beside an NCCL one for the two small control exchanges
    (12 doubles, 5 counts per rank): host tensors, no device round trips.
    Created collectively on first use."""
    if dist.get_backend(group) != "nccl":
        return group
    key = id(group)
    if key not in _CTRL_GROUPS:
        ranks = None if group is None else dist.get_process_group_ranks(group)
        _CTRL_GROUPS[key] = dist.new_group(ranks=ranks, backend="gloo")
    return _CTRL_GROUPS[key]


_PINNED = {}


def _pinned(dev, key, rows):
    """A reused pinned host buffer of at least `rows` points."""
    buf = _PINNED.get((dev, key))
    if buf is None or buf.shape[0] < rows:
        buf = torch.empty((max(rows, 1 << 16), 2), dtype=torch.float64, pin_memory=True)
        _PINNED[(dev, key)] = buf
    return buf


def _pinned_copy(t, key):
    """Starts the copy of device points t into a pinned buffer (on the
    current stream); the caller synchronises before reading it."""
    out = _pinned(t.device, key, t.shape[0])[: t.shape[0]]
    out.copy_(t, non_blocking=True)
    return out


def _to_host(gathered, counts):
    """The gathered chains on the host: device runs go through one reused
    pinned buffer (a pageable .cpu() per run stages every byte twice)."""
    if not gathered or not gathered[0].is_cuda:
        return gathered
    buf = _pinned(gathered[0].device, "peers", sum(c[0] for c in counts))
    out, off = [], 0
    for g, c in zip(gathered, counts):
        out.append(buf[off: off + c[0]])
        out[-1].copy_(g[: c[0]], non_blocking=True)
        off += c[0]
    torch.cuda.current_stream(dev).synchronize()
    return out


def _device_for(group) -> torch.device:
    backend = dist.get_backend(group)
    if backend == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def sharded_convex_hull(ops: ShardOps, chunk_count: int = 1024, group=None):
    """Returns the global hull on rank 0 (None elsewhere)."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    dev = _device_for(group)
    ctrl = _ctrl_group(group)  # host-side exchanges of the small control data

    # exchange 1: extreme candidates (8 coords + 4 indices; indices < 2^53
    # travel exactly as float64)
    q, idx = ops.extremes()
    mine = torch.from_numpy(np.concatenate([np.asarray(q, np.float64).reshape(8),
                                            np.asarray(idx, np.float64)]))
    allq = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(allq, mine, group=ctrl)
    arr = torch.stack(allq).numpy()
    fold = getattr(ops, "fold", None) or fold_extremes  # (duck-typed ops may not have one)
    quad = fold(arr[:, :8], arr[:, 8:].astype(np.int64))

    # per-rank discard + sort + SPA against the global quad (a CUDA tensor
    # from GpuShardOps, numpy from the CPU ops of the tests)
    ch, kc = ops.chains(quad, chunk_count)
    ch = (ch if isinstance(ch, torch.Tensor)
          else torch.from_numpy(np.ascontiguousarray(ch, np.float64))).reshape(-1, 2)
    # rank 0's own chains never need the exchange: their copy to the host
    # starts now and overlaps it
    own = _pinned_copy(ch, "own") if rank == 0 and ch.is_cuda else None

    # exchange 2: chains to rank 0 (sizes and region counts first, then
    # padded payloads)
    cnt = torch.tensor([ch.shape[0]] + list(kc), dtype=torch.int64)
    counts = [torch.empty_like(cnt) for _ in range(world)]
    dist.all_gather(counts, cnt, group=ctrl)
    counts = [[int(x) for x in c.tolist()] for c in counts]
    width = max(max(c[0] for c in counts), 1)
    if ch.shape[0] == width and ch.device == dev and ch.is_contiguous():
        buf = ch  # (the widest rank sends its chains as they are)
    else:
        buf = torch.empty((width, 2), dtype=torch.float64, device=dev)  # rows past a rank's count are never read
        if ch.shape[0]:
            buf[: ch.shape[0]] = ch.to(dev)
    gathered = [torch.empty_like(buf) for _ in range(world)] if rank == 0 else None
    if dist.get_backend(group) == "nccl":
        # NCCL gather: emulate with all_gather (the payload is tiny), into
        # one flat tensor (one launch, no per-rank output list)
        flat = torch.empty((world * width, 2), dtype=torch.float64, device=dev)
        dist.all_gather_into_tensor(flat, buf, group=group)
        gathered = list(flat.view(world, width, 2)) if rank == 0 else None
    else:
        dist.gather(buf, gathered, dst=0, group=group)
    if rank != 0:
        return None
    if len(frame_vertices(quad)) > 2:
        # each region's sorted runs merged, the ring closed with the global
        # frame, Melkman on the host (the chains are ~35K points per rank)
        peers = _to_host(gathered[1:], counts[1:])
        if own is not None:
            torch.cuda.current_stream(ch.device).synchronize()
            mine_host = own.numpy()
        else:
            mine_host = gathered[0][: counts[0][0]].numpy()
        runs = [(mine_host, counts[0][1:])] + [(g[: c[0]].numpy(), c[1:])
                                              for g, c in zip(peers, counts[1:])]
        return ops.merge(runs, quad)
    frame = torch.from_numpy(frame_vertices(quad)).to(dev)
    union = torch.cat([g[: c[0]] for g, c in zip(gathered, counts)] + [frame], dim=0)
    return ops.finish(union.numpy() if dev.type == "cpu" else union, chunk_count)
