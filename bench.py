#!/usr/bin/env python3
"""Benchmark of the B200 CudaChain hull path (BASELINE.json metric:
"Mpoints/s end-to-end hull (20M uniform pts); HBM GB/s of discard kernels").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one full convex_hull of a synthetic point set (the reference's own
generator, bit-identical): extremes -> classify/discard -> region sort ->
SPA -> chains to host -> Melkman, result on the host.

* value: Mpoints/s with the input already resident in HBM (chgpu_hull_device),
  timed with CUDA events on the library's stream, max over ranks.
* e2e: the same metric through the C ABI with the input in pinned HOST
  memory (chgpu_hull), host->device copy and the chain/hull read-back inside
  the timed region.
* roofline: the dominant kernel (the onesweep radix pass) plus the discard
  kernels (K1 + K2), algorithmic bytes / CUDA-event time, against
  MEASURED_PEAKS.json hbm_gbs.
* cpu_baseline: the reference C++ path (oracle/_ref, compiled from the
  unmodified sources) on this host's cores, on the same input.

N > 1 (torchrun): weak scaling, each rank owns a 20M-point shard of one
global set (shard r = generate(dist, n, seed + r)); the step is the sharded
hull (paper_1508_05488_b200/sharded.py) and value counts all ranks' points.
The input is 320 MB per rank, larger than the 126 MB L2, so no L2 flush is
needed between steps.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Mpoints/s end-to-end hull (20M uniform pts)"
UNIT = "Mpoints/s"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.p:
            time.sleep(0.25)
            self.p.terminate()
            try:
                self.out, _ = self.p.communicate(timeout=5)
            except Exception:
                self.p.kill()

    def summary(self):
        rows = []
        for line in (self.out or "").strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                rows.append(parts)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(rows[0][1]) if rows[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(rows)}


# Per-launch DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) of
# the pipeline's kernels from the committed ncu --set full captures of this
# workload (profiles/, tools/round_measure.sh); None when absent.
TRAFFIC_FILE = os.path.join(ROOT, "profiles", "round1", "traffic.json")


def measured_traffic(kernel_key: str):
    try:
        with open(TRAFFIC_FILE) as f:
            t = json.load(f)
        return t.get(kernel_key)
    except Exception:
        return None


def cpu_baseline(pts: np.ndarray, steps: int = 3):
    """The reference CPU path (oracle/_ref) on this host; port if absent."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from pyoracle import Oracle, RefLib
    cores = os.cpu_count() or 1
    if RefLib.available():
        ref = RefLib()
        kind = "reference"
        run = lambda par: ref.convex_hull(pts, 1024, par)  # noqa: E731
    else:
        orc = Oracle()
        kind, cores = "port", 1
        run = lambda par: orc.convex_hull(pts, 1024)  # noqa: E731
    run(0)  # warm-up (page faults, allocator)
    ts = []
    for _ in range(steps):
        t0 = time.perf_counter()
        run(0)
        ts.append(time.perf_counter() - t0)
    t_all = statistics.median(ts)
    t0 = time.perf_counter()
    run(1)
    t_one = time.perf_counter() - t0
    n = len(pts)
    return {"value": n / t_all / 1e6, "unit": UNIT, "cores": cores, "kind": kind,
            "sample": f"{n} points, convex_hull chunk_count=1024, median of {steps} runs "
                      f"(parallelism=0 = all {cores} host threads), generation excluded",
            "value_1thread": n / t_one / 1e6, "ms_all_cores": t_all * 1e3,
            "ms_1thread": t_one * 1e3}


def run_reference(args, rank, world):
    """--impl reference: the reference's own CPU implementation of the path."""
    import paper_1508_05488_b200 as P
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from pyoracle import Oracle, RefLib
    pts = P.generate(args.dist, args.n, args.seed)
    cores = os.cpu_count() or 1
    if RefLib.available():
        ref, kind = RefLib(), "reference"
        step = lambda: ref.convex_hull(pts, args.chunk_count, 0)  # noqa: E731
    else:
        orc, kind, cores = Oracle(), "port", 1
        step = lambda: orc.convex_hull(pts, args.chunk_count)  # noqa: E731
    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = (time.perf_counter() - t0) / args.steps
    v = args.n / dt / 1e6
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": f"{args.n} {args.dist} points seed {args.seed}",
                       "chunk_count": args.chunk_count, "parallelism": "cpu threads"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": kind,
                             "sample": f"{args.n} points per step, all host threads"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--dist", default="uniform_square")
    ap.add_argument("--n", type=int, default=20_000_000)
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--chunk-count", type=int, default=1024)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="exchange backend for N > 1 (gloo: testing several ranks on one GPU)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    import paper_1508_05488_b200 as P
    from paper_1508_05488_b200.sharded import GpuShardOps, sharded_convex_hull

    local = local % max(1, torch.cuda.device_count())  # gloo testing: ranks may share a GPU
    torch.cuda.set_device(local)
    if world > 1:
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    ctx = P.Context(local)
    cfg = P.PipelineConfig(chunk_count=args.chunk_count)

    # Input: this rank's shard, generated on the host (bit-identical to the
    # reference generator), resident in HBM and in pinned host memory.
    pts = P.generate(args.dist, args.n, args.seed + rank)
    d_pts = torch.from_numpy(pts).to(f"cuda:{local}")
    h_pin = torch.empty((args.n, 2), dtype=torch.float64, pin_memory=True)
    h_pin.numpy()[:] = pts
    ctx.reserve(args.n)
    torch.cuda.synchronize()

    stream = torch.cuda.ExternalStream(ctx.stream)

    def step_device():
        if world == 1:
            return ctx.convex_hull_device(d_pts.data_ptr(), args.n, cfg, copy=False)
        ops = GpuShardOps(ctx, d_pts, rank * args.n)
        return sharded_convex_hull(ops, args.chunk_count)

    def step_host():
        if world == 1:
            return ctx.convex_hull(h_pin.numpy(), cfg, copy=False)
        # host-resident shard: copy in, then the sharded step
        d_pts.copy_(h_pin, non_blocking=True)
        torch.cuda.synchronize()
        ops = GpuShardOps(ctx, d_pts, rank * args.n)
        return sharded_convex_hull(ops, args.chunk_count)

    def timed(fn, steps):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        out = None
        for _ in range(steps):
            out = fn()
        e1.record(stream)
        e1.synchronize()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        if world > 1:
            t = torch.tensor([ms], dtype=torch.float64,
                             device=f"cuda:{local}" if args.backend == "nccl" else "cpu")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms, out

    for _ in range(args.warmup):
        last = step_device()
    # correctness guard for the measured configuration (single GPU)
    diag = last.diag if world == 1 else None

    with ClockSampler(local) as clk:
        ms, res = timed(step_device, args.steps)
    for _ in range(2):
        step_host()
    ms_e2e, res_e2e = timed(step_host, args.steps)
    clocks = clk.summary()

    total_pts = args.n * world
    value = total_pts / (ms * 1e-3) / 1e6
    e2e_value = total_pts / (ms_e2e * 1e-3) / 1e6

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference generator, bit-identical)",
            "config": {"workload": f"{args.n} {args.dist} points per GPU, seed {args.seed}",
                       "chunk_count": args.chunk_count, "input_bytes": args.n * 16,
                       "l2": "input 320 MB > 126 MB L2 (no flush needed)",
                       "parallelism": f"shard{world}" if world > 1 else "single"},
            "clocks": clocks}

    if rank == 0 and world == 1:
        r = res
        d = r.diag
        s1 = sum(d.region_counts[1:])
        hbm, src = peaks()
        t = d.times_ms
        n = args.n
        # K2 writes each survivor as an 8-byte filter key + a 4-byte input
        # index on the pre-filtered path, as a 16-byte (k, v) record on the
        # sort path
        surv_b = 12 if d.spa_path == 1 else 16
        disc_bytes = 32 * n + surv_b * s1
        disc_ms = t["t_k1_ms"] + t["t_k2_ms"]
        kernels = {
            "k1_extremes": {"ms": t["t_k1_ms"], "bytes": 16 * n,
                            "basis": "16 B/pt read"},
            ("k2_classify_survivors" if d.spa_path == 1 else "k2_classify_compact"):
                {"ms": t["t_k2_ms"], "bytes": 16 * n + surv_b * s1,
                 "basis": f"16 B/pt read + {surv_b} B/survivor write"},
        }
        if d.spa_path == 1:
            lb = d.filter_log2nb
            nb = 4 * (1 << lb)
            nc = d.n_candidates
            kernels.update({
                "k3_bin_scan": {"ms": t["t_binscan_ms"], "bytes": 24 * nb,
                                "basis": "12 B/bin read + 12 B/bin write"},
                "k3_filter": {"ms": t["t_filter_ms"], "bytes": 8 * s1 + 36 * nc,
                              "basis": "8 B/survivor key read + per candidate 4 B index "
                                       "+ 16 B point read, 16 B record write",
                              "candidates": nc},
                "k3_bin_sort": {"ms": t["t_binsort_ms"],
                                "basis": "bins above 32 candidates sorted in place"},
                "k4_spa_chunks_emit": {"ms": t["t_spa_kernel_ms"],
                                       "bytes": 16 * nc + 32 * sum(d.kept_counts),
                                       "basis": "16 B/candidate read + 16 B/kept scratch "
                                                "+ 16 B/kept point write"},
            })
        else:
            pass_ms = t["t_passes_ms"] / max(d.sort_passes, 1)
            kernels.update({
                "k3_hist": {"ms": t["t_hist_ms"], "bytes": 8 * s1, "basis": "8 B/record read"},
                "k3_radix_pass": {"ms": pass_ms, "launches": d.sort_passes, "bytes": 32 * s1,
                                  "basis": "16 B/record read + 16 B/record write"},
                "k3_ties": {"ms": t["t_ties_ms"]},
                "k4_spa": {"ms": t["t_spa_kernel_ms"], "bytes": 8 * s1 + 2 * s1
                           + 16 * sum(d.kept_counts),
                           "basis": "8 B/record read + 16 B/kept write (+ flags)"},
            })
        for kv in kernels.values():
            if kv.get("bytes") and kv.get("ms"):
                kv["gbs"] = kv["bytes"] / (kv["ms"] * 1e-3) / 1e9
        kernels["d2h_chains_ms"] = t["t_d2h_ms"]
        kernels["host_melkman_ms"] = t["t_host_ms"]
        dom_name, dom = max(((k, v) for k, v in kernels.items()
                             if isinstance(v, dict) and v.get("gbs")), key=lambda kv: kv[1]["ms"])
        line["roofline"] = {
            "bound": "hbm", "kernel": dom_name,
            "achieved": dom["gbs"], "peak": hbm, "unit": "GB/s",
            "peak_source": src, "frac": dom["gbs"] / hbm,
            "traffic": measured_traffic(dom_name),
            "algorithmic_bytes": f"{dom.get('basis', 'bytes moved')}: {dom['bytes']} B per launch",
            "discard_kernels": {"kernels": "k_extremes_partial (+ last-block merge), k_classify_survivors",
                                "achieved": disc_bytes / (disc_ms * 1e-3) / 1e9,
                                "frac": disc_bytes / (disc_ms * 1e-3) / 1e9 / hbm,
                                "bytes": disc_bytes, "ms": disc_ms},
            "spa_path": ["sort", "prefilter", "prefilter->sort"][d.spa_path],
            "per_kernel": kernels,
        }
        line["stats"] = {"n_after_round1": r.stats.n_after_round1,
                         "n_after_spa": r.stats.n_after_spa, "n_hull": r.stats.n_hull,
                         "frac_after_round1": r.stats.n_after_round1 / n}
        line["gpu_launches"] = d.launches * args.steps
        # device -> host: the kept chains (the host finisher builds the hull),
        # or on the convex fast path the finished hull alone
        d2h = 16 * (r.stats.n_hull if d.convex_fast_path else sum(d.kept_counts))
        line["e2e"] = {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": n * 16,
                       "d2h_bytes_per_step": d2h, "ms_per_step": ms_e2e,
                       "h2d_ms": res_e2e.diag.times_ms["t_h2d_ms"]}
        if not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(pts)
    elif rank == 0:
        line["e2e"] = {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": args.n * 16,
                       "d2h_bytes_per_step": 0, "ms_per_step": ms_e2e}
        line["hull_vertices"] = int(len(res)) if res is not None else None
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    ctx.close()


if __name__ == "__main__":
    main()
