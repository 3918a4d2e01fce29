#!/usr/bin/env python3
"""Benchmark of the B200 CudaChain hull path (BASELINE.json metric:
"Mpoints/s end-to-end hull (20M uniform pts); HBM GB/s of discard kernels").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one full convex_hull of a synthetic point set (the reference's own
generator, bit-identical): extremes -> classify/discard -> SPA pre-filter ->
chunk SPA -> chains to host -> Melkman, the hull on the host.

Workloads (identical `config` in both arms):
* N = 1: BASELINE configs[1], 20M uniform_square points, seed 42.
* N > 1 (torchrun, one rank per GPU): BASELINE configs[4], the 1B-point
  uniform_square set (seed 42) split into N contiguous index ranges; rank r
  generates exactly its range (chgpu_generate_range). The step is the sharded
  hull (paper_1508_05488_b200/sharded.py: NCCL exchange of the extreme
  candidates, per-rank discard + SPA against the global quad, chains gathered,
  rank-0 merge); value counts all 1B points ("scaling": "strong").

Keys of our line:
* value: Mpoints/s with the input resident in HBM (chgpu_hull_device), CUDA
  events on the library's stream around K steps, max over ranks.
* e2e: the same metric through the C ABI with the input in pinned HOST memory
  (chgpu_hull: H2D inside the timed region, overlapped with K1), and
  e2e.pageable the same through the C++ drop-in chainhull::convex_hull
  (libchainhull.so) on pageable host memory, as a std::vector caller has it.
* roofline: the kernel with the largest time (K2) against MEASURED_PEAKS.json
  hbm_gbs, algorithmic bytes / its in-step CUDA-event time, plus the discard
  kernels K1 + K2 on SURVEY §8(d)'s basis (32 n + 16 s1).
* parity: the measured step's hull and counters against the reference's own
  outputs (tests/golden/big.json, big_1b.json), outside the timed region.
* cpu_baseline: the reference C++ path (oracle/_ref, the unmodified sources)
  on this host's cores, median of 5 after one warm-up, with
  mallopt(M_MMAP_THRESHOLD, 256 MB) as tests/acceptance.cpp:376 does.

--impl reference: the reference's own CPU implementation (oracle/_ref) on the
same config; it imports nothing from the product (inputs come from the
reference's own generate()). Under torchrun only rank 0 runs it.

The input (320 MB per 20M points) exceeds the 126 MB L2, so no L2 flush is
needed between steps.
"""
from __future__ import annotations

import argparse
import ctypes
import hashlib
import json
import os
import platform
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Mpoints/s end-to-end hull (20M uniform pts)"
UNIT = "Mpoints/s"
N_SINGLE = 20_000_000        # BASELINE configs[1]
N_SHARDED = 1_000_000_000    # BASELINE configs[4]
REF_SAMPLE_SHARDED = 50_000_000  # reference arm's bounded sample of configs[4]


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def workload(args, world):
    """The config dict both arms print (identical by construction)."""
    sharded = world > 1 or args.sharded
    n = args.n if args.n else (N_SHARDED if sharded else N_SINGLE)
    shards = world
    name = ("BASELINE configs[4]" if sharded and n == N_SHARDED and args.dist == "uniform_square"
            else "BASELINE configs[1]" if not sharded and n == N_SINGLE
            and args.dist == "uniform_square" else "custom")
    return {"workload": f"{n} {args.dist} points, seed {args.seed}"
                        + (f", {shards} contiguous shard{'s' if shards > 1 else ''}"
                           if sharded else ""),
            "baseline_config": name, "n_points": n, "distribution": args.dist, "seed": args.seed,
            "chunk_count": args.chunk_count, "shards": shards,
            "parallelism": f"shard{shards}" if sharded else "single",
            "l2": (f"input {16 * n // shards // 1_000_000} MB per GPU > 126 MB L2 (no flush needed)"
                   if 16 * n // shards > 126_000_000 else "input fits in L2 (not flushed)")}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def set_mallopt():
    """mallopt(M_MMAP_THRESHOLD, 256 MB), as the reference's acceptance
    harness does before timing (tests/acceptance.cpp:376)."""
    try:
        libc = ctypes.CDLL("libc.so.6")
        return bool(libc.mallopt(-3, 256 << 20))  # M_MMAP_THRESHOLD = -3
    except OSError:
        return False


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()


def golden_for(n, dist, seed, chunk_count):
    """The reference's own hull + counters for this input (tests/golden)."""
    gdir = os.path.join(ROOT, "tests", "golden")
    try:
        with open(os.path.join(gdir, "big.json")) as f:
            for g in json.load(f):
                if (g["n"], g["dist"], g["seed"], g["chunk_count"]) == (n, dist, seed, chunk_count):
                    return g
        with open(os.path.join(gdir, "big_1b.json")) as f:
            g = json.load(f)
            if (g["n"], g["dist"], g["seed"], g["chunk_count"]) == (n, dist, seed, chunk_count):
                return g
    except (OSError, ValueError, KeyError):
        pass
    return None


def check_parity(hull, counts, n, dist, seed, chunk_count, sharded):
    """'bit-exact' when the hull bytes (and, on one GPU, all four counters)
    equal the reference's; raises on a mismatch; 'unpinned' without a golden."""
    g = golden_for(n, dist, seed, chunk_count)
    if g is None:
        return "unpinned (no golden for this input)"
    if sha(hull) != g["hull_sha"] or len(hull) != g["hull_n"]:
        raise SystemExit(f"PARITY FAILURE: hull differs from the reference ({len(hull)} vs "
                         f"{g['hull_n']} vertices)")
    if not sharded and list(counts) != list(g["counts"]):
        raise SystemExit(f"PARITY FAILURE: counters {list(counts)} != reference {g['counts']}")
    return ("bit-exact (hull sha256 == reference)" if sharded
            else "bit-exact (hull sha256 and n_input/n_after_round1/n_after_spa/n_hull == reference)")


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.p = None
        self.out = ""

    def __enter__(self):
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.2)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        if self.p:
            time.sleep(0.1)
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


# Per-launch DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) of the
# pipeline's kernels from the committed ncu --set full captures of this
# workload (profiles/); None when absent.
TRAFFIC_FILE = os.path.join(ROOT, "profiles", "round2", "traffic.json")


def measured_traffic(kernel_key: str):
    try:
        with open(TRAFFIC_FILE) as f:
            return json.load(f).get(kernel_key)
    except Exception:
        return None


def ref_lib():
    """The reference (oracle/_ref) or, where it was not built, the C port."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from pyoracle import Oracle, RefLib
    if RefLib.available():
        return RefLib(), "reference"
    return Oracle(), "port"


def ref_step(lib, kind, pts, chunk_count, parallelism):
    if kind == "reference":
        return lib.convex_hull(pts, chunk_count, parallelism)[0]
    return lib.convex_hull(pts, chunk_count)


def cpu_baseline(pts: np.ndarray, chunk_count: int):
    """The reference CPU path (oracle/_ref) on this host, same input: median
    of 5 after one warm-up at parallelism = 0 (all host threads), and at
    parallelism = 1 (median of 3), generation excluded."""
    lib, kind = ref_lib()
    mall = set_mallopt()
    cores = os.cpu_count() or 1

    def timed(par, reps):
        ref_step(lib, kind, pts, chunk_count, par)  # warm-up (page faults, allocator)
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            ref_step(lib, kind, pts, chunk_count, par)
            ts.append(time.perf_counter() - t0)
        return statistics.median(ts)

    t_all = timed(0, 5)
    t_one = timed(1, 3)
    n = len(pts)
    return {"value": n / t_all / 1e6, "unit": UNIT, "cores": cores if kind == "reference" else 1,
            "kind": kind, "cpu_model": cpu_model(), "nproc": cores,
            "sample": f"the same {n} points, convex_hull chunk_count={chunk_count}, "
                      f"parallelism=0 (all {cores} host threads), median of 5 after 1 warm-up; "
                      f"mallopt(M_MMAP_THRESHOLD, 256 MB) {'applied' if mall else 'unavailable'}; "
                      f"generation excluded",
            "value_1thread": n / t_one / 1e6, "ms_all_cores": t_all * 1e3,
            "ms_1thread": t_one * 1e3}


def run_reference(args, rank, world):
    """--impl reference: the reference's own CPU implementation of the path
    (oracle/_ref, the unmodified sources) on this host's cores. Imports
    nothing from the product: the input comes from the reference's own
    generate()."""
    if rank != 0:
        return
    cfg = workload(args, world)
    n = cfg["n_points"]
    lib, kind = ref_lib()
    mall = set_mallopt()
    cores = os.cpu_count() or 1
    # a bounded sample of configs[4]: its first REF_SAMPLE_SHARDED points
    # (uniform_square draws two values per point in order, so the prefix of
    # the 1B set is generate(m)); configs[1] runs whole
    m = min(n, REF_SAMPLE_SHARDED) if (world > 1 or args.sharded) else n
    pts = lib.generate(args.dist, m, args.seed)
    for _ in range(args.warmup):
        ref_step(lib, kind, pts, args.chunk_count, 0)
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        ref_step(lib, kind, pts, args.chunk_count, 0)
        ts.append(time.perf_counter() - t0)
    dt = sum(ts) / len(ts)
    v = m / dt / 1e6
    sample = (f"{m} points per step" + (f" (the first {m} of the {n}-point set)" if m < n else "")
              + f", convex_hull chunk_count={args.chunk_count}, parallelism=0 (all {cores} host "
              f"threads), mean of {args.steps} steps after {args.warmup} warm-up; "
              f"mallopt(M_MMAP_THRESHOLD, 256 MB) {'applied' if mall else 'unavailable'}")
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "strong" if (world > 1 or args.sharded) else "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (the reference's generate())", "impl": "reference",
            "config": cfg,
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores if kind == "reference" else 1,
                             "kind": kind, "cpu_model": cpu_model(), "nproc": cores,
                             "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def capi_lib():
    """libchainhull.so (the C++ drop-in) through its C entry
    (include/chainhull_capi.h)."""
    import paper_1508_05488_b200 as P
    P.load_library()  # libchgpu.so first (libchainhull.so's dependency)
    L = ctypes.CDLL(os.path.join(ROOT, "paper_1508_05488_b200", "libchainhull.so"))
    sz = ctypes.c_size_t
    L.chainhull_capi_convex_hull.argtypes = [ctypes.c_void_p, sz, sz, sz, ctypes.c_int,
                                             ctypes.c_void_p, sz, ctypes.POINTER(sz),
                                             ctypes.POINTER(sz)]
    return L


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--dist", default="uniform_square")
    ap.add_argument("--npoints", dest="n", type=int, default=0, help="points in the whole set (default: the "
                    "BASELINE config for the GPU count)")
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--chunk-count", type=int, default=1024)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-pageable", action="store_true")
    ap.add_argument("--sharded", action="store_true",
                    help="run the N > 1 code path (NCCL exchanges, rank-0 merge) even at one rank")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="exchange backend for N > 1 (gloo: several ranks on one GPU, testing)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    sharded = world > 1 or args.sharded
    if sharded and "MASTER_ADDR" not in os.environ:  # --sharded without torchrun
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(29500 + os.getpid() % 2000),
                          RANK="0", WORLD_SIZE="1")

    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    import paper_1508_05488_b200 as P
    from paper_1508_05488_b200.sharded import GpuShardOps, sharded_convex_hull

    cfg = workload(args, world)
    n_total = cfg["n_points"]
    local = local % max(1, torch.cuda.device_count())  # gloo testing: ranks may share a GPU
    torch.cuda.set_device(local)
    if sharded:
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    ctx = P.Context(local)
    pcfg = P.PipelineConfig(chunk_count=args.chunk_count)

    # This rank's contiguous shard of the set, generated on the host
    # (bit-identical to the reference generator) straight into pinned memory,
    # then resident in HBM.
    begin = n_total * rank // world
    n = n_total * (rank + 1) // world - begin
    h_pin = torch.empty((n, 2), dtype=torch.float64, pin_memory=True)
    P.generate(args.dist, n_total, args.seed, begin=begin, count=n, out=h_pin.numpy())
    d_pts = h_pin.to(f"cuda:{local}")
    ctx.reserve(n)
    torch.cuda.synchronize()
    stream = torch.cuda.ExternalStream(ctx.stream)
    ops = GpuShardOps(ctx, d_pts, begin) if sharded else None

    def step_device():
        if not sharded:
            return ctx.convex_hull_device(d_pts.data_ptr(), n, pcfg, copy=False)
        return sharded_convex_hull(ops, args.chunk_count)

    def step_host():
        if not sharded:
            return ctx.convex_hull(h_pin.numpy(), pcfg, copy=False)
        # host-resident shard: copy it in on the library stream, then the
        # sharded step
        with torch.cuda.stream(stream):
            d_pts.copy_(h_pin, non_blocking=True)
        return sharded_convex_hull(ops, args.chunk_count)

    def timed(fn, steps):
        if sharded:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        outs = []
        e0.record(stream)
        for _ in range(steps):
            outs.append(fn())
        e1.record(stream)
        e1.synchronize()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        if sharded:
            t = torch.tensor([ms], dtype=torch.float64,
                             device=f"cuda:{local}" if args.backend == "nccl" else "cpu")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms, outs

    for _ in range(args.warmup):
        step_device()
    with ClockSampler(local) as clk:
        ms, outs = timed(step_device, args.steps)
        res = outs[-1]
        # parity of the measured configuration, outside the timed region
        if not sharded:
            r = res
            counts = [r.stats.n_input, r.stats.n_after_round1, r.stats.n_after_spa, r.stats.n_hull]
            parity = check_parity(r.hull.vertices, counts, n_total, args.dist, args.seed,
                                  args.chunk_count, sharded=False)
        elif rank == 0:
            parity = check_parity(res, [n_total, None, None, len(res)], n_total, args.dist,
                                  args.seed, args.chunk_count, sharded=True)
        for _ in range(2):
            step_host()
        ms_e2e, outs_e2e = timed(step_host, args.steps)
        res_e2e = outs_e2e[-1]
    clocks = clk.summary()

    value = n_total / (ms * 1e-3) / 1e6
    e2e_value = n_total / (ms_e2e * 1e-3) / 1e6
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong" if sharded else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference generator, bit-identical)", "config": cfg,
            "clocks": clocks}

    if rank == 0 and not sharded:
        r = res
        line["parity"] = parity
        hbm, src = peaks()
        # the discard stage (K1 + K2, one CUDA-event interval when K2 is
        # launched programmatically) from every timed step's StageStats
        disc_steps = [o.stats.t_extremes_ms + o.stats.t_classify_ms for o in outs]
        # per-kernel breakdown: three extra steps with per-kernel events on
        # (each event query costs host time, so the timed steps run without)
        ctx.set_stage_times(True)
        for _ in range(3):
            rd = step_device()
        h2d_ms = step_host().diag.times_ms["t_h2d_ms"]
        ctx.set_stage_times(False)
        d = rd.diag
        s1 = sum(d.region_counts[1:])
        t = dict(d.times_ms)
        t["t_k1_ms"] = statistics.median(disc_steps) if d.k1k2_overlapped else t["t_k1_ms"]
        # K2 writes each survivor as one 8-byte filter key (bin, segment
        # position, w >> 32) on the pre-filtered path, as a 16-byte (k, v)
        # record on the sort path
        surv_b = 8 if d.spa_path == 1 else 16
        disc_ms = t["t_k1_ms"] + t["t_k2_ms"]
        if d.k1k2_overlapped:
            # K2 launched programmatically behind K1 (its CTAs start while
            # K1's last block merges the quad): one CUDA-event interval for
            # the discard stage. Algorithmic bytes on SURVEY §8(d)'s basis
            # (K1 16 B/pt; K2 16 B/pt + 16 B/survivor); K2 actually writes
            # surv_b B per survivor (bytes_moved).
            kernels = {
                "k1k2_discard": {"ms": t["t_k1_ms"], "bytes": 32 * n + 16 * s1,
                                 "bytes_moved": 32 * n + surv_b * s1,
                                 "basis": "SURVEY 8(d): K1 16 B/pt read + K2 16 B/pt read + 16 B/"
                                          f"survivor write (moved: {surv_b} B/survivor); "
                                          "k_extremes_partial + k_classify_survivors, "
                                          "programmatically overlapped"},
            }
        else:
            kernels = {
                "k1_extremes": {"ms": t["t_k1_ms"], "bytes": 16 * n, "basis": "16 B/pt read"},
                ("k2_classify_survivors" if d.spa_path == 1 else "k2_classify_compact"):
                    {"ms": t["t_k2_ms"], "bytes": 16 * n + surv_b * s1,
                     "basis": f"16 B/pt read + {surv_b} B/survivor write"},
            }
        if d.spa_path == 1:
            nc = d.n_candidates
            kernels.update({
                "k3_bin_scan": {"ms": t["t_binscan_ms"], "bytes": 24 * 4 * (1 << d.filter_log2nb),
                                "basis": "12 B/bin read + 12 B/bin write"},
                "k3_filter": {"ms": t["t_filter_ms"], "bytes": 8 * s1 + 32 * nc,
                              "basis": "8 B/survivor key read + per candidate 16 B point read, "
                                       "16 B record write",
                              "candidates": nc},
                "k4_chunk_spa": {"ms": t["t_spa_kernel_ms"],
                                 "bytes": 16 * nc + 32 * sum(d.kept_counts),
                                 "basis": "k_spa_small + k_spa_finish: 16 B/candidate read "
                                          "+ 16 B/kept scratch + 16 B/kept point write",
                                 "of_which_finish_ms": t["t_binsort_ms"]},
            })
        else:
            pass_ms = t["t_passes_ms"] / max(d.sort_passes, 1)
            kept = sum(d.kept_counts)
            kernels.update({
                # (the bucket passes take their digit bases from the column
                # scans: no global histogram, this interval is the setup)
                "k3_setup": {"ms": t["t_hist_ms"]},
                "k3_radix_pass": {"ms": pass_ms, "launches": d.sort_passes, "bytes": 40 * s1,
                                  "basis": "per pass: k_upsweep 8 B/record read + k_colscan + "
                                           "k_onesweep 16 B/record read + 16 B/record write"},
                "k3_ties": {"ms": t["t_ties_ms"]},
                "k4_spa": {"ms": t["t_spa_kernel_ms"], "bytes": 8 * s1 + 24 * kept,
                           "basis": "k_spa_tile: 8 B/record read (v) + per kept record 8 B read "
                                    "(k) + 16 B point write"},
            })
        for kv in kernels.values():
            if kv.get("bytes") and kv.get("ms"):
                kv["gbs"] = kv["bytes"] / (kv["ms"] * 1e-3) / 1e9
        kernels["d2h_chains_ms"] = t["t_d2h_ms"]
        kernels["host_melkman_ms"] = t["t_host_ms"]
        kernels["note"] = ("k1k2_discard: median over the timed steps (StageStats); the other stages "
                           "from 3 extra steps with per-kernel events on")
        dom_name, dom = max(((k, v) for k, v in kernels.items()
                             if isinstance(v, dict) and v.get("gbs")), key=lambda kv: kv[1]["ms"])
        # SURVEY §8(d) basis of the discard kernels: 32 n + 16 s1
        disc_bytes = 32 * n + 16 * s1
        disc_bytes_written = 32 * n + surv_b * s1
        line["roofline"] = {
            "bound": "hbm", "kernel": dom_name,
            "achieved": dom["gbs"], "peak": hbm, "unit": "GB/s",
            "peak_source": src, "frac": dom["gbs"] / hbm,
            "traffic": measured_traffic(dom_name),
            "algorithmic_bytes": f"{dom.get('basis', 'bytes moved')}: {dom['bytes']} B per launch",
            "discard_kernels": {
                "kernels": "k_extremes_partial (+ last-block merge), k_classify_survivors"
                           + (" (programmatically overlapped)" if d.k1k2_overlapped else ""),
                "basis": "SURVEY 8(d): 32 B/pt + 16 B/survivor",
                "bytes": disc_bytes, "ms": disc_ms,
                "achieved": disc_bytes / (disc_ms * 1e-3) / 1e9,
                "frac": disc_bytes / (disc_ms * 1e-3) / 1e9 / hbm,
                "bytes_moved": disc_bytes_written,
                "frac_bytes_moved": disc_bytes_written / (disc_ms * 1e-3) / 1e9 / hbm},
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
        e2e = {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": n * 16,
               "d2h_bytes_per_step": d2h, "ms_per_step": ms_e2e,
               "h2d_ms": h2d_ms,
               "source": "pinned host memory through the C ABI (chgpu_hull)"}
        if not args.no_pageable:
            # the C++ drop-in chainhull::convex_hull on pageable memory (a
            # std::vector's), timed on the host clock (synchronous API)
            L = capi_lib()
            h_page = np.array(h_pin.numpy(), copy=True)  # pageable
            nh = ctypes.c_size_t()
            cnt = (ctypes.c_size_t * 4)()

            def page_step():
                st = L.chainhull_capi_convex_hull(h_page.ctypes.data, n, args.chunk_count, 0, 1,
                                                  None, 0, ctypes.byref(nh), cnt)
                if st:
                    raise SystemExit(f"chainhull_capi_convex_hull failed ({st})")
            for _ in range(2):
                page_step()
            t0 = time.perf_counter()
            for _ in range(args.steps):
                page_step()
            ms_page = (time.perf_counter() - t0) * 1e3 / args.steps
            if list(cnt) != [r.stats.n_input, r.stats.n_after_round1, r.stats.n_after_spa,
                             r.stats.n_hull]:
                raise SystemExit("PARITY FAILURE: C++ drop-in counters differ")
            e2e["pageable"] = {"value": n / (ms_page * 1e-3) / 1e6, "unit": UNIT,
                               "ms_per_step": ms_page, "h2d_bytes_per_step": n * 16,
                               "d2h_bytes_per_step": d2h,
                               "source": "pageable host memory through the C++ drop-in "
                                         "chainhull::convex_hull (libchainhull.so), host clock"}
        line["e2e"] = e2e
        if not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(h_pin.numpy(), args.chunk_count)
    elif rank == 0:
        line["parity"] = parity
        line["e2e"] = {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": n_total * 16,
                       "d2h_bytes_per_step": 16 * len(res_e2e), "ms_per_step": ms_e2e,
                       "source": "each rank's shard from pinned host memory, copied in inside "
                                 "the timed region, then the sharded step"}
        line["hull_vertices"] = int(len(res)) if res is not None else None
    if rank == 0:
        print(json.dumps(line), flush=True)
    if sharded:
        dist.barrier()
        dist.destroy_process_group()
    # torch's tensors (and the pinned-memory events its copies recorded on the
    # library stream) go before the context that owns that stream
    torch.cuda.synchronize()
    del ops, d_pts, h_pin, stream
    import gc
    gc.collect()
    ctx.close()


if __name__ == "__main__":
    main()
