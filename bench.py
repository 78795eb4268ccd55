#!/usr/bin/env python
"""Benchmark: all-points exact KNN self-join (HybridKNN-Join hot path) on B200.

Metric (BASELINE.json): KNN self-join points/sec, K=32, on the metric's own config
C5 (BASELINE.json configs[4]: 100M uniform 4-D points, K=32, the 1/2/4/8-GPU scaling
run; synthetic, seed 1). --config C2/NS/... runs the other shapes.
One step = one full run_hybrid pass (variance reorder -> eps_mean -> distance
histogram -> grid build -> split -> fused range-join + top-K -> exact fallback)
over the whole dataset.

  value : device-resident points/s (dataset already in HBM; results left in HBM)
  e2e   : the same through the public C ABI with host buffers: pinned H2D of the
          dataset + knnj_run + D2H of ids/dist, every step
  --impl reference : the reference's own CPU implementation (oracle/_ref, the
          unmodified library built from /root/reference) on a bounded query sample.

Launch: python bench.py [--gpus N --steps K --warmup W]; N>1 under torchrun
(queries sharded by contiguous cell ranges, dataset + grid replicated; the only
exchange is an all-reduce of the 100 histogram counters).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "KNN self-join points/sec (end-to-end, K=32) at 1/2/4/8 B200 vs CPU ref"
PHASES = ("ms_total", "ms_reorder", "ms_eps_mean", "ms_histogram", "ms_grid", "ms_split", "ms_join",
          "ms_fallback", "ms_join_kernel", "ms_hist_kernel", "ms_join_build", "ms_download")
UNIT = "points/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C5")
    ap.add_argument("--size", type=int, default=0, help="override |D| (testing only)")
    ap.add_argument("--cpu-sample", type=int, default=0, help="reference query sample per step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[1]))
                mx = float(r[2])
                for i, nm in enumerate(names):
                    if r[4 + i].lower().startswith("active"):
                        reasons.add(nm)
            except (ValueError, IndexError):
                pass
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def load_peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


def profile_traffic(config: str):
    """dram bytes per launch of the join kernel from the committed ncu --set full capture
    of this workload (profiles/join_traffic.json, keyed by config), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "join_traffic.json")) as f:
            d = json.load(f)
    except (OSError, ValueError):
        return None
    e = d.get(config)
    return e.get("dram_bytes_per_launch") if isinstance(e, dict) else None


# ---------------------------------------------------------------------------- reference arm
def calibrated_sample(ref, h, N, k, cores, seconds, seed):
    """Query-sample size that keeps the reference's kd-tree queries busy for about
    `seconds` on `cores` threads (a 20k-query probe sets the rate)."""
    rng = np.random.default_rng(seed + 99)
    probe = np.sort(rng.choice(N, min(N, 20000), replace=False)).astype(np.uint32)
    _, _, secs = ref.kd_query(h, probe, k, cores)
    rate = probe.size / max(secs, 1e-6)
    return int(min(N, max(20000, rate * seconds)))


def cpu_reference(X, k, sample, seed=1, seconds=15.0):
    """The reference's RefImpl (SparseOnly: reorder + kd-tree) on a query sample
    against the FULL dataset, all host threads; the sample is sized to ~`seconds` of
    query time unless given. Returns (points/s, cores, detail)."""
    from oracle.oracle import Ref, ref_available
    if not ref_available():
        return None
    ref = Ref()
    h, t_reorder, t_build = ref.kd_create(X, min(6, X.shape[1]))
    cores = ref.hardware_concurrency()
    if not sample:
        sample = calibrated_sample(ref, h, X.shape[0], k, cores, seconds, seed)
    rng = np.random.default_rng(seed)
    q = np.sort(rng.choice(X.shape[0], sample, replace=False)).astype(np.uint32)
    _, _, secs = ref.kd_query(h, q, k, cores)
    return dict(handle=h, ref=ref, rate=sample / secs, secs=secs, cores=cores,
                t_reorder=t_reorder, t_build=t_build, q=q)


def cpu_hybrid_reduced(cfgd, size=None):
    """The reference's Hybrid mode (the paper's algorithm, run_hybrid with every phase)
    at a reduced |D| of the same distribution: its eps histogram is quadratic in |D|, so
    the full size is out of reach on the host. points/s over
    measured_total and over the call's wall time, all host threads."""
    from oracle.oracle import Ref, ref_available
    from paper_1810_04758_b200.synthetic import generate
    if not ref_available():
        return None
    size = size or {"C1": cfgd["size"], "C3": 100_000, "C4": 400_000}.get(cfgd["key"], 500_000)
    Xs = generate(cfgd["spec"], size, cfgd["dims"], seed=1)
    ref = Ref()
    t = time.perf_counter()
    o = ref.run(Xs, k=cfgd["k"], mode="hybrid", seed=1, workers=0, buffer_size=100_000_000)
    wall = time.perf_counter() - t
    return {"points": size, "value": size / o["measured_total"], "unit": UNIT,
            "measured_total_s": o["measured_total"], "wall_s": wall,
            "cores": ref.hardware_concurrency(),
            "note": f"reference Hybrid (run_hybrid) on {size} points of the same distribution; "
                    f"value = points / measured_total (reorder + eps + split + "
                    f"max(dense, sparse) + reassign + merge, orchestrator.cpp:245-248)"}


def run_reference(args, cfgd, X):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle.oracle import Ref, ref_available
    if not ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return
    k = cfgd["k"]
    ref = Ref()
    h, t_reorder, t_build = ref.kd_create(X, min(6, X.shape[1]))
    cores = ref.hardware_concurrency()
    # each step a bounded sample: ~3 s of kd-tree queries on all host threads
    sample = args.cpu_sample or calibrated_sample(ref, h, X.shape[0], k, cores, 3.0, 1234)
    rng = np.random.default_rng(1234)
    times = []
    for step in range(args.warmup + args.steps):
        q = np.sort(rng.choice(X.shape[0], sample, replace=False)).astype(np.uint32)
        _, _, secs = ref.kd_query(h, q, k, cores)
        if step >= args.warmup:
            times.append(secs)
    ref.kd_destroy(h)
    per_step = statistics.mean(times)
    value = sample / per_step
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_step * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": cfgd["name"], "points": X.shape[0], "dims": X.shape[1], "k": k,
                   "distribution": cfgd["spec"], "sample_queries_per_step": sample},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": f"{sample} seeded random queries per step against all "
                                   f"{X.shape[0]} points; reference SparseOnly/RefImpl (kd-tree, "
                                   f"run_sparse_knn) on {cores} threads; kd build "
                                   f"{t_build:.1f}s and reorder {t_reorder:.1f}s excluded like the "
                                   f"reference's measured_total"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


# ---------------------------------------------------------------------------- our arm
def run_ours(args, cfgd, X):
    import torch
    import torch.distributed as dist

    from paper_1810_04758_b200 import Engine, RunConfig
    rank, world, local = dist_env()
    # one process per GPU; KNNJ_DIST_BACKEND=gloo runs all ranks on the visible GPUs
    # round-robin (a multi-rank smoke of the sharded path on a 1-GPU box)
    backend = os.environ.get("KNNJ_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    N, n = X.shape
    k = cfgd["k"]
    eng = Engine(local)
    print(f"[bench] rank {rank}/{world} on cuda:{local} backend={backend if world > 1 else '-'}",
          file=sys.stderr)
    stream = torch.cuda.ExternalStream(eng.lib.knnj_stream(eng.h), device=torch.device("cuda", local))
    lib = eng.lib

    # pinned host buffers for the e2e leg
    nbytes_in = N * n * 8
    p_in = lib.knnj_alloc_pinned(nbytes_in)
    Xp = np.ctypeslib.as_array((np.ctypeslib.ctypes.c_double * (N * n)).from_address(p_in)).reshape(N, n)
    Xp[:] = X
    p_ids = lib.knnj_alloc_pinned(N * k * 4)
    p_dist = lib.knnj_alloc_pinned(N * k * 8)
    p_prov = lib.knnj_alloc_pinned(N)

    cfg = RunConfig(k=k, mode="hybrid", seed=1)
    eng.set_points((p_in, N, n))
    shard = None
    if world > 1:
        from paper_1810_04758_b200.distributed import torch_allreduce
        shard = (rank, world, torch_allreduce())

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(fn, steps):
        infos = []
        barrier()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(steps):
            infos.append(fn())
        ev1.record(stream)
        ev1.synchronize()
        barrier()
        ms = ev0.elapsed_time(ev1) / steps
        if world > 1:
            t = torch.tensor([ms], device="cuda" if backend == "nccl" else "cpu")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms, infos

    def step_device():
        r = eng.run(cfg, out=(0, 0, 0), want_hist=False, shard=shard)
        return r.info

    def step_e2e():
        eng.set_points((p_in, N, n))
        r = eng.run(cfg, out=(p_ids, p_dist, p_prov), want_hist=False, shard=shard)
        return r.info

    for _ in range(args.warmup):
        step_device()
    with ClockSampler(local) as clk:
        ms, infos = timed(step_device, args.steps)
    for _ in range(1):
        step_e2e()
    ms_e2e, infos_e2e = timed(step_e2e, args.steps)

    # Roofline of the dominant kernel (the fused join), per launch, as SURVEY.md §8(d)
    # defines the work: 3n flops (one sub + one FMA per dimension) per candidate pair of
    # the reference's 3^m walk (its candidates_examined counter, counted exactly by the
    # pass build over every level-0 row, before the box filter). Screens, rechecks and the
    # FP16 hi/lo split are not credited. The denominator is the pipe the kernel runs on:
    # the measured dense bf16 tensor peak (MEASURED_PEAKS.json) for the tcgen05 screen, the
    # FFMA peak measured live on this GPU for the SIMT kernel.
    info = infos[-1]
    join_ms = statistics.mean(i["ms_join_kernel"] for i in infos)
    hist_ms = statistics.mean(i["ms_hist_kernel"] for i in infos)
    cand = info["join_candidate_pairs"]   # this rank's level-0 join pairs (dense + sparse rows)
    screened = info["join_screened_pairs"]
    owned = [i["n_owned"] for i in infos_e2e]
    d2h = int(owned[-1]) * (k * 12 + 1 + 4 * (world > 1))
    flops = 3.0 * n * cand
    peak_c = np.ctypeslib.ctypes.c_double()
    eng._check(lib.knnj_fp32_peak(eng.h, np.ctypeslib.ctypes.byref(peak_c)))
    fp32_peak = peak_c.value
    peaks = load_peaks()
    if info["join_tensor_cores"]:
        peak = peaks.get("bf16_tflops", 1590.0)
        peak_src = ("MEASURED_PEAKS.json bf16_tflops (dense, burst; fp16 runs at the bf16 rate)"
                    if "bf16_tflops" in peaks else "B200_PROFILING.md fallback 1.59 PFLOP/s")
        bound = "tensor"
    else:
        peak = fp32_peak
        peak_src = "FFMA microbenchmark measured live on this GPU (no FP32 figure in MEASURED_PEAKS.json)"
        bound = "fp32"
    achieved = flops / (join_ms * 1e-3) / 1e12
    hist_pairs = info["hist_query_count"] * (N - 1)
    # whole-run check: t_ideal = max(F / P_fp32, B / BW_hbm) with
    # F = 3n (histogram pairs + join pairs + eps_mean pairs), B = the algorithmic bytes.
    # Above 1 means the run skips work the formula counts (capped histogram, box filter,
    # tensor-core screen): a work-avoidance ratio, not a utilisation.
    pairs_mean = min(10 * N, 1_000_000)
    F_run = 3.0 * n * (hist_pairs + cand + pairs_mean)
    B_run = N * n * 4 + N * 8 + info["grid_cells"] * 24 + N * k * 12
    bw = peaks.get("hbm_gbs", 6545.0) * 1e9
    t_ideal = max(F_run / (fp32_peak * 1e12), B_run / bw)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        c = cpu_reference(X, k, args.cpu_sample)
        if c is not None:
            c["ref"].kd_destroy(c["handle"])
            cpu = {"value": c["rate"], "unit": UNIT, "cores": c["cores"], "kind": "reference",
                   "sample": f"{len(c['q'])} seeded random queries against all {N} points, "
                             f"reference SparseOnly/RefImpl kd-tree (the faster reference CPU "
                             f"mode), {c['secs']:.2f}s of queries on {c['cores']} threads; kd build "
                             f"{c['t_build']:.1f}s and reorder {c['t_reorder']:.1f}s excluded like the "
                             f"reference's measured_total"}
            hyb = cpu_hybrid_reduced(cfgd)
            if hyb is not None:
                cpu["hybrid_reduced"] = hyb
    if rank == 0:
        line = {
            "metric": METRIC, "value": N / (ms * 1e-3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": cfgd["name"], "points": N, "dims": n, "k": k,
                       "distribution": cfgd["spec"], "seed": 1,
                       "parallelism": f"cell-range query shards x{world}" if world > 1 else "1 GPU",
                       "l2": "inputs (%.0f MB FP64) exceed the 126 MB L2" % (N * n * 8 / 1e6),
                       "eps_used": info["eps_used"], "grid_cells": info["grid_cells"],
                       "candidates_per_query": info["candidates_examined"] / max(1, info["q_gpu"]),
                       "hist_bins_counted": info["hist_bins_counted"]},
            "e2e": {"value": N / (ms_e2e * 1e-3), "unit": UNIT, "h2d_bytes_per_step": N * n * 8,
                    "d2h_bytes_per_step": d2h, "ms_per_step": ms_e2e,
                    "path": "knnj_set_points (pinned H2D) + knnj_run%s + D2H of ids/dist/prov" %
                            ("_shard" if world > 1 else "")},
            "roofline": {"bound": bound,
                         "kernel": "k_tc<JOIN> (tcgen05 fused range-join + screened top-K)"
                                   if bound == "tensor" else "k_join (SIMT fused range-join + top-K)",
                         "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": profile_traffic(cfgd["key"]),
                         "peak_source": peak_src,
                         "algorithmic_flops_per_launch": flops,
                         "flops_definition": "SURVEY.md 8(d): 3n flops per candidate pair of the "
                                             "reference 3^m walk (candidates_examined over all "
                                             "level-0 rows, before the box filter)",
                         "kernel_ms": join_ms, "candidate_pairs": cand,
                         "screened_pairs": screened,
                         "fp32_peak_measured": fp32_peak},
            "run_roofline": {"F_flops": F_run, "B_bytes": B_run, "t_ideal_s": t_ideal,
                             "t_measured_s": ms * 1e-3,
                             "t_ideal_over_measured": t_ideal / (ms * 1e-3),
                             "definition": "SURVEY.md 8(d): F = 3n (N_hq (|D|-1) + sum C_q + "
                                           "P_mean) against the measured FFMA peak, B against "
                                           "MEASURED_PEAKS hbm_gbs; above 1 = work the run "
                                           "avoids (capped histogram, box filter, tensor screen)"},
            "phases_ms": {k2: statistics.mean(i[k2] for i in infos) for k2 in PHASES},
            "phases_ms_e2e": {k2: statistics.mean(i[k2] for i in infos_e2e) for k2 in PHASES},
            "kth_bound": {"bound2": info["kth_bound2"], "rows_retried": info["bound_retried"]},
            "hist_pairs_per_s": hist_pairs / (hist_ms * 1e-3) if hist_ms > 0 else None,
            "gpu_launches": int(info["kernel_launches"]),
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line))
    for p in (p_in, p_ids, p_dist, p_prov):
        lib.knnj_free_pinned(p)
    eng.close()
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    from paper_1810_04758_b200.synthetic import CONFIGS, generate
    cfgd = dict(CONFIGS[args.config])
    cfgd["key"] = args.config
    cfgd["name"] = f"{args.config}: " + {
        "C1": "synthetic uniform 2-D, 100k points, K=5",
        "C2": "SuSy-shaped synthetic 18-D, 5M points, K=32, clustered (Gaussian mixture)",
        "C3": "Songs-shaped synthetic 90-D, 500k points, K=16 (mixture)",
        "C4": "exponentially-distributed skewed 6-D, 20M points, K=64",
        "C5": "uniform 4-D, 100M points, K=32, cell-range sharded across 1/2/4/8 B200 "
              "(BASELINE.json configs[4], the metric's scaling run)",
        "NS": "north-star: SuSy-shaped clustered 18-D, 10M points, K=32",
    }.get(args.config, args.config)
    if args.size:
        cfgd["size"] = args.size
    X = generate(cfgd["spec"], cfgd["size"], cfgd["dims"], seed=1)
    if args.impl == "reference":
        run_reference(args, cfgd, X)
    else:
        run_ours(args, cfgd, X)


if __name__ == "__main__":
    main()
