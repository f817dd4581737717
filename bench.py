"""Benchmark: slimLS iterations/s on the BASELINE headline workload.

Workload (BASELINE.json configs[1], the config the metric is quoted on):
2D parallel-beam tomography, 256x256 image (n = 65,536), 180 views over
[0, pi) x 362 rays, Siddon CSR fp64, 10-ellipse phantom, 1% noise, one
block = one view (ell = 362), r = 10, lambda = 1e-3 (alpha = 1000),
random_cyclic sampling.  A "step" is one slimLS iteration.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

* warm-up: max(W, r + 1) untimed steps so the memory window is full when
  the timed region starts (the same slim_run call continues into it);
* value: K / device time of steps W'+1 .. W'+K (CUDA events on the
  x-chain stream, all streams joined at the end), operator resident in
  HBM; per-iteration working set (Gram ring 254 MB + two factor buffers
  + CSR 180 MB) exceeds the 126 MB L2, so no flush is inserted;
* e2e: the public ``run()`` on a fresh host-resident operator, timed by
  wall clock including the operator upload and the history / x download;
* cpu_baseline / --impl reference: the oracle port of the reference's
  algorithm (dense fetch, vstack, full Gram, LAPACK Cholesky) on the
  host cores, a bounded sample (window fill + 3 steady-state steps).

N > 1 (torchrun): replicas only -- every rank runs an independent
replica (sampler seed base + rank, like the reference harness), timing
is the max over ranks, value = all ranks' steps / that time.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "slim iterations/s and rows/s at 1/2/4/8 B200; HBM GB/s vs roofline"
CFG = dict(grid=256, n_views=180, rays=362, r=10, alpha=1000.0, seed=2, sampler_seed=7962)


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except OSError:
        return {}


# FP64 DMMA/DFMA peak is not in MEASURED_PEAKS.json; measured on this pool
# by tools/microbench/fp64_rates.cu (profiles/fp64_peak_r01.txt)
FP64_PEAK_TFLOPS = 37.1


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("gloo")
        return world, rank, local, dist
    return 1, 0, 0, None


def _max_over_ranks(dist, v: float) -> float:
    if dist is None:
        return v
    import torch

    t = torch.tensor([v], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _barrier(dist):
    if dist is not None:
        dist.barrier()


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    QUERY = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.QUERY}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.5)  # let nvidia-smi attach before the timed region starts
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, flag in zip(names, parts[4:8]):
                if flag.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def build_problem(threads=None):
    from paper_1912_07962_b200 import problems

    return problems.tomo2d(grid=CFG["grid"], n_views=CFG["n_views"], rays=CFG["rays"],
                           seed=CFG["seed"], threads=threads)


def cpu_sample(prob, r, alpha, seed, steady=3):
    """Oracle port on the host: window fill + ``steady`` full-window steps."""
    from oracle import slimls_oracle as orc

    op = prob.op
    K = r + 1 + steady
    idx = orc.sampler_indices("random_cyclic", op.n_blocks, seed, K)
    fetch = orc.csr_fetch([op.csr_block(i) for i in range(1, op.n_blocks + 1)], prob.b)
    t0 = time.perf_counter()
    traj = orc.run_slimls(fetch, op.n_blocks, op.n_cols, idx, np.full(K, alpha), r=r)
    total = time.perf_counter() - t0
    per_step = float(np.mean(traj.wall_times[-steady:]))
    return {"value": 1.0 / per_step, "unit": "it/s", "cores": os.cpu_count(), "kind": "port",
            "sample": f"oracle restatement of the reference (dense fetch + vstack + full Gram + "
                      f"LAPACK Cholesky), {K} steps ({r + 1}-step window fill, then {steady} "
                      f"full-window steps timed), {total:.1f} s total, "
                      f"OpenBLAS threads = all {os.cpu_count()} host cores"}


def run_reference(args, world, rank, dist):
    if rank != 0:
        return
    prob = build_problem()
    cb = cpu_sample(prob, CFG["r"], CFG["alpha"], CFG["sampler_seed"])
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": "it/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 / cb["value"], "higher_is_better": True,
            "scaling": "replicas", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": _config_dict(world), "rows_per_s": cb["value"] * CFG["rays"],
            "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": "it/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _config_dict(world):
    return {"workload": "configs[1]: 2D parallel-beam tomography 256x256, 180 views x 362 rays, "
                        "Siddon CSR fp64, r=10, lambda=1e-3, random_cyclic",
            "n": CFG["grid"] ** 2, "m": CFG["n_views"] * CFG["rays"], "ell": CFG["rays"],
            "r": CFG["r"], "lambda": 1.0 / CFG["alpha"], "dual_system_N": (CFG["r"] + 1) * CFG["rays"],
            "parallelism": f"replicas{world}" if world > 1 else "single",
            "l2": "per-iteration working set > 126 MB L2 (no flush)"}


def run_ours(args, world, rank, local, dist):
    import paper_1912_07962_b200 as slim

    dev = local
    prob = build_problem()
    op, b, xt = prob.op, prob.b, prob.x_true
    r, alpha = CFG["r"], CFG["alpha"]
    seed = CFG["sampler_seed"] + rank
    D = int(os.environ.get("SLIM_BATCH", "8"))
    wprime = -(-max(args.warmup, r + 1) // D) * D  # whole factorization batches
    total = wprime + args.steps
    M = op.n_blocks
    # upload + kernel warm-up (untimed)
    slim.run("slimls", op, slim.Sampler("random_cyclic", M, seed), slim.Schedule("constant", alpha),
             epochs=(r + 2) / M, r=r, device=dev)
    timing = {"start_step": wprime + 1}
    _barrier(dist)
    with ClockSampler(dev) as clk:
        traj = slim.run("slimls", op, slim.Sampler("random_cyclic", M, seed),
                        slim.Schedule("constant", alpha), epochs=total / M, r=r,
                        references={"x_true": xt}, record_every=1, device=dev, timing=timing)
    _barrier(dist)
    assert traj.status == "ok" and len(traj.ks) == total + 1
    t_win = _max_over_ranks(dist, timing["window_ms"] / 1e3)
    value = world * args.steps / t_win
    # ---- roofline of the dominant kernel (tile Cholesky), per launch ----
    N = (r + 1) * CFG["rays"]
    per_launch = args.steps / max(1, timing["cholesky_count"])  # systems per batched launch
    flops_chol = per_launch * N ** 3 / 3.0
    chol_ms = timing["cholesky_ms"] / max(1, timing["cholesky_count"])
    achieved = flops_chol / (chol_ms * 1e-3) / 1e12
    agg = (N ** 3 / 3.0) * args.steps / (timing["window_ms"] * 1e-3) / 1e12
    traffic = None
    try:  # dram bytes per launch from the committed ncu --set full capture
        with open(os.path.join(ROOT, "profiles", "ncu_chol_r01.json")) as fh:
            prof = json.load(fh)
        if int(prof.get("systems_per_launch", 0)) == int(round(per_launch)):
            traffic = prof["dram_bytes_per_launch"]
    except (OSError, ValueError, KeyError):
        pass
    roofline = {"bound": "tensor", "achieved": achieved, "peak": FP64_PEAK_TFLOPS,
                "unit": "TFLOP/s", "frac": achieved / FP64_PEAK_TFLOPS, "traffic": traffic,
                "kernel": f"k_chol_tiles (fp64 DMMA tile-DAG Cholesky, {per_launch:g} systems "
                          f"of N=3982 interleaved per launch)",
                "algorithmic_per_launch": f"{per_launch:g} x N^3/3 = {flops_chol:.4g} flop",
                "peak_source": "FP64 DMMA peak measured on this pool (tools/microbench/fp64_rates.cu)",
                "aggregate_tflops_over_window": agg,
                "aggregate_frac": agg / FP64_PEAK_TFLOPS,
                "avg_launch_ms": chol_ms, "launches": timing["cholesky_count"]}
    # ---- e2e through the public API, host-resident fresh operator ----
    e2e = None
    if not args.quick:
        op2 = slim.SparseBlockOperator([op.csr_block(i) for i in range(1, M + 1)], b)
        h2d = sum(p[0].nbytes + p[1].nbytes + p[2].nbytes for p in op2._parts) + b.nbytes \
            + 2 * xt.nbytes + total * 16
        t0 = time.perf_counter()
        tr2 = slim.run("slimls", op2, slim.Sampler("random_cyclic", M, seed),
                       slim.Schedule("constant", alpha), epochs=total / M, r=r,
                       references={"x_true": xt}, record_every=1, device=dev)
        wall = time.perf_counter() - t0
        del op2
        wall = _max_over_ranks(dist, wall)
        d2h = (total + 1) * (5 + 1) * 8 + xt.nbytes
        e2e = {"value": world * total / wall, "unit": "it/s",
               "h2d_bytes_per_step": int(h2d / total), "d2h_bytes_per_step": int(d2h / total),
               "what": f"public run() on a fresh host operator: CSR upload + per-block CSC build + "
                       f"{total} steps + history/x download, wall clock"}
        assert tr2.status == "ok"
    if rank != 0:
        return
    cb = cpu_sample(prob, r, alpha, CFG["sampler_seed"]) if world == 1 and not args.quick else None
    line = {"metric": METRIC, "value": value, "unit": "it/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_win / args.steps,
            "higher_is_better": True, "scaling": "weak" if world > 1 else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": _config_dict(world), "rows_per_s": value * CFG["rays"],
            "roofline": roofline, "cpu_baseline": cb, "e2e": e2e,
            "gpu_launches": int(timing["launches"]), "clocks": clk.summary(),
            "kernel_ms_per_step": {
                "gram": timing["gram_ms"] / max(1, timing["gram_count"]),
                "cholesky": chol_ms,
                "x_chain": timing["x_chain_ms"] / max(1, timing["x_chain_count"])},
            "final_rel_err_x_true": float(traj.rel_errors["x_true"][-1])}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=96)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--quick", action="store_true",
                    help="skip the CPU baseline and the e2e leg (profiling runs)")
    args = ap.parse_args()
    world, rank, local, dist = _dist()
    if args.impl == "reference":
        run_reference(args, world, rank, dist)
    else:
        run_ours(args, world, rank, local, dist)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
