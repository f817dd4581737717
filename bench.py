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
import gc
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "slim iterations/s and rows/s at 1/2/4/8 B200; HBM GB/s vs roofline"

# BASELINE.json configs (1-based here); lambda = 1 / alpha
CONFIGS = {
    1: dict(workload="configs[0]: dense Gaussian LS 20,000 x 1,000 fp64, ell=100, r=5, "
                     "lambda=1e-2, random_cyclic", r=5, alpha=100.0, scheme="random_cyclic",
            dtype="f64"),
    2: dict(workload="configs[1]: 2D parallel-beam tomography 256x256, 180 views x 362 rays, "
                     "Siddon CSR fp64, r=10, lambda=1e-3, random_cyclic", r=10, alpha=1000.0,
            scheme="random_cyclic", dtype="f64"),
    3: dict(workload="configs[2]: 2D tomography 1024x1024, 720 views x 1448 rays, Siddon CSR "
                     "fp32 values / int32 indices, r=8, lambda=1e-3, random_cyclic", r=8,
            alpha=1000.0, scheme="random_cyclic", dtype="f32 values, f64 arithmetic"),
    4: dict(workload="configs[3]: 3D parallel-beam tomography 128^3, 180 directions x 128x128 "
                     "detector, 8 sub-blocks of 2048 rays per view, CSR fp32, r=5, lambda=1e-3, "
                     "random_cyclic", r=5, alpha=1000.0, scheme="random_cyclic",
            dtype="f32 values, f64 arithmetic"),
    5: dict(workload="configs[4]: streaming dense LS n=65,536, m=4,194,304, splitmix64 rows "
                     "generated in-kernel (fp32), ell=256, r=20, lambda=1e-2, single pass",
            r=20, alpha=100.0, scheme="cyclic", dtype="f32 values, f64 arithmetic"),
}
SAMPLER_SEED = 7962


def build_config(cfg_id, threads=None):
    """(op, b, x_true) of a BASELINE config at full size."""
    from paper_1912_07962_b200 import problems

    if cfg_id == 1:
        return problems.gaussian_dense()
    if cfg_id == 2:
        p = problems.tomo2d(grid=256, n_views=180, rays=362, seed=2, threads=threads)
    elif cfg_id == 3:
        p = problems.tomo2d(grid=1024, n_views=720, rays=1448, seed=3, dtype=np.float32,
                            threads=threads)
    elif cfg_id == 4:
        p = problems.tomo3d(grid=128, n_views=180, side=128, sub_rows=2048, seed=4,
                            threads=threads)
    else:
        return problems.generated_dense()
    return p.op, p.b, p.x_true


def batch_size(n_sys: int) -> int:
    """Systems per batched factorization (same rule as slim_create)."""
    env = os.environ.get("SLIM_BATCH")
    if env:
        return max(1, min(16, int(env)))
    return 8 if n_sys <= 2048 else (16 if n_sys <= 6144 else 4)


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except OSError:
        return {}


# FP64 DMMA/DFMA peak is not in MEASURED_PEAKS.json; measured on this pool
# by tools/microbench/fp64_rates.cu (profiles/fp64_peak_r01.txt)
FP64_PEAK_TFLOPS = 37.1
# int8 tcgen05 peak (kind::i8, M=128 N=256, smem operands) and the ceiling of
# the factorization's own MMA shape (M=128 N=64), measured on this pool by
# tools/microbench/i8_rates.cu (profiles/i8_peak_r01.txt)
I8_PEAK_TOPS = 4579.0
I8_N64_CEIL_TOPS = 3056.0


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


def oracle_fetch(op, b):
    """The oracle's fetch for the operator (reference arithmetic)."""
    from oracle import slimls_oracle as orc
    from paper_1912_07962_b200.linops import GeneratedBlockOperator, SparseBlockOperator

    if isinstance(op, GeneratedBlockOperator):
        return orc.gen_fetch(op.seed, op.n_cols, op.block_rows, b)
    if isinstance(op, SparseBlockOperator):
        return orc.csr_fetch([op.csr_block(i) for i in range(1, op.n_blocks + 1)], b)
    return orc.dense_fetch(op.matrix, b, op.block_rows)


def cpu_sample(cfg_id, op, b, r, alpha, scheme, seed, steady=3):
    """The reference algorithm (oracle port) on the host: the window is filled
    with r fetched blocks (untimed), then ``steady`` full-window steps are
    timed, each including its block fetch as in the reference loop."""
    from collections import deque

    from oracle import slimls_oracle as orc

    idx = orc.sampler_indices(scheme, op.n_blocks, seed, r + steady)
    n = op.n_cols
    if cfg_id in (3, 4):
        # dense fetch infeasible (12-34 GB per block): sparse dual-form restatement
        import scipy.sparse as sp

        mats = [sp.csr_matrix((d.astype(float), ix, ip), shape=shp)
                for ip, ix, d, shp in (op.csr_block(int(i)) for i in set(idx.tolist()))]
        lookup = dict(zip(sorted(set(idx.tolist())), mats))
        x = np.zeros(n)
        window = deque(maxlen=r + 1)
        for k in range(r):
            window.append(lookup[int(idx[k])])
        times = []
        ell = op.block_rows
        for k in range(r, r + steady):
            i = int(idx[k])
            t0 = time.perf_counter()
            a = lookup[i]
            window.append(a)
            res = a @ x - b[(i - 1) * ell:i * ell]
            mat = sp.vstack(list(window)).tocsr()
            g = (mat @ mat.T).toarray() * alpha
            g[np.diag_indices_from(g)] += 1.0
            y = np.zeros(mat.shape[0])
            y[-ell:] = res
            import scipy.linalg

            w = scipy.linalg.solve(g, y, assume_a="pos")
            x = x - alpha * (mat.T @ w)
            times.append(time.perf_counter() - t0)
        what = ("sparse dual-form restatement of the reference step (the reference's dense "
                "block fetch needs 12-34 GB per block here)")
    else:
        fetch = oracle_fetch(op, b)
        st = orc._State(x=np.zeros(n), window=deque(maxlen=r + 1), div_limit_sq=np.inf)
        for k in range(r):
            st.window.append((int(idx[k]), fetch(int(idx[k]))[0]))
        times = []
        for k in range(r, r + steady):
            i = int(idx[k])
            t0 = time.perf_counter()
            a, bb = fetch(i)
            orc.slimls_step(st, i, a, bb, alpha)
            times.append(time.perf_counter() - t0)
        what = ("oracle restatement of the reference step (block fetch, vstack, full Gram, "
                "LAPACK Cholesky solve)")
    per_step = float(np.mean(times))
    return {"value": 1.0 / per_step, "unit": "it/s", "cores": os.cpu_count(), "kind": "port",
            "sample": f"{what}; window prefilled with {r} blocks (untimed), {steady} full-window "
                      f"steps timed ({sum(times):.1f} s), BLAS threads = all {os.cpu_count()} "
                      f"host cores"}


def run_reference(args, world, rank, dist):
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    op, b, _ = build_config(args.config)
    cb = cpu_sample(args.config, op, b, cfg["r"], cfg["alpha"], cfg["scheme"], SAMPLER_SEED)
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": "it/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 / cb["value"], "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": _config_dict(args.config, op, world),
            "rows_per_s": cb["value"] * op.block_rows, "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": "it/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _config_dict(cfg_id, op, world, sharded=False, factor="replicated"):
    cfg = CONFIGS[cfg_id]
    return {"workload": cfg["workload"], "n": op.n_cols, "m": op.n_rows, "ell": op.block_rows,
            "r": cfg["r"], "lambda": 1.0 / cfg["alpha"],
            "dual_system_N": (cfg["r"] + 1) * op.block_rows,
            "parallelism": (f"columns{world}" + ("-rr" if factor == "round_robin" else "")
                            if sharded else f"replicas{world}") if world > 1 else "single",
            "l2": "per-iteration working set > 126 MB L2 (no flush)"}


def run_ours(args, world, rank, local, dist):
    import paper_1912_07962_b200 as slim

    dev = local
    cfg = CONFIGS[args.config]
    op, b, xt = build_config(args.config)
    r, alpha, scheme = cfg["r"], cfg["alpha"], cfg["scheme"]
    ell, M = op.block_rows, op.n_blocks
    seed = SAMPLER_SEED + rank
    N = (r + 1) * ell
    D = batch_size(N)
    wprime = -(-max(args.warmup, r + 1) // D) * D  # whole factorization batches
    total = wprime + args.steps
    if scheme == "cyclic" and total > M:
        raise SystemExit(f"config {args.config}: {total} steps exceed one pass ({M} blocks)")

    sharded = world > 1 and args.shard == "columns"
    if sharded:
        from paper_1912_07962_b200.parallel import NcclShard

        import torch

        torch.cuda.set_device(dev)
        shard = NcclShard.from_torch(op.n_cols, round_robin=args.factor == "round_robin")
        seed = SAMPLER_SEED  # one solve: every shard walks the same index trace
    else:
        shard = None

    def sampler():
        return slim.Sampler(scheme, M, seed)

    # upload + kernel warm-up (untimed).  The device-timed leg starts with the
    # whole operator in HBM (uploaded up front, no host streaming); the e2e
    # leg below measures the streamed default on a fresh operator.
    prev = os.environ.get("SLIM_HOST_STREAMING")
    os.environ["SLIM_HOST_STREAMING"] = "0"
    slim.run("slimls", op, sampler(), slim.Schedule("constant", alpha),
             epochs=min(r + 2, M) / M, r=r, device=dev, shard=shard)
    if prev is None:
        os.environ.pop("SLIM_HOST_STREAMING")
    else:
        os.environ["SLIM_HOST_STREAMING"] = prev
    timing = {"start_step": wprime + 1, "probe_reps": 0 if args.bare else 24}
    _barrier(dist)
    with ClockSampler(dev) as clk:
        traj = slim.run("slimls", op, sampler(), slim.Schedule("constant", alpha),
                        epochs=total / M, r=r, references={"x_true": xt}, record_every=1,
                        device=dev, timing=timing, shard=shard)
    _barrier(dist)
    assert traj.status == "ok" and len(traj.ks) == total + 1
    t_win = _max_over_ranks(dist, timing["window_ms"] / 1e3)
    # replicas: every rank solves its own problem; columns: all ranks one solve
    value = (1 if sharded else world) * args.steps / t_win
    # ---- roofline of the dominant kernel (batched tile Cholesky), per launch ----
    # systems per batched launch; the algorithmic flops are those of the tiles
    # the launches factor (a step recomputes only the tiles its new block
    # reaches), counted by the library per launch
    per_launch = args.steps / max(1, timing["cholesky_count"])
    flops_chol = timing["cholesky_flops"] / max(1, timing["cholesky_count"])
    chol_ms = timing["cholesky_ms"] / max(1, timing["cholesky_count"])
    achieved = flops_chol / (chol_ms * 1e-3) / 1e12
    agg = timing["cholesky_flops"] / (timing["window_ms"] * 1e-3) / 1e12
    traffic = None
    try:  # dram bytes per launch from the committed ncu --set full capture
        with open(os.path.join(ROOT, "profiles", f"ncu_chol_cfg{args.config}.json")) as fh:
            prof = json.load(fh)
        if int(prof.get("systems_per_launch", 0)) == int(round(per_launch)):
            traffic = prof["dram_bytes_per_launch"]
    except (OSError, ValueError, KeyError):
        pass
    i8ops = timing.get("cholesky_i8ops", 0.0) / max(1, timing["cholesky_count"])
    if i8ops > 0:
        # int8 tensor-core factorization: the tile updates are exact int32
        # digit-pair products (QD (QD + 1) / 2 per 64^3 update); POTRF/TRSM
        # stay fp64
        qd, dbits = timing["cholesky_digits"]
        pairs = qd * (qd + 1) // 2
        ach_i8 = i8ops / (chol_ms * 1e-3) / 1e12
        roofline = {"bound": "tensor", "achieved": ach_i8, "peak": I8_PEAK_TOPS,
                    "unit": "TOPS (int8)", "frac": ach_i8 / I8_PEAK_TOPS, "traffic": traffic,
                    "kernel": f"k_chol_i8 (tile-DAG Cholesky, updates on tcgen05 kind::i8 with "
                              f"TMEM accumulators, {per_launch:g} systems of N={N} per launch)",
                    "algorithmic_per_launch": f"{i8ops:.4g} int8 ops ({pairs} digit-pair products "
                                              f"({qd} digits: 7-bit lead, {dbits}-bit rest) x "
                                              f"2*64^3 per 64x64x64 tile update; the launch "
                                              f"factors {flops_chol:.4g} fp64-equivalent flop)",
                    "peak_source": "int8 tcgen05 peak measured on this pool, M=128 N=256 "
                                   "(tools/microbench/i8_rates.cu, profiles/i8_peak_r01.txt)",
                    "shape_ceiling_tops": I8_N64_CEIL_TOPS,
                    "frac_of_shape_ceiling": ach_i8 / I8_N64_CEIL_TOPS,
                    "fp64_equivalent_tflops": achieved,
                    "fp64_equivalent_frac_of_dmma_peak": achieved / FP64_PEAK_TFLOPS,
                    "aggregate_tflops_over_window": agg,
                    "avg_launch_ms": chol_ms, "launches": timing["cholesky_count"]}
    else:
        roofline = {"bound": "tensor", "achieved": achieved, "peak": FP64_PEAK_TFLOPS,
                    "unit": "TFLOP/s", "frac": achieved / FP64_PEAK_TFLOPS, "traffic": traffic,
                    "kernel": f"k_chol_tiles (fp64 DMMA tile-DAG Cholesky, {per_launch:g} systems "
                              f"of N={N} interleaved per launch)",
                    "algorithmic_per_launch": f"{flops_chol:.4g} flop (tiles factored, 2*64^3 per "
                                              f"tile update; from scratch a system is N^3/3 = "
                                              f"{N ** 3 / 3.0:.4g})",
                    "peak_source": "FP64 DMMA peak measured on this pool "
                                   "(tools/microbench/fp64_rates.cu, profiles/fp64_peak_r01.txt)",
                    "aggregate_tflops_over_window": agg,
                    "aggregate_frac": agg / FP64_PEAK_TFLOPS,
                    "avg_launch_ms": chol_ms, "launches": timing["cholesky_count"]}
    # ---- operator-streaming kernels alone (K1, K5, CSR K2), cold L2 ----
    hbm_peak = float(_peaks().get("hbm_gbs", 0.0)) or 7700.0
    streaming = {"peak_gbs": hbm_peak,
                 "peak_source": "MEASURED_PEAKS.json hbm_gbs" if _peaks().get("hbm_gbs")
                 else "B200_PROFILING.md fallback",
                 "how": "probe after the timed run: 24 launches, each on a different window of "
                        "resident blocks, L2 flushed (256 MB read) between launches, one CUDA "
                        "event pair per launch on the x-chain stream; bytes = operator bytes the "
                        "launch must read once + vectors read/written (algorithmic)"}
    for name, (us, nbytes) in timing.get("streaming", {}).items():
        gbs = nbytes / (us * 1e-6) / 1e9
        streaming[name] = {"us_per_launch": us, "bytes_per_launch": nbytes, "achieved_gbs": gbs,
                           "frac": gbs / hbm_peak}
    # ---- e2e through the public API, host-resident fresh operator ----
    e2e = None
    if not args.quick and not args.bare and not sharded:
        op2, b2, _ = (op, b, xt) if args.config == 5 else build_config(args.config)
        if args.config == 5:
            op2 = op.with_rhs(b)  # fresh operator object: no cached device state
        h2d = _operator_bytes(op2) + 2 * xt.nbytes + total * 16
        walls = []
        while True:  # short runs are repeated on fresh operators, median reported
            gc.collect()  # the previous operator's context is released here, untimed
            t0 = time.perf_counter()
            tr2 = slim.run("slimls", op2, sampler(), slim.Schedule("constant", alpha),
                           epochs=total / M, r=r, references={"x_true": xt}, record_every=1,
                           device=dev)
            walls.append(time.perf_counter() - t0)
            if len(walls) == 5 or sum(walls) > 2.0:
                break
            op2 = op2.with_rhs(op2.rhs)  # same arrays, no cached device state
        wall = float(np.median(walls))
        print("e2e walls (s): " + " ".join(f"{w:.4f}" for w in walls), file=sys.stderr)
        del op2
        wall = _max_over_ranks(dist, wall)
        d2h = (total + 1) * (5 + 1) * 8 + xt.nbytes
        e2e = {"value": world * total / wall, "unit": "it/s",
               "h2d_bytes_per_step": int(h2d / total), "d2h_bytes_per_step": int(d2h / total),
               "what": f"public run() on a fresh host operator: operator upload (streamed "
                       f"block by block in first-use order, + per-block CSC build for CSR) + "
                       f"{total} steps + history/x download, wall clock, median of "
                       f"{len(walls)} fresh operators"}
        assert tr2.status == "ok"
    # ---- device projector: tomography operators traced in HBM ----
    projector = None
    if args.config in (2, 3, 4) and not sharded and not args.bare:
        projector = _projector_leg(args, dev, b, xt, r, alpha, scheme, total, M, sampler)
    if rank != 0:
        return
    cb = None
    if world == 1 and not args.quick and not args.bare:
        cb = cpu_sample(args.config, op, b, r, alpha, scheme, SAMPLER_SEED)
    line = {"metric": METRIC, "value": value, "unit": "it/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_win / args.steps,
            "higher_is_better": True, "scaling": "strong" if sharded else "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": _config_dict(args.config, op, world, sharded, args.factor),
            "rows_per_s": value * ell, "roofline": roofline, "streaming": streaming,
            "cpu_baseline": cb, "e2e": e2e, "device_projector": projector,
            "gpu_launches": int(timing["launches"]), "clocks": clk.summary(),
            "kernel_ms_per_step": {
                "gram": timing["gram_ms"] / max(1, timing["gram_count"]),
                "cholesky": chol_ms,
                "x_chain": timing["x_chain_ms"] / max(1, timing["x_chain_count"])},
            "final_rel_err_x_true": float(traj.rel_errors["x_true"][-1])}
    print(json.dumps(line), flush=True)


def _projector_leg(args, dev, b, xt, r, alpha, scheme, total, M, sampler):
    """Device Siddon projector: trace time of the whole operator (count pass,
    scan, fill, per-block CSC) and e2e through the public API with the
    operator traced on the device inside the timed region (only b and the
    geometry cross PCIe)."""
    import torch

    import paper_1912_07962_b200 as slim
    from paper_1912_07962_b200 import problems, tomo

    geom, grid, dtype, ell, rmap = problems.projector_config(args.config)
    builds = []
    for _ in range(3):
        gc.collect()
        op = tomo.ProjectorOperator(geom, grid, dtype=dtype, block_rows=ell, ray_of_row=rmap)
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        dop = op.device_context(r, dev)
        torch.cuda.synchronize(dev)
        builds.append(time.perf_counter() - t0)
        nnz = dop.nnz()
        del dop, op
    vb = np.dtype(dtype).itemsize
    m = b.shape[0]
    csr_bytes = nnz * (4 + vb) + (m + 1) * 8
    t_build = float(np.median(builds))
    out = {"what": "slim_build_projector + slim_finalize_operator on a fresh context: count pass, "
                   "row-pointer scan, fill pass, per-block CSC; wall clock, median of 3",
           "nnz": nnz, "build_ms": 1e3 * t_build, "csr_bytes": csr_bytes,
           "csr_write_gbs": csr_bytes / t_build / 1e9,
           "rays_per_s": m / t_build}
    if args.quick:
        return out
    walls = []
    for _ in range(3):
        gc.collect()
        t0 = time.perf_counter()
        op = tomo.ProjectorOperator(geom, grid, dtype=dtype, block_rows=ell, ray_of_row=rmap,
                                    b=b)
        tr = slim.run("slimls", op, sampler(), slim.Schedule("constant", alpha),
                      epochs=total / M, r=r, references={"x_true": xt}, record_every=1,
                      device=dev)
        walls.append(time.perf_counter() - t0)
        assert tr.status == "ok"
        del op
    wall = float(np.median(walls))
    out["e2e"] = {"value": total / wall, "unit": "it/s",
                  "h2d_bytes_per_step": int((b.nbytes + 2 * xt.nbytes + total * 16) / total),
                  "d2h_bytes_per_step": int(((total + 1) * 6 * 8 + xt.nbytes) / total),
                  "what": f"public run() on a fresh ProjectorOperator (geometry + b on the host): "
                          f"device trace of the operator + CSC + {total} steps + history/x "
                          f"download, wall clock, median of 3"}
    return out


def _operator_bytes(op) -> int:
    parts = getattr(op, "_parts", None)
    if parts is not None:
        return sum(p[0].nbytes + p[1].nbytes + p[2].nbytes for p in parts) + op.rhs.nbytes
    a = getattr(op, "matrix", None)
    if a is not None:
        return a.nbytes + op.rhs.nbytes
    return op.rhs.nbytes  # generated: only b crosses the bus


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=176,
                    help="timed steps (default 176: with the warm-up batch one epoch of configs[1], the reference K = 180)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2, choices=sorted(CONFIGS),
                    help="BASELINE config (1-based); 2 = configs[1], the metric's config")
    ap.add_argument("--shard", default="replicas", choices=["replicas", "columns"],
                    help="N > 1: independent replicas (default) or one column-sharded solve "
                         "(NCCL allreduce of Gram panel / residual / norm partials per step)")
    ap.add_argument("--factor", default="replicated", choices=["replicated", "round_robin"],
                    help="--shard columns: every rank factors every system (replicated) or "
                         "batch B is factored on rank B mod N only (SURVEY 8f.1)")
    ap.add_argument("--bare", action="store_true",
                    help="only the timed steps (no streaming probe, projector leg, e2e or CPU "
                         "legs): for ncu launch lists whose kernel shares are the step's")
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
