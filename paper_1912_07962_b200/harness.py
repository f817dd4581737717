"""Experiment driver: problems, replicates, CSV outputs (reference harness.py).

``run_experiment`` runs the configured slimLS solve for ``replicates``
sampler streams (seed ``base_seed + i``, harness.py:147) on the GPU and
writes the reference's three CSV files with the same columns, ordering and
number formatting (``%.17g``, harness.py:40-66, 217-313):

* ``<out>_metrics.csv``     one row per (replicate, recorded step)
* ``<out>_aggregate.csv``   per-step median and 5/95th percentiles
* ``<out>_replicates.csv``  per-replicate final status

Replicates run one after another on the device (``workers`` > 1 would
fork host processes in the reference; the device run is already parallel).
"""

from __future__ import annotations

import csv
import os
import time
from dataclasses import dataclass

import numpy as np

from . import problems
from .config import ExperimentConfig
from .linops import DenseBlockOperator, SparseBlockOperator
from .sampling import Sampler
from .slimfile import load_stream_file
from .solvers import Schedule, Trajectory, run

DESK_MAX_N = 2000

METRIC_COLUMNS = (
    "replicate", "k", "epoch_fraction", "rel_err_true", "rel_err_xls", "rel_err_xhat",
    "sampled_residual_norm", "alpha_k", "wall_time_seconds", "status",
)
_REF_COLUMN = {"x_true": "rel_err_true", "x_ls": "rel_err_xls", "x_hat": "rel_err_xhat"}


def _fmt(value) -> str:
    if value is None:
        return ""
    if isinstance(value, str):
        return value
    if isinstance(value, (int, np.integer)):
        return str(int(value))
    v = float(value)
    if np.isnan(v):
        return "nan"
    return f"{v:.17g}"


def build_problem(cfg: ExperimentConfig):
    """(operator-with-rhs, b, x_true or None) for the configured problem."""
    kind = cfg.problem_kind
    if kind == "gaussian":
        # reference tomo.gaussian_testproblem (tomo.py:336-356): N(0, 1), x_true = 1
        g = np.random.Generator(np.random.Philox(key=cfg.problem_seed))
        a = g.standard_normal((cfg.m, cfg.n))
        x_true = np.ones(cfg.n)
        clean = a @ x_true
        b = problems.scaled_noise(clean, cfg.noise_level, g) if cfg.noise_level > 0 else clean
        return DenseBlockOperator(a, cfg.m // cfg.blocks, b), b, x_true
    if kind == "generated":
        op, b, xt = problems.generated_dense(n=cfg.n, m=cfg.m, ell=cfg.m // cfg.blocks,
                                             seed=cfg.problem_seed, noise=cfg.noise_level)
        return op, b, xt
    if kind == "baseline":
        import importlib
        import sys

        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        if root not in sys.path:
            sys.path.insert(0, root)
        bench = importlib.import_module("bench")
        return bench.build_config(cfg.baseline_config)
    if kind == "tomo2d":
        rays = cfg.rays_per_view or cfg.grid
        angles = np.linspace(-cfg.half_angle, cfg.half_angle, cfg.views)  # tomo.py:207-209
        parts = [problems.siddon2d_block(a, cfg.grid, rays) for a in angles]
        x_true = problems.shepp_logan_2d(cfg.grid)
        return _tomo_rhs(parts, x_true, cfg)
    if kind == "tomo3d":
        side = cfg.detector_side or cfg.grid
        g = np.random.Generator(np.random.Philox(key=cfg.problem_seed))  # tomo.py:212-216
        raw = g.standard_normal((cfg.views, 3))
        dirs = raw / np.linalg.norm(raw, axis=1, keepdims=True)
        parts = [problems.siddon3d_block(d, cfg.grid, side) for d in dirs]
        x_true = problems.shepp_logan_3d(cfg.grid)
        return _tomo_rhs(parts, x_true, cfg)
    op = load_stream_file(cfg.path)
    return op, op.rhs, None


def _tomo_rhs(parts, x_true, cfg):
    op = SparseBlockOperator(parts)
    clean = np.concatenate([problems._csr_matvec(ip, ix, d, x_true) for ip, ix, d, _ in parts])
    if cfg.noise_level > 0:  # tomo.py:323-333
        g = np.random.Generator(np.random.Philox(key=cfg.problem_seed))
        eps = g.standard_normal(clean.shape[0])
        eps *= cfg.noise_level * np.linalg.norm(clean) / np.linalg.norm(eps)
        b = clean + eps
    else:
        b = clean
    return op.with_rhs(b), b, x_true


def build_schedule(cfg: ExperimentConfig) -> Schedule:
    sched = Schedule(cfg.schedule_kind, cfg.alpha, cfg.ramp_length, cfg.decay_exponent)
    if sched.kind == "ramp" and sched.ramp_length is None:
        sched = sched.with_ramp_length(cfg.r + 1)
    return sched


def build_references(cfg: ExperimentConfig, op, b, x_true) -> dict:
    """x_true, plus x_ls at desk scale (harness.py:116-141).  x_hat needs the
    reference's theory validator (out of scope) and is dropped with a notice."""
    refs = {}
    wanted = set(cfg.error_references)
    if "x_true" in wanted and x_true is not None:
        refs["x_true"] = np.asarray(x_true, dtype=float)
    if "x_hat" in wanted:
        print("note: x_hat needs the theory validator (not on the B200 path); dropping it")
    if "x_ls" in wanted:
        if op.n_cols > DESK_MAX_N:
            print(f"note: n = {op.n_cols} exceeds the desk-scale guard {DESK_MAX_N}; "
                  "dropping references ['x_ls']")
        else:
            a = np.vstack([op.fetch_block(i).a_block for i in range(1, op.n_blocks + 1)])
            refs["x_ls"] = np.linalg.lstsq(a, np.asarray(b, float), rcond=None)[0]
    return refs


@dataclass
class ExperimentResult:
    metrics_path: str
    aggregate_path: str
    replicates_path: str
    trajectories: list
    n_diverged: int


def run_experiment(cfg: ExperimentConfig, device: int = 0) -> ExperimentResult:
    cfg.validate()
    op, b, x_true = build_problem(cfg)
    references = build_references(cfg, op, b, x_true)
    t0 = time.perf_counter()
    trajectories = []
    for rep in range(cfg.replicates):
        sampler = Sampler(cfg.scheme, op.n_blocks, seed=cfg.base_seed + rep)
        trajectories.append(run(
            cfg.method, op, sampler, build_schedule(cfg), epochs=cfg.epochs, r=cfg.r,
            lam=cfg.lam, references=references, record_every=cfg.record_every,
            store_iterates=cfg.store_iterates, inner=cfg.inner, device=device))
    elapsed = time.perf_counter() - t0
    paths = write_outputs(cfg.output, cfg, trajectories, references)
    n_div = sum(1 for t in trajectories if t.status == "diverged")
    print(f"{cfg.method}: {cfg.replicates} replicate(s), "
          f"{int(round(cfg.epochs * op.n_blocks))} step(s) each, {n_div} diverged, "
          f"{elapsed:.2f} s")
    return ExperimentResult(*paths, trajectories, n_div)


def write_outputs(prefix, cfg, trajectories: list, references: dict):
    """The reference's CSV files, byte-compatible layout (harness.py:217-313)."""
    os.makedirs(os.path.dirname(prefix) or ".", exist_ok=True)
    metrics_path = f"{prefix}_metrics.csv"
    aggregate_path = f"{prefix}_aggregate.csv"
    replicates_path = f"{prefix}_replicates.csv"
    have = {_REF_COLUMN[name] for name in references}

    with open(metrics_path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(METRIC_COLUMNS)
        for rep, traj in enumerate(trajectories):
            for j, k in enumerate(traj.ks):
                row = [rep, int(k), _fmt(traj.epoch_fraction[j])]
                for name in ("x_true", "x_ls", "x_hat"):
                    row.append(_fmt(traj.rel_errors[name][j]) if _REF_COLUMN[name] in have else "")
                row += [_fmt(traj.residual_norms[j]), _fmt(traj.alphas[j]),
                        _fmt(traj.wall_times[j]), traj.row_status[j]]
                w.writerow(row)

    per_k: dict = {}
    epoch_at: dict = {}
    for traj in trajectories:
        for j, k in enumerate(traj.ks):
            bucket = per_k.setdefault(int(k), {name: [] for name in references} | {"residual": []})
            epoch_at[int(k)] = float(traj.epoch_fraction[j])
            for name in references:
                bucket[name].append(traj.rel_errors[name][j])
            bucket["residual"].append(traj.residual_norms[j])
    agg_columns = ["k", "epoch_fraction", "n_replicates"]
    for name in ("x_true", "x_ls", "x_hat"):
        col = _REF_COLUMN[name]
        agg_columns += [f"median_{col}", f"p5_{col}", f"p95_{col}"]
    agg_columns += ["median_sampled_residual_norm"]
    with open(aggregate_path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(agg_columns)
        for k in sorted(per_k):
            bucket = per_k[k]
            row = [k, _fmt(epoch_at[k]), len(bucket["residual"])]
            for name in ("x_true", "x_ls", "x_hat"):
                if name in references:
                    vals = np.asarray(bucket[name], dtype=float)
                    with np.errstate(invalid="ignore"):
                        row += [_fmt(np.median(vals)), _fmt(np.percentile(vals, 5)),
                                _fmt(np.percentile(vals, 95))]
                else:
                    row += ["", "", ""]
            res = np.asarray(bucket["residual"], dtype=float)
            row.append(_fmt(np.median(res)) if res.size else "")
            w.writerow(row)

    with open(replicates_path, "w", newline="") as fh:
        w = csv.writer(fh)
        header = ["replicate", "status", "diverged_at", "final_k"]
        header += [f"final_{_REF_COLUMN[n]}" for n in ("x_true", "x_ls", "x_hat")]
        w.writerow(header)
        for rep, traj in enumerate(trajectories):
            row = [rep, traj.status, "" if traj.diverged_at is None else traj.diverged_at,
                   int(traj.ks[-1])]
            for name in ("x_true", "x_ls", "x_hat"):
                row.append(_fmt(traj.rel_errors[name][-1]) if name in references else "")
            w.writerow(row)
    return metrics_path, aggregate_path, replicates_path
