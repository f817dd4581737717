"""slimLS driver: the reference's ``run`` entry point on the B200 path.

``run`` keeps the signature, validation order, exception types and the
``Trajectory`` record of the reference (solvers.py:438-588).  The loop
itself (solvers.py:560-574) is executed by one ``slim_run`` call of the
C-ABI: the sampler trace and the alpha_k schedule are precomputed on the
host, the operator already lives in HBM, and history rows come back at the
end.  Only the slimLS family is on this path:

* ``slimls`` with identity C and ``inner`` in {"auto", "dual"};
* ``damped_block_kaczmarz`` = slimLS with r = 0 (solvers.py:294-302);
* ``slimtik`` with ``lam == 0`` = slimLS (solvers.py:413-414).

Everything else raises ``ValueError`` -- there is no CPU fallback.
"""

from __future__ import annotations

import copy
import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .linops import RowBlockOperator, StreamOrderError, device_operator

DIVERGENCE_FACTOR = 1e12
DUAL_MAX_ALPHA = 1e8

METHODS = (
    "slimls", "sg", "kaczmarz", "block_kaczmarz", "damped_block_kaczmarz",
    "recursive_ls", "olbfgs", "slimtik",
)
DEVICE_METHODS = ("slimls", "damped_block_kaczmarz", "slimtik", "sg")


class DivergenceError(RuntimeError):
    """Iterate became non-finite or exceeded the divergence threshold."""


@dataclass
class Schedule:
    """Damping sequence alpha_k, k >= 1 (solvers.py:93-130)."""

    kind: str = "constant"
    alpha: float = 1.0
    ramp_length: int | None = None
    decay_exponent: float = 1.0

    def __post_init__(self):
        if self.kind not in ("constant", "ramp", "decay"):
            raise ValueError(f"unknown schedule kind {self.kind!r}")
        if not self.alpha > 0:
            raise ValueError("alpha must be > 0")
        if self.kind == "ramp" and self.ramp_length is not None and self.ramp_length < 1:
            raise ValueError("ramp_length must be >= 1")

    def alpha_at(self, k: int) -> float:
        if k < 1:
            raise ValueError("step index k is 1-based")
        if self.kind == "constant":
            return self.alpha
        if self.kind == "ramp":
            length = self.ramp_length or 1
            if k >= length:
                return self.alpha
            return self.alpha * (k / length)
        return self.alpha / k**self.decay_exponent

    def with_ramp_length(self, length: int) -> "Schedule":
        return Schedule(self.kind, self.alpha, length, self.decay_exponent)


@dataclass
class Trajectory:
    """Recorded metrics of one solver run (solvers.py:438-455)."""

    ks: np.ndarray
    epoch_fraction: np.ndarray
    alphas: np.ndarray
    residual_norms: np.ndarray
    rel_errors: dict
    wall_times: np.ndarray
    row_status: list
    x_final: np.ndarray
    status: str = "ok"
    diverged_at: int | None = None
    iterates: list | None = None

    def rel_error(self, name: str) -> np.ndarray:
        return self.rel_errors[name]


def _validate(method, op, sampler, epochs, r, reg, lam, inner, record_every, schedule):
    """Same checks, same order and messages as solvers.py:504-524."""
    if method not in METHODS:
        raise ValueError(f"unknown method {method!r}, want one of {METHODS}")
    if epochs < 0:
        raise ValueError("epochs must be >= 0")
    if record_every < 1:
        raise ValueError("record_every must be >= 1")
    if r < 0:
        raise ValueError("memory level r must be >= 0")
    steps = int(round(epochs * op.n_blocks))
    if op.access_mode == "single_pass":
        if sampler.scheme != "cyclic":
            raise ValueError("single-pass operators require cyclic sampling")
        if steps > op.n_blocks:
            raise ValueError("single-pass operators cannot be revisited; at most one epoch")
    if method == "kaczmarz" and op.block_rows != 1:
        raise ValueError("kaczmarz operates on single rows; need ell = 1")
    if method not in DEVICE_METHODS:
        raise ValueError(f"method {method!r} is not on the B200 slimLS path; "
                         f"supported: {DEVICE_METHODS}")
    if method == "damped_block_kaczmarz" and r != 0:
        raise ValueError("damped block Kaczmarz keeps no memory; create the state with r=0")
    if method == "slimtik" and lam != 0.0:
        if lam < 0:
            raise ValueError("lambda must be >= 0")
        raise ValueError("slimtik with lam > 0 is not on the B200 slimLS path")
    # sg (solvers.py:245-250) takes no window, regularizer or inner solve
    if method != "sg" and reg is not None and not getattr(reg, "is_identity", False):
        raise ValueError("only the identity regularizer C = I is on the B200 dual path")
    if method != "sg" and inner not in ("auto", "dual"):
        raise ValueError(f"inner solve {inner!r} is not on the B200 path; use 'auto' or 'dual'")
    if schedule.kind == "ramp" and schedule.ramp_length is None:
        schedule = schedule.with_ramp_length(r + 1)
    return steps, schedule


def _check_dual_alphas(method, inner, alphas):
    """The reference's auto dispatch sends alpha_k > 1e8 to the n x n
    ``direct_step`` (innersolve.py:356, 377-380; solvers.py:230-237): the dual
    system I + alpha M M^T is then too ill-conditioned to trust.  The device
    path solves only the dual form, so ``inner="auto"`` refuses such a
    schedule instead of silently changing the route; ``inner="dual"`` (the
    reference's explicit dual route) is honoured."""
    if method == "sg" or inner != "auto" or alphas.size == 0:
        return
    k = int(np.argmax(alphas))
    if alphas[k] > DUAL_MAX_ALPHA:
        raise ValueError(
            f"alpha_{k + 1} = {alphas[k]:g} > {DUAL_MAX_ALPHA:g}: the reference's auto dispatch "
            "takes the direct (n x n normal-equation) route there, which is not on the B200 "
            "path; pass inner='dual' to solve the dual system anyway")


def run(method: str, op: RowBlockOperator, sampler, schedule: Schedule, *, epochs: float,
        r: int = 0, reg=None, lam: float = 0.0, olbfgs_memory: int = 10,
        x0: np.ndarray | None = None, references: dict | None = None, record_every: int = 1,
        store_iterates: bool = False, inner: str = "auto", device: int = 0,
        timing: dict | None = None, shard=None) -> Trajectory:
    """Execute ``epochs * M`` sampled slimLS steps on the GPU and record metrics.

    Deterministic given the sampler seed (fixed-order device reductions).
    Rows are recorded at k = 0, every ``record_every``-th step, the final
    step, and a divergence step if one occurs (solvers.py:497-503).

    ``timing`` (optional dict, used by bench.py): on input ``start_step``
    selects the first timed step; on output it receives the device time of
    steps start_step..K, per-kernel-class event timings and the number of
    kernels launched in that window.

    ``shard`` (optional, see :mod:`.parallel`): run this process's column
    shard of a sharded solve; x0 / references are sliced to the shard and
    ``Trajectory.x_final`` holds the shard's slice of x.
    """
    steps, schedule = _validate(method, op, sampler, epochs, r, reg, lam, inner, record_every,
                                schedule)
    big_m = op.n_blocks
    x0 = np.zeros(op.n_cols) if x0 is None else np.asarray(x0, dtype=float).reshape(-1)
    if x0.shape != (op.n_cols,):
        raise ValueError(f"x0 has shape {x0.shape}, expected ({op.n_cols},)")
    alphas = np.array([schedule.alpha_at(k) for k in range(1, steps + 1)], dtype=float)
    for k in range(steps):
        if not alphas[k] > 0:
            raise ValueError(f"schedule produced alpha_{k + 1} = {alphas[k]} <= 0")
    _check_dual_alphas(method, inner, alphas)
    # the whole trace is drawn up front; the sampler's state before the draws
    # is kept so a diverged run leaves it where the reference's would be
    # (solvers.py:560-570 draws one index per executed step)
    sampler_before = copy.deepcopy(sampler) if steps else None
    idx = sampler.indices(steps) if steps else np.zeros(0, dtype=np.int64)
    idx = np.ascontiguousarray(idx, dtype=np.int64)

    references = references or {}
    ref_items = [(name, np.ascontiguousarray(np.asarray(v, dtype=float).reshape(-1)),
                  float(np.linalg.norm(v))) for name, v in references.items()]
    for name, vec, _ in ref_items:
        if vec.shape != (op.n_cols,):
            raise ValueError(f"reference {name!r} has shape {vec.shape}, expected ({op.n_cols},)")

    stream_state = getattr(op, "_next", None) if op.access_mode == "single_pass" else None
    if stream_state is not None and steps > 0 and stream_state != 1:
        raise StreamOrderError(f"single-pass stream expected block {stream_state}, got 1")

    x0_full = x0
    r_dev = 0 if method == "sg" else r  # sg keeps no window (r only sets the ramp length)
    if shard is not None:
        c0, c1 = shard.col0, shard.col1
        dop = shard.device_operator(op, r_dev, device)
        x0 = np.ascontiguousarray(x0[c0:c1])
        dev_refs = [np.ascontiguousarray(v[c0:c1]) for _, v, _ in ref_items]
    else:
        dop = device_operator(op, r_dev, device)
        dev_refs = [v for _, v, _ in ref_items]
    dop.call("slim_set_method", _lib.SLIM_METHOD_SG if method == "sg" else _lib.SLIM_METHOD_SLIMLS)
    x0c = np.ascontiguousarray(x0)
    dop.call("slim_set_x", _lib.dptr(x0c))
    refp = (C.POINTER(C.c_double) * max(1, len(ref_items)))(*[_lib.dptr(v) for v in dev_refs])
    dop.call("slim_set_references", len(ref_items), refp)
    limit = DIVERGENCE_FACTOR * (1.0 + float(np.linalg.norm(x0_full)))
    dop.call("slim_set_divergence_limit", C.c_double(limit))

    ncol = _lib.SLIM_HIST_FIXED + len(ref_items)
    cap = steps // record_every + 2
    hist = np.zeros((cap, ncol))
    iters = np.zeros((cap, x0.shape[0])) if store_iterates else None
    n_rows = C.c_int64(0)
    status = C.c_int32(0)
    div_at = C.c_int64(0)
    if timing is not None:
        dop.call("slim_set_profiling", 1)
        dop.call("slim_set_timing_start", int(timing.get("start_step", 1)))
    dop.call("slim_run", _lib.i64ptr(idx), _lib.dptr(alphas), steps, record_every,
             _lib.dptr(hist), C.byref(n_rows), C.byref(status), C.byref(div_at),
             _lib.dptr(iters) if iters is not None else None)
    if timing is not None:
        dop.call("slim_set_profiling", 0)
        ms, cnt = C.c_double(0), C.c_int64(0)
        for which, key in ((0, "gram"), (1, "cholesky"), (2, "x_chain"), (3, "window")):
            dop.call("slim_timing", which, C.byref(ms), C.byref(cnt))
            timing[key + "_ms"] = ms.value
            timing[key + "_count"] = cnt.value
        dop.call("slim_timing", 4, C.byref(ms), C.byref(cnt))
        timing["launches"] = cnt.value
        dop.call("slim_timing", 5, C.byref(ms), C.byref(cnt))
        timing["cholesky_flops"] = ms.value
        dop.call("slim_timing", 6, C.byref(ms), C.byref(cnt))
        timing["cholesky_i8ops"] = ms.value
        dop.call("slim_timing", 7, C.byref(ms), C.byref(cnt))
        timing["cholesky_digits"] = (int(ms.value), int(cnt.value))  # (count, trailing bits)
        dop.call("slim_timing", 9, C.byref(ms), C.byref(cnt))
        timing["cholesky_pairs"] = (int(ms.value), int(cnt.value))  # (pairs per update, QX)
        reps = int(timing.get("probe_reps", 0))
        if reps > 0:  # operator-streaming kernels alone, cold L2 (bench "streaming")
            timing["streaming"] = {}
            us, nbytes = C.c_double(0), C.c_double(0)
            for kid, name in ((0, "residual"), (1, "mtw"), (2, "gram")):
                try:
                    dop.call("slim_probe_stream", kid, reps, C.byref(us), C.byref(nbytes))
                except ValueError:  # generated blocks: the Gram is the tensor-core kernel
                    continue
                timing["streaming"][name] = (us.value, nbytes.value)
    x_final = np.empty(x0.shape[0])
    dop.call("slim_get_x", _lib.dptr(x_final))
    if status.value and sampler_before is not None:
        _rewind_sampler(sampler, sampler_before, int(div_at.value))
    if stream_state is not None:
        op._next = stream_state + (int(div_at.value) if status.value else steps)
    return _trajectory(hist[: n_rows.value], iters, x0_full, ref_items, big_m, status.value,
                       div_at.value, x_final, store_iterates)


def _rewind_sampler(sampler, before, consumed: int):
    """Put ``sampler`` in the state of ``before`` advanced by ``consumed`` draws."""
    state = copy.deepcopy(before.__dict__)
    sampler.__dict__.clear()
    sampler.__dict__.update(state)
    if consumed:
        sampler.indices(consumed)


def _trajectory(rows, iters, x0, ref_items, big_m, status, div_at, x_final, store_iterates):
    ks = [0]
    efrac = [0.0]
    alphas = [np.nan]
    resid = [np.nan]
    stamps = [0.0]
    statuses = ["ok"]
    rel = {name: [] for name, _, _ in ref_items}
    for name, vec, nrm in ref_items:
        diff = float(np.linalg.norm(x0 - vec))
        rel[name].append(diff / nrm if nrm > 0 else diff)
    iterates = [x0.copy()] if store_iterates else None
    for i, row in enumerate(rows):
        k = int(row[0])
        ks.append(k)
        efrac.append(k / big_m)
        alphas.append(float(row[1]))
        resid.append(float(row[2]))
        stamps.append(float(row[3]) * 1e-9)
        statuses.append("diverged" if row[4] != 0 else "ok")
        for q, (name, _, nrm) in enumerate(ref_items):
            diff = float(row[_lib.SLIM_HIST_FIXED + q])
            rel[name].append(diff / nrm if nrm > 0 else diff)
        if store_iterates:
            iterates.append(np.array(iters[i]))
    wall = [0.0] + [stamps[i] - stamps[i - 1] for i in range(1, len(stamps))]
    return Trajectory(
        ks=np.asarray(ks, dtype=np.int64), epoch_fraction=np.asarray(efrac),
        alphas=np.asarray(alphas), residual_norms=np.asarray(resid),
        rel_errors={n: np.asarray(v) for n, v in rel.items()}, wall_times=np.asarray(wall),
        row_status=statuses, x_final=x_final, status="diverged" if status else "ok",
        diverged_at=int(div_at) if status else None, iterates=iterates)


def dual_step(stacked_blocks, rhs_residual, alpha: float, device: int = 0) -> np.ndarray:
    """Secondary seam: ``innersolve.dual_step`` (innersolve.py:305-321) on the GPU."""
    mats = [np.atleast_2d(np.asarray(m, dtype=float)) for m in stacked_blocks]
    ell = mats[-1].shape[0]
    if any(m.shape[0] != ell for m in mats):
        raise ValueError("the device dual step needs equal block heights")
    mat = np.ascontiguousarray(np.vstack(mats))
    res = np.ascontiguousarray(np.asarray(rhs_residual, dtype=float).reshape(-1))
    if res.shape[0] != ell:
        raise ValueError(f"rhs_residual has {res.shape[0]} entries, newest block has {ell} rows")
    if not alpha > 0:
        raise ValueError("alpha must be > 0")
    s = np.empty(mat.shape[1])
    rc = _lib.lib().slim_dual_step(device, _lib.dptr(mat), mat.shape[0], mat.shape[1],
                                   _lib.dptr(res), ell, C.c_double(alpha), _lib.dptr(s))
    _lib.check(rc, None)
    return s


def potrf(g: np.ndarray, device: int = 0) -> np.ndarray:
    """Lower Cholesky factor of an SPD matrix by the tile-DAG kernel."""
    g = np.ascontiguousarray(np.asarray(g, dtype=float))
    n = g.shape[0]
    out = np.empty_like(g)
    _lib.check(_lib.lib().slim_potrf(device, _lib.dptr(g), n, _lib.dptr(out)), None)
    return out
