"""CPU oracle for the slimLS hot path -- TEST INFRASTRUCTURE ONLY.

This module is the *checker*, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  The product package
``paper_1912_07962_b200`` must never import anything under ``oracle/``.

It restates, in plain NumPy/SciPy, the reference algorithm of
``arxiv/paper_1912_07962`` (package ``slimsolve``) for exactly the path
the B200 build accelerates: ``solvers.run("slimls", ...)`` with identity
regularizer, ``lam = 0`` and ``inner = "auto"``.  Every function cites the
reference file:line it follows (paths relative to the reference's
``pkg/src/slimsolve/``).  The arithmetic is the reference's own: dense
block fetch, ``vstack`` of the window, full Gram recompute every step,
``scipy.linalg.solve(assume_a="pos")`` for the dual system and
``np.linalg.inv`` for the single-block route.  That keeps the oracle's
cost structure equal to the reference's, so it doubles as the CPU
baseline ("port") that ``bench.py --impl reference`` times.

Pinning: ``tests/test_oracle_golden.py`` checks this restatement against
vectors produced by the reference itself (``tests/golden/make_golden.py``
imports ``slimsolve`` from ``/root/reference/pkg/src`` in the build
container and commits the outputs as ``tests/golden/*.npz``).
"""

from __future__ import annotations

import time
from collections import deque
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg

# solvers.py:47 / innersolve.py:356
DIVERGENCE_FACTOR = 1e12
DUAL_MAX_ALPHA = 1e8
SOLVE_CACHE_MAX_ENTRIES = 512  # solvers.py:187

SCHEMES = ("cyclic", "random_cyclic", "uniform_iid")  # sampling.py:35


# ---------------------------------------------------------------------------
# Sampling (sampling.py:38-84)
# ---------------------------------------------------------------------------


def fisher_yates(m: int, rng: np.random.Generator) -> np.ndarray:
    """Backward Fisher-Yates over 1..m with scalar bounded draws.

    Follows sampling.py:38-44: one ``rng.integers(0, i + 1)`` call per
    position i = m-1 .. 1, swapping perm[i] and perm[j].
    """
    perm = np.arange(1, m + 1, dtype=np.int64)
    for i in range(m - 1, 0, -1):
        j = int(rng.integers(0, i + 1))
        perm[i], perm[j] = perm[j], perm[i]
    return perm


class OracleSampler:
    """Restatement of ``Sampler`` (sampling.py:47-84)."""

    def __init__(self, scheme: str, n_blocks: int, seed: int = 0):
        if scheme not in SCHEMES:
            raise ValueError(f"unknown scheme {scheme!r}")
        if n_blocks < 1:
            raise ValueError("n_blocks must be >= 1")
        self.scheme = scheme
        self.n_blocks = int(n_blocks)
        # Philox 4x64 keyed directly by the seed (sampling.py:58)
        self.rng = np.random.Generator(np.random.Philox(key=int(seed)))
        self.position = 0
        self._perm = None

    def next_index(self) -> int:  # sampling.py:62-75
        m = self.n_blocks
        if self.scheme == "cyclic":
            idx = self.position % m + 1
        elif self.scheme == "uniform_iid":
            idx = int(self.rng.integers(1, m + 1))
        else:
            off = self.position % m
            if off == 0:
                self._perm = fisher_yates(m, self.rng)
            idx = int(self._perm[off])
        self.position += 1
        return idx

    def indices(self, count: int) -> np.ndarray:  # sampling.py:77-79
        return np.array([self.next_index() for _ in range(count)], dtype=np.int64)


def sampler_indices(scheme: str, n_blocks: int, seed: int, count: int) -> np.ndarray:
    return OracleSampler(scheme, n_blocks, seed).indices(count)


# ---------------------------------------------------------------------------
# Schedule (solvers.py:93-130)
# ---------------------------------------------------------------------------


def schedule_alpha(kind: str, alpha: float, k: int, ramp_length=None,
                   decay_exponent: float = 1.0) -> float:
    """alpha_k, k >= 1 (solvers.py:117-127)."""
    if kind == "constant":
        return alpha
    if kind == "ramp":
        length = ramp_length or 1
        if k >= length:
            return alpha
        return alpha * (k / length)
    return alpha / k**decay_exponent


# ---------------------------------------------------------------------------
# Inner solves (innersolve.py:209-215, 276-321, 340-381)
# ---------------------------------------------------------------------------


def stack_window(mats) -> np.ndarray:
    """``_stack`` (innersolve.py:209-215): vstack copy, oldest first."""
    mats = [np.atleast_2d(np.asarray(m, dtype=float)) for m in mats]
    return np.vstack(mats) if len(mats) > 1 else mats[0]


def dual_system(mat: np.ndarray, alpha: float) -> np.ndarray:
    """``_dual_system`` (innersolve.py:298-302): G = alpha (M M^T) + I."""
    g = mat @ mat.T
    g *= alpha
    g[np.diag_indices_from(g)] += 1.0
    return g


def dual_step(mats, residual: np.ndarray, alpha: float) -> np.ndarray:
    """``dual_step`` (innersolve.py:305-321): s = alpha M^T G^{-1} [0..0; r]."""
    mat = stack_window(mats)
    rows = mat.shape[0]
    residual = np.asarray(residual, dtype=float).reshape(-1)
    y = np.zeros(rows)
    y[rows - residual.shape[0]:] = residual
    w = scipy.linalg.solve(dual_system(mat, alpha), y, assume_a="pos")
    return alpha * (mat.T @ w)


def direct_step(mats, residual: np.ndarray, alpha: float) -> np.ndarray:
    """``direct_step``/``solve_normal`` (innersolve.py:276-295, 340-350)."""
    newest = np.atleast_2d(np.asarray(mats[-1], dtype=float))
    gradient = newest.T @ np.asarray(residual, dtype=float).reshape(-1)
    mat = stack_window(mats)
    n = mat.shape[1]
    system = mat.T @ mat + np.eye(n) / alpha
    return scipy.linalg.solve(system, gradient, assume_a="pos")


def solve_step_auto(mats, residual: np.ndarray, alpha: float) -> np.ndarray:
    """``solve_step(method="auto")`` for identity C (innersolve.py:359-381)."""
    rows = sum(np.atleast_2d(np.asarray(m)).shape[0] for m in mats)
    n = np.atleast_2d(np.asarray(mats[0])).shape[1]
    if rows <= n and alpha <= DUAL_MAX_ALPHA:
        return dual_step(mats, residual, alpha)
    return direct_step(mats, residual, alpha)


# ---------------------------------------------------------------------------
# Driver (solvers.py:161-242, 438-588)
# ---------------------------------------------------------------------------


@dataclass
class OracleTrajectory:
    """Field-for-field restatement of ``Trajectory`` (solvers.py:438-455)."""

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


@dataclass
class _State:
    x: np.ndarray
    window: deque
    div_limit_sq: float
    last_residual_norm: float = float("nan")
    inv_cache: dict = field(default_factory=dict)


def _dual_single_block(st: _State, index: int, a: np.ndarray, residual, alpha):
    """``_dual_single_block`` (solvers.py:190-210), cache per (index, alpha)."""
    key = (index, alpha)
    inv = st.inv_cache.get(key)
    if inv is None:
        system = alpha * (a @ a.T)
        system[np.diag_indices_from(system)] += 1.0
        inv = np.linalg.inv(system)
        if len(st.inv_cache) < SOLVE_CACHE_MAX_ENTRIES:
            st.inv_cache[key] = inv
    return alpha * (a.T @ (inv @ residual))


def slimls_step(st: _State, index: int, a: np.ndarray, b: np.ndarray, alpha: float):
    """``slimls_step`` (solvers.py:213-242) with identity C and inner="auto".

    Returns False when the new iterate trips the divergence check of
    ``_finish`` (solvers.py:169-177); the iterate is stored either way.
    """
    st.window.append((index, a))  # push before the solve (solvers.py:227)
    residual = a @ st.x - b  # _sampled_residual, solvers.py:180-183
    st.last_residual_norm = float(np.sqrt(residual @ residual))
    if len(st.window) == 1 and a.shape[0] <= a.shape[1] and alpha <= DUAL_MAX_ALPHA:
        s = _dual_single_block(st, index, a, residual, alpha)
    else:
        s = solve_step_auto([m for _, m in st.window], residual, alpha)
    st.x = st.x - s
    norm_sq = float(st.x @ st.x)
    return norm_sq <= st.div_limit_sq


def sg_step(st: _State, index: int, a: np.ndarray, b: np.ndarray, alpha: float):
    """``sg_step`` (solvers.py:245-250): x - alpha A_k^T (A_k x - b_k), the
    memoryless subset of the slimLS chain (no window, no solve)."""
    residual = a @ st.x - b  # _sampled_residual, solvers.py:180-183
    st.last_residual_norm = float(np.sqrt(residual @ residual))
    st.x = st.x - alpha * (a.T @ residual)
    norm_sq = float(st.x @ st.x)
    return norm_sq <= st.div_limit_sq


def run_slimls(fetch, n_blocks: int, n_cols: int, indices, alphas, *, r: int = 0,
               x0=None, references=None, record_every: int = 1,
               store_iterates: bool = False, method: str = "slimls") -> OracleTrajectory:
    """Restatement of ``run`` (solvers.py:480-588) for the slimLS path.

    ``fetch(i)`` returns the dense block (a_block (ell, n), b_block (ell,))
    for 1-based index i, like ``RowBlockOperator.fetch_block``
    (linops.py:192-206 / 270-279).  ``indices``/``alphas`` are the
    precomputed sampler trace and alpha_k sequence, so the step count is
    ``len(indices)``.
    """
    indices = np.asarray(indices, dtype=np.int64)
    alphas = np.asarray(alphas, dtype=float)
    steps = int(indices.shape[0])
    x0 = np.zeros(n_cols) if x0 is None else np.asarray(x0, dtype=float).reshape(-1)
    x0_norm = float(np.linalg.norm(x0))
    limit = DIVERGENCE_FACTOR * (1.0 + x0_norm)  # solvers.py:144-146
    st = _State(x=x0.copy(), window=deque(maxlen=r + 1), div_limit_sq=limit * limit)

    references = references or {}
    ref_items = [(name, np.asarray(v, dtype=float), float(np.linalg.norm(v)))
                 for name, v in references.items()]
    ks, efrac, al, resid, wall, statuses = [], [], [], [], [], []
    rel = {name: [] for name, _, _ in ref_items}
    iterates = [] if store_iterates else None

    def record(k, alpha, status, dt):  # solvers.py:543-554
        ks.append(k)
        efrac.append(k / n_blocks)
        al.append(alpha)
        resid.append(st.last_residual_norm if k else np.nan)
        wall.append(dt)
        statuses.append(status)
        for name, vec, nrm in ref_items:
            diff = float(np.linalg.norm(st.x - vec))
            rel[name].append(diff / nrm if nrm > 0 else diff)
        if iterates is not None:
            iterates.append(st.x.copy())

    status, diverged_at = "ok", None
    record(0, np.nan, "ok", 0.0)
    t_prev = time.perf_counter()
    for k in range(1, steps + 1):
        idx = int(indices[k - 1])
        a, b = fetch(idx)
        alpha = float(alphas[k - 1])
        if not alpha > 0:
            raise ValueError(f"schedule produced alpha_{k} = {alpha} <= 0")
        ok = (sg_step if method == "sg" else slimls_step)(st, idx, a, b, alpha)
        if not ok:  # solvers.py:563-570
            status, diverged_at = "diverged", k
            now = time.perf_counter()
            record(k, alpha, "diverged", now - t_prev)
            break
        if k % record_every == 0 or k == steps:
            now = time.perf_counter()
            record(k, alpha, "ok", now - t_prev)
            t_prev = now

    return OracleTrajectory(
        ks=np.asarray(ks, dtype=np.int64), epoch_fraction=np.asarray(efrac),
        alphas=np.asarray(al), residual_norms=np.asarray(resid),
        rel_errors={n: np.asarray(v) for n, v in rel.items()},
        wall_times=np.asarray(wall), row_status=statuses, x_final=st.x.copy(),
        status=status, diverged_at=diverged_at, iterates=iterates)


# ---------------------------------------------------------------------------
# Block fetch helpers (linops.py:84-88, 192-206, 270-279)
# ---------------------------------------------------------------------------


def dense_fetch(a: np.ndarray, b: np.ndarray, ell: int):
    """Block i = rows [(i-1) ell, i ell) of a dense matrix (linops.py:84-88)."""
    a = np.ascontiguousarray(a, dtype=float)
    b = np.asarray(b, dtype=float)

    def fetch(i):
        s = (i - 1) * ell
        return a[s:s + ell], b[s:s + ell]
    return fetch


def csr_fetch(blocks, b: np.ndarray):
    """Per-block CSR densified on every fetch, like linops.py:270-279.

    ``blocks`` is a list of (indptr, indices, data, (ell, n)) tuples;
    values of any float dtype are widened to fp64 (the reference stores
    fp64, linops.py:236) and densified with scipy's ``toarray`` exactly
    as the reference does.
    """
    import scipy.sparse as sp

    b = np.asarray(b, dtype=float)
    mats = [sp.csr_matrix((np.asarray(d, dtype=float), ix, ip), shape=shape)
            for ip, ix, d, shape in blocks]
    ell = mats[0].shape[0]

    def fetch(i):
        return mats[i - 1].toarray(), b[(i - 1) * ell:i * ell]
    return fetch


# ---------------------------------------------------------------------------
# configs[4] generator (BASELINE.json configs[4])
# A[i, j] = fp32((2u - 1) / sqrt(n)), u = (splitmix64(seed ^ (i n + j)) >> 11) 2^-53
# The reference has no generator operator; this is the RowBlockOperator
# subclass the survey prescribes, restated independently of the product.
# ---------------------------------------------------------------------------

_M64 = (1 << 64) - 1


def splitmix64_scalar(z: int) -> int:
    """Published splitmix64 finaliser on a Python int (reference for tests)."""
    z = (z + 0x9E3779B97F4A7C15) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def gen_entry_scalar(seed: int, i: int, j: int, n: int) -> float:
    z = splitmix64_scalar(seed ^ ((i * n + j) & _M64))
    u = (z >> 11) * 2.0**-53
    return float(np.float32((2.0 * u - 1.0) / np.sqrt(float(n))))


def gen_rows(seed: int, row0: int, rows: int, n: int) -> np.ndarray:
    """Vectorised generator rows [row0, row0 + rows) as fp64 of the fp32 values."""
    i = (np.uint64(row0) + np.arange(rows, dtype=np.uint64))[:, None]
    j = np.arange(n, dtype=np.uint64)[None, :]
    with np.errstate(over="ignore"):
        z = np.uint64(seed) ^ (i * np.uint64(n) + j)
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    u = (z >> np.uint64(11)).astype(np.float64) * 2.0**-53
    return ((2.0 * u - 1.0) / np.sqrt(float(n))).astype(np.float32).astype(np.float64)


def gen_fetch(seed: int, n: int, ell: int, b: np.ndarray):
    """fetch(i) of the generated operator, like linops.py:192-206."""
    b = np.asarray(b, dtype=float)

    def fetch(i):
        s = (i - 1) * ell
        return gen_rows(seed, s, ell, n), b[s:s + ell]
    return fetch


# ---------------------------------------------------------------------------
# Sparse dual-form restatement for full-size tomography (configs[2]/[3]).
# The reference densifies every fetched block (linops.py:278), which needs
# 12-34 GB per block at those sizes; this restatement performs the same
# arithmetic steps of slimls_step / dual_step (solvers.py:213-242,
# innersolve.py:298-321) with the window kept sparse: G = alpha (M M^T) + I
# formed densely from the sparse product, LAPACK Cholesky solve, s = alpha
# M^T w.  Cross-validated against the reference at reduced size by
# tests/test_oracle_golden.py::test_sparse_restatement_matches_reference.
# ---------------------------------------------------------------------------


def run_slimls_sparse(blocks, b, indices, alphas, *, r=0, x0=None, references=None,
                      record_every=1, step_times=None, threads_at=None):
    """``step_times`` (optional list) receives each step's wall time (the
    bench's CPU legs); ``threads_at(k)`` (optional) is called before step k
    to set the BLAS thread count (the reference arm's thread sweep)."""
    import scipy.sparse as sp

    mats = [sp.csr_matrix((np.asarray(d, dtype=float), ix, ip), shape=shp)
            for ip, ix, d, shp in blocks]
    ell, n = mats[0].shape
    b = np.asarray(b, dtype=float)
    indices = np.asarray(indices, dtype=np.int64)
    alphas = np.asarray(alphas, dtype=float)
    steps = int(indices.shape[0])
    x = np.zeros(n) if x0 is None else np.asarray(x0, dtype=float).copy()
    limit = DIVERGENCE_FACTOR * (1.0 + float(np.linalg.norm(x)))
    window = deque(maxlen=r + 1)
    inv_cache = {}
    references = references or {}
    refs = [(k, np.asarray(v, float), float(np.linalg.norm(v))) for k, v in references.items()]
    ks, resid, rel = [0], [np.nan], {k: [] for k, _, _ in refs}
    status, diverged_at = "ok", None

    def rec():
        for name, vec, nrm in refs:
            d = float(np.linalg.norm(x - vec))
            rel[name].append(d / nrm if nrm > 0 else d)

    rec()
    for k in range(1, steps + 1):
        if threads_at is not None:
            threads_at(k)
        t0 = time.perf_counter()
        idx = int(indices[k - 1])
        alpha = float(alphas[k - 1])
        a = mats[idx - 1]
        window.append((idx, a))
        res = a @ x - b[(idx - 1) * ell: idx * ell]
        rn = float(np.sqrt(res @ res))
        if len(window) == 1 and ell <= n and alpha <= DUAL_MAX_ALPHA:
            key = (idx, alpha)
            inv = inv_cache.get(key)
            if inv is None:
                system = alpha * (a @ a.T).toarray()
                system[np.diag_indices_from(system)] += 1.0
                inv = np.linalg.inv(system)
                if len(inv_cache) < SOLVE_CACHE_MAX_ENTRIES:
                    inv_cache[key] = inv
            s = alpha * (a.T @ (inv @ res))
        else:
            mat = sp.vstack([m for _, m in window]).tocsr()
            g = (mat @ mat.T).toarray()
            g *= alpha
            g[np.diag_indices_from(g)] += 1.0
            y = np.zeros(mat.shape[0])
            y[-ell:] = res
            w = scipy.linalg.solve(g, y, assume_a="pos")
            s = alpha * (mat.T @ w)
        x = x - s
        ok = float(x @ x) <= limit * limit
        if step_times is not None:
            step_times.append(time.perf_counter() - t0)
        if not ok or k % record_every == 0 or k == steps:
            ks.append(k)
            resid.append(rn)
            rec()
        if not ok:
            status, diverged_at = "diverged", k
            break
    return OracleTrajectory(
        ks=np.asarray(ks, dtype=np.int64), epoch_fraction=np.asarray(ks) / len(mats),
        alphas=np.concatenate([[np.nan], alphas[np.asarray(ks[1:], dtype=np.int64) - 1]]),
        residual_norms=np.asarray(resid), rel_errors={k: np.asarray(v) for k, v in rel.items()},
        wall_times=np.zeros(len(ks)), row_status=["ok"] * len(ks), x_final=x, status=status,
        diverged_at=diverged_at)
