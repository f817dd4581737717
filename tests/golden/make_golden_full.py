"""Full-size golden runs on the BASELINE configurations (run once, in the
build container, where ``/root/reference`` is importable).

    PYTHONPATH=/root/reference/pkg/src OPENBLAS_NUM_THREADS=4 \
        python tests/golden/make_golden_full.py cfg1 cfg2      # reference run()
    python tests/golden/make_golden_full.py cfg5 cfg3 cfg4    # (cfg5: reference run(),
                                                              #  cfg3/4: sparse restatement)

Each case runs the whole trajectory the GPU parity tests compare against
(tests/test_gpu_full_runs.py), with record_every = 1:

* cfg1 -- configs[0] dense Gaussian, K = 2000 (10 epochs), the unmodified
  reference ``slimsolve.run`` on the regenerated matrix;
* cfg2 -- configs[1] 256^2 tomography, K = 180 (one epoch), reference
  ``run`` on a reference ``SparseBlockOperator`` holding exactly the CSR
  blocks the GPU path uploads (same bits; the operator's sha256 is stored);
* cfg5 -- configs[4] generated rows at full n = 65,536 (m = 4,194,304),
  K = 30 cyclic single-pass steps (window of 21 full from k = 21) through a
  generator ``RowBlockOperator`` subclass of the reference (the contract of
  linops.py:75-100).  b is stored for the 30 blocks the pass touches;
* cfg3 / cfg4 -- configs[2] (1024^2, N = 13,032) and configs[3] (128^3,
  N = 12,288) at full size with the window full and evicting (K = 16 / 12):
  the reference cannot densify these blocks (12-34 GB each), so the
  trajectory comes from the oracle's sparse dual-form restatement, which
  tests/test_oracle_golden.py pins to the reference at reduced size.

For n >= 1M the final iterate is stored as (a) 65,536 entries at seeded
positions and (b) 16 Gaussian projections v_j . x (v_j from Philox key
4242 + j); the test estimates ||x - x_ref|| from both.  Histories
(residual norms, relative errors) are stored per step.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
REF_SRC = "/root/reference/pkg/src"

from tests.golden_cases import operator_digest  # noqa: E402

N_PROJ = 16
N_SAMPLE = 65536


def projections(x: np.ndarray) -> np.ndarray:
    n = x.shape[0]
    return np.array([np.random.Generator(np.random.Philox(key=4242 + j)).standard_normal(n) @ x
                     for j in range(N_PROJ)])


def sample_positions(n: int) -> np.ndarray:
    g = np.random.Generator(np.random.Philox(key=777))
    return np.sort(g.choice(n, size=min(n, N_SAMPLE), replace=False)).astype(np.int64)


def _traj(prefix, traj, full_x=True):
    d = {f"{prefix}/ks": np.asarray(traj.ks), f"{prefix}/alphas": np.asarray(traj.alphas),
         f"{prefix}/residual_norms": np.asarray(traj.residual_norms),
         f"{prefix}/status": np.array(traj.status),
         f"{prefix}/diverged_at": np.array(-1 if traj.diverged_at is None else traj.diverged_at)}
    for name, v in traj.rel_errors.items():
        d[f"{prefix}/rel/{name}"] = np.asarray(v)
    x = np.asarray(traj.x_final)
    d[f"{prefix}/x_norm"] = np.array(np.linalg.norm(x))
    if full_x:
        d[f"{prefix}/x_final"] = x
    else:
        pos = sample_positions(x.shape[0])
        d[f"{prefix}/x_pos"] = pos
        d[f"{prefix}/x_sample"] = x[pos]
        d[f"{prefix}/x_proj"] = projections(x)
    return d


def _save(name, d):
    path = os.path.join(HERE, f"full_{name}.npz")
    np.savez_compressed(path, **d)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)", flush=True)


def _reference():
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import slimsolve  # noqa: F401
    return slimsolve


def cfg1():
    _reference()
    from slimsolve.linops import DenseBlockOperator
    from slimsolve.sampling import Sampler
    from slimsolve.solvers import Schedule, run

    from paper_1912_07962_b200 import problems
    op, b, xt = problems.gaussian_dense()
    a = op.matrix
    t = time.time()
    traj = run("slimls", DenseBlockOperator(a, 100, b), Sampler("random_cyclic", 200, seed=7962),
               Schedule("constant", 100.0), epochs=10, r=5, references={"x_true": xt},
               record_every=1)
    print(f"cfg1 reference run: {time.time() - t:.1f} s", flush=True)
    d = _traj("cfg1", traj)
    d["cfg1/A_check"] = np.array([a.sum(), np.abs(a).sum(), b.sum(), xt.sum()])
    d["cfg1/K"] = np.array(2000)
    _save("cfg1", d)


def cfg2():
    _reference()
    import scipy.sparse as sp
    from slimsolve.linops import SparseBlockOperator as RefSparse
    from slimsolve.sampling import Sampler
    from slimsolve.solvers import Schedule, run

    import bench
    op, b, xt = bench.build_config(2)
    blocks = [sp.csr_matrix((d.astype(np.float64), ix, ip), shape=shp)
              for ip, ix, d, shp in (op.csr_block(i) for i in range(1, op.n_blocks + 1))]
    rop = RefSparse(blocks, b)
    K = 180
    t = time.time()
    traj = run("slimls", rop, Sampler("random_cyclic", 180, seed=7962),
               Schedule("constant", 1000.0), epochs=1, r=10, references={"x_true": xt},
               record_every=1)
    print(f"cfg2 reference run: {time.time() - t:.1f} s", flush=True)
    d = _traj("cfg2", traj)
    d["cfg2/op_sha256"] = np.array(operator_digest(op))
    d["cfg2/b_sum"] = np.array([b.sum(), np.abs(b).sum(), xt.sum()])
    d["cfg2/K"] = np.array(K)
    _save("cfg2", d)


def cfg5():
    _reference()
    from slimsolve.linops import RowBlockOperator, SampleBlock
    from slimsolve.sampling import Sampler
    from slimsolve.solvers import Schedule, run

    from oracle import slimls_oracle as orc

    n, m, ell, seed, K, r = 65536, 4194304, 256, 1912, 30, 20
    x_true = np.random.Generator(np.random.Philox(key=seed)).standard_normal(n)
    # b on the rows the K-step pass touches: A x_true (fp64 sums of the fp32
    # entries) + 0.5% Gaussian noise (Philox key seed + 1) scaled over those rows
    rows = K * ell
    clean = np.concatenate([orc.gen_rows(seed, s, ell, n) @ x_true for s in range(0, rows, ell)])
    eps = np.random.Generator(np.random.Philox(key=seed + 1)).standard_normal(rows)
    eps *= 0.005 * np.linalg.norm(clean) / np.linalg.norm(eps)
    b_used = clean + eps

    class GeneratedOperator(RowBlockOperator):
        """Generator subclass of the reference base class: block i is rows
        [(i-1) ell, i ell) of the splitmix64 matrix, generated on fetch."""

        access_mode = "random_access"

        def __init__(self):
            self.n_rows, self.n_cols, self.block_rows, self.n_blocks = m, n, ell, m // ell

        def has_rhs(self):
            return True

        def fetch_block(self, i):
            self._check_index(i)
            s, e = self.row_range(i)
            if e > rows:
                raise IndexError("golden rhs covers only the first K blocks")
            return SampleBlock(i, orc.gen_rows(seed, s, ell, n), b_used[s:e])

    t = time.time()
    traj = run("slimls", GeneratedOperator(), Sampler("cyclic", m // ell, seed=0),
               Schedule("constant", 100.0), epochs=K / (m // ell), r=r,
               references={"x_true": x_true}, record_every=1)
    print(f"cfg5 reference run: {time.time() - t:.1f} s", flush=True)
    d = _traj("cfg5", traj)
    d["cfg5/b_used"] = b_used
    d["cfg5/K"] = np.array(K)
    _save("cfg5", d)


def _sparse_case(name, cfg_id, K, r, alpha):
    import bench
    from oracle import slimls_oracle as orc

    t = time.time()
    op, b, xt = bench.build_config(cfg_id)
    print(f"{name}: operator built in {time.time() - t:.1f} s", flush=True)
    M = op.n_blocks
    idx = orc.sampler_indices("random_cyclic", M, 7962, K)
    t = time.time()
    traj = orc.run_slimls_sparse([op.csr_block(i) for i in range(1, M + 1)], b, idx,
                                 np.full(K, alpha), r=r, references={"x_true": xt})
    print(f"{name}: sparse restatement run {time.time() - t:.1f} s", flush=True)
    d = _traj(name, traj, full_x=False)
    d[f"{name}/op_sha256"] = np.array(operator_digest(op))
    d[f"{name}/b_sum"] = np.array([b.sum(), np.abs(b).sum(), xt.sum()])
    d[f"{name}/indices"] = idx
    d[f"{name}/K"] = np.array(K)
    _save(name, d)


def cfg3():
    _sparse_case("cfg3", 3, K=16, r=8, alpha=1000.0)


def cfg4():
    _sparse_case("cfg4", 4, K=12, r=5, alpha=1000.0)


if __name__ == "__main__":
    for arg in sys.argv[1:]:
        globals()[arg]()
