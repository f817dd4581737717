"""Measured parity margins of the fp64 paths (GPU box): relative iterate error
vs the oracle for the tight (1e-10) cases of tests/test_gpu_parity.py.

usage: [SLIM_LIB=...] python tools/parity_margins.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_1912_07962_b200 as slim  # noqa: E402
from oracle import slimls_oracle as orc  # noqa: E402
from paper_1912_07962_b200 import problems  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def tomo_reduced():
    prob = problems.tomo2d(grid=64, n_views=45, rays=90, seed=2)
    op, K = prob.op, 30
    traj = slim.run("slimls", op, slim.Sampler("random_cyclic", op.n_blocks, 11),
                    slim.Schedule("constant", 1000.0), epochs=K / op.n_blocks, r=10)
    idx = orc.sampler_indices("random_cyclic", op.n_blocks, 11, K)
    fetch = orc.csr_fetch([op.csr_block(i) for i in range(1, op.n_blocks + 1)], prob.b)
    ref = orc.run_slimls(fetch, op.n_blocks, op.n_cols, idx, np.full(K, 1000.0), r=10)
    return rel(traj.x_final, ref.x_final)


def full(cfg, r, alpha, K, sparse):
    op, b, xt = bench.build_config(cfg)
    M = op.n_blocks
    traj = slim.run("slimls", op, slim.Sampler("random_cyclic", M, 7962),
                    slim.Schedule("constant", alpha), epochs=K / M, r=r)
    idx = orc.sampler_indices("random_cyclic", M, 7962, K)
    al = np.full(K, alpha)
    if sparse:
        ref = orc.run_slimls_sparse([op.csr_block(i) for i in range(1, M + 1)], b, idx, al, r=r)
    else:
        ref = orc.run_slimls(bench.oracle_fetch(op, b), M, op.n_cols, idx, al, r=r)
    return rel(traj.x_final, ref.x_final)


if __name__ == "__main__":
    lib = os.environ.get("SLIM_LIB", "default")
    for name, fn in (("tomo 64^2 reduced (kappa ~1e6), 30 steps", tomo_reduced),
                     ("configs[0] 300 steps", lambda: full(1, 5, 100.0, 300, False)),
                     ("configs[1] full size, 14 steps", lambda: full(2, 10, 1000.0, 14, False)),
                     ("configs[3] full size, 3 steps", lambda: full(4, 5, 1000.0, 3, True))):
        print(f"{os.path.basename(lib)}: {name}: rel iterate error vs oracle {fn():.2e} (bar 1e-10)",
              flush=True)
