"""Repeat the in-process sharded runs (LocalGroup, P shards on one device)
and compare every repetition with the unsharded run: a race in the shard
exchange or the upload path shows up as a repetition that differs.

usage: python tools/shard_stress.py [reps] [P]   (GPU box)
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1912_07962_b200 as slim  # noqa: E402
from paper_1912_07962_b200 import problems  # noqa: E402
from paper_1912_07962_b200.parallel import LocalGroup  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    P = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    prob = problems.tomo2d(grid=48, n_views=30, rays=68, seed=6)
    op, xt = prob.op, prob.x_true
    M, K, r, alpha = op.n_blocks, 40, 6, 1000.0
    kw = dict(epochs=K / M, r=r, references={"x_true": xt})
    single = slim.run("slimls", op, slim.Sampler("random_cyclic", M, 5),
                      slim.Schedule("constant", alpha), **kw)
    bad = 0
    for rep in range(reps):
        for rr in (False, True):
            group = LocalGroup(P, round_robin=rr)
            try:
                full, per = group.run("slimls", op.with_rhs(op.rhs), lambda: slim.Sampler("random_cyclic", M, 5),
                                      slim.Schedule("constant", alpha), **kw)
            except Exception as exc:  # a corrupted exchange can make the dual system indefinite
                bad += 1
                print(f"rep {rep} P={P} round_robin={rr}: {type(exc).__name__}: {exc}", flush=True)
                continue
            err = np.linalg.norm(full.x_final - single.x_final) / np.linalg.norm(single.x_final)
            if not err <= 1e-10:
                bad += 1
                k_bad = int(np.argmax(~np.isclose(full.residual_norms, single.residual_norms, rtol=1e-9)))
                print(f"rep {rep} P={P} round_robin={rr}: relative difference {err:.3e}; "
                      f"residual history first differs at row {k_bad}", flush=True)
    print(f"{reps} repetitions x 2 modes, P = {P}: {bad} differing runs")


main()
