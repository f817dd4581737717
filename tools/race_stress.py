"""Repetition stress for the hand-synchronized kernels (compute-sanitizer is
closed on this GPU pool): the same run on fresh device contexts many times
must give bit-identical iterates -- a race in the factorization's epoch
flags, the cluster solves or the last-CTA reductions shows up as a run that
differs -- and must stay within 1e-10 of the CPU oracle.

    python tools/race_stress.py --config 2 --steps 48 --reps 12
"""

import argparse
import gc
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--steps", type=int, default=48)
    ap.add_argument("--reps", type=int, default=12)
    ap.add_argument("--oracle", action="store_true")
    args = ap.parse_args()
    import paper_1912_07962_b200 as slim

    op, b, xt = bench.build_config(args.config)
    cfg = bench.CONFIGS[args.config]
    first, bad = None, 0
    for rep in range(args.reps):
        gc.collect()
        op2 = op.with_rhs(b)
        # alternate streamed and pre-uploaded operators and vary nothing else
        os.environ["SLIM_HOST_STREAMING"] = "1" if rep % 2 else "0"
        t = slim.run("slimls", op2, slim.Sampler(cfg["scheme"], op.n_blocks, 7962),
                     slim.Schedule("constant", cfg["alpha"]), epochs=args.steps / op.n_blocks,
                     r=cfg["r"], references={"x_true": xt})
        if first is None:
            first = t
        same = (np.array_equal(t.x_final, first.x_final)
                and np.array_equal(t.residual_norms, first.residual_norms, equal_nan=True))
        bad += 0 if same else 1
        print(f"config {args.config} rep {rep}: bit-identical to rep 0: {same}", flush=True)
        del op2, t
    if args.oracle:
        from oracle import slimls_oracle as orc
        idx = orc.sampler_indices(cfg["scheme"], op.n_blocks, 7962, args.steps)
        ref = orc.run_slimls(bench.oracle_fetch(op, b), op.n_blocks, op.n_cols, idx,
                             np.full(args.steps, cfg["alpha"]), r=cfg["r"])
        err = np.linalg.norm(first.x_final - ref.x_final) / np.linalg.norm(ref.x_final)
        print(f"config {args.config}: relative error vs oracle {err:.2e}", flush=True)
    print(f"config {args.config}: {args.reps} runs, {bad} differing", flush=True)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
