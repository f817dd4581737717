"""A/B of the batched factorization's ticket order on one GPU.

    python tools/chol_order_sweep.py --config 3 --orders 1:32,2:16,2:32,3:32,4:32

For each cols:band setting (SLIM_CHOL_COLS / SLIM_CHOL_BAND) a fresh device
context runs warm-up + K timed steps of the bench workload; prints it/s
and the mean factorization launch time (CUDA events on its stream).
"""

import argparse
import gc
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--steps", type=int, default=32)
    ap.add_argument("--orders", default="1:32,2:16,2:32,3:32,4:32")
    ap.add_argument("--repeat", type=int, default=2)
    args = ap.parse_args()
    import paper_1912_07962_b200 as slim

    os.environ["SLIM_HOST_STREAMING"] = "0"
    op, b, xt = bench.build_config(args.config)
    cfg = bench.CONFIGS[args.config]
    r, alpha, scheme = cfg["r"], cfg["alpha"], cfg["scheme"]
    N = (r + 1) * op.block_rows
    D = bench.batch_size(N)
    wprime = -(-(r + 1) // D) * D
    total = wprime + args.steps
    for rep in range(args.repeat):
        for spec in args.orders.split(","):
            cols, band = spec.split(":")
            os.environ["SLIM_CHOL_COLS"], os.environ["SLIM_CHOL_BAND"] = cols, band
            gc.collect()
            op2 = op.with_rhs(b)
            timing = {"start_step": wprime + 1}
            traj = slim.run("slimls", op2, slim.Sampler(scheme, op.n_blocks, bench.SAMPLER_SEED),
                            slim.Schedule("constant", alpha), epochs=total / op.n_blocks, r=r,
                            references={"x_true": xt}, timing=timing)
            assert traj.status == "ok"
            chol = timing["cholesky_ms"] / max(1, timing["cholesky_count"])
            print(f"rep {rep} cols={cols} band={band}: {args.steps / (timing['window_ms'] / 1e3):8.2f} "
                  f"it/s, factorization launch {chol:7.3f} ms, x_final[0..2] {traj.x_final[:2]}",
                  flush=True)
            del op2, traj


if __name__ == "__main__":
    main()
