"""Split the e2e wall time of a public run() on a fresh operator into the
device-operator registration and the run itself, streamed vs pre-uploaded.

usage: python tools/e2e_split.py [config]   (GPU box)
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1912_07962_b200 as slim  # noqa: E402
from paper_1912_07962_b200 import linops  # noqa: E402


def one(op, spec, total, M):
    t0 = time.perf_counter()
    dop = linops.device_operator(op, spec["r"], 0)
    t1 = time.perf_counter()
    tr = slim.run("slimls", op, slim.Sampler(spec["scheme"], M, 7962), slim.Schedule("constant", spec["alpha"]),
                  epochs=total / M, r=spec["r"], record_every=1)
    t2 = time.perf_counter()
    assert tr.status == "ok"
    del dop
    return 1e3 * (t1 - t0), 1e3 * (t2 - t1)


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    spec = bench.CONFIGS[cfg]
    op, b, xt = bench.build_config(cfg)
    M, total = op.n_blocks, 112
    slim.run("slimls", op, slim.Sampler(spec["scheme"], M, 1), slim.Schedule("constant", spec["alpha"]),
             epochs=4 / M, r=spec["r"])
    for mode in ("1", "0", "1"):
        os.environ["SLIM_HOST_STREAMING"] = mode
        for rep in range(3):
            op2 = op.with_rhs(op.rhs)
            reg, run = one(op2, spec, total, M)
            print(f"streaming={mode} rep {rep}: device_operator {reg:8.2f} ms  run {run:8.2f} ms  "
                  f"total {reg + run:8.2f} ms  ({total / (reg + run) * 1e3:7.1f} it/s)", flush=True)


main()
