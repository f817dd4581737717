"""Where the wall time of the bench's e2e leg goes: per C-ABI call and the
Python around it, for a public run() of `total` steps on a fresh operator.

usage: python tools/e2e_trace.py [config] [total]   (GPU box)
"""
import collections
import gc
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1912_07962_b200 as slim  # noqa: E402
from paper_1912_07962_b200 import linops  # noqa: E402


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    total = int(sys.argv[2]) if len(sys.argv) > 2 else 32
    spec = bench.CONFIGS[cfg]
    op, b, xt = bench.build_config(cfg)
    M = op.n_blocks
    slim.run("slimls", op, slim.Sampler(spec["scheme"], M, 1), slim.Schedule("constant", spec["alpha"]),
             epochs=12 / M, r=spec["r"])
    acc = collections.OrderedDict()
    orig = linops.DeviceOperator.call

    def timed(self, name, *a):
        t0 = time.perf_counter()
        try:
            return orig(self, name, *a)
        finally:
            acc[name] = acc.get(name, 0.0) + time.perf_counter() - t0

    linops.DeviceOperator.call = timed
    orig_init = linops.DeviceOperator.__init__

    def timed_init(self, *a, **k):
        t0 = time.perf_counter()
        orig_init(self, *a, **k)
        acc["DeviceOperator.__init__ (slim_create)"] = acc.get("DeviceOperator.__init__ (slim_create)", 0.0) + time.perf_counter() - t0

    linops.DeviceOperator.__init__ = timed_init
    for rep in range(3):
        gc.collect()
        acc.clear()
        op2 = bench._fresh(op)
        t0 = time.perf_counter()
        tr = slim.run("slimls", op2, slim.Sampler(spec["scheme"], M, 7962),
                      slim.Schedule("constant", spec["alpha"]), epochs=total / M, r=spec["r"],
                      references={"x_true": xt}, record_every=1)
        wall = time.perf_counter() - t0
        assert tr.status == "ok"
        print(f"rep {rep}: wall {1e3 * wall:8.2f} ms ({total / wall:6.1f} it/s); C calls "
              f"{1e3 * sum(acc.values()):8.2f} ms, python around them {1e3 * (wall - sum(acc.values())):7.2f} ms")
        for k, v in acc.items():
            if v > 2e-4:
                print(f"    {k:44s} {1e3 * v:9.2f} ms")
        del op2, tr


main()
