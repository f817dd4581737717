"""Where the end-to-end time of a public run() goes (one configuration).

usage: python tools/e2e_phases.py [config]   (GPU box)
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1912_07962_b200 as slim  # noqa: E402
from paper_1912_07962_b200 import _lib, linops  # noqa: E402


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    spec = bench.CONFIGS[cfg]
    op, b, xt = bench.build_config(cfg)
    M, r, alpha = op.n_blocks, spec["r"], spec["alpha"]
    total = 112
    # warm the CUDA context / module load
    slim.run("slimls", op, slim.Sampler(spec["scheme"], M, 1), slim.Schedule("constant", alpha),
             epochs=4 / M, r=r)
    op2, b2, _ = bench.build_config(cfg)
    src = op2
    t = {}
    t0 = time.perf_counter()
    if isinstance(src, linops.SparseBlockOperator):
        rowptr, col, val = src.global_csr()
        t["global_csr"] = time.perf_counter() - t0
        t1 = time.perf_counter()
        dop = linops.DeviceOperator(n_rows=src.n_rows, n_cols=src.n_cols, ell=src.block_rows, r=r,
                                    layout=_lib.SLIM_CSR_PERBLOCK, dtype=src.dtype)
        t["slim_create"] = time.perf_counter() - t1
        t1 = time.perf_counter()
        bb = np.ascontiguousarray(src.rhs, dtype=float)
        dop.call("slim_upload_csr", _lib.i64ptr(rowptr), _lib.i32ptr(col),
                 _lib.vptr(np.ascontiguousarray(val)), _lib.dptr(bb))
        t["upload_csr"] = time.perf_counter() - t1
        t1 = time.perf_counter()
        dop.call("slim_finalize_operator")
        t["finalize"] = time.perf_counter() - t1
        del dop
    t2 = time.perf_counter()
    tr = slim.run("slimls", op2, slim.Sampler(spec["scheme"], M, 7962),
                  slim.Schedule("constant", alpha), epochs=total / M, r=r,
                  references={"x_true": xt}, record_every=1)
    t["public_run_total"] = time.perf_counter() - t2
    t3 = time.perf_counter()
    tr = slim.run("slimls", op2, slim.Sampler(spec["scheme"], M, 7962),
                  slim.Schedule("constant", alpha), epochs=total / M, r=r,
                  references={"x_true": xt}, record_every=1)
    t["public_run_cached_operator"] = time.perf_counter() - t3
    for k, v in t.items():
        print(f"{k:28s} {1e3 * v:9.2f} ms")
    print("status", tr.status)


main()
