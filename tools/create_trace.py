import sys, time
sys.path.insert(0, '.')
import bench
from paper_1912_07962_b200 import linops, _lib
op, b, xt = bench.build_config(int(sys.argv[1]))
for i in range(3):
    t = time.perf_counter()
    dop = linops.DeviceOperator(n_rows=op.n_rows, n_cols=op.n_cols, ell=op.block_rows, r=int(sys.argv[2]),
                                layout=_lib.SLIM_CSR_PERBLOCK, dtype=op.dtype)
    t1 = time.perf_counter()
    del dop
    t2 = time.perf_counter()
    print(f"create {1e3*(t1-t):.1f} ms destroy {1e3*(t2-t1):.1f} ms", flush=True)
