"""Timeline of one tile-DAG Cholesky (debug): where the critical path goes."""
import ctypes as C
import json
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1912_07962_b200 import _lib  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 3982
rng = np.random.default_rng(0)
a = rng.standard_normal((N, N + 50)) / np.sqrt(N)
g = a @ a.T * 1000.0 + np.eye(N)
T = (N + 63) // 64
nt = T * (T + 1) // 2  # buffer sized for tiles; tasks use the first T(T-1)/2+1
tr = np.zeros(4 * nt, dtype=np.uint64)
L = np.empty_like(g)
ms = C.c_double(0)
_lib.check(_lib.lib().slim_potrf_traced(0, _lib.dptr(g), N, _lib.dptr(L),
                                        tr.ctypes.data_as(C.POINTER(C.c_uint64)), C.byref(ms)))
tr = tr.reshape(nt, 4).astype(np.int64)[: T * (T - 1) // 2 + 1]
t0 = tr[:, 0].min()
tr = tr - t0
# ticket -> task, same order as task_order_one() in chol.cu
order = [(0, 0)]
for j in range(T):
    if j + 2 < T:
        order.append((j + 2, j))
    if j + 1 < T:
        order.append((j + 1, j + 1))
    order += [(i, j) for i in range(j + 3, T)]
pair = {j: t for t, (i, jj) in enumerate(order) if i == jj for j in [jj]}
err = np.abs(L - np.linalg.cholesky(g)).max()
print(f"N={N} T={T} event time {ms.value:.3f} ms, trace span {tr[:, 3].max() / 1e3:.1f} us, max|L-Lref|={err:.2e}")
potrf, sub, gap = [], [], []
for j in range(T - 1):
    a, b = tr[pair[j]], tr[pair[j + 1]]
    potrf.append(a[2] - a[1])
    sub.append(a[3] - a[2])
    gap.append(b[1] - a[3])
for name, v in (("potrf", potrf), ("publish+sub trsm", sub), ("-> next diag ready", gap)):
    v = np.asarray(v) / 1e3
    print(f"  {name:20s} mean {v.mean():7.2f} us  median {np.median(v):7.2f}  max {v.max():7.2f}")
print("  diag publish times (us):", (tr[[pair[j] for j in range(0, T, max(1, T // 12))], 2] / 1e3).round(1).tolist())
print("  dispatch percentiles (us):", [round(float(np.percentile(tr[:, 0], q)) / 1e3, 1) for q in (0, 25, 50, 75, 100)])
