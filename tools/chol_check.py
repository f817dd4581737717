"""Factor random SPD dual-like systems with the device tile Cholesky
(slim_potrf_traced) and compare with LAPACK; prints error and launch time.

usage: [SLIM_CHOL=dmma|i8] python tools/chol_check.py N [N ...]   (GPU box)
"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1912_07962_b200 import _lib  # noqa: E402


def main():
    mode = os.environ.get("SLIM_CHOL", "i8")
    for N in [int(a) for a in sys.argv[1:]] or [100, 600, 1000, 3982]:
        rng = np.random.default_rng(N)
        a = rng.standard_normal((N, N + 50)) / np.sqrt(N)
        a[::7] *= 30.0  # uneven row scales
        g = a @ a.T * 1000.0 + np.eye(N)
        T = (N + 63) // 64
        tr = np.zeros(4 * T * (T + 1) // 2, dtype=np.uint64)
        L = np.empty_like(g)
        ms = C.c_double(0)
        times = []
        for _ in range(3):
            _lib.check(_lib.lib().slim_potrf_traced(0, _lib.dptr(g), N, _lib.dptr(L),
                                                    tr.ctypes.data_as(C.POINTER(C.c_ulonglong)),
                                                    C.byref(ms)))
            times.append(ms.value)
        Lr = np.linalg.cholesky(g)
        Lg = np.tril(L)
        rel = np.abs(Lg - Lr).max() / np.abs(Lr).max()
        resid = np.abs(Lg @ Lg.T - g).max() / np.abs(g).max()
        # solve check, like the x-chain: w = G^-1 y
        y = rng.standard_normal(N)
        w = np.linalg.solve(Lg.T, np.linalg.solve(Lg, y))
        wr = np.linalg.solve(g, y)
        werr = np.linalg.norm(w - wr) / np.linalg.norm(wr)
        fl = N ** 3 / 3
        print(f"{mode} N={N}: max|L-Lref|/max|L| {rel:.2e}  backward {resid:.2e}  "
              f"solve {werr:.2e}  ms {min(times):.3f}  ({fl / min(times) / 1e9:.2f} TF/s fp64-eq)",
              flush=True)


if __name__ == "__main__":
    main()
