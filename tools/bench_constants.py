"""||A x_true|| of the large tomography configs (configs[2], configs[3]).

bench.py's reference arm builds only the views its bounded sample touches
(with the reference's own projector, no libslimb200.so) and scales the 1%
noise with these whole-operator norms, so its b matches the full problem's
noise convention (tomo.py:323-333).  Computed once with the host projector:

    python tools/bench_constants.py
"""

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_1912_07962_b200 import problems

    for cfg, mk in ((3, lambda: problems.tomo2d(grid=1024, n_views=720, rays=1448, seed=3,
                                                dtype=np.float32)),
                    (4, lambda: problems.tomo3d(grid=128, n_views=180, side=128, sub_rows=2048,
                                                seed=4))):
        p = mk()
        clean = np.concatenate([problems._csr_matvec(ip, ix, d.astype(np.float64), p.x_true)
                                for ip, ix, d, _ in (p.op.csr_block(i)
                                                     for i in range(1, p.op.n_blocks + 1))])
        print(f"{cfg}: {float(np.linalg.norm(clean))!r}", flush=True)
        del p, clean


if __name__ == "__main__":
    main()
