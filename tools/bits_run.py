"""Save x_final of a short BASELINE-config run (for bit-for-bit comparison of
two library builds: SLIM_LIB=... python tools/bits_run.py 2 48 out.npy)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

cfg_id, K, out = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
import paper_1912_07962_b200 as slim  # noqa: E402
op, b, xt = bench.build_config(cfg_id)
cfg = bench.CONFIGS[cfg_id]
t = slim.run("slimls", op, slim.Sampler(cfg["scheme"], op.n_blocks, 7962),
             slim.Schedule("constant", cfg["alpha"]), epochs=K / op.n_blocks, r=cfg["r"],
             references={"x_true": xt})
np.save(out, t.x_final)
