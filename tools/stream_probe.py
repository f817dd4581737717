"""Cold-L2 probe of the operator-streaming kernels (slim_probe_stream) on a
BASELINE config, for kernel A/B (e.g. SLIM_MTW_QUAD variants):

    SLIM_MTW_QUAD=2 python tools/stream_probe.py --config 3
"""

import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--reps", type=int, default=24)
    args = ap.parse_args()
    import paper_1912_07962_b200 as slim
    from paper_1912_07962_b200.linops import device_operator

    os.environ["SLIM_HOST_STREAMING"] = "0"
    op, b, xt = bench.build_config(args.config)
    cfg = bench.CONFIGS[args.config]
    slim.run("slimls", op, slim.Sampler(cfg["scheme"], op.n_blocks, 7962),
             slim.Schedule("constant", cfg["alpha"]), epochs=(cfg["r"] + 2) / op.n_blocks, r=cfg["r"])
    dop = device_operator(op, cfg["r"], 0)
    peak = float(bench._peaks().get("hbm_gbs", 6543.7))
    tag = os.environ.get("SLIM_MTW_QUAD", "default")
    for kid, name in ((0, "residual"), (1, "mtw"), (2, "gram")):
        us, nb = C.c_double(0), C.c_double(0)
        try:
            dop.call("slim_probe_stream", kid, args.reps, C.byref(us), C.byref(nb))
        except ValueError:
            continue
        gbs = nb.value / (us.value * 1e-6) / 1e9
        print(f"config {args.config} quad={tag} {name:8s}: {us.value:8.1f} us  {nb.value / 1e6:8.1f} MB  "
              f"{gbs:7.0f} GB/s  {gbs / peak:5.1%}", flush=True)


if __name__ == "__main__":
    main()
