"""Small slimLS runs for compute-sanitizer (memcheck / racecheck / synccheck).

    compute-sanitizer --tool memcheck python tools/sanitize_run.py dense
    compute-sanitizer --tool racecheck python tools/sanitize_run.py tomo

`dense`: configs[0]-shaped dense run at reduced size (4000 x 400, ell = 40,
r = 5, 2 epochs: window fill, eviction, tile reuse, the int8 factorization,
DMMA Gram, dense M^T w).  `tomo`: configs[1]-shaped CSR tomography at
reduced size (48^2 image, 40 views x 68 rays, r = 8, host-streamed blocks,
per-block CSC build, CSR Gram, fused M^T w + finish, cluster solves).
`gen`: generated rows with the tcgen05 3xTF32 Gram (n = 4096, ell = 256).
`file`: a .slim stream file read into HBM by the library.
Each run is checked against the CPU oracle so a sanitizer-perturbed run
that computes garbage is caught too.
"""

import os
import sys
import tempfile

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def _check(traj, ref, tol):
    err = np.linalg.norm(traj.x_final - ref.x_final) / np.linalg.norm(ref.x_final)
    print(f"relative error vs oracle {err:.2e}", flush=True)
    assert err <= tol, err


def main(kind):
    import paper_1912_07962_b200 as slim
    from oracle import slimls_oracle as orc
    from paper_1912_07962_b200 import problems

    if kind in ("dense", "file"):
        g = np.random.Generator(np.random.Philox(key=1912))
        a = g.standard_normal((4000, 400)) / np.sqrt(1000.0)
        xt = g.standard_normal(400)
        b = a @ xt + 0.01 * g.standard_normal(4000)
        K, r = (200, 5) if kind == "dense" else (100, 3)
        op = slim.DenseBlockOperator(a, 40, b)
        scheme = "random_cyclic" if kind == "dense" else "cyclic"
        if kind == "file":
            from paper_1912_07962_b200.slimfile import FileStreamOperator, write_stream_file
            path = os.path.join(tempfile.mkdtemp(), "s.slim")
            write_stream_file(path, op)
            op = FileStreamOperator(path)
        traj = slim.run("slimls", op, slim.Sampler(scheme, 100, 7962),
                        slim.Schedule("constant", 100.0), epochs=K / 100, r=r,
                        references={"x_true": xt})
        idx = orc.sampler_indices(scheme, 100, 7962, K)
        ref = orc.run_slimls(orc.dense_fetch(a, b, 40), 100, 400, idx, np.full(K, 100.0), r=r,
                             references={"x_true": xt})
        _check(traj, ref, 1e-10)
    elif kind == "tomo":
        prob = problems.tomo2d(grid=48, n_views=40, rays=68, seed=5)
        op, K, r = prob.op, 60, 8
        traj = slim.run("slimls", op, slim.Sampler("random_cyclic", op.n_blocks, 3),
                        slim.Schedule("constant", 1000.0), epochs=K / op.n_blocks, r=r,
                        references={"x_true": prob.x_true})
        idx = orc.sampler_indices("random_cyclic", op.n_blocks, 3, K)
        fetch = orc.csr_fetch([op.csr_block(i) for i in range(1, op.n_blocks + 1)], prob.b)
        ref = orc.run_slimls(fetch, op.n_blocks, op.n_cols, idx, np.full(K, 1000.0), r=r,
                             references={"x_true": prob.x_true})
        _check(traj, ref, 1e-10)
    elif kind == "gen":
        n, ell, m, K, r = 4096, 256, 256 * 12, 10, 6
        op, b, xt = problems.generated_dense(n=n, m=m, ell=ell, seed=44)
        traj = slim.run("slimls", op, slim.Sampler("random_cyclic", op.n_blocks, 2),
                        slim.Schedule("constant", 100.0), epochs=K / op.n_blocks, r=r,
                        references={"x_true": xt})
        idx = orc.sampler_indices("random_cyclic", op.n_blocks, 2, K)
        ref = orc.run_slimls(orc.gen_fetch(44, n, ell, b), op.n_blocks, n, idx, np.full(K, 100.0),
                             r=r, references={"x_true": xt})
        _check(traj, ref, 1e-5)
    print(f"sanitize_run {kind}: ok", flush=True)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "dense")
