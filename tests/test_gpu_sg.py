"""The plain sampled-gradient method ``sg`` (solvers.py:245-250) on the
device: the memoryless subset of the slimLS chain (residual, s = A_k^T r,
x update), SURVEY.md 8f.4. Checked against the reference's own golden runs
(tests/golden/sg_runs.npz) and the CPU oracle, for dense, CSR, generated and
column-sharded operators. Tolerance: fp64 iterates within 1e-10 relative.
"""

import numpy as np
import pytest

from tests import golden_cases as gc

pytestmark = pytest.mark.gpu

RTOL = 1e-10


@pytest.fixture(scope="module")
def slim():
    import paper_1912_07962_b200 as slim
    from paper_1912_07962_b200 import _lib
    _lib.lib()
    return slim


@pytest.mark.parametrize("name", gc.SG_CASES)
def test_sg_matches_reference(slim, name):
    c = gc.dense_case(name)
    op = slim.DenseBlockOperator(c["A"], int(c["ell"]), c["b"])
    ramp = int(c["sched_ramp"])
    sched = slim.Schedule(str(c["sched_kind"]), float(c["sched_alpha"]),
                          None if ramp < 0 else ramp, float(c["sched_decay"]))
    traj = slim.run("sg", op, slim.Sampler(str(c["scheme"]), op.n_blocks, int(c["seed"])), sched,
                    epochs=float(c["epochs"]), r=int(c["r"]), x0=c.get("x0"),
                    references=c["refs"], record_every=int(c["record_every"]),
                    store_iterates="iterates" in c)
    assert np.array_equal(traj.ks, c["ks"])
    assert traj.status == str(c["status"])
    assert (traj.diverged_at or -1) == int(c["diverged_at"])
    assert traj.row_status == list(c["row_status"])
    np.testing.assert_array_equal(traj.alphas, c["alphas"])
    scale = max(1.0, float(np.abs(c["x_final"]).max()))
    np.testing.assert_allclose(traj.x_final, c["x_final"], rtol=RTOL, atol=RTOL * 1e-2 * scale)
    np.testing.assert_allclose(traj.residual_norms, c["residual_norms"], rtol=RTOL, equal_nan=True)
    for key, vals in c["rel"].items():
        np.testing.assert_allclose(traj.rel_errors[key], vals, rtol=RTOL)
    if "iterates" in c:
        np.testing.assert_allclose(np.asarray(traj.iterates), c["iterates"], rtol=RTOL, atol=1e-12)


def test_sg_csr_tomography_vs_oracle(slim):
    from oracle import slimls_oracle as orc
    from paper_1912_07962_b200 import problems
    prob = problems.tomo2d(grid=48, n_views=40, rays=68, seed=7)
    op, K, alpha, seed = prob.op, 80, 0.01, 3
    traj = slim.run("sg", op, slim.Sampler("random_cyclic", op.n_blocks, seed),
                    slim.Schedule("constant", alpha), epochs=K / op.n_blocks,
                    references={"x_true": prob.x_true})
    idx = orc.sampler_indices("random_cyclic", op.n_blocks, seed, K)
    fetch = orc.csr_fetch([op.csr_block(i) for i in range(1, op.n_blocks + 1)], prob.b)
    ref = orc.run_slimls(fetch, op.n_blocks, op.n_cols, idx, np.full(K, alpha),
                         references={"x_true": prob.x_true}, method="sg")
    err = np.linalg.norm(traj.x_final - ref.x_final) / np.linalg.norm(ref.x_final)
    assert err <= RTOL, err
    np.testing.assert_allclose(traj.residual_norms, ref.residual_norms, rtol=RTOL, equal_nan=True)


def test_sg_generated_vs_oracle(slim):
    from oracle import slimls_oracle as orc
    from paper_1912_07962_b200 import problems
    n, ell, m, K = 1024, 64, 64 * 40, 30
    op, b, xt = problems.generated_dense(n=n, m=m, ell=ell, seed=77)
    traj = slim.run("sg", slim.SinglePassAdapter(op), slim.Sampler("cyclic", op.n_blocks, 0),
                    slim.Schedule("constant", 0.5), epochs=K / op.n_blocks,
                    references={"x_true": xt})
    idx = orc.sampler_indices("cyclic", op.n_blocks, 0, K)
    ref = orc.run_slimls(orc.gen_fetch(77, n, ell, b), op.n_blocks, n, idx, np.full(K, 0.5),
                         references={"x_true": xt}, method="sg")
    err = np.linalg.norm(traj.x_final - ref.x_final) / np.linalg.norm(ref.x_final)
    assert err <= RTOL, err


def test_sg_sharded_equals_single(slim):
    from paper_1912_07962_b200 import problems
    from paper_1912_07962_b200.parallel import LocalGroup
    prob = problems.tomo2d(grid=48, n_views=30, rays=68, seed=6)
    op, K = prob.op, 50
    kw = dict(epochs=K / op.n_blocks, references={"x_true": prob.x_true})
    single = slim.run("sg", op, slim.Sampler("random_cyclic", op.n_blocks, 5),
                      slim.Schedule("constant", 0.01), **kw)
    full, _ = LocalGroup(2).run("sg", op, lambda: slim.Sampler("random_cyclic", op.n_blocks, 5),
                                slim.Schedule("constant", 0.01), **kw)
    err = np.linalg.norm(full.x_final - single.x_final) / np.linalg.norm(single.x_final)
    assert err <= RTOL, err


def test_sg_then_slimls_on_shared_context(slim):
    """The method is set per run: an sg run and a damped-BK run (both r = 0)
    share one device context without interfering."""
    c = gc.dense_case("sg_dense")
    op = slim.DenseBlockOperator(c["A"], int(c["ell"]), c["b"])
    mk = lambda: slim.Sampler("cyclic", op.n_blocks, 0)
    a1 = slim.run("sg", op, mk(), slim.Schedule("constant", 0.01), epochs=1)
    slim.run("damped_block_kaczmarz", op, mk(), slim.Schedule("constant", 2.0), epochs=1)
    a2 = slim.run("sg", op, mk(), slim.Schedule("constant", 0.01), epochs=1)
    np.testing.assert_array_equal(a1.x_final, a2.x_final)
