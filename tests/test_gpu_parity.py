"""GPU parity: the CUDA path (through the C-ABI) against the reference's
golden vectors and the CPU oracle on the same seeded inputs.

Tolerances (north_star): fp64 iterates within 1e-10 relative, fp32-matrix
configs within 1e-4 relative after K steps.
"""

import numpy as np
import pytest

from tests import golden_cases as gc

pytestmark = pytest.mark.gpu

RTOL64 = 1e-10
QX_DEFAULT = 1  # kernels.h SLIM_QX


@pytest.fixture(scope="module")
def slim():
    import paper_1912_07962_b200 as slim
    from paper_1912_07962_b200 import _lib
    _lib.lib()  # fail loudly if the extension is missing
    return slim


def _run_dense_case(slim, c, **kw):
    op = slim.DenseBlockOperator(c["A"], int(c["ell"]), c["b"])
    scheme = str(c["scheme"])
    if kw.pop("single_pass", False):
        op = slim.SinglePassAdapter(op)
    kind = str(c["sched_kind"])
    ramp = int(c["sched_ramp"])
    sched = slim.Schedule(kind, float(c["sched_alpha"]), None if ramp < 0 else ramp,
                          float(c["sched_decay"]))
    return slim.run("slimls", op, slim.Sampler(scheme, op.n_blocks, int(c["seed"])), sched,
                    epochs=float(c["epochs"]), r=int(c["r"]), x0=c.get("x0"),
                    references=c["refs"], record_every=int(c["record_every"]),
                    store_iterates="iterates" in c, **kw)


def _assert_traj(traj, c, rtol=RTOL64):
    assert np.array_equal(traj.ks, c["ks"])
    assert traj.status == str(c["status"])
    assert (traj.diverged_at or -1) == int(c["diverged_at"])
    assert traj.row_status == list(c["row_status"])
    np.testing.assert_array_equal(traj.epoch_fraction, c["epoch_fraction"])
    np.testing.assert_array_equal(traj.alphas, c["alphas"])
    scale = max(1.0, float(np.abs(c["x_final"]).max()))
    np.testing.assert_allclose(traj.x_final, c["x_final"], rtol=rtol, atol=rtol * 1e-2 * scale)
    np.testing.assert_allclose(traj.residual_norms, c["residual_norms"], rtol=rtol, equal_nan=True)
    for name, vals in c["rel"].items():
        np.testing.assert_allclose(traj.rel_errors[name], vals, rtol=rtol)
    assert np.all(np.diff(np.cumsum(traj.wall_times)) >= 0)


@pytest.mark.parametrize("name", gc.DENSE_CASES)
def test_dense_runs_match_reference(slim, name):
    c = gc.dense_case(name)
    traj = _run_dense_case(slim, c, single_pass=(name == "single_pass"))
    _assert_traj(traj, c)
    if "iterates" in c:
        np.testing.assert_allclose(np.asarray(traj.iterates), c["iterates"], rtol=RTOL64,
                                   atol=1e-12)


@pytest.mark.parametrize("name", ["tomo2d", "tomo3d"])
def test_tomo_runs_match_reference(slim, name):
    c = gc.tomo_case(name)
    op = slim.SparseBlockOperator(c["blocks"], c["b"])
    k = len(c["indices"])
    scheme = "random_cyclic" if name == "tomo2d" else "uniform_iid"
    seed = 7 if name == "tomo2d" else 3
    traj = slim.run("slimls", op, slim.Sampler(scheme, op.n_blocks, seed),
                    slim.Schedule("constant", float(c["alpha"])),
                    epochs=k / op.n_blocks, r=int(c["r"]), references={"x_true": c["x_true"]})
    np.testing.assert_allclose(traj.x_final, c["x_final"], rtol=RTOL64,
                               atol=RTOL64 * np.abs(c["x_final"]).max())
    np.testing.assert_allclose(traj.rel_errors["x_true"], c["rel"]["x_true"], rtol=RTOL64)
    np.testing.assert_allclose(traj.residual_norms, c["residual_norms"], rtol=RTOL64,
                               equal_nan=True)


def test_dual_step_seam_matches_reference(slim):
    d = gc.load("dual_step.npz")
    for q in range(4):
        m = d[f"{q}/M"]
        ell = int(d[f"{q}/ell"])
        blocks = [m[i:i + ell] for i in range(0, m.shape[0], ell)]
        s = slim.dual_step(blocks, d[f"{q}/residual"], float(d[f"{q}/alpha"]))
        np.testing.assert_allclose(s, d[f"{q}/s"], rtol=1e-10, atol=1e-13)


@pytest.mark.parametrize("n", [1, 5, 63, 64, 65, 130, 257, 600, 1000])
def test_potrf_matches_numpy(slim, n):
    rng = np.random.default_rng(n)
    a = rng.standard_normal((n, n + 3))
    g = a @ a.T + n * np.eye(n)
    L = slim.potrf(g)
    ref = np.linalg.cholesky(g)
    np.testing.assert_allclose(L, ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())


def test_potrf_rejects_indefinite(slim):
    g = np.eye(70)
    g[40, 40] = -1.0
    with pytest.raises(np.linalg.LinAlgError):
        slim.potrf(g)


def test_same_seed_bit_identical(slim):
    c = gc.dense_case("dense_dual")
    t1 = _run_dense_case(slim, c)
    t2 = _run_dense_case(slim, c)
    assert np.array_equal(t1.x_final, t2.x_final)
    for name in t1.rel_errors:
        assert np.array_equal(t1.rel_errors[name], t2.rel_errors[name])
    assert np.array_equal(t1.residual_norms, t2.residual_norms, equal_nan=True)


def test_errors_map_to_reference_exceptions(slim):
    c = gc.dense_case("ramp")
    op = slim.DenseBlockOperator(c["A"], 6, c["b"])
    smp = slim.Sampler("cyclic", op.n_blocks, 0)
    with pytest.raises(ValueError, match="unknown method"):
        slim.run("nope", op, smp, slim.Schedule(), epochs=1)
    with pytest.raises(ValueError, match="epochs"):
        slim.run("slimls", op, smp, slim.Schedule(), epochs=-1)
    with pytest.raises(ValueError, match="record_every"):
        slim.run("slimls", op, smp, slim.Schedule(), epochs=1, record_every=0)
    with pytest.raises(ValueError, match="memory level"):
        slim.run("slimls", op, smp, slim.Schedule(), epochs=1, r=-1)
    with pytest.raises(ValueError, match="not on the B200"):
        slim.run("olbfgs", op, smp, slim.Schedule(), epochs=1)
    sp = slim.SinglePassAdapter(op)
    with pytest.raises(ValueError, match="cyclic"):
        slim.run("slimls", sp, slim.Sampler("uniform_iid", op.n_blocks, 0), slim.Schedule(),
                 epochs=1)
    with pytest.raises(ValueError, match="one epoch"):
        slim.run("slimls", sp, slim.Sampler("cyclic", op.n_blocks, 0), slim.Schedule(), epochs=2)
    # a consumed single-pass stream cannot be replayed
    slim.run("slimls", sp, slim.Sampler("cyclic", op.n_blocks, 0), slim.Schedule(), epochs=1)
    with pytest.raises(slim.StreamOrderError):
        slim.run("slimls", sp, slim.Sampler("cyclic", op.n_blocks, 0), slim.Schedule(), epochs=1)


def test_specialisations(slim):
    """damped_block_kaczmarz == slimls(r=0); slimtik(lam=0) == slimls (bitwise)."""
    c = gc.dense_case("r0")
    op = slim.DenseBlockOperator(c["A"], 6, c["b"])
    kw = dict(epochs=2, references={"x_true": np.ones(40)})
    base = slim.run("slimls", op, slim.Sampler("random_cyclic", 15, 3),
                    slim.Schedule("constant", 2.0), r=0, **kw)
    dbk = slim.run("damped_block_kaczmarz", op, slim.Sampler("random_cyclic", 15, 3),
                   slim.Schedule("constant", 2.0), r=0, **kw)
    assert np.array_equal(base.x_final, dbk.x_final)
    t1 = slim.run("slimls", op, slim.Sampler("random_cyclic", 15, 3),
                  slim.Schedule("constant", 2.0), r=2, **kw)
    t2 = slim.run("slimtik", op, slim.Sampler("random_cyclic", 15, 3),
                  slim.Schedule("constant", 2.0), r=2, lam=0.0, **kw)
    assert np.array_equal(t1.x_final, t2.x_final)


# ---------------------------------------------------------------------------
# against the CPU oracle on BASELINE-shaped inputs (reduced where the oracle
# would take minutes)
# ---------------------------------------------------------------------------


def _oracle_run(op_dense_fetch, nb, n, idx, alpha, r, refs, record_every=1):
    from oracle import slimls_oracle as orc
    return orc.run_slimls(op_dense_fetch, nb, n, idx, np.full(len(idx), alpha), r=r,
                          references=refs, record_every=record_every)


def test_config1_vs_oracle(slim):
    """configs[0] at full size, 300 steps (window full from step 6)."""
    from oracle import slimls_oracle as orc
    from paper_1912_07962_b200 import problems
    op, b, xt = problems.gaussian_dense()
    K = 300
    traj = slim.run("slimls", op, slim.Sampler("random_cyclic", 200, 7962),
                    slim.Schedule("constant", 100.0), epochs=K / 200, r=5,
                    references={"x_true": xt}, record_every=10)
    idx = orc.sampler_indices("random_cyclic", 200, 7962, K)
    ref = _oracle_run(orc.dense_fetch(op.matrix, b, 100), 200, 1000, idx, 100.0, 5,
                      {"x_true": xt}, record_every=10)
    np.testing.assert_allclose(traj.x_final, ref.x_final, rtol=RTOL64,
                               atol=RTOL64 * np.abs(ref.x_final).max())
    np.testing.assert_allclose(traj.rel_errors["x_true"], ref.rel_errors["x_true"], rtol=RTOL64)
    np.testing.assert_allclose(traj.residual_norms, ref.residual_norms, rtol=RTOL64,
                               equal_nan=True)


def _tomo_vs_oracle(slim, prob, K, r, alpha, seed, rtol):
    from oracle import slimls_oracle as orc
    op = prob.op
    traj = slim.run("slimls", op, slim.Sampler("random_cyclic", op.n_blocks, seed),
                    slim.Schedule("constant", alpha), epochs=K / op.n_blocks, r=r,
                    references={"x_true": prob.x_true})
    idx = orc.sampler_indices("random_cyclic", op.n_blocks, seed, K)
    fetch = orc.csr_fetch([op.csr_block(i) for i in range(1, op.n_blocks + 1)], prob.b)
    ref = _oracle_run(fetch, op.n_blocks, op.n_cols, idx, alpha, r, {"x_true": prob.x_true})
    err = np.linalg.norm(traj.x_final - ref.x_final) / np.linalg.norm(ref.x_final)
    assert err <= rtol, err
    np.testing.assert_allclose(traj.rel_errors["x_true"], ref.rel_errors["x_true"], rtol=rtol)
    np.testing.assert_allclose(traj.residual_norms, ref.residual_norms, rtol=rtol, equal_nan=True)


def test_config2_reduced_vs_oracle(slim):
    """configs[1] geometry at 64^2 (n = 4096, 45 views x 90 rays), r = 10,
    lambda = 1e-3: eviction exercised, kappa ~ 1e6 dual system."""
    from paper_1912_07962_b200 import problems
    prob = problems.tomo2d(grid=64, n_views=45, rays=90, seed=2)
    _tomo_vs_oracle(slim, prob, K=30, r=10, alpha=1000.0, seed=11, rtol=RTOL64)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_refined_six_digit_factorization_vs_oracle(slim, monkeypatch, dtype):
    """The six-digit int8 factorization with one refinement step of w against
    the fp64 Gram ring (the default for dual systems above 6144 rows; forced
    here with SLIM_REFINE=1 on the kappa ~ 1e6 reduced tomography) holds the
    fp64 bar, is bit-identical run to run, and reports its layout."""
    from oracle import slimls_oracle as orc
    from paper_1912_07962_b200 import problems
    monkeypatch.setenv("SLIM_REFINE", "1")
    prob = problems.tomo2d(grid=64, n_views=45, rays=90, seed=2, dtype=dtype)
    op, K, r, alpha, seed = prob.op, 30, 10, 1000.0, 11
    runs = []
    for _ in range(2):
        timing = {"start_step": 1}
        fresh = op.with_rhs(op.rhs)
        runs.append(slim.run("slimls", fresh, slim.Sampler("random_cyclic", op.n_blocks, seed),
                             slim.Schedule("constant", alpha), epochs=K / op.n_blocks, r=r,
                             references={"x_true": prob.x_true}, timing=timing))
        assert timing["cholesky_digits"][0] == 6 and timing["cholesky_pairs"] == (21, 0)
    np.testing.assert_array_equal(runs[0].x_final, runs[1].x_final)
    idx = orc.sampler_indices("random_cyclic", op.n_blocks, seed, K)
    fetch = orc.csr_fetch([op.csr_block(i) for i in range(1, op.n_blocks + 1)], prob.b)
    ref = _oracle_run(fetch, op.n_blocks, op.n_cols, idx, alpha, r, {"x_true": prob.x_true})
    err = np.linalg.norm(runs[0].x_final - ref.x_final) / np.linalg.norm(ref.x_final)
    print(f"six digits + refinement ({np.dtype(dtype).name} values): relative iterate error vs oracle {err:.2e}")
    assert err <= RTOL64, err
    np.testing.assert_allclose(runs[0].residual_norms, ref.residual_norms, rtol=RTOL64, equal_nan=True)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_fixed_point_csr_gram_general_sparse(slim, monkeypatch, dtype):
    """The record / fixed-point CSR Gram kernel (k_gram_rowexp + k_gram_lut +
    k_gram_csr_fx; chosen from 2^18 nonzeros per block, forced here) on a
    general sparse operator: signed entries, ~6 entries per column and block
    (the path past the two packed entries), row scales spread over 10^-3 .. 10^3,
    an empty row and an empty column.  Same bar as the fp64 kernel, and the
    two kernels' iterates agree far inside it."""
    import scipy.sparse as sp
    from oracle import slimls_oracle as orc
    g = np.random.Generator(np.random.Philox(key=77))
    n, ell, nb, r, alpha, K = 384, 48, 12, 4, 50.0, 30
    blocks = []
    for _ in range(nb):
        a = sp.random(ell, n, density=0.12, random_state=g, data_rvs=g.standard_normal, format="csr")
        a = sp.diags(10.0 ** g.uniform(-3, 3, ell)) @ a
        a = a.tolil()
        a[5, :] = 0.0          # an empty row
        a[:, 17] = 0.0         # an empty column
        a = a.tocsr()
        a.sort_indices()
        blocks.append(a.astype(dtype))
    xt = g.standard_normal(n)
    b = np.concatenate([blk.astype(float) @ xt for blk in blocks])
    b = b + 1e-3 * np.abs(b).mean() * g.standard_normal(b.shape)
    xs = {}
    for lut in ("1", "0"):
        monkeypatch.setenv("SLIM_GRAM_LUT", lut)
        op = slim.SparseBlockOperator(blocks, b)
        xs[lut] = slim.run("slimls", op, slim.Sampler("random_cyclic", nb, 4),
                           slim.Schedule("constant", alpha), epochs=K / nb, r=r)
    parts = [(blk.indptr, blk.indices, blk.data, blk.shape) for blk in blocks]
    idx = orc.sampler_indices("random_cyclic", nb, 4, K)
    ref = _oracle_run(orc.csr_fetch(parts, b), nb, n, idx, alpha, r, {})
    nrm = np.linalg.norm(ref.x_final)
    err = {k: np.linalg.norm(v.x_final - ref.x_final) / nrm for k, v in xs.items()}
    diff = np.linalg.norm(xs["1"].x_final - xs["0"].x_final) / nrm
    print(f"general sparse ({np.dtype(dtype).name}): fixed-point Gram vs oracle {err['1']:.2e}, "
          f"fp64 Gram vs oracle {err['0']:.2e}, the two kernels differ by {diff:.2e}")
    assert err["1"] <= RTOL64 and err["0"] <= RTOL64
    np.testing.assert_allclose(xs["1"].residual_norms, ref.residual_norms, rtol=RTOL64, equal_nan=True)


def test_fp32_tomo_reduced_vs_oracle(slim):
    """configs[2] style: fp32 values / int32 indices, fp64 accumulation (1e-4 bar;
    the oracle sees the same fp32-rounded values)."""
    from paper_1912_07962_b200 import problems
    prob = problems.tomo2d(grid=48, n_views=40, rays=68, seed=5, dtype=np.float32)
    _tomo_vs_oracle(slim, prob, K=25, r=8, alpha=1000.0, seed=3, rtol=1e-4)


def test_block_residual(slim):
    from paper_1912_07962_b200 import problems
    from paper_1912_07962_b200.linops import device_operator
    from paper_1912_07962_b200 import _lib
    prob = problems.tomo2d(grid=32, n_views=10, rays=46, seed=9)
    dop = device_operator(prob.op, 2)
    x = np.random.default_rng(0).standard_normal(prob.op.n_cols)
    r = np.empty(46)
    nrm = np.zeros(1)
    dop.call("slim_block_residual", 4, _lib.dptr(x), _lib.dptr(r), _lib.dptr(nrm))
    blk = prob.op.fetch_block(4)
    ref = blk.a_block @ x - blk.b_block
    np.testing.assert_allclose(r, ref, rtol=1e-12, atol=1e-12)


# ---------------------------------------------------------------------------
# configs[4]: generated operator (splitmix64 rows, never stored)
# ---------------------------------------------------------------------------


def test_generated_device_rows_bit_exact(slim):
    """Device generator == host generator: A x computed both ways agrees to
    fp64 summation-order level, and one generated block's residual matches."""
    from paper_1912_07962_b200.linops import GeneratedBlockOperator, device_operator
    from paper_1912_07962_b200 import _lib
    from oracle import slimls_oracle as orc
    n, ell, m = 3000, 40, 400
    op = GeneratedBlockOperator(m, n, ell, seed=5)
    x = np.random.default_rng(1).standard_normal(n)
    dev = op.apply_device(x)
    host = orc.gen_rows(5, 0, m, n) @ x
    np.testing.assert_allclose(dev, host, rtol=1e-12, atol=1e-13)
    op = op.with_rhs(host)
    dop = device_operator(op, 2)
    r = np.empty(ell)
    nrm = np.zeros(1)
    dop.call("slim_block_residual", 7, _lib.dptr(x), _lib.dptr(r), _lib.dptr(nrm))
    ref = orc.gen_rows(5, 6 * ell, ell, n) @ x - host[6 * ell:7 * ell]
    np.testing.assert_allclose(r, ref, atol=1e-12)


def test_generated_run_vs_oracle(slim):
    """configs[4] shape at reduced size: n = 2048, ell = 64, r = 20, lambda = 1e-2,
    cyclic single pass; window fills at step 21, 30 steps checked."""
    from oracle import slimls_oracle as orc
    from paper_1912_07962_b200 import problems
    n, ell, m, K, r = 2048, 64, 64 * 48, 30, 20
    op, b, xt = problems.generated_dense(n=n, m=m, ell=ell, seed=1912)
    traj = slim.run("slimls", slim.SinglePassAdapter(op), slim.Sampler("cyclic", op.n_blocks, 0),
                    slim.Schedule("constant", 100.0), epochs=K / op.n_blocks, r=r,
                    references={"x_true": xt})
    idx = orc.sampler_indices("cyclic", op.n_blocks, 0, K)
    ref = orc.run_slimls(orc.gen_fetch(1912, n, ell, b), op.n_blocks, n, idx, np.full(K, 100.0),
                         r=r, references={"x_true": xt})
    err = np.linalg.norm(traj.x_final - ref.x_final) / np.linalg.norm(ref.x_final)
    assert err <= 1e-10, err
    np.testing.assert_allclose(traj.rel_errors["x_true"], ref.rel_errors["x_true"], rtol=1e-10)
    np.testing.assert_allclose(traj.residual_norms, ref.residual_norms, rtol=1e-10, equal_nan=True)


# ---------------------------------------------------------------------------
# BASELINE configs at FULL size: the first steps against the oracle (the
# dense-fetch oracle for configs[1]/[4], the sparse dual-form restatement for
# configs[2]/[3] whose dense blocks would need 12-34 GB each)
# ---------------------------------------------------------------------------


def _full_vs_oracle(slim, op, b, xt, r, alpha, scheme, K, rtol, sparse=False):
    from oracle import slimls_oracle as orc
    M = op.n_blocks
    traj = slim.run("slimls", op, slim.Sampler(scheme, M, 7962), slim.Schedule("constant", alpha),
                    epochs=K / M, r=r, references={"x_true": xt})
    idx = orc.sampler_indices(scheme, M, 7962, K)
    al = np.full(K, alpha)
    if sparse:
        ref = orc.run_slimls_sparse([op.csr_block(i) for i in range(1, M + 1)], b, idx, al, r=r,
                                    references={"x_true": xt})
    else:
        import bench
        ref = orc.run_slimls(bench.oracle_fetch(op, b), M, op.n_cols, idx, al, r=r,
                             references={"x_true": xt})
    err = np.linalg.norm(traj.x_final - ref.x_final) / np.linalg.norm(ref.x_final)
    print(f"relative iterate error vs oracle after {K} steps: {err:.2e}")
    assert err <= rtol, err
    np.testing.assert_allclose(traj.rel_errors["x_true"], ref.rel_errors["x_true"], rtol=rtol)
    np.testing.assert_allclose(traj.residual_norms, ref.residual_norms, rtol=rtol, equal_nan=True)
    return err


def test_config2_full_size_vs_oracle(slim):
    """configs[1] at full size: window fill (11 steps) + 3 full-window steps."""
    import bench
    op, b, xt = bench.build_config(2)
    _full_vs_oracle(slim, op, b, xt, 10, 1000.0, "random_cyclic", 14, RTOL64)


def test_config3_full_size_first_steps(slim):
    """configs[2] (1024^2, 720 x 1448, fp32 CSR) at full size, 3 steps vs the
    sparse restatement (fp32 bar 1e-4; fp64 arithmetic gives ~1e-12)."""
    import bench
    op, b, xt = bench.build_config(3)
    _full_vs_oracle(slim, op, b, xt, 8, 1000.0, "random_cyclic", 3, 1e-10, sparse=True)


def test_config4_full_size_first_steps(slim):
    """configs[3] (128^3, 180 x 128^2 rays in 2048-row sub-blocks, fp32 CSR)."""
    import bench
    op, b, xt = bench.build_config(4)
    _full_vs_oracle(slim, op, b, xt, 5, 1000.0, "random_cyclic", 3, 1e-10, sparse=True)


def test_config5_full_size_first_steps(slim):
    """configs[4] (n = 65,536 generated rows) at full size, 3 single-pass steps.
    The Gram runs as 3xTF32 on tcgen05 (fp32-matrix bar 1e-4; tested at 1e-5)."""
    import bench
    op, b, xt = bench.build_config(5)
    _full_vs_oracle(slim, op, b, xt, 20, 100.0, "cyclic", 3, 1e-5)


@pytest.mark.parametrize("tc", ["1", "0"])
def test_generated_tensor_core_gram(slim, tc, monkeypatch):
    """ell = 256 generated blocks: tcgen05 3xTF32 Gram (1e-5) and the fp64 DMMA
    fallback (SLIM_GRAM_TC=0, 1e-10) against the oracle, window filled (r = 6)."""
    from oracle import slimls_oracle as orc
    from paper_1912_07962_b200 import problems
    monkeypatch.setenv("SLIM_GRAM_TC", tc)
    n, ell, m, K, r = 8192, 256, 256 * 16, 12, 6
    op, b, xt = problems.generated_dense(n=n, m=m, ell=ell, seed=44)
    traj = slim.run("slimls", op, slim.Sampler("random_cyclic", op.n_blocks, 2),
                    slim.Schedule("constant", 100.0), epochs=K / op.n_blocks, r=r,
                    references={"x_true": xt})
    idx = orc.sampler_indices("random_cyclic", op.n_blocks, 2, K)
    ref = orc.run_slimls(orc.gen_fetch(44, n, ell, b), op.n_blocks, n, idx, np.full(K, 100.0),
                         r=r, references={"x_true": xt})
    err = np.linalg.norm(traj.x_final - ref.x_final) / np.linalg.norm(ref.x_final)
    assert err <= (1e-5 if tc == "1" else 1e-10), err
    np.testing.assert_allclose(traj.rel_errors["x_true"], ref.rel_errors["x_true"],
                               rtol=1e-5 if tc == "1" else 1e-10)


# ---------------------------------------------------------------------------
# column sharding through the real GPU path: P shards on one device (local
# group, one host thread per shard) against the unsharded run
# ---------------------------------------------------------------------------


def _sharded_vs_single(slim, op, xt, scheme, seed, alpha, r, K, P, round_robin=False):
    from oracle import slimls_oracle as orc
    from paper_1912_07962_b200.parallel import LocalGroup
    M = op.n_blocks
    kw = dict(epochs=K / M, r=r, references={"x_true": xt})
    single = slim.run("slimls", op, slim.Sampler(scheme, M, seed), slim.Schedule("constant", alpha),
                      **kw)
    group = LocalGroup(P, round_robin=round_robin)
    full, per = group.run("slimls", op, lambda: slim.Sampler(scheme, M, seed),
                          slim.Schedule("constant", alpha), **kw)
    # the sharded run against the CPU oracle too (not only against the unsharded run)
    import bench
    idx = orc.sampler_indices(scheme, M, seed, K)
    ref = orc.run_slimls(bench.oracle_fetch(op, op.rhs), M, op.n_cols, idx, np.full(K, alpha), r=r,
                         references={"x_true": xt})
    err_o = np.linalg.norm(full.x_final - ref.x_final) / np.linalg.norm(ref.x_final)
    print(f"{P} shards{' round-robin' if round_robin else ''}: relative error vs oracle {err_o:.2e}")
    assert err_o <= 1e-10, err_o
    np.testing.assert_allclose(full.rel_errors["x_true"], ref.rel_errors["x_true"], rtol=1e-10)
    err = np.linalg.norm(full.x_final - single.x_final) / np.linalg.norm(single.x_final)
    assert err <= 1e-10, err
    np.testing.assert_allclose(full.rel_errors["x_true"], single.rel_errors["x_true"], rtol=1e-10)
    np.testing.assert_allclose(full.residual_norms, single.residual_norms, rtol=1e-10,
                               equal_nan=True)
    for t in per[1:]:  # every shard records the same global history
        np.testing.assert_array_equal(t.rel_errors["x_true"], per[0].rel_errors["x_true"])
        assert np.array_equal(t.ks, per[0].ks)


@pytest.mark.parametrize("P", [2, 4])
def test_sharded_dense(slim, P):
    c = gc.dense_case("dense_dual")
    op = slim.DenseBlockOperator(c["A"], 20, c["b"])
    _sharded_vs_single(slim, op, c["refs"]["x_true"], "random_cyclic", 11, 100.0, 4, 60, P)


@pytest.mark.parametrize("P", [2, 3])
def test_sharded_csr_tomography(slim, P):
    from paper_1912_07962_b200 import problems
    prob = problems.tomo2d(grid=48, n_views=30, rays=68, seed=6)
    _sharded_vs_single(slim, prob.op, prob.x_true, "random_cyclic", 5, 1000.0, 6, 40, P)


@pytest.mark.parametrize("P", [2, 3])
def test_sharded_round_robin_tomography(slim, P):
    """factorizations distributed over the shards (batch B on
    rank B mod P), w allreduced from its owner."""
    from paper_1912_07962_b200 import problems
    prob = problems.tomo2d(grid=48, n_views=30, rays=68, seed=6)
    _sharded_vs_single(slim, prob.op, prob.x_true, "random_cyclic", 5, 1000.0, 6, 60, P,
                       round_robin=True)


@pytest.mark.parametrize("round_robin", [False, True])
def test_sharded_tomography_with_refinement(slim, monkeypatch, round_robin):
    """Column shards with the six-digit factorization and its refinement step
    forced (SLIM_REFINE=1; the default for dual systems above 6144 rows): the
    refinement reads the allreduced Gram ring on the x-chain of the rank that
    solves the step, replicated or round-robin."""
    from paper_1912_07962_b200 import problems
    monkeypatch.setenv("SLIM_REFINE", "1")
    prob = problems.tomo2d(grid=48, n_views=30, rays=68, seed=6)
    op = prob.op.with_rhs(prob.op.rhs)  # fresh contexts: the variant is chosen at creation
    _sharded_vs_single(slim, op, prob.x_true, "random_cyclic", 5, 1000.0, 6, 40, 2,
                       round_robin=round_robin)


def test_sharded_round_robin_dense(slim):
    c = gc.dense_case("dense_dual")
    op = slim.DenseBlockOperator(c["A"], 20, c["b"])
    _sharded_vs_single(slim, op, c["refs"]["x_true"], "random_cyclic", 11, 100.0, 4, 60, 2,
                       round_robin=True)


def test_sharded_generated(slim):
    from paper_1912_07962_b200 import problems
    op, b, xt = problems.generated_dense(n=1536, m=64 * 30, ell=64, seed=9)
    _sharded_vs_single(slim, op, xt, "cyclic", 0, 100.0, 8, 20, 2)


# ---------------------------------------------------------------------------
# host streaming: blocks copied to HBM inside the run, in first-use order
# ---------------------------------------------------------------------------


def _run_fresh(slim, make_op, monkeypatch, streaming, scheme, seed, alpha, r, K, refs):
    monkeypatch.setenv("SLIM_HOST_STREAMING", "1" if streaming else "0")
    op = make_op()
    return slim.run("slimls", op, slim.Sampler(scheme, op.n_blocks, seed),
                    slim.Schedule("constant", alpha), epochs=K / op.n_blocks, r=r,
                    references=refs)


def test_host_streaming_csr_bit_identical(slim, monkeypatch):
    """Streamed CSR (values, columns and per-block CSC built inside the run)
    gives the same bits as the operator uploaded and converted up front."""
    from paper_1912_07962_b200 import problems
    prob = problems.tomo2d(grid=48, n_views=40, rays=68, seed=4)
    mk = lambda: slim.SparseBlockOperator([prob.op.csr_block(i) for i in range(1, 41)], prob.b)
    a = _run_fresh(slim, mk, monkeypatch, True, "random_cyclic", 5, 1000.0, 6, 70,
                   {"x_true": prob.x_true})
    b = _run_fresh(slim, mk, monkeypatch, False, "random_cyclic", 5, 1000.0, 6, 70,
                   {"x_true": prob.x_true})
    np.testing.assert_array_equal(a.x_final, b.x_final)
    np.testing.assert_array_equal(a.residual_norms, b.residual_norms)


def test_host_streaming_dense_bit_identical(slim, monkeypatch):
    c = gc.dense_case("cfg1_reduced")
    mk = lambda: slim.DenseBlockOperator(c["A"], int(c["ell"]), c["b"])
    a = _run_fresh(slim, mk, monkeypatch, True, "uniform_iid", 3, 50.0, 4, 60, c["refs"])
    b = _run_fresh(slim, mk, monkeypatch, False, "uniform_iid", 3, 50.0, 4, 60, c["refs"])
    np.testing.assert_array_equal(a.x_final, b.x_final)


def test_host_streaming_rejects_bad_column(slim, monkeypatch):
    from paper_1912_07962_b200 import problems
    prob = problems.tomo2d(grid=16, n_views=6, rays=23, seed=1)
    parts = [tuple(np.array(p) if isinstance(p, np.ndarray) else p for p in prob.op.csr_block(i))
             for i in range(1, 7)]
    ip, ix, d, shp = parts[3]
    ix = ix.copy()
    ix[0] = 10_000  # out of range, only seen when block 4 is first sampled
    parts[3] = (ip, ix, d, shp)
    monkeypatch.setenv("SLIM_HOST_STREAMING", "1")
    op = slim.SparseBlockOperator(parts, prob.b)
    with pytest.raises(ValueError, match="column index"):
        slim.run("slimls", op, slim.Sampler("cyclic", 6, 0), slim.Schedule("constant", 10.0),
                 epochs=1.0, r=1)


def test_streaming_probe_keeps_solver_state(slim):
    """slim_probe_stream (bench 'streaming') measures the operator-streaming
    kernels on scratch only: a run after the probe continues bit-identically."""
    import ctypes as C
    from paper_1912_07962_b200 import _lib, problems
    from paper_1912_07962_b200.linops import device_operator
    prob = problems.tomo2d(grid=32, n_views=20, rays=46, seed=3)
    op = prob.op
    mk = lambda: slim.Sampler("random_cyclic", op.n_blocks, 2)
    kw = dict(epochs=30 / op.n_blocks, r=3)
    ref = slim.run("slimls", op, mk(), slim.Schedule("constant", 1000.0), **kw)
    dop = device_operator(op, 3, 0)
    us, nbytes = C.c_double(0), C.c_double(0)
    for kid in (0, 1, 2):
        dop.call("slim_probe_stream", kid, 4, C.byref(us), C.byref(nbytes))
        assert us.value > 0 and nbytes.value > 0
    again = slim.run("slimls", op, mk(), slim.Schedule("constant", 1000.0), **kw)
    np.testing.assert_array_equal(again.x_final, ref.x_final)
    with pytest.raises(ValueError):
        dop.call("slim_probe_stream", 3, 4, C.byref(us), C.byref(nbytes))


def test_factorization_digit_layout_reported(slim):
    """slim_timing which = 7 reports the compile-time digit layout of k_chol_i8
    (seven digits, 8-bit trailing width by default), and the int8 op count of
    the profiled launches (which = 6) is the layout's digit pairs times the
    tile-update flops: QD (QD + 1) / 2 products of 2 * 64^3 per update."""
    c = gc.dense_case("dense_dual")
    op = slim.DenseBlockOperator(c["A"], int(c["ell"]), c["b"])
    timing = {"start_step": 1}
    traj = slim.run("slimls", op, slim.Sampler("random_cyclic", op.n_blocks, 5),
                    slim.Schedule("constant", 100.0), epochs=2.0, r=3, timing=timing)
    assert traj.status == "ok"
    qd, dbits = timing["cholesky_digits"]
    # the layout is a compile-time choice (SLIM_QD / SLIM_DBITS via
    # SLIM_NVCC_EXTRA); the default build is seven digits of 8-bit width
    import os
    extra = os.environ.get("SLIM_NVCC_EXTRA", "")
    want_qd = int(extra.split("SLIM_QD=")[1].split()[0]) if "SLIM_QD=" in extra else 7
    want_db = int(extra.split("SLIM_DBITS=")[1].split()[0]) if "SLIM_DBITS=" in extra else 8
    assert (qd, dbits) == (want_qd, want_db)
    pairs, qx = timing["cholesky_pairs"]
    want_qx = int(extra.split("SLIM_QX=")[1].split()[0]) if "SLIM_QX=" in extra else QX_DEFAULT
    assert qx == want_qx
    # digit pairs (a, b) in [1, qd]^2 with a + b <= qd + 1 + qx
    assert pairs == sum(min(qd, qd + 1 + qx - a) for a in range(1, qd + 1))
    if timing["cholesky_i8ops"] > 0:  # SLIM_CHOL=dmma reports 0
        updates = timing["cholesky_i8ops"] / (pairs * 2 * 64 ** 3)
        assert updates == int(updates) and updates >= 1
