"""Drop-in contract details on the GPU path: reference-shaped operators
through ``run()``, the sampler position after a divergence, the NCCL shard
path at world size 1, and dual systems past the int8 factorization's tile
limit (fp64 DMMA fallback)."""

import ctypes as C

import numpy as np
import pytest

from tests import golden_cases as gc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def slim():
    import paper_1912_07962_b200 as slim
    from paper_1912_07962_b200 import _lib
    _lib.lib()
    return slim


# ---------------------------------------------------------------------------
# stand-ins with the reference operator surface (linops.py:142-331): the GPU
# box has no /root/reference, so these mirror its attributes exactly
# ---------------------------------------------------------------------------


class RefDense:
    """Surface of the reference ``DenseBlockOperator`` (linops.py:142-206)."""

    access_mode = "random_access"

    def __init__(self, a, ell, b):
        self._a = np.array(a, dtype=float)
        self._a.flags.writeable = False
        self._b = np.array(b, dtype=float)
        self.n_rows, self.n_cols = self._a.shape
        self.block_rows = ell
        self.n_blocks = self.n_rows // ell

    @property
    def matrix(self):
        return self._a

    @property
    def rhs(self):
        return self._b

    def has_rhs(self):
        return True

    def fetch_block(self, i):
        raise AssertionError("the device path must not fetch blocks one by one")


class RefSparse:
    """Surface of the reference ``SparseBlockOperator`` (linops.py:209-299);
    its ``matrix`` densifies everything, which the device path must avoid."""

    access_mode = "random_access"

    def __init__(self, blocks, b):
        import scipy.sparse as sp
        self._blocks = [sp.csr_matrix(blk) for blk in blocks]
        self.block_rows, self.n_cols = self._blocks[0].shape
        self.n_blocks = len(blocks)
        self.n_rows = self.block_rows * self.n_blocks
        self._b = np.array(b, dtype=float)

    def sparse_block(self, i):
        return self._blocks[i - 1]

    @property
    def matrix(self):
        raise AssertionError("densified the whole reference operator")

    @property
    def rhs(self):
        return self._b

    def has_rhs(self):
        return True

    def fetch_block(self, i):
        raise AssertionError("the device path must not fetch blocks one by one")


class RefSinglePass:
    """Surface of the reference ``SinglePassAdapter`` (linops.py:302-331)."""

    access_mode = "single_pass"

    def __init__(self, op):
        self._op = op
        self.n_rows, self.n_cols = op.n_rows, op.n_cols
        self.n_blocks, self.block_rows = op.n_blocks, op.block_rows
        self._next = 1

    def has_rhs(self):
        return True


def _assert_same(traj, c, rtol=1e-10):
    np.testing.assert_array_equal(traj.ks, c["ks"])
    np.testing.assert_allclose(traj.x_final, c["x_final"], rtol=rtol,
                               atol=rtol * np.abs(c["x_final"]).max())
    for name, vals in c["rel"].items():
        np.testing.assert_allclose(traj.rel_errors[name], vals, rtol=rtol)


def test_reference_dense_operator_through_run(slim):
    c = gc.dense_case("dense_dual")
    op = RefDense(c["A"], int(c["ell"]), c["b"])
    traj = slim.run("slimls", op, slim.Sampler("random_cyclic", op.n_blocks, int(c["seed"])),
                    slim.Schedule("constant", float(c["sched_alpha"])), epochs=float(c["epochs"]),
                    r=int(c["r"]), references=c["refs"])
    _assert_same(traj, c)


def test_reference_sparse_operator_through_run(slim):
    c = gc.tomo_case("tomo2d")
    import scipy.sparse as sp
    blocks = [sp.csr_matrix((d, ix, ip), shape=shp) for ip, ix, d, shp in c["blocks"]]
    op = RefSparse(blocks, c["b"])
    k = len(c["indices"])
    traj = slim.run("slimls", op, slim.Sampler("random_cyclic", op.n_blocks, 7),
                    slim.Schedule("constant", float(c["alpha"])), epochs=k / op.n_blocks,
                    r=int(c["r"]), references={"x_true": c["x_true"]})
    np.testing.assert_allclose(traj.x_final, c["x_final"], rtol=1e-10,
                               atol=1e-10 * np.abs(c["x_final"]).max())
    np.testing.assert_allclose(traj.rel_errors["x_true"], c["rel"]["x_true"], rtol=1e-10)


def test_reference_single_pass_adapter_through_run(slim):
    c = gc.dense_case("single_pass")
    op = RefSinglePass(RefDense(c["A"], int(c["ell"]), c["b"]))
    traj = slim.run("slimls", op, slim.Sampler("cyclic", op.n_blocks, 0),
                    slim.Schedule("constant", float(c["sched_alpha"])), epochs=1.0,
                    r=int(c["r"]), references=c["refs"])
    _assert_same(traj, c)
    assert op._next == op.n_blocks + 1  # the stream was consumed in order


@pytest.mark.parametrize("scheme", ["uniform_iid", "random_cyclic"])
def test_sampler_position_after_divergence(slim, scheme):
    """The reference draws one index per executed step and stops at the
    divergence step (solvers.py:560-570): the caller's sampler must end there."""
    c = gc.dense_case("diverge_late")
    op = slim.DenseBlockOperator(c["A"], int(c["ell"]), c["b"])
    smp = slim.Sampler(scheme, op.n_blocks, 3)
    traj = slim.run("slimls", op, smp, slim.Schedule("constant", 1.0), epochs=4, r=1)
    assert traj.status == "diverged"
    k = traj.diverged_at
    assert smp.position == k
    fresh = slim.Sampler(scheme, op.n_blocks, 3)
    fresh.indices(k)
    np.testing.assert_array_equal(smp.indices(25), fresh.indices(25))


def test_nccl_world_size_one_bit_identical(slim):
    """NcclShard with one rank: dlopen, ncclCommInitRank, ncclCommSplit and
    every per-step ncclAllReduce run for real; the result is the unsharded
    run's, bit for bit."""
    from paper_1912_07962_b200 import _lib
    from paper_1912_07962_b200.parallel import NcclShard
    c = gc.dense_case("dense_dual")
    for rr in (False, True):
        buf = C.create_string_buffer(128)  # a unique id serves one communicator
        _lib.check(_lib.lib().slim_nccl_unique_id(buf))
        op = slim.DenseBlockOperator(c["A"], int(c["ell"]), c["b"])
        shard = NcclShard(0, 1, 0, op.n_cols, bytes(buf.raw))
        shard.round_robin = rr
        kw = dict(epochs=3.0, r=4, references={"x_true": c["refs"]["x_true"]})
        one = slim.run("slimls", op, slim.Sampler("random_cyclic", op.n_blocks, 11),
                       slim.Schedule("constant", 100.0), shard=shard, **kw)
        ref = slim.run("slimls", slim.DenseBlockOperator(c["A"], int(c["ell"]), c["b"]),
                       slim.Sampler("random_cyclic", op.n_blocks, 11),
                       slim.Schedule("constant", 100.0), **kw)
        np.testing.assert_array_equal(one.x_final, ref.x_final)
        np.testing.assert_array_equal(one.rel_errors["x_true"], ref.rel_errors["x_true"])
        np.testing.assert_array_equal(one.residual_norms, ref.residual_norms)


def test_potrf_beyond_int8_tile_limit(slim):
    """T = 294 tile rows (N = 18,816) exceeds the int8 path's exact-int32
    bound (CHOL_I8_TMAX = 293): the fp64 DMMA factorization takes over."""
    n = 294 * 64
    rng = np.random.default_rng(294)
    r = rng.standard_normal((n, n))
    g = r + r.T
    g[np.diag_indices(n)] += 4.0 * np.sqrt(n) + 10.0
    L = slim.potrf(g)
    ref = np.linalg.cholesky(g)
    err = np.abs(L - ref).max() / np.abs(ref).max()
    print(f"potrf N={n}: max |L - L_lapack| / max |L| = {err:.2e}")
    assert err <= 1e-12


def test_run_beyond_int8_tile_limit_vs_oracle(slim):
    """(r + 1) ell = 19,000 rows (T = 297): a run through the DMMA
    factorization against the oracle (rows > n, so the reference takes its
    direct route; the dual system is the same linear map)."""
    from oracle import slimls_oracle as orc
    g = np.random.Generator(np.random.Philox(key=297))
    ell, r, nb, n, K, alpha = 1900, 9, 12, 1500, 12, 0.05
    a = g.standard_normal((ell * nb, n)) / np.sqrt(n)
    xt = g.standard_normal(n)
    b = a @ xt + 0.01 * g.standard_normal(ell * nb)
    op = slim.DenseBlockOperator(a, ell, b)
    traj = slim.run("slimls", op, slim.Sampler("random_cyclic", nb, 4),
                    slim.Schedule("constant", alpha), epochs=K / nb, r=r,
                    references={"x_true": xt})
    idx = orc.sampler_indices("random_cyclic", nb, 4, K)
    ref = orc.run_slimls(orc.dense_fetch(a, b, ell), nb, n, idx, np.full(K, alpha), r=r,
                         references={"x_true": xt})
    err = np.linalg.norm(traj.x_final - ref.x_final) / np.linalg.norm(ref.x_final)
    print(f"N = 19,000 run (DMMA factorization): relative error vs oracle {err:.2e}")
    assert err <= 1e-10
    np.testing.assert_allclose(traj.rel_errors["x_true"], ref.rel_errors["x_true"], rtol=1e-10)
