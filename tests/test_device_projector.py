"""Device Siddon projector (csrc/siddon.cu) against the
reference-pinned host projector and the reference's own golden blocks.

The bar is bit-exact: same row pointers, same columns, and the same values
(fp64 identical; fp32 = the fp64 value rounded once), because the device
tracer performs the host restatement's floating-point operations in the
same order (tomo.py:219-301). Runs on a device-traced operator are then
bit-identical to runs on the host-built one.
"""

import numpy as np
import pytest

from tests import golden_cases as gc


@pytest.fixture(scope="module")
def tomo():
    from paper_1912_07962_b200 import build
    build.build()
    from paper_1912_07962_b200 import tomo
    return tomo


def _geom_2d(tomo, angles, rays, spacing=1.0):
    return tomo.parallel_2d_geometry(np.asarray(angles, dtype=float), rays, spacing)


def _dirs_3d(count, seed):
    g = np.random.Generator(np.random.Philox(key=seed))
    raw = g.standard_normal((count, 3))
    axial = np.array([[0.0, 0.0, 1.0], [1.0, 0.0, 0.0], [0.0, -1.0, 0.0], [0.0, 0.0, -1.0],
                      [np.sqrt(0.5), np.sqrt(0.5), 0.0], [-0.6, 0.0, 0.8]])
    d = np.vstack([axial, raw / np.linalg.norm(raw, axis=1, keepdims=True)])
    return d / np.linalg.norm(d, axis=1, keepdims=True)


# ---- host side (no GPU): the operator's host view and validation ----------

def test_host_blocks_are_the_host_projector(tomo):
    from paper_1912_07962_b200 import problems
    geom = _geom_2d(tomo, [0.0, 33.5, 90.0, -45.0], 23)
    op = tomo.ProjectorOperator(geom, 16)
    for i, ang in enumerate(geom.angles, start=1):
        ip, ix, d, shp = op.csr_block(i)
        rip, rix, rd, rshp = problems.siddon2d_block(ang, 16, 23)
        assert shp == rshp
        assert np.array_equal(ip, rip) and np.array_equal(ix, rix) and np.array_equal(d, rd)


def test_build_projector_host_matches_reference_golden(tomo):
    d = gc.load("projector.npz")
    angles = [float(d[f"p2d/{i}/angle"]) for i in range(9)]
    op = tomo.build_projector(_geom_2d(tomo, angles, 23), 16)
    for i in range(9):
        rip, rix, rd, _ = gc.csr_blocks(d, f"p2d/{i}")[0]
        ip, ix, dd, _ = op.csr_block(i + 1)
        assert np.array_equal(ip, rip) and np.array_equal(ix, rix)
        np.testing.assert_allclose(dd, rd, rtol=1e-14, atol=1e-14)


def test_geometry_validation_messages(tomo):
    with pytest.raises(ValueError, match="lie in"):
        tomo.parallel_2d_geometry([-90.0], 4)
    with pytest.raises(ValueError, match="unit vectors"):
        tomo.parallel_3d_geometry([[1.0, 1.0, 0.0]], 4)
    with pytest.raises(ValueError, match="desk-scale"):
        tomo.build_projector(tomo.parallel_3d_geometry([[0.0, 0.0, 1.0]], 4), 65)
    geom = _geom_2d(tomo, [0.0, 10.0], 10)
    with pytest.raises(ValueError, match="do not split"):
        tomo.ProjectorOperator(geom, 8, block_rows=3)
    with pytest.raises(ValueError, match="ray_of_row"):
        tomo.ProjectorOperator(geom, 8, ray_of_row=np.zeros(5, dtype=np.int32))


# ---- device ----------------------------------------------------------------

def _assert_blocks_equal(op, dtype):
    for i in range(1, op.n_blocks + 1):
        dip, dix, dd = op.device_block(i)
        hip, hix, hd, _ = op.csr_block(i)
        assert np.array_equal(dip, hip), f"block {i} rowptr"
        assert np.array_equal(dix, hix), f"block {i} columns"
        assert dd.dtype == dtype
        assert np.array_equal(dd, hd.astype(dtype)), f"block {i} values"


@pytest.mark.gpu
@pytest.mark.parametrize("spacing", [1.0, 0.7, 1.9])
def test_device_2d_bit_exact(tomo, spacing):
    angles = np.concatenate([[0.0, 90.0, 45.0, -45.0, 30.0, -60.0, 89.99, -89.99, 1e-9],
                             np.linspace(-89.0, 90.0, 17)])
    geom = _geom_2d(tomo, angles, 46, spacing)
    op = tomo.build_projector(geom, 32, device=0)
    _assert_blocks_equal(op, np.float64)


@pytest.mark.gpu
def test_device_2d_reference_golden(tomo):
    d = gc.load("projector.npz")
    angles = [float(d[f"p2d/{i}/angle"]) for i in range(9)]
    op = tomo.build_projector(_geom_2d(tomo, angles, 23), 16, device=0)
    for i in range(9):
        rip, rix, rd, _ = gc.csr_blocks(d, f"p2d/{i}")[0]
        ip, ix, dd = op.device_block(i + 1)
        assert np.array_equal(ip, rip) and np.array_equal(ix, rix)
        np.testing.assert_allclose(dd, rd, rtol=1e-14, atol=1e-14)


@pytest.mark.gpu
def test_device_3d_reference_golden(tomo):
    d = gc.load("projector.npz")
    dirs = np.stack([d[f"p3d/{i}/dir"] for i in range(7)])
    op = tomo.build_projector(tomo.parallel_3d_geometry(dirs, 6), 6, device=0)
    for i in range(7):
        rip, rix, rd, _ = gc.csr_blocks(d, f"p3d/{i}")[0]
        ip, ix, dd = op.device_block(i + 1)
        assert np.array_equal(ip, rip) and np.array_equal(ix, rix)
        np.testing.assert_allclose(dd, rd, rtol=1e-14, atol=1e-14)


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_device_3d_permuted_subblocks_bit_exact(tomo, dtype):
    dirs = _dirs_3d(10, 3)
    side, grid = 12, 10
    geom = tomo.parallel_3d_geometry(dirs, side, 0.9)
    g = np.random.Generator(np.random.Philox(key=4))
    rpv = side * side
    rmap = np.concatenate([g.permutation(rpv) for _ in range(len(dirs))]).astype(np.int32)
    op = tomo.build_projector(geom, grid, device=0, dtype=dtype, block_rows=36, ray_of_row=rmap)
    assert op.n_blocks == len(dirs) * rpv // 36
    _assert_blocks_equal(op, dtype)


@pytest.mark.gpu
def test_device_apply_matches_host(tomo):
    geom = _geom_2d(tomo, np.linspace(-89.0, 90.0, 30), 60)
    op = tomo.build_projector(geom, 40, device=0)
    x = np.random.Generator(np.random.Philox(key=8)).standard_normal(op.n_cols)
    host = op.to_host()
    ref = np.concatenate([host.sparse_block(i) @ x for i in range(1, op.n_blocks + 1)])
    np.testing.assert_allclose(op.apply_device(x), ref, rtol=1e-13, atol=1e-13)


@pytest.mark.gpu
def test_run_on_device_projector_equals_host_operator(tomo):
    """slimLS on the device-traced operator is bit-identical to the same run on
    the host-built operator, and matches the CPU oracle (1e-10)."""
    import paper_1912_07962_b200 as slim
    from oracle import slimls_oracle as orc
    from paper_1912_07962_b200 import problems
    grid, views, rays = 48, 40, 68
    geom = _geom_2d(tomo, problems.angles_0_pi(views), rays)
    op = tomo.build_projector(geom, grid, device=0)
    xt = problems.random_ellipses(grid, 6, 3)
    clean = op.apply_device(xt)
    b = problems.scaled_noise(clean, 0.01, problems._rng(5))
    op = op.with_rhs(b)
    host = op.to_host()
    K, r, alpha, seed = 30, 6, 1000.0, 13
    kw = dict(epochs=K / op.n_blocks, r=r, references={"x_true": xt})
    t_dev = slim.run("slimls", op, slim.Sampler("random_cyclic", op.n_blocks, seed),
                     slim.Schedule("constant", alpha), **kw)
    t_host = slim.run("slimls", host, slim.Sampler("random_cyclic", op.n_blocks, seed),
                      slim.Schedule("constant", alpha), **kw)
    assert np.array_equal(t_dev.x_final, t_host.x_final)
    idx = orc.sampler_indices("random_cyclic", op.n_blocks, seed, K)
    blocks = [host.csr_block(i) for i in range(1, op.n_blocks + 1)]
    ref = orc.run_slimls(orc.csr_fetch(blocks, b), op.n_blocks, op.n_cols, idx,
                         np.full(K, alpha), r=r, references={"x_true": xt})
    err = np.linalg.norm(t_dev.x_final - ref.x_final) / np.linalg.norm(ref.x_final)
    assert err <= 1e-10


@pytest.mark.gpu
def test_device_config1_full_size_bit_exact(tomo):
    """configs[1]'s whole operator (180 views x 362 rays on 256^2)."""
    from paper_1912_07962_b200 import problems
    geom = _geom_2d(tomo, problems.angles_0_pi(180), 362)
    op = tomo.build_projector(geom, 256, device=0)
    _assert_blocks_equal(op, np.float64)
    nnz = sum(int(op.device_block(i)[0][-1]) for i in range(1, op.n_blocks + 1))
    assert nnz == 15018524


@pytest.mark.gpu
def test_device_config2_views_bit_exact(tomo):
    """configs[2] (1024^2, 720 views x 1448 rays, fp32 values): a spread of views."""
    from paper_1912_07962_b200 import problems
    geom = _geom_2d(tomo, problems.angles_0_pi(720), 1448)
    op = tomo.build_projector(geom, 1024, device=0, dtype=np.float32)
    for i in (1, 2, 181, 360, 361, 362, 540, 719, 720):
        dip, dix, dd = op.device_block(i)
        hip, hix, hd, _ = op.csr_block(i)
        assert np.array_equal(dip, hip) and np.array_equal(dix, hix)
        assert np.array_equal(dd, hd.astype(np.float32))


def test_permuted_subblocks_match_problem_generator(tomo):
    """ray_of_row reproduces configs[3]'s sub-block construction (problems.tomo3d)."""
    from paper_1912_07962_b200 import problems
    prob = problems.tomo3d(grid=8, n_views=4, side=8, sub_rows=16, ellipsoids=3, seed=2,
                           dtype=np.float64)
    dirs, rmap = problems.tomo3d_geometry(4, 8, 16, 2)
    op = tomo.ProjectorOperator(tomo.parallel_3d_geometry(dirs, 8), 8, block_rows=16,
                                ray_of_row=rmap)
    assert op.n_blocks == prob.op.n_blocks
    for i in range(1, op.n_blocks + 1):
        a, b = op.csr_block(i), prob.op.csr_block(i)
        for u, v in zip(a[:3], b[:3]):
            assert np.array_equal(u, v)
