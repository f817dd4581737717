"""Problem-setup pins (host side): the Siddon projector vs the reference's."""

import numpy as np
import pytest

from tests import golden_cases as gc


@pytest.fixture(scope="module")
def problems():
    from paper_1912_07962_b200 import build
    build.build()
    from paper_1912_07962_b200 import problems
    return problems


def _compare(mine, ref):
    ip, ix, d, shp = mine
    rip, rix, rd, rshp = ref
    assert tuple(shp) == tuple(rshp)
    assert np.array_equal(ip, rip)
    assert np.array_equal(ix, rix)
    np.testing.assert_allclose(d, rd, rtol=1e-14, atol=1e-14)


def test_siddon2d_matches_reference(problems):
    d = gc.load("projector.npz")
    for i in range(9):
        ref = gc.csr_blocks(d, f"p2d/{i}")[0]
        mine = problems.siddon2d_block(float(d[f"p2d/{i}/angle"]), 16, 23)
        _compare(mine, ref)


def test_siddon3d_matches_reference(problems):
    d = gc.load("projector.npz")
    for i in range(7):
        ref = gc.csr_blocks(d, f"p3d/{i}")[0]
        mine = problems.siddon3d_block(d[f"p3d/{i}/dir"], 6, 6)
        _compare(mine, ref)


def test_tomo_golden_blocks_reproduced(problems):
    """The 2D golden run's operator is regenerated exactly by our projector."""
    c = gc.tomo_case("tomo2d")
    for blk, ang in zip(c["blocks"], c["angles"]):
        _compare(problems.siddon2d_block(float(ang), int(c["grid"]), int(c["rays"])), blk)


def test_angles_mapping():
    from paper_1912_07962_b200.problems import angles_0_pi
    a = angles_0_pi(180)
    assert a[0] == 0.0 and a[90] == 90.0 and a[91] == -89.0
    assert np.all(a > -90) and np.all(a <= 90)


def test_column_shard_builders_match_slicing():
    """bench.py's column-sharded runs build each rank's slice view by view
    (problems.tomo2d / tomo3d col_range): the same CSR bits as slicing the
    whole operator, and the whole problem's b."""
    import numpy as np

    from paper_1912_07962_b200 import problems
    from paper_1912_07962_b200.parallel import shard_operator

    full = problems.tomo2d(grid=48, n_views=20, rays=68, seed=5, dtype=np.float32)
    part = problems.tomo2d(grid=48, n_views=20, rays=68, seed=5, dtype=np.float32,
                           col_range=(1000, 2000))
    ref = shard_operator(full.op, 1000, 2000)
    assert np.array_equal(full.b, part.b) and part.op.n_cols == 1000
    for i in range(1, 21):
        a, c = ref.csr_block(i), part.op.csr_block(i)
        assert np.array_equal(a[0] - a[0][0], c[0] - c[0][0])
        assert np.array_equal(a[1], c[1]) and np.array_equal(a[2], c[2])
    f3 = problems.tomo3d(grid=12, n_views=6, side=8, sub_rows=16, seed=4)
    p3 = problems.tomo3d(grid=12, n_views=6, side=8, sub_rows=16, seed=4, col_range=(300, 900))
    r3 = shard_operator(f3.op, 300, 900)
    assert np.array_equal(f3.b, p3.b) and f3.op.n_blocks == p3.op.n_blocks
    for i in range(1, f3.op.n_blocks + 1):
        a, c = r3.csr_block(i), p3.op.csr_block(i)
        assert np.array_equal(a[1], c[1]) and np.array_equal(a[2], c[2])
