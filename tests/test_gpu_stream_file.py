""".slim stream files on the device path (reference
linops.py:334-429): records go from the file through the pinned ring
straight into HBM, one block at a time, never through a host copy of the
matrix."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

from tests import golden_cases as gc

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def slim():
    import paper_1912_07962_b200 as slim
    from paper_1912_07962_b200 import _lib
    _lib.lib()
    return slim


def test_stream_file_run_matches_reference(slim, tmp_path):
    """The reference's single-pass golden run, fed from a .slim file."""
    from paper_1912_07962_b200.slimfile import FileStreamOperator, write_stream_file
    c = gc.dense_case("single_pass")
    path = tmp_path / "sp.slim"
    write_stream_file(path, slim.DenseBlockOperator(c["A"], int(c["ell"]), c["b"]))
    st = FileStreamOperator(path)
    traj = slim.run("slimls", st, slim.Sampler("cyclic", st.n_blocks, 0),
                    slim.Schedule("constant", float(c["sched_alpha"])), epochs=1.0,
                    r=int(c["r"]), references=c["refs"])
    np.testing.assert_array_equal(traj.ks, c["ks"])
    np.testing.assert_allclose(traj.x_final, c["x_final"], rtol=1e-10,
                               atol=1e-10 * np.abs(c["x_final"]).max())
    np.testing.assert_allclose(traj.rel_errors["x_true"], c["rel"]["x_true"], rtol=1e-10)
    assert st._next == st.n_blocks + 1  # consumed, like the reference stream
    with pytest.raises(slim.StreamOrderError):
        slim.run("slimls", st, slim.Sampler("cyclic", st.n_blocks, 0),
                 slim.Schedule("constant", 1.0), epochs=1.0, r=1)
    # same bits as the in-memory single-pass operator
    mem = slim.run("slimls", slim.SinglePassAdapter(
        slim.DenseBlockOperator(c["A"], int(c["ell"]), c["b"])),
        slim.Sampler("cyclic", st.n_blocks, 0), slim.Schedule("constant", float(c["sched_alpha"])),
        epochs=1.0, r=int(c["r"]), references=c["refs"])
    np.testing.assert_array_equal(traj.x_final, mem.x_final)


def test_stream_file_errors(slim, tmp_path):
    from paper_1912_07962_b200.slimfile import FileStreamOperator, write_stream_file
    g = np.random.default_rng(1)
    op = slim.DenseBlockOperator(g.standard_normal((12, 5)), 3, g.standard_normal(12))
    path = tmp_path / "t.slim"
    write_stream_file(path, op)
    raw = path.read_bytes()
    cut = tmp_path / "cut.slim"
    cut.write_bytes(raw[:-8])  # last record short by one rhs entry
    st = FileStreamOperator(cut)
    with pytest.raises(ValueError, match="truncated record 4"):
        slim.run("slimls", st, slim.Sampler("cyclic", 4, 0), slim.Schedule("constant", 1.0),
                 epochs=1.0, r=1)
    bad = tmp_path / "bad.slim"
    bad.write_bytes(b"SLIM2" + raw[5:])
    with pytest.raises(ValueError, match="bad magic"):
        FileStreamOperator(bad)


_CHILD = r"""
import json, resource, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_1912_07962_b200 as slim
from paper_1912_07962_b200.slimfile import FileStreamOperator
st = FileStreamOperator(sys.argv[2])
xt = np.load(sys.argv[3])
before = resource.getrusage(resource.RUSAGE_SELF).ru_maxrss
traj = slim.run("slimls", st, slim.Sampler("cyclic", st.n_blocks, 0),
                slim.Schedule("constant", 50.0), epochs=1.0, r=3, references={"x_true": xt})
after = resource.getrusage(resource.RUSAGE_SELF).ru_maxrss
np.save(sys.argv[4], traj.x_final)
print(json.dumps({"rss_before_kb": before, "rss_after_kb": after,
                  "rel": [float(v) for v in traj.rel_errors["x_true"]]}))
"""


def test_multi_gb_stream_file_never_held_on_host(slim, tmp_path):
    """A 2.2 GB file (34 blocks of 256 x 32,768 fp64 rows) run end to end in
    a fresh process whose peak RSS grows by far less than the matrix; the
    iterate matches the oracle fed block by block from the same file."""
    from oracle import slimls_oracle as orc
    from paper_1912_07962_b200.linops import GeneratedBlockOperator
    from paper_1912_07962_b200.slimfile import FileStreamOperator, write_stream_file
    n, ell, nb = 32768, 256, 34
    gen = GeneratedBlockOperator(nb * ell, n, ell, seed=77)
    xt = np.random.Generator(np.random.Philox(key=77)).standard_normal(n)

    class _WithRhs(GeneratedBlockOperator):
        def fetch_block(self, i):  # b computed block by block: no m x n array anywhere
            a = self.block_values(i).astype(np.float64)
            noise = np.random.Generator(np.random.Philox(key=1000 + i)).standard_normal(ell)
            return slim.SampleBlock(i, a, a @ xt + 0.01 * noise)

    src = _WithRhs(nb * ell, n, ell, 77)
    path = tmp_path / "big.slim"
    write_stream_file(path, src)
    size = os.path.getsize(path)
    assert size > 2 * 2 ** 30
    np.save(tmp_path / "xt.npy", xt)
    out = subprocess.run([sys.executable, "-c", _CHILD, ROOT, str(path), str(tmp_path / "xt.npy"),
                          str(tmp_path / "x.npy")], capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    info = json.loads(out.stdout.strip().splitlines()[-1])
    grew_mb = (info["rss_after_kb"] - info["rss_before_kb"]) / 1024
    print(f"stream file {size / 2**30:.2f} GiB: peak RSS grew by {grew_mb:.0f} MB during run()")
    assert grew_mb < 0.25 * size / 2 ** 20
    # oracle: blocks read one at a time from the file
    st = FileStreamOperator(path)

    def fetch(i):
        blk = st.fetch_block(i)
        return blk.a_block, blk.b_block
    ref = orc.run_slimls(fetch, nb, n, np.arange(1, nb + 1), np.full(nb, 50.0), r=3,
                         references={"x_true": xt})
    x = np.load(tmp_path / "x.npy")
    err = np.linalg.norm(x - ref.x_final) / np.linalg.norm(ref.x_final)
    print(f"multi-GB stream file: relative iterate error vs oracle {err:.2e}")
    assert err <= 1e-10
    np.testing.assert_allclose(info["rel"], ref.rel_errors["x_true"], rtol=1e-10)
    del gen
