"""Config schema (reference config.py) and harness CSV outputs (harness.py)."""

import ast
import csv
import io

import numpy as np
import pytest

from tests import golden_cases as gc


def test_reference_config_files_parse_identically():
    from paper_1912_07962_b200.config import parse_config
    d = gc.load("harness.npz")
    names = sorted({k.split("/")[1] for k in d.files if k.startswith("cfgfile/")})
    assert len(names) == 4
    for name in names:
        ours = parse_config(str(d[f"cfgfile/{name}/text"])).__dict__
        ref = ast.literal_eval(str(d[f"cfgfile/{name}/parsed"]))
        for key, val in ref.items():
            mine = ours[key]
            if isinstance(val, (list, tuple)):
                assert tuple(mine) == tuple(val), (name, key)
            else:
                assert mine == val, (name, key, mine, val)


def test_config_errors():
    from paper_1912_07962_b200.config import ConfigError, parse_config
    with pytest.raises(ConfigError, match="unknown config section"):
        parse_config("[nope]\nx = 1\n")
    with pytest.raises(ConfigError, match="unknown key"):
        parse_config("[problem]\nwhatever = 1\n")
    with pytest.raises(ConfigError, match="bad value"):
        parse_config("[problem]\nm = ten\n")
    with pytest.raises(ConfigError, match="not divisible"):
        parse_config("[problem]\nkind = gaussian\nm = 10\nblocks = 3\n")
    cfg = parse_config("[problem]\nkind = baseline\nconfig = 3\n")
    assert cfg.baseline_config == 3


def _rows(text):
    return list(csv.reader(io.StringIO(text)))


def _compare_csv(ours, ref, skip_cols=("wall_time_seconds",)):
    a, b = _rows(ours), _rows(ref)
    assert a[0] == b[0] and len(a) == len(b)
    for ra, rb in zip(a[1:], b[1:]):
        for col, x, y in zip(a[0], ra, rb):
            if col in skip_cols:
                continue
            try:
                fx, fy = float(x), float(y)
            except ValueError:
                assert x == y, (col, x, y)
                continue
            if np.isnan(fy):
                assert np.isnan(fx)
            else:
                assert abs(fx - fy) <= 1e-10 * max(1.0, abs(fy)), (col, x, y)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["gauss", "wedge"])
def test_harness_csv_matches_reference(name, tmp_path):
    from paper_1912_07962_b200.config import parse_config
    from paper_1912_07962_b200.harness import run_experiment
    d = gc.load("harness.npz")
    cfg = parse_config(str(d[f"{name}/cfg_text"])).with_overrides(output=str(tmp_path / name))
    res = run_experiment(cfg)
    for kind, path in (("metrics", res.metrics_path), ("aggregate", res.aggregate_path),
                       ("replicates", res.replicates_path)):
        _compare_csv(open(path).read(), str(d[f"{name}/{kind}"]))


def test_slim_container_roundtrip(tmp_path):
    from paper_1912_07962_b200 import DenseBlockOperator
    from paper_1912_07962_b200.linops import StreamOrderError
    from paper_1912_07962_b200.slimfile import FileStreamOperator, load_stream_file, write_stream_file
    g = np.random.default_rng(0)
    op = DenseBlockOperator(g.standard_normal((12, 5)), 3, g.standard_normal(12))
    path = tmp_path / "p.slim"
    write_stream_file(path, op)
    back = load_stream_file(path)
    assert np.array_equal(back.matrix, op.matrix) and np.array_equal(back.rhs, op.rhs)
    with FileStreamOperator(path) as st:
        assert st.fetch_block(1).a_block.shape == (3, 5)
        with pytest.raises(StreamOrderError):
            st.fetch_block(3)


def test_auto_dispatch_refuses_direct_route_alphas():
    """alpha_k > 1e8 sends the reference's auto dispatch to the n x n direct
    route (innersolve.py:356, 377-380); the device path raises ValueError
    before touching the GPU instead of silently solving the dual form."""
    import numpy as np
    import pytest

    import paper_1912_07962_b200 as slim

    rng = np.random.default_rng(0)
    op = slim.DenseBlockOperator(rng.standard_normal((40, 10)), 4, rng.standard_normal(40))
    with pytest.raises(ValueError, match="direct"):
        slim.run("slimls", op, slim.Sampler("cyclic", op.n_blocks, 0),
                 slim.Schedule("constant", 2e8), epochs=1, r=2)
    with pytest.raises(ValueError, match="direct"):  # a decaying schedule starting above 1e8
        slim.run("slimls", op, slim.Sampler("cyclic", op.n_blocks, 0),
                 slim.Schedule("decay", 4e8, decay_exponent=1.0), epochs=1, r=2)
