"""Column sharding host logic on CPU: world_size-2 gloo processes run the
sharded decomposition (partial residuals / Gram panels / norms exchanged by
allreduce, factorization replicated, x update local) with NumPy arithmetic
and must reproduce the unsharded oracle; the shard slicing helpers are the
product's (paper_1912_07962_b200.parallel)."""

import os
import socket

import numpy as np
import pytest
import scipy.linalg
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

from oracle import slimls_oracle as orc
from paper_1912_07962_b200.parallel import column_ranges, shard_operator, slice_csr_columns


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _allreduce(v):
    t = torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64))
    dist.all_reduce(t)
    return t.numpy()


def _sharded_run(a_shard, b, ell, idx, alpha, r, rank, xt_shard, round_robin=False, world=1,
                 batch=1):
    """slimLS on one column shard; exchanges by gloo allreduce. With
    ``round_robin`` (slim_set_factor_round_robin) only rank
    (k - 1) // batch mod world factors step k's system and solves for w; the
    others add zeros in an allreduce of w."""
    n_p = a_shard.shape[1]
    x = np.zeros(n_p)
    window = []
    history = []
    for k, i in enumerate(idx, start=1):
        blk = a_shard[(i - 1) * ell:i * ell]
        window = (window + [blk])[-(r + 1):]
        res = blk @ x - (b[(i - 1) * ell:i * ell] if rank == 0 else 0.0)
        res = _allreduce(res)
        mat = np.vstack(window)
        g = _allreduce(mat @ mat.T)  # Gram partials over this shard's columns
        g *= alpha
        g[np.diag_indices_from(g)] += 1.0
        y = np.zeros(mat.shape[0])
        y[-ell:] = res
        if not round_robin:
            w = scipy.linalg.solve(g, y, assume_a="pos")  # replicated
        else:
            own = ((k - 1) // batch) % world == rank
            w = scipy.linalg.solve(g, y, assume_a="pos") if own else np.zeros_like(y)
            w = _allreduce(w)  # the owner's w, exactly
        x = x - alpha * (mat.T @ w)  # local
        norms = _allreduce(np.array([x @ x, (x - xt_shard) @ (x - xt_shard)]))
        history.append((float(np.sqrt(res @ res)), float(np.sqrt(norms[1]))))
    return x, history


def _worker(rank, world, port, out, round_robin=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = np.random.Generator(np.random.Philox(key=3))
    m, n, ell, r, alpha, K = 240, 60, 12, 3, 50.0, 25
    a = g.standard_normal((m, n)) / np.sqrt(n)
    xt = g.standard_normal(n)
    b = a @ xt + 0.01 * g.standard_normal(m)
    c0, c1 = column_ranges(n, world)[rank]
    idx = orc.sampler_indices("random_cyclic", m // ell, 11, K)
    x, hist = _sharded_run(a[:, c0:c1], b, ell, idx, alpha, r, rank, xt[c0:c1],
                           round_robin=round_robin, world=world, batch=4)
    xs = [None] * world
    dist.all_gather_object(xs, x)
    if rank == 0:
        out.put((np.concatenate(xs), hist))
    dist.destroy_process_group()


@pytest.mark.parametrize("round_robin", [False, True])
def test_column_sharded_decomposition_matches_oracle(round_robin):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(p, world, port, q, round_robin))
             for p in range(world)]
    for p in procs:
        p.start()
    x, hist = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = np.random.Generator(np.random.Philox(key=3))
    m, n, ell, r, alpha, K = 240, 60, 12, 3, 50.0, 25
    a = g.standard_normal((m, n)) / np.sqrt(n)
    xt = g.standard_normal(n)
    b = a @ xt + 0.01 * g.standard_normal(m)
    idx = orc.sampler_indices("random_cyclic", m // ell, 11, K)
    ref = orc.run_slimls(orc.dense_fetch(a, b, ell), m // ell, n, idx, np.full(K, alpha), r=r,
                         references={"x_true": xt})
    np.testing.assert_allclose(x, ref.x_final, rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose([h[0] for h in hist], ref.residual_norms[1:], rtol=1e-10)
    np.testing.assert_allclose(np.array([h[1] for h in hist]) / np.linalg.norm(xt),
                               ref.rel_errors["x_true"][1:], rtol=1e-10)


def test_column_ranges_cover():
    for n, p in [(10, 3), (65536, 8), (7, 7)]:
        rr = column_ranges(n, p)
        assert rr[0][0] == 0 and rr[-1][1] == n
        assert all(rr[i][1] == rr[i + 1][0] for i in range(p - 1))
    with pytest.raises(ValueError):
        column_ranges(3, 4)


def test_csr_column_slices_reassemble():
    import scipy.sparse as sp
    a = sp.random(40, 50, density=0.2, format="csr", random_state=2)
    parts = [slice_csr_columns(a.indptr, a.indices, a.data, a.shape, c0, c1)
             for c0, c1 in column_ranges(50, 4)]
    full = np.hstack([sp.csr_matrix((d, ix, ip), shape=shp).toarray() for ip, ix, d, shp in parts])
    assert np.array_equal(full, a.toarray())


def test_shard_operator_dense_and_sparse():
    from paper_1912_07962_b200 import DenseBlockOperator, SparseBlockOperator
    import scipy.sparse as sp
    g = np.random.default_rng(0)
    a = g.standard_normal((12, 9))
    b = g.standard_normal(12)
    op = DenseBlockOperator(a, 4, b)
    sh = shard_operator(op, 3, 7)
    assert np.array_equal(sh.matrix, a[:, 3:7]) and np.array_equal(sh.rhs, b)
    blocks = [sp.random(4, 9, density=0.5, format="csr", random_state=s) for s in range(3)]
    sop = SparseBlockOperator(blocks, b)
    ssh = shard_operator(sop, 2, 9)
    for i in range(1, 4):
        assert np.allclose(ssh.fetch_block(i).a_block, sop.fetch_block(i).a_block[:, 2:9])


def test_bench_spawns_ranks_for_gpus_n():
    """bench.py --gpus 2 without torchrun launches two ranks itself (gloo host
    plumbing on 127.0.0.1); the reference arm runs on rank 0 only and prints
    exactly one JSON line with n_gpus = 2."""
    import json
    import subprocess
    import sys

    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--gpus", "2", "--config", "1", "--steps", "3", "--warmup", "1"],
                         capture_output=True, text=True, env=env, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    rec = json.loads(lines[0])
    assert rec["impl"] == "reference" and rec["n_gpus"] == 2 and rec["steps"] == 3
    assert rec["repo_native_loaded"] == []  # the reference arm never loads libslimb200.so
    assert rec["cpu_baseline"]["kind"] == "reference"
