"""Column-sharded slimLS: one exchange of partial sums per step.

Shard p owns the columns [col0, col1) of A and the matching slices of x
and of every reference vector.  Per step the shards allreduce (sum):

* the new Gram panel A_k M_k^T (x-independent, on the Gram stream),
* the residual partials A_k[:, p] x_p (rank 0 subtracts b_k),
* the norm partials ||x_p||^2, ||x_p - ref_p||^2 (divergence, history);

the dual-system factorization is replicated (identical inputs,
deterministic kernels) and s_p = alpha M_k[:, p]^T w, x_p -= s_p are local.
For 2D/3D tomography the C-order column ranges are image-row / z slabs.

Communicators:

* :class:`NcclShard` -- one process per GPU, NCCL over NVLink/NVSwitch; the
  unique id is broadcast with ``torch.distributed``;
* :class:`LocalGroup` -- P shards on ONE device in one process, one host
  thread per shard (tests; emulates the exchange with a host barrier and a
  rank-ordered sum kernel -- no kernel waits on another shard's kernel).
"""

from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass

import numpy as np

from . import _lib
from .linops import (DenseBlockOperator, DeviceOperator, GeneratedBlockOperator,
                     SinglePassAdapter, SparseBlockOperator, device_operator)


def column_ranges(n: int, nranks: int) -> list[tuple[int, int]]:
    """Balanced contiguous column ranges, rank order."""
    if nranks < 1 or nranks > n:
        raise ValueError(f"cannot split {n} columns over {nranks} shards")
    edges = [(n * p) // nranks for p in range(nranks + 1)]
    return [(edges[p], edges[p + 1]) for p in range(nranks)]


def slice_csr_columns(indptr, indices, data, shape, c0, c1):
    """CSR restricted to columns [c0, c1), column indices shifted to the shard."""
    indptr = np.asarray(indptr, dtype=np.int64)
    indices = np.asarray(indices)
    keep = (indices >= c0) & (indices < c1)
    cs = np.zeros(indices.shape[0] + 1, dtype=np.int64)
    np.cumsum(keep, out=cs[1:])
    counts = cs[indptr[1:]] - cs[indptr[:-1]]
    nip = np.zeros(shape[0] + 1, dtype=np.int64)
    np.cumsum(counts, out=nip[1:])
    return (nip, (indices[keep] - c0).astype(np.int32), np.asarray(data)[keep],
            (shape[0], c1 - c0))


def shard_operator(op, c0: int, c1: int):
    """The operator restricted to columns [c0, c1) (same rows, same b)."""
    src = op.source if isinstance(op, SinglePassAdapter) else op
    if isinstance(src, GeneratedBlockOperator):
        raise TypeError("generated operators are sharded on the device (GeneratedShard)")
    if isinstance(src, SparseBlockOperator):
        parts = [slice_csr_columns(*src.csr_block(i), c0, c1)
                 for i in range(1, src.n_blocks + 1)]
        out = SparseBlockOperator(parts, src.rhs, dtype=src.dtype)
    else:
        a = getattr(src, "matrix", None)
        if a is None:
            a = np.vstack([src.fetch_block(i).a_block for i in range(1, src.n_blocks + 1)])
        out = DenseBlockOperator(np.ascontiguousarray(a[:, c0:c1]), src.block_rows, src.rhs,
                                 dtype=a.dtype)
    return SinglePassAdapter(out) if isinstance(op, SinglePassAdapter) else out


@dataclass
class _Shard:
    rank: int
    nranks: int
    col0: int
    col1: int

    def _attach(self, dop):  # pragma: no cover - overridden
        raise NotImplementedError

    def device_operator(self, op, r: int, device: int):
        src = op.source if isinstance(op, SinglePassAdapter) else op
        cache = src.__dict__.setdefault("_slim_shard_cache", {})
        key = (device, r, self.col0, self.col1, id(getattr(src, "_b", None)), id(self))
        dop = cache.get(key)
        if dop is None:
            if isinstance(src, GeneratedBlockOperator):
                dop = DeviceOperator(n_rows=src.n_rows, n_cols=self.col1 - self.col0,
                                     ell=src.block_rows, r=r, layout=_lib.SLIM_GEN_SPLITMIX64,
                                     dtype=np.float32, device=device, gen_seed=src.seed,
                                     gen_n_total=src.n_cols, col_offset=self.col0)
                b = np.ascontiguousarray(src.rhs)
                dop.call("slim_set_rhs", _lib.dptr(b))
                dop.call("slim_finalize_operator")
            else:
                dop = device_operator(shard_operator(src, self.col0, self.col1), r, device)
            self._attach(dop)
            cache[key] = dop
        # factorizations round-robin over the shards (batch B on
        # rank B mod P), w allreduced from its owner instead of replicated solves
        dop.call("slim_set_factor_round_robin", 1 if getattr(self, "round_robin", False) else 0)
        return dop


class LocalGroup:
    """P column shards on one device, driven by one host thread each."""

    def __init__(self, nranks: int, round_robin: bool = False):
        self.nranks = int(nranks)
        self.round_robin = bool(round_robin)
        self.handle = _lib.lib().slim_local_group_create(self.nranks)
        if not self.handle:
            raise ValueError("a local shard group holds 1..8 shards")

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            try:
                _lib.lib().slim_local_group_destroy(h)
            except Exception:  # pragma: no cover
                pass
            self.handle = None

    def shard(self, rank: int, n: int) -> "LocalShard":
        c0, c1 = column_ranges(n, self.nranks)[rank]
        sh = LocalShard(rank, self.nranks, c0, c1, self)
        sh.round_robin = self.round_robin
        return sh

    def run(self, method, op, make_sampler, schedule, **kw):
        """Run every shard in its own thread; returns (trajectory of rank 0 with
        the concatenated x_final, list of per-shard trajectories)."""
        from .solvers import run

        n = op.n_cols
        shards = [self.shard(p, n) for p in range(self.nranks)]
        for sh in shards:  # upload serially (device allocation), attach comm
            sh.device_operator(op, kw.get("r", 0), kw.get("device", 0))
        out = [None] * self.nranks
        err = []

        def worker(p):
            try:
                out[p] = run(method, op, make_sampler(), schedule, shard=shards[p], **kw)
            except BaseException as exc:  # pragma: no cover - surfaced below
                err.append(exc)

        threads = [threading.Thread(target=worker, args=(p,)) for p in range(self.nranks)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        if err:
            raise err[0]
        full = out[0]
        full.x_final = np.concatenate([t.x_final for t in out])
        return full, out


@dataclass
class LocalShard(_Shard):
    group: LocalGroup = None

    def _attach(self, dop):
        dop.call("slim_comm_init_local", C.c_void_p(self.group.handle), self.rank)

    def __hash__(self):
        return id(self)


@dataclass
class NcclShard(_Shard):
    """This process's shard of an NCCL-connected solve (one process per GPU)."""

    uid: bytes = b""

    @classmethod
    def from_torch(cls, n: int, round_robin: bool = False):
        """Create the shard for this torch.distributed rank (NCCL id broadcast);
        ``round_robin``: factorizations distributed over the ranks (8f.1)."""
        import torch.distributed as dist

        rank, world = dist.get_rank(), dist.get_world_size()
        obj = [None]
        if rank == 0:
            buf = C.create_string_buffer(128)
            _lib.check(_lib.lib().slim_nccl_unique_id(buf))
            obj[0] = bytes(buf.raw)
        dist.broadcast_object_list(obj, src=0)
        c0, c1 = column_ranges(n, world)[rank]
        sh = cls(rank, world, c0, c1, obj[0])
        sh.round_robin = bool(round_robin)
        return sh

    def _attach(self, dop):
        buf = C.create_string_buffer(self.uid, 128)
        dop.call("slim_comm_init", buf, self.nranks, self.rank)

    def __hash__(self):
        return id(self)
