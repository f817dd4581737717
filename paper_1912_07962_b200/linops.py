"""Row-block operators (reference linops.py) backed by device storage.

The classes keep the reference's public surface -- ``n_rows``, ``n_cols``,
``n_blocks``, ``block_rows``, ``access_mode``, 1-based ``fetch_block``,
``row_range``, ``with_rhs``, ``apply``/``apply_adjoint`` -- so problem code
written against ``slimsolve.linops`` runs unchanged.  What differs is
where the hot path reads the matrix: instead of densifying a block per
fetch (linops.py:270-279) the operator is uploaded once into HBM
(row-major dense, or per-block CSR plus per-block CSC) and the device
loop reads blocks in place.

Operators from the reference package itself are also accepted by
:func:`device_operator` (duck-typed on ``matrix``/``sparse_block``/``rhs``).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import os

import numpy as np

from . import _lib


class StreamOrderError(RuntimeError):
    """A single-pass operator was asked for an out-of-order block."""


@dataclass(frozen=True)
class SampleBlock:
    """One sampled pair (A_k, b_k) plus the 1-based block index (linops.py:34-55)."""

    block_index: int
    a_block: np.ndarray
    b_block: np.ndarray

    def __post_init__(self):
        if self.a_block.shape[0] != self.b_block.shape[0]:
            raise ValueError(
                "a_block and b_block row counts disagree: "
                f"{self.a_block.shape[0]} vs {self.b_block.shape[0]}")

    @property
    def n_rows(self) -> int:
        return self.a_block.shape[0]

    @property
    def n_cols(self) -> int:
        return self.a_block.shape[1]


def _check_partition(m: int, ell: int) -> int:
    if ell < 1:
        raise ValueError(f"block size must be >= 1, got {ell}")
    if m % ell != 0:
        raise ValueError(f"m = {m} is not divisible by block size ell = {ell}; "
                         "only uniform partitions are supported")
    return m // ell


class RowBlockOperator:
    n_rows: int
    n_cols: int
    n_blocks: int
    block_rows: int
    access_mode: str

    def row_range(self, i: int) -> tuple[int, int]:
        self._check_index(i)
        start = (i - 1) * self.block_rows
        return start, start + self.block_rows

    def _check_index(self, i: int):
        if not 1 <= i <= self.n_blocks:
            raise IndexError(f"block index {i} out of range 1..{self.n_blocks}")

    def fetch_block(self, i: int) -> SampleBlock:
        raise NotImplementedError

    def has_rhs(self) -> bool:
        raise NotImplementedError

    def _require_random_access(self, what: str):
        if self.access_mode != "random_access":
            raise RuntimeError(f"{what} requires a random_access operator")

    def apply(self, x: np.ndarray) -> np.ndarray:
        self._require_random_access("apply")
        x = np.asarray(x, dtype=float)
        if x.shape != (self.n_cols,):
            raise ValueError(f"x has shape {x.shape}, expected ({self.n_cols},)")
        out = np.empty(self.n_rows)
        for i in range(1, self.n_blocks + 1):
            s, e = self.row_range(i)
            out[s:e] = self.fetch_block(i).a_block @ x
        return out

    def blocks(self):
        for i in range(1, self.n_blocks + 1):
            yield self.fetch_block(i)


class DenseBlockOperator(RowBlockOperator):
    """Random-access dense operator (linops.py:142-206).

    ``dtype`` may be float32 for the single-precision matrix configs;
    products are always accumulated in fp64 on the device.
    """

    access_mode = "random_access"

    def __init__(self, a: np.ndarray, ell: int, b: np.ndarray | None = None, dtype=np.float64):
        a = np.array(a, dtype=dtype, order="C")
        if a.ndim != 2:
            raise ValueError("A must be a 2-D array")
        a.flags.writeable = False
        self._a = a
        self.n_rows, self.n_cols = a.shape
        self.block_rows = int(ell)
        self.n_blocks = _check_partition(self.n_rows, self.block_rows)
        self._b = None
        if b is not None:
            self._bind_rhs(b)

    def _bind_rhs(self, b):
        b = np.array(b, dtype=float).reshape(-1)
        if b.shape != (self.n_rows,):
            raise ValueError(f"b has length {b.shape[0]}, expected {self.n_rows}")
        b.flags.writeable = False
        self._b = b

    def with_rhs(self, b) -> "DenseBlockOperator":
        op = DenseBlockOperator.__new__(DenseBlockOperator)
        op._a = self._a
        op.n_rows, op.n_cols = self.n_rows, self.n_cols
        op.block_rows, op.n_blocks = self.block_rows, self.n_blocks
        op._b = None
        op._bind_rhs(b)
        return op

    def has_rhs(self) -> bool:
        return self._b is not None

    @property
    def matrix(self) -> np.ndarray:
        return self._a

    @property
    def rhs(self) -> np.ndarray:
        if self._b is None:
            raise ValueError("operator has no right-hand side bound")
        return self._b

    def fetch_block(self, i: int) -> SampleBlock:
        self._check_index(i)
        if self._b is None:
            raise ValueError("operator has no right-hand side bound; use with_rhs(b)")
        s, e = self.row_range(i)
        return SampleBlock(i, np.asarray(self._a[s:e], dtype=float), self._b[s:e])


def _as_csr_parts(blk):
    """(indptr int64, indices int32, data, shape) from scipy or a tuple."""
    if isinstance(blk, tuple):
        indptr, indices, data, shape = blk
    else:
        blk = blk.tocsr()
        indptr, indices, data, shape = blk.indptr, blk.indices, blk.data, blk.shape
    return (np.asarray(indptr, dtype=np.int64), np.asarray(indices, dtype=np.int32),
            np.asarray(data), (int(shape[0]), int(shape[1])))


class SparseBlockOperator(RowBlockOperator):
    """Random-access operator over per-block CSR matrices (linops.py:209-299).

    Blocks may be scipy sparse matrices or ``(indptr, indices, data,
    shape)`` tuples; float32 data (configs 3/4) is kept in float32 on the
    device and widened to fp64 inside every product.
    """

    access_mode = "random_access"

    def __init__(self, blocks: list, b: np.ndarray | None = None, dtype=None):
        if not blocks:
            raise ValueError("need at least one block")
        parts = [_as_csr_parts(blk) for blk in blocks]
        ell, n = parts[0][3]
        for p in parts:
            if p[3] != (ell, n):
                raise ValueError("all blocks must share the same shape")
        if dtype is None:
            dtype = np.float32 if all(p[2].dtype == np.float32 for p in parts) else np.float64
        self.dtype = np.dtype(dtype)
        self._parts = [(ip, ix, np.asarray(d, dtype=self.dtype), shp) for ip, ix, d, shp in parts]
        self.block_rows = ell
        self.n_cols = n
        self.n_blocks = len(parts)
        self.n_rows = ell * self.n_blocks
        self._b = None
        if b is not None:
            self._bind_rhs(b)

    _bind_rhs = DenseBlockOperator._bind_rhs

    def with_rhs(self, b) -> "SparseBlockOperator":
        op = SparseBlockOperator.__new__(SparseBlockOperator)
        op.__dict__.update({k: v for k, v in self.__dict__.items() if not k.startswith("_slim")})
        op._b = None
        op._bind_rhs(b)
        return op

    def has_rhs(self) -> bool:
        return self._b is not None

    @property
    def rhs(self) -> np.ndarray:
        if self._b is None:
            raise ValueError("operator has no right-hand side bound")
        return self._b

    def csr_block(self, i: int):
        self._check_index(i)
        return self._parts[i - 1]

    def sparse_block(self, i: int):
        import scipy.sparse as sp

        ip, ix, d, shp = self.csr_block(i)
        return sp.csr_matrix((d.astype(float), ix, ip), shape=shp)

    def fetch_block(self, i: int) -> SampleBlock:
        self._check_index(i)
        if self._b is None:
            raise ValueError("operator has no right-hand side bound; use with_rhs(b)")
        s, e = self.row_range(i)
        return SampleBlock(i, self.sparse_block(i).toarray(), self._b[s:e])

    def global_csr(self):
        """Concatenated (rowptr int64 (m+1), col int32, val) of all blocks."""
        nnz = np.array([p[0][-1] - p[0][0] for p in self._parts], dtype=np.int64)
        rowptr = np.empty(self.n_rows + 1, dtype=np.int64)
        rowptr[0] = 0
        col = np.empty(int(nnz.sum()), dtype=np.int32)
        val = np.empty(int(nnz.sum()), dtype=self.dtype)
        off = 0
        ell = self.block_rows
        for i, (ip, ix, d, _) in enumerate(self._parts):
            rowptr[i * ell + 1:(i + 1) * ell + 1] = off + (ip[1:] - ip[0])
            col[off:off + nnz[i]] = ix[ip[0]:ip[-1]]
            val[off:off + nnz[i]] = d[ip[0]:ip[-1]]
            off += int(nnz[i])
        return rowptr, col, val


class SinglePassAdapter(RowBlockOperator):
    """Random-access operator exposed as a strict single-pass stream (linops.py:302-331)."""

    access_mode = "single_pass"

    def __init__(self, op: RowBlockOperator):
        if op.access_mode != "random_access":
            raise ValueError("can only adapt a random_access operator")
        self._op = op
        self.n_rows, self.n_cols = op.n_rows, op.n_cols
        self.n_blocks, self.block_rows = op.n_blocks, op.block_rows
        self._next = 1

    def has_rhs(self) -> bool:
        return self._op.has_rhs()

    def fetch_block(self, i: int) -> SampleBlock:
        self._check_index(i)
        if i != self._next:
            raise StreamOrderError(f"single-pass stream expected block {self._next}, got {i}")
        self._next += 1
        return self._op.fetch_block(i)

    @property
    def source(self):
        return self._op


def splitmix64(z: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser on uint64 arrays (wrapping arithmetic)."""
    z = z + np.uint64(0x9E3779B97F4A7C15)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def generated_rows(seed: int, row0: int, rows: int, n: int, col0: int = 0,
                   cols: int | None = None) -> np.ndarray:
    """A[i, j] = fp32((2u - 1) / sqrt(n)), u = (splitmix64(seed ^ (i n + j)) >> 11) 2^-53.

    Host evaluation of the configs[4] generator; bit-identical to the device
    kernel (every operation is exactly rounded IEEE fp64, then one fp32 cast).
    """
    cols = n - col0 if cols is None else cols
    i = (np.uint64(row0) + np.arange(rows, dtype=np.uint64))[:, None]
    j = (np.uint64(col0) + np.arange(cols, dtype=np.uint64))[None, :]
    with np.errstate(over="ignore"):
        z = splitmix64(np.uint64(seed) ^ (i * np.uint64(n) + j))
    u = (z >> np.uint64(11)).astype(np.float64) * 2.0**-53
    return ((2.0 * u - 1.0) / np.sqrt(float(n))).astype(np.float32)


class GeneratedBlockOperator(RowBlockOperator):
    """configs[4] streaming operator: rows generated from (seed, i, j), never stored.

    ``fetch_block`` evaluates the generator on the host (for inspection and
    the oracle); the device path generates each sampled block in-kernel
    into a ring of window blocks.
    """

    access_mode = "random_access"

    def __init__(self, n_rows: int, n_cols: int, ell: int, seed: int, b=None):
        self.n_rows, self.n_cols = int(n_rows), int(n_cols)
        self.block_rows = int(ell)
        self.n_blocks = _check_partition(self.n_rows, self.block_rows)
        self.seed = int(seed)
        self._b = None
        if b is not None:
            self._bind_rhs(b)

    _bind_rhs = DenseBlockOperator._bind_rhs

    def with_rhs(self, b) -> "GeneratedBlockOperator":
        return GeneratedBlockOperator(self.n_rows, self.n_cols, self.block_rows, self.seed, b)

    def has_rhs(self) -> bool:
        return self._b is not None

    @property
    def rhs(self) -> np.ndarray:
        if self._b is None:
            raise ValueError("operator has no right-hand side bound")
        return self._b

    def block_values(self, i: int) -> np.ndarray:
        s, _ = self.row_range(i)
        return generated_rows(self.seed, s, self.block_rows, self.n_cols)

    def fetch_block(self, i: int) -> SampleBlock:
        self._check_index(i)
        if self._b is None:
            raise ValueError("operator has no right-hand side bound; use with_rhs(b)")
        s, e = self.row_range(i)
        return SampleBlock(i, self.block_values(i).astype(np.float64), self._b[s:e])

    def apply_device(self, x: np.ndarray, device: int = 0) -> np.ndarray:
        """A x over all rows by the device generator (fp64 accumulation)."""
        dop = DeviceOperator(n_rows=self.n_rows, n_cols=self.n_cols, ell=self.block_rows, r=0,
                             layout=_lib.SLIM_GEN_SPLITMIX64, dtype=np.float32, device=device,
                             gen_seed=self.seed, gen_n_total=self.n_cols)
        x = np.ascontiguousarray(np.asarray(x, dtype=float))
        out = np.empty(self.n_rows)
        dop.call("slim_gen_apply", _lib.dptr(x), _lib.dptr(out))
        return out


# ---------------------------------------------------------------------------
# device binding
# ---------------------------------------------------------------------------


class DeviceOperator:
    """Owns one C-ABI context holding the operator in HBM."""

    # slim_desc.flags of the contexts created next (parallel.LocalShard sets
    # SLIM_FLAG_FP64_FACTOR for in-process groups of three or more shards)
    default_flags = 0

    def __init__(self, *, n_rows, n_cols, ell, r, layout, dtype, device=0, gen_seed=0,
                 gen_n_total=0, col_offset=0):
        L = _lib.lib()
        d = _lib.SlimDesc()
        d.n_rows, d.n_cols, d.block_rows, d.memory_r = n_rows, n_cols, ell, r
        d.value_dtype = _lib.SLIM_F32 if np.dtype(dtype) == np.float32 else _lib.SLIM_F64
        d.layout = layout
        d.device = int(device)
        d.flags = int(DeviceOperator.default_flags)
        d.gen_seed = int(gen_seed)
        d.gen_n_total = int(gen_n_total)
        d.col_offset = int(col_offset)
        ctx = C.c_void_p()
        rc = L.slim_create(C.byref(ctx), C.byref(d))
        if rc != _lib.SLIM_OK:
            if ctx:
                L.slim_destroy(ctx)
            _lib.check(rc, None)
        self.ctx = ctx
        self.n_rows, self.n_cols, self.ell, self.r = n_rows, n_cols, ell, r
        self.n_blocks = n_rows // ell
        self.dtype = np.dtype(dtype)
        self.layout = layout

    def __del__(self):
        ctx = getattr(self, "ctx", None)
        if ctx:
            try:
                _lib.lib().slim_destroy(ctx)
            except Exception:  # pragma: no cover - interpreter shutdown
                pass
            self.ctx = None

    def call(self, name, *args):
        rc = getattr(_lib.lib(), name)(self.ctx, *args)
        _lib.check(rc, self.ctx)

    def nnz(self) -> int:
        """Stored nonzeros of a CSR operator (0 for dense / generated)."""
        out = C.c_int64(0)
        self.call("slim_nnz", C.byref(out))
        return out.value


def _dense_source(op):
    a = getattr(op, "matrix", None)
    if isinstance(a, np.ndarray) and a.ndim == 2:
        return a
    return None


def _stream_file_path(src):
    """Path of a single-pass .slim stream operator, else None."""
    if getattr(src, "access_mode", None) != "single_pass":
        return None
    path = getattr(src, "device_path", None)
    if path is None and type(src).__name__ == "FileStreamOperator":
        path = getattr(src, "_path", None)  # the reference's class (linops.py:374-386)
    return os.fspath(path) if path is not None else None


def device_operator(op, r: int, device: int = 0) -> DeviceOperator:
    """Upload ``op`` (once per (device, r)) and return its device context."""
    src = op.source if isinstance(op, SinglePassAdapter) else getattr(op, "_op", op)
    path = _stream_file_path(src)
    if path is not None:
        # a .slim stream (ours or the reference's FileStreamOperator): the
        # library reads each record from the file into HBM when its block is
        # first sampled; the matrix never passes through host memory
        cache = src.__dict__.setdefault("_slim_device_cache", {})
        key = (int(device), int(r), "file", path)
        if key not in cache:
            dop = DeviceOperator(n_rows=src.n_rows, n_cols=src.n_cols, ell=src.block_rows, r=r,
                                 layout=_lib.SLIM_DENSE_ROWMAJOR, dtype=np.float64, device=device)
            dop.call("slim_attach_stream_file", os.fsencode(path))
            cache[key] = dop
        return cache[key]
    if hasattr(src, "device_context"):  # tomo.ProjectorOperator: traced on the device
        return src.device_context(r, device)
    cache = src.__dict__.setdefault("_slim_device_cache", {})
    key = (int(device), int(r), id(getattr(src, "_b", None)))
    dop = cache.get(key)
    if dop is not None:
        return dop
    b = np.ascontiguousarray(np.asarray(src.rhs if hasattr(src, "rhs") else None, dtype=float))
    m, n, ell = src.n_rows, src.n_cols, src.block_rows
    if isinstance(src, GeneratedBlockOperator):
        dop = DeviceOperator(n_rows=m, n_cols=n, ell=ell, r=r, layout=_lib.SLIM_GEN_SPLITMIX64,
                             dtype=np.float32, device=device, gen_seed=src.seed, gen_n_total=n)
        dop.call("slim_set_rhs", _lib.dptr(b))
        dop.call("slim_finalize_operator")
        cache[key] = dop
        return dop
    if hasattr(src, "sparse_block") and not isinstance(src, SparseBlockOperator):
        # a reference SparseBlockOperator (linops.py:209-299): take its CSR
        # blocks as they are -- never its ``matrix`` property, which densifies
        # the whole operator -- and upload them like our own sparse operator
        mine = SparseBlockOperator([src.sparse_block(i) for i in range(1, src.n_blocks + 1)],
                                   src.rhs)
        dop = device_operator(mine, r, device)
        dop.host_op = mine  # keeps the registered host arrays alive
        cache[key] = dop
        return dop
    # host streaming (default): the operator is registered by pointer and each
    # block is copied to HBM inside slim_run right before the batch that first
    # samples it, overlapped with the device work of earlier batches; the
    # host arrays are kept alive by the device operator
    streaming = os.environ.get("SLIM_HOST_STREAMING", "1") != "0"
    a = _dense_source(src)
    if a is not None:
        dtype = np.float32 if a.dtype == np.float32 else np.float64
        dop = DeviceOperator(n_rows=m, n_cols=n, ell=ell, r=r, layout=_lib.SLIM_DENSE_ROWMAJOR,
                             dtype=dtype, device=device)
        a_c = np.ascontiguousarray(a, dtype=dtype)
        if streaming:
            dop.call("slim_set_host_streaming", 1)
            dop.host_refs = (a_c, b)
        dop.call("slim_upload_dense", _lib.vptr(a_c), _lib.dptr(b))
    elif streaming and isinstance(src, SparseBlockOperator):
        dop = DeviceOperator(n_rows=m, n_cols=n, ell=ell, r=r, layout=_lib.SLIM_CSR_PERBLOCK,
                             dtype=src.dtype, device=device)
        dop.call("slim_set_host_streaming", 1)
        refs = [b]
        nb = src.n_blocks
        ptrs = np.empty((3, nb), dtype=np.uintp)
        for i in range(1, nb + 1):
            ip, ix, d, _ = src.csr_block(i)
            ip = np.ascontiguousarray(ip, dtype=np.int64)
            ix = np.ascontiguousarray(ix, dtype=np.int32)
            d = np.ascontiguousarray(d, dtype=src.dtype)
            ptrs[0, i - 1] = ip.ctypes.data
            ptrs[1, i - 1] = ix.ctypes.data
            ptrs[2, i - 1] = d.ctypes.data
            refs.append((ip, ix, d))
        # one registration call for all blocks (the host arrays stay alive in refs)
        dop.call("slim_upload_csr_blocks", nb, C.c_void_p(ptrs[0].ctypes.data),
                 C.c_void_p(ptrs[1].ctypes.data), C.c_void_p(ptrs[2].ctypes.data), _lib.dptr(b))
        dop.host_refs = refs
    else:
        if isinstance(src, SparseBlockOperator):
            rowptr, col, val = src.global_csr()
            dtype = src.dtype
        else:  # generic random-access operator: densify once on the host
            blocks = [np.asarray(src.fetch_block(i).a_block, dtype=float)
                      for i in range(1, src.n_blocks + 1)]
            a = np.vstack(blocks)
            dop = DeviceOperator(n_rows=m, n_cols=n, ell=ell, r=r,
                                 layout=_lib.SLIM_DENSE_ROWMAJOR, dtype=np.float64, device=device)
            dop.call("slim_upload_dense", _lib.vptr(a), _lib.dptr(b))
            dop.call("slim_finalize_operator")
            cache[key] = dop
            return dop
        dop = DeviceOperator(n_rows=m, n_cols=n, ell=ell, r=r, layout=_lib.SLIM_CSR_PERBLOCK,
                             dtype=dtype, device=device)
        val = np.ascontiguousarray(val, dtype=dtype)
        dop.call("slim_upload_csr", _lib.i64ptr(rowptr), _lib.i32ptr(col), _lib.vptr(val),
                 _lib.dptr(b))
    dop.call("slim_finalize_operator")
    cache[key] = dop
    return dop
