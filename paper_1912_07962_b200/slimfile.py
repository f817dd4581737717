"""``.slim`` stream containers on the B200 path (reference format:
linops.py:334-429).

Byte layout (the interchange contract, unchanged): the 5-byte magic
``SLIM1``, then m, n, M, ell as little-endian uint64 (37 bytes), then M
records; record i is block i's ell x n fp64 entries (row-major) followed by
its ell fp64 right-hand-side entries.

What is different from the reference is where a record goes.  The
reference's ``FileStreamOperator`` reads each record into host memory on
``fetch_block``.  Here ``run()`` hands the PATH to the C-ABI
(``slim_attach_stream_file``): the library reads each record once, when its
block is first sampled, through the pinned staging ring straight into HBM,
overlapped with the device work of earlier steps.  The host never holds
more than the ring (8 x 4 MB), whatever the file size.  ``fetch_block``
stays available for host-side inspection with the reference's single-pass
rules and error messages.
"""

from __future__ import annotations

import os

import numpy as np

from .linops import DenseBlockOperator, RowBlockOperator, SampleBlock, StreamOrderError

STREAM_MAGIC = b"SLIM1"
# magic + (m, n, M, ell): one structured little-endian record
_HEAD = np.dtype([("magic", "S5"), ("m", "<u8"), ("n", "<u8"), ("M", "<u8"), ("ell", "<u8")])


def _record_bytes(n: int, ell: int) -> int:
    return 8 * ell * (n + 1)


def read_stream_header(path) -> tuple[int, int, int, int]:
    """(m, n, M, ell) of a container, validated like linops.py:360-371."""
    raw = np.fromfile(path, dtype=np.uint8, count=_HEAD.itemsize)
    if raw.size < _HEAD.itemsize:
        raise ValueError(f"{path}: truncated header")
    head = raw.view(_HEAD)[0]
    if bytes(head["magic"]) != STREAM_MAGIC:
        raise ValueError(f"{path}: bad magic {bytes(head['magic'])!r}, expected {STREAM_MAGIC!r}")
    m, n, big_m, ell = (int(head[k]) for k in ("m", "n", "M", "ell"))
    if big_m * ell != m:
        raise ValueError(f"{path}: header inconsistent, M*ell != m")
    return m, n, big_m, ell


def write_stream_file(path, op: RowBlockOperator):
    """Write a random-access operator with its rhs, one record per block
    (only one block is ever held in memory; generated operators included)."""
    op._require_random_access("write_stream_file")
    head = np.zeros(1, dtype=_HEAD)
    head[0] = (STREAM_MAGIC, op.n_rows, op.n_cols, op.n_blocks, op.block_rows)
    with open(path, "wb") as fh:
        head.tofile(fh)
        for i in range(1, op.n_blocks + 1):
            blk = op.fetch_block(i)
            np.asarray(blk.a_block, dtype="<f8").tofile(fh)
            np.asarray(blk.b_block, dtype="<f8").tofile(fh)


class FileStreamOperator(RowBlockOperator):
    """Single-pass operator over a ``.slim`` file (linops.py:374-415).

    On the device path the file is streamed record by record into HBM by
    the library (``device_path``); ``fetch_block`` serves host reads, in
    order, each block once.
    """

    access_mode = "single_pass"

    def __init__(self, path):
        self.path = os.fspath(path)
        self.n_rows, self.n_cols, self.n_blocks, self.block_rows = read_stream_header(self.path)
        self._rec = _record_bytes(self.n_cols, self.block_rows)
        self._next = 1
        self._open = True

    @property
    def device_path(self) -> str:
        return self.path

    def close(self):
        self._open = False

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def has_rhs(self) -> bool:
        return True

    def fetch_block(self, i: int) -> SampleBlock:
        self._check_index(i)
        if i != self._next:
            raise StreamOrderError(f"single-pass stream expected block {self._next}, got {i}")
        ell, n = self.block_rows, self.n_cols
        rec = np.fromfile(self.path, dtype="<f8", count=ell * (n + 1),
                          offset=_HEAD.itemsize + (i - 1) * self._rec)
        if rec.size != ell * (n + 1):
            raise ValueError(f"{self.path}: truncated record {i}")
        self._next += 1
        return SampleBlock(i, rec[:ell * n].reshape(ell, n), rec[ell * n:])

    @property
    def rhs(self):
        raise RuntimeError("rhs of a stream is only available block by block")


def load_stream_file(path) -> DenseBlockOperator:
    """Whole container as a random-access dense operator (linops.py:418-429)."""
    m, n, big_m, ell = read_stream_header(path)
    body = np.fromfile(path, dtype="<f8", count=big_m * ell * (n + 1),
                       offset=_HEAD.itemsize)
    if body.size != big_m * ell * (n + 1):
        raise ValueError(f"{path}: truncated record {body.size // (ell * (n + 1)) + 1}")
    # a record is ell*n block entries, then ell rhs entries
    flat = body.reshape(big_m, ell * (n + 1))
    return DenseBlockOperator(flat[:, :ell * n].reshape(m, n), ell, flat[:, ell * n:].reshape(m))
