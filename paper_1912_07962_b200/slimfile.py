"""The reference's streamed-matrix container (``.slim``, linops.py:334-429).

Fixed header: magic ``SLIM1`` then m, n, M, ell as little-endian uint64;
then M records of ell*n fp64 block entries followed by ell fp64 right-hand
side entries, row-major.  ``FileStreamOperator`` is single-pass (blocks in
order 1..M, each once); for the device path the stream is consumed once in
order and uploaded (the device keeps the operator resident).
"""

from __future__ import annotations

import struct

import numpy as np

from .linops import DenseBlockOperator, RowBlockOperator, SampleBlock, StreamOrderError

STREAM_MAGIC = b"SLIM1"
_HEADER = struct.Struct("<5sQQQQ")


def write_stream_file(path, op: RowBlockOperator):
    """Write a random-access operator with its rhs (linops.py:346-357)."""
    op._require_random_access("write_stream_file")
    with open(path, "wb") as fh:
        fh.write(_HEADER.pack(STREAM_MAGIC, op.n_rows, op.n_cols, op.n_blocks, op.block_rows))
        for i in range(1, op.n_blocks + 1):
            blk = op.fetch_block(i)
            fh.write(np.ascontiguousarray(blk.a_block, dtype="<f8").tobytes())
            fh.write(np.ascontiguousarray(blk.b_block, dtype="<f8").tobytes())


def read_stream_header(path) -> tuple[int, int, int, int]:
    with open(path, "rb") as fh:
        raw = fh.read(_HEADER.size)
    if len(raw) < _HEADER.size:
        raise ValueError(f"{path}: truncated header")
    magic, m, n, big_m, ell = _HEADER.unpack(raw)
    if magic != STREAM_MAGIC:
        raise ValueError(f"{path}: bad magic {magic!r}, expected {STREAM_MAGIC!r}")
    if big_m * ell != m:
        raise ValueError(f"{path}: header inconsistent, M*ell != m")
    return m, n, big_m, ell


class FileStreamOperator(RowBlockOperator):
    """Single-pass operator reading blocks from a container file (linops.py:374-415)."""

    access_mode = "single_pass"

    def __init__(self, path):
        self._path = path
        self.n_rows, self.n_cols, self.n_blocks, self.block_rows = read_stream_header(path)
        self._fh = open(path, "rb")
        self._fh.seek(_HEADER.size)
        self._next = 1

    def close(self):
        if self._fh is not None:
            self._fh.close()
            self._fh = None

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
        raw = self._fh.read((ell * n + ell) * 8)
        if len(raw) != (ell * n + ell) * 8:
            raise ValueError(f"{self._path}: truncated record {i}")
        a = np.frombuffer(raw, dtype="<f8", count=ell * n).reshape(ell, n)
        b = np.frombuffer(raw, dtype="<f8", offset=ell * n * 8, count=ell)
        self._next += 1
        return SampleBlock(i, a, b)

    def consume_all(self) -> DenseBlockOperator:
        """Read the remaining stream once, in order, into a resident operator."""
        if self._next != 1:
            raise StreamOrderError(f"single-pass stream expected block {self._next}, got 1")
        a = np.empty((self.n_rows, self.n_cols))
        b = np.empty(self.n_rows)
        ell = self.block_rows
        for i in range(1, self.n_blocks + 1):
            blk = self.fetch_block(i)
            a[(i - 1) * ell:i * ell] = blk.a_block
            b[(i - 1) * ell:i * ell] = blk.b_block
        self._next = 1  # the device copy now serves the pass
        return DenseBlockOperator(a, ell, b)

    @property
    def rhs(self):
        raise RuntimeError("rhs of a stream is only available block by block")


def load_stream_file(path) -> DenseBlockOperator:
    """Whole container as a random-access dense operator (linops.py:418-429)."""
    with FileStreamOperator(path) as stream:
        return stream.consume_all()
