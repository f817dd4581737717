"""Block-index selection, bit-exact with the reference ``Sampler``
(sampling.py:35-84).

An index trace is a pure function of (scheme, M, seed): the three schemes
draw 1-based block indices from the Philox 4x64 stream keyed by the seed,
with the reference's draw sequence (one bounded draw per step for
``uniform_iid``; one backward Fisher-Yates shuffle per epoch for
``random_cyclic``; no draws for ``cyclic``). The B200 driver takes the whole
run's trace up front (:meth:`Sampler.indices`) and the device loop walks it
without host round trips.
"""

from __future__ import annotations

import numpy as np

SCHEMES = ("cyclic", "random_cyclic", "uniform_iid")


def _shuffled(m: int, rng: np.random.Generator) -> np.ndarray:
    """1..m permuted by a backward Fisher-Yates pass: position i (from m - 1
    down to 1) swaps with a uniform draw from [0, i] (sampling.py:38-44)."""
    order = np.arange(1, m + 1, dtype=np.int64)
    for i in range(m - 1, 0, -1):
        j = int(rng.integers(0, i + 1))
        order[[i, j]] = order[[j, i]]
    return order


class Sampler:
    """Stateful index source with the reference attributes (``scheme``,
    ``n_blocks``, ``seed``, ``rng``, ``position``); single-threaded."""

    def __init__(self, scheme: str, n_blocks: int, seed: int = 0):
        if scheme not in SCHEMES:
            raise ValueError(f"unknown scheme {scheme!r}, want one of {SCHEMES}")
        if n_blocks < 1:
            raise ValueError("n_blocks must be >= 1")
        self.scheme, self.n_blocks, self.seed = scheme, int(n_blocks), int(seed)
        self.rng = np.random.Generator(np.random.Philox(key=self.seed))
        self.position = 0
        self._order = None  # the current epoch's permutation (random_cyclic)

    def _draw_cyclic(self) -> int:
        return self.position % self.n_blocks + 1

    def _draw_iid(self) -> int:
        return int(self.rng.integers(1, self.n_blocks + 1))

    def _draw_permuted(self) -> int:
        slot = self.position % self.n_blocks
        if slot == 0:  # a new epoch: a fresh permutation
            self._order = _shuffled(self.n_blocks, self.rng)
        return int(self._order[slot])

    def _draw(self) -> int:
        if self.scheme == "cyclic":
            return self._draw_cyclic()
        if self.scheme == "uniform_iid":
            return self._draw_iid()
        return self._draw_permuted()

    def next_index(self) -> int:
        idx = self._draw()
        self.position += 1
        return idx

    def indices(self, count: int) -> np.ndarray:
        """The next ``count`` indices, as ``count`` calls of next_index."""
        if self.scheme == "cyclic":  # no draws: closed form
            out = (self.position + np.arange(count, dtype=np.int64)) % self.n_blocks + 1
            self.position += count
            return out
        return np.fromiter((self.next_index() for _ in range(count)), dtype=np.int64, count=count)

    @property
    def epochs_completed(self) -> float:
        return self.position / self.n_blocks
