"""Block-index selection, bit-exact with the reference ``Sampler``.

Same three schemes over 1-based block indices and the same Philox 4x64
stream keyed by the seed (reference sampling.py:35-84), so an index trace
is a pure function of (scheme, M, seed).  The B200 driver consumes the
trace up front: :meth:`Sampler.indices` gives the whole run's sequence,
which the device loop then walks without any host round trip.
"""

from __future__ import annotations

import numpy as np

SCHEMES = ("cyclic", "random_cyclic", "uniform_iid")


def _fisher_yates(m: int, rng: np.random.Generator) -> np.ndarray:
    """Backward shuffle of 1..m, one bounded draw per position (sampling.py:38-44)."""
    perm = np.arange(1, m + 1, dtype=np.int64)
    for i in range(m - 1, 0, -1):
        j = int(rng.integers(0, i + 1))
        perm[i], perm[j] = perm[j], perm[i]
    return perm


class Sampler:
    """Stateful index source (sampling.py:47-84); single-threaded."""

    def __init__(self, scheme: str, n_blocks: int, seed: int = 0):
        if scheme not in SCHEMES:
            raise ValueError(f"unknown scheme {scheme!r}, want one of {SCHEMES}")
        if n_blocks < 1:
            raise ValueError("n_blocks must be >= 1")
        self.scheme = scheme
        self.n_blocks = int(n_blocks)
        self.seed = int(seed)
        self.rng = np.random.Generator(np.random.Philox(key=self.seed))
        self.position = 0
        self._epoch_perm: np.ndarray | None = None

    def next_index(self) -> int:
        m = self.n_blocks
        if self.scheme == "cyclic":
            idx = self.position % m + 1
        elif self.scheme == "uniform_iid":
            idx = int(self.rng.integers(1, m + 1))
        else:
            offset = self.position % m
            if offset == 0:
                self._epoch_perm = _fisher_yates(m, self.rng)
            idx = int(self._epoch_perm[offset])
        self.position += 1
        return idx

    def indices(self, count: int) -> np.ndarray:
        """The next ``count`` indices (same sequence as repeated next_index)."""
        if self.scheme == "cyclic":
            out = (self.position + np.arange(count, dtype=np.int64)) % self.n_blocks + 1
            self.position += count
            return out
        return np.array([self.next_index() for _ in range(count)], dtype=np.int64)

    @property
    def epochs_completed(self) -> float:
        return self.position / self.n_blocks
