"""Counter-based SplitMix64 streams (test/bench input infrastructure).

This module holds NO arithmetic of the rendering method. It only turns a
(seed, stream, counter) triple into reproducible random numbers, so that the
CUDA path's tests, ``bench.py`` and the oracle tests see the same synthetic
inputs (SURVEY.md §8(d) "Synthetic inputs": SplitMix64, uniform f32 from the
top 24 bits, normals by Box-Muller in f64).
"""
from __future__ import annotations

import numpy as np

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def _mix(z: np.ndarray) -> np.ndarray:
    z = z.copy()
    z ^= z >> np.uint64(30)
    z *= _M1
    z ^= z >> np.uint64(27)
    z *= _M2
    z ^= z >> np.uint64(31)
    return z


class Stream:
    """One independent SplitMix64 stream; draws advance an internal counter."""

    def __init__(self, seed: int, stream: int = 0):
        with np.errstate(over="ignore"):
            base = _mix(np.array([(seed * 0x100000001B3 + stream * 0x2545F4914F6CDD1D) & (2**64 - 1)],
                                 dtype=np.uint64))[0]
        self._base = np.uint64(base)
        self._ctr = 0

    def u64(self, n: int) -> np.ndarray:
        idx = np.arange(self._ctr + 1, self._ctr + 1 + n, dtype=np.uint64)
        self._ctr += n
        with np.errstate(over="ignore"):
            return _mix(self._base + idx * _GOLDEN)

    def uniform(self, n: int, lo: float = 0.0, hi: float = 1.0) -> np.ndarray:
        """Uniform in [lo, hi): f32 mantissa from the top 24 bits, returned as f64."""
        u = (self.u64(n) >> np.uint64(40)).astype(np.float64) * (1.0 / 16777216.0)
        return lo + (hi - lo) * u

    def normal(self, n: int, mean: float = 0.0, std: float = 1.0) -> np.ndarray:
        """Box-Muller in f64 (one normal per pair of uniforms)."""
        u1 = self.uniform(n)
        u2 = self.uniform(n)
        r = np.sqrt(-2.0 * np.log1p(-u1))  # 1-u1 in (0,1]
        return mean + std * r * np.cos(2.0 * np.pi * u2)

    def integers(self, n: int, lo: int, hi: int) -> np.ndarray:
        """Integers in [lo, hi)."""
        span = np.uint64(hi - lo)
        return (self.u64(n) % span).astype(np.int64) + lo
