"""Host-side seeded randomness for weights and the initial latent.

The reference draws every parameter and the x_T latent from one splitmix64
stream (pkg/src/pab_engine/numerics.py:161-215).  splitmix64 is counter
based: draw k of a stream at state s is mix(s + k * GOLDEN), so any slice of
the stream can be produced independently.  The host class below reproduces
the stream bit-for-bit; ``model.init_model(..., device="cuda")`` uses the same
counter formulation inside a CUDA kernel (csrc/init.cu) so that billion-
parameter configs are generated on the GPU instead of in numpy.
"""

from __future__ import annotations

import math

import numpy as np

from .errors import ValidationError

GOLDEN = 0x9E3779B97F4A7C15
MIX_A = 0xBF58476D1CE4E5B9
MIX_B = 0x94D049BB133111EB
MASK64 = (1 << 64) - 1


def splitmix_finalize(z: np.ndarray) -> np.ndarray:
    """The splitmix64 output function on a uint64 array (wrapping arithmetic)."""
    z = z.astype(np.uint64, copy=False)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(MIX_A)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(MIX_B)
    return z ^ (z >> np.uint64(31))


def counter_draws(state: int, start: int, n: int) -> np.ndarray:
    """Draws ``start+1 .. start+n`` of a stream whose current state is ``state``."""
    k = np.arange(start + 1, start + n + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        states = np.uint64(state & MASK64) + k * np.uint64(GOLDEN)
    return splitmix_finalize(states)


class RandomStream:
    """splitmix64 stream (same API and bit stream as the reference class)."""

    def __init__(self, state: int):
        self.state = int(state) & MASK64

    def next_u64(self) -> int:
        self.state = (self.state + GOLDEN) & MASK64
        return int(counter_draws(self.state, -1, 1)[0])

    def advance(self, n: int) -> int:
        """Skip ``n`` draws; returns the state before skipping."""
        before = self.state
        self.state = (self.state + n * GOLDEN) & MASK64
        return before

    def _raw(self, n: int) -> np.ndarray:
        before = self.advance(n)
        return counter_draws(before, 0, n)

    def uniform(self, n: int, lo: float = 0.0, hi: float = 1.0) -> np.ndarray:
        if not lo < hi:
            raise ValidationError(f"uniform needs lo < hi, got [{lo}, {hi})")
        mant = (self._raw(n) >> np.uint64(11)).astype(np.float64)
        return lo + (mant * 2.0**-53) * (hi - lo)

    def normal(self, n: int) -> np.ndarray:
        """Box-Muller on (first half, second half) of 2*ceil(n/2) draws."""
        half = (n + 1) // 2
        mant = self._raw(2 * half) >> np.uint64(11)
        u_radius = (mant[:half].astype(np.float64) + 1.0) * 2.0**-53
        u_angle = mant[half:].astype(np.float64) * 2.0**-53
        radius = np.sqrt(-2.0 * np.log(u_radius))
        angle = (2.0 * math.pi) * u_angle
        out = np.empty(2 * half, dtype=np.float64)
        out[0::2] = radius * np.cos(angle)
        out[1::2] = radius * np.sin(angle)
        return out[:n]
