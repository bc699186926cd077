"""Oracle restatement of the reference RNG layer (TEST INFRASTRUCTURE ONLY).

Follows /root/reference/pkg/src/lowrank/rng.py:
  * stream = numpy Philox4x64-10 keyed by the 64-bit seed (rng.py:25-28)
  * normals by Box-Muller over one uniform block of 2*ceil(n/2): the first
    half feeds the radius as 1-u, the second half the angle; cos values go to
    even slots, sin values to odd slots (rng.py:38-55)
  * gaussian_block fills column by column then stores row-major (rng.py:77-94)
  * derive(tag) = (seed * 0x9E3779B97F4A7C15 + tag + 1) mod 2^63 (rng.py:72-74)
"""

from __future__ import annotations

import numpy as np

_GOLDEN = 0x9E3779B97F4A7C15
_MASK63 = (1 << 63) - 1


class Stream:
    def __init__(self, seed: int):
        self.seed = int(seed)
        self.drawn = 0
        self._bits = np.random.Generator(np.random.Philox(key=self.seed))

    def uniforms(self, count: int) -> np.ndarray:
        self.drawn += count
        return self._bits.random(count)

    def normals(self, count: int) -> np.ndarray:
        half = (count + 1) // 2
        u = self.uniforms(2 * half)
        rho = np.sqrt(-2.0 * np.log(1.0 - u[:half]))
        theta = 2.0 * np.pi * u[half:]
        out = np.empty(2 * half)
        out[0::2] = rho * np.cos(theta)
        out[1::2] = rho * np.sin(theta)
        return out[:count]

    def sample_distinct(self, universe: int, count: int) -> np.ndarray:
        self.drawn += count
        return self._bits.choice(universe, size=count, replace=False, shuffle=False)

    def shuffle_index(self, n: int) -> np.ndarray:
        self.drawn += n
        return self._bits.permutation(n)

    def derive(self, tag: int) -> "Stream":
        return Stream((self.seed * _GOLDEN + tag + 1) & _MASK63)


def gaussian_block(stream: Stream, rows: int, cols: int) -> np.ndarray:
    if rows < 1 or cols < 1:
        raise ValueError(f"gaussian matrix needs rows, cols >= 1, got {rows}x{cols}")
    flat = stream.normals(rows * cols)
    return np.ascontiguousarray(flat.reshape((cols, rows)).T)
