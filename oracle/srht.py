"""Subsampled randomized Hadamard transform (§2.1.1):

  "Theta consists of selecting (uniformly at random) s rows from the product
   of the Walsh-Hadamard transform with a diagonal matrix D with random
   i.i.d. Rademacher (+-1) entries on the diagonal."

Readings: natural / Sylvester ordering H[r,t] = (-1)^popcount(r&t)
(G-6); zero-pad n to N = 2^ceil(log2 n) (G-7); rows without replacement,
sorted (G-8); Theta = (1/sqrt(s)) P H_N D so that E||Theta x||^2 = ||x||^2
and Theta is an isometry at s = N (G-9); RNG per oracle/rng.py (G-10).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
import math

import numpy as np

from . import rng


def next_pow2(n: int) -> int:
    return 1 << max(0, (int(n) - 1).bit_length())


def fwht(x: np.ndarray) -> np.ndarray:
    """Textbook radix-2 fast Walsh-Hadamard transform, natural order,
    unnormalized: for h = 1, 2, 4, ...: (a, b) <- (a + b, a - b) on pairs
    (j, j+h).  Works along axis 0 (vector or matrix of columns)."""
    y = np.array(x, dtype=np.float64, copy=True)
    N = y.shape[0]
    assert N & (N - 1) == 0, "length must be a power of two"
    rest = y.shape[1:]
    h = 1
    while h < N:
        v = y.reshape((N // (2 * h), 2, h) + rest)
        a = v[:, 0].copy()
        b = v[:, 1]
        v[:, 0] += b
        v[:, 1] = a - b
        h *= 2
    return y


def hadamard_dense(N: int) -> np.ndarray:
    """H[r, t] = (-1)^popcount(r & t), written out entry by entry."""
    r = np.arange(N)[:, None]
    t = np.arange(N)[None, :]
    a = r & t
    pc = np.zeros_like(a)
    while a.any():
        pc += a & 1
        a = a >> 1
    return np.where(pc % 2 == 1, -1.0, 1.0)


class SRHT:
    """Theta in R^{s x n}: rows, signs, scale = 1/sqrt(s)."""

    def __init__(self, n: int, s: int, seed: int):
        self.n = int(n)
        self.N = next_pow2(n)
        if not (1 <= s <= self.N):
            raise ValueError("InvalidSketchSize: need 1 <= s <= N")
        self.s = int(s)
        self.seed = int(seed)
        self.rows = rng.rows(seed, self.N, s)
        self.signs = rng.signs(seed, self.N)          # length N (padding too)
        self.scale = 1.0 / math.sqrt(s)

    def apply(self, x: np.ndarray) -> np.ndarray:
        """Theta x for a vector, or column by column for a matrix."""
        x = np.asarray(x, dtype=np.float64)
        if x.ndim == 2:
            return np.stack([self.apply(x[:, j]) for j in range(x.shape[1])], axis=1)
        if x.shape[0] != self.n:
            raise ValueError("DimensionMismatch")
        pad = np.zeros(self.N)
        pad[: self.n] = x * self.signs[: self.n]   # D [x; 0]
        y = fwht(pad)                               # H_N D [x; 0]
        return self.scale * y[self.rows]            # (1/sqrt s) P H_N D [x; 0]

    def row_entry(self, r: int, x: np.ndarray) -> float:
        """One sketch entry (Theta x)_r for sampled row r, by definition
        sum_t H[r,t] D_tt x_t / sqrt(s) -- O(n), used for full-size spot
        checks where the full FWHT is too slow."""
        t = np.arange(self.n, dtype=np.int64)
        a = np.int64(r) & t
        # popcount parity of (r & t)
        par = np.zeros(self.n, dtype=np.int64)
        while a.any():
            par ^= a & 1
            a >>= 1
        hs = np.where(par == 1, -1.0, 1.0) * self.signs[: self.n]
        return float(self.scale * np.dot(hs, x))
