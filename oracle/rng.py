"""Counter-based RNG for the SRHT (reading G-10; "selecting
(uniformly at random) s rows ... diagonal matrix D with random i.i.d.
Rademacher (+-1) entries").  The paper names no generator; this is the fixed,
fully integer spec both sides implement independently:

  mix64(z)      the SplitMix64 output mixer (Steele, Lea & Flood 2014)
  phi           0x9E3779B97F4A7C15, the SplitMix64 increment
  key(seed,tag) mix64(seed ^ tag), tag = ASCII "SIGN" / "ROWS"
  h(key, i)     mix64(key + (i+1)*phi)   (= output i of SplitMix64(state=key))

  sign  D_tt = -1  iff bit 63 of h(key_SIGN, t) is set,   t in [0, N)
  rows  Floyd's sampling without replacement (G-8): for j = N-s .. N-1,
        q = h(key_ROWS, j-N+s), t = floor(q*(j+1) / 2^64); take j if t was
        already taken, else t.  Finally sort ascending.

All arithmetic is mod 2^64 on Python ints / numpy uint64: bit-exact.
TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
import numpy as np

MASK = (1 << 64) - 1
PHI = 0x9E3779B97F4A7C15
M1 = 0xBF58476D1CE4E5B9
M2 = 0x94D049BB133111EB
TAG_SIGN = 0x5349474E   # "SIGN"
TAG_ROWS = 0x524F5753   # "ROWS"


def mix64(z: int) -> int:
    z &= MASK
    z = ((z ^ (z >> 30)) * M1) & MASK
    z = ((z ^ (z >> 27)) * M2) & MASK
    return z ^ (z >> 31)


def splitmix64_stream(state: int, count: int):
    """Plain SplitMix64 generator: state += phi; yield mix64(state)."""
    out = []
    for _ in range(count):
        state = (state + PHI) & MASK
        out.append(mix64(state))
    return out


def key(seed: int, tag: int) -> int:
    return mix64((seed & MASK) ^ tag)


def h(k: int, i: int) -> int:
    return mix64((k + (i + 1) * PHI) & MASK)


def _mix64_np(z):
    z = z.astype(np.uint64, copy=True)
    with np.errstate(over="ignore"):
        z ^= z >> np.uint64(30)
        z *= np.uint64(M1)
        z ^= z >> np.uint64(27)
        z *= np.uint64(M2)
        z ^= z >> np.uint64(31)
    return z


def signs(seed: int, N: int, start: int = 0, count: int = None) -> np.ndarray:
    """D_tt in {+1,-1} (int8) for t in [start, start+count)."""
    if count is None:
        count = N - start
    k = np.uint64(key(seed, TAG_SIGN))
    t = np.arange(start, start + count, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = k + (t + np.uint64(1)) * np.uint64(PHI)
    hv = _mix64_np(z)
    neg = (hv >> np.uint64(63)).astype(bool)
    return np.where(neg, -1, 1).astype(np.int8)


def rows(seed: int, N: int, s: int) -> np.ndarray:
    """s distinct row indices in [0, N), sorted ascending (Floyd)."""
    return rows_from_key(key(seed, TAG_ROWS), N, s)


def rows_from_key(k: int, N: int, s: int) -> np.ndarray:
    """Floyd's sampling driven by the SplitMix64 stream of state k (q_i =
    h(k, i) = output i of SplitMix64(state = k))."""
    if not (1 <= s <= N):
        raise ValueError("need 1 <= s <= N")
    chosen = set()
    for j in range(N - s, N):
        q = h(k, j - N + s)
        t = (q * (j + 1)) >> 64
        chosen.add(j if t in chosen else t)
    return np.array(sorted(chosen), dtype=np.int64)
