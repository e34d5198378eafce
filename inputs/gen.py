"""Counter-based seeded input generators (numpy, host side).  See package docstring."""
from __future__ import annotations

import numpy as np

_M64 = (1 << 64) - 1
_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_C1 = np.uint64(0xBF58476D1CE4E5B9)
_C2 = np.uint64(0x94D049BB133111EB)


def splitmix64(x):
    """splitmix64 finaliser on uint64 (scalar int or numpy array), wrapping mod 2^64."""
    if isinstance(x, (int, np.integer)):
        z = (int(x) + 0x9E3779B97F4A7C15) & _M64
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
        return z ^ (z >> 31)
    z = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z + _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _C1
        z = (z ^ (z >> np.uint64(27))) * _C2
    return z ^ (z >> np.uint64(31))


def mulhi64(x, p: int):
    """floor(x * p / 2^64) for uint64 x and p < 2^32, exact (split x into 32-bit halves)."""
    if isinstance(x, (int, np.integer)):
        return (int(x) * int(p)) >> 64
    x = np.asarray(x, dtype=np.uint64)
    pp = np.uint64(p)
    lo = x & np.uint64(0xFFFFFFFF)
    hi = x >> np.uint64(32)
    with np.errstate(over="ignore"):
        t = hi * pp + ((lo * pp) >> np.uint64(32))   # < 2^64, no wrap (p < 2^32)
    return t >> np.uint64(32)


def uniform_residues(n: int, seed: int, p: int, start: int = 0,
                     chunk: int = 1 << 24) -> np.ndarray:
    """Flat uint32 array r[j] = mulhi64(splitmix64(splitmix64(seed) ^ (start+j)), p), j < n."""
    if not (2 <= p < (1 << 32)):
        raise ValueError("p must be in [2, 2^32)")
    key = np.uint64(splitmix64(int(seed)))
    out = np.empty(n, dtype=np.uint32)
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        j = np.arange(start + s, start + e, dtype=np.uint64)
        out[s:e] = mulhi64(splitmix64(j ^ key), p).astype(np.uint32)
    return out


def uniform_matrix(m: int, k: int, seed: int, p: int) -> np.ndarray:
    """m x k uint32 matrix of uniform residues mod p (row-major flat index i*k+t)."""
    return uniform_residues(m * k, seed, p).reshape(m, k)


def uniform_matrix_ext(m: int, k: int, seed: int, p: int) -> np.ndarray:
    """m x k x 2 uint32 array: GF(p^2) matrix as interleaved (re, im) residue pairs."""
    return uniform_residues(2 * m * k, seed, p).reshape(m, k, 2)


def uniform_matrix_quat(m: int, k: int, seed: int, p: int) -> np.ndarray:
    """m x k x 4 uint32 array: a quaternion matrix over GF(p) as interleaved (x1, x2, x3, x4)
    = x1 + x2 i + x3 j + x4 k (flat index 4 (i k + t) + c)."""
    return uniform_residues(4 * m * k, seed, p).reshape(m, k, 4)


def vandermonde_points(m: int, seed: int, p: int) -> np.ndarray:
    """m seeded evaluation points x_i in [1, p)."""
    return (uniform_residues(m, seed ^ 0x5A5A5A5A, p - 1) + 1).astype(np.uint32)


def vandermonde_matrix(x: np.ndarray, k: int, p: int) -> np.ndarray:
    """A[i][t] = x_i^t mod p (t = 0..k-1), uint32.  Powers are built column by column.

    For GF(p^2) pass x as an (m, 2) array of (re, im) with i^2 = -1; returns (m, k, 2).
    """
    x = np.asarray(x, dtype=np.int64)
    if x.ndim == 1:
        m = x.shape[0]
        out = np.empty((k, m), dtype=np.uint32)
        cur = np.ones(m, dtype=np.int64)
        for t in range(k):
            out[t] = cur
            cur = (cur * x) % p
        return np.ascontiguousarray(out.T)
    m = x.shape[0]
    out = np.empty((k, m, 2), dtype=np.uint32)
    cr = np.ones(m, dtype=np.int64)
    ci = np.zeros(m, dtype=np.int64)
    xr, xi = x[:, 0], x[:, 1]
    for t in range(k):
        out[t, :, 0] = cr
        out[t, :, 1] = ci
        cr, ci = (cr * xr - ci * xi) % p, (cr * xi + ci * xr) % p
    return np.ascontiguousarray(out.transpose(1, 0, 2))


def constant_matrix(m: int, k: int, c: int, p: int) -> np.ndarray:
    """A[i][t] = c mod p (overflow-stress input: drives each limb to a chosen extreme)."""
    return np.full((m, k), c % p, dtype=np.uint32)
