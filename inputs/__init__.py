"""Seeded synthetic inputs shared by the oracle tests, the CUDA parity tests and bench.py.

This module holds NONE of the method's arithmetic (no products, no pre-additions,
no skew-unitary matrices).  It only turns (seed, index) into residues.

Generator (SURVEY.md §8(d) "Synthetic inputs"): a counter-based PRNG,

    A_flat[j] = mulhi64(splitmix64(splitmix64(seed) ^ j), p)

where ``mulhi64(x, p) = (x * p) >> 64`` maps a 64-bit word to [0, p) with bias
<= p / 2^64.  ``j`` is the flat row-major position (j = i*k + t for an m x k
matrix with leading dimension k).  For GF(p^2) inputs stored as interleaved
(re, im) pairs the flat index of the real part is 2*(i*k+t) and of the
imaginary part 2*(i*k+t)+1, i.e. the same formula over the interleaved array.

The paper (§7) measures on square random matrices over
Z/131071Z without stating the distribution; uniform residues stand in.

The same generator exists on the GPU (``inputs/gen.cu`` -> ``inputs/_gen.so``)
so that multi-GiB inputs can be made in HBM; tests check both agree bit for bit.
"""
from .gen import (splitmix64, mulhi64, uniform_residues, uniform_matrix,
                  uniform_matrix_ext, uniform_matrix_quat, vandermonde_points, vandermonde_matrix,
                  constant_matrix)

__all__ = ["splitmix64", "mulhi64", "uniform_residues", "uniform_matrix",
           "uniform_matrix_ext", "uniform_matrix_quat", "vandermonde_points", "vandermonde_matrix",
           "constant_matrix"]
