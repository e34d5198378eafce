"""ORACLE -- TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously correct CPU implementation of what the hot path computes,
written from the paper (arXiv 2101.01025, PAPER.md).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / ``--impl reference`` legs may
import, call, link or execute anything here.  The CUDA product path
(``paper_2101_01025_b200``) never imports it and shares no code, header, table or constant
generator with it; the only shared module is ``inputs`` (seeded generators, no method
arithmetic).

Contents
- oracle.c / liboracle.so (O1): classical Low(A phi(A)) mod p in uint64, OpenMP over rows:
  phi = transpose over GF(p), phi = conjugate transpose over GF(p)[i]/(i^2+1) and over the
  quaternions H_GF(p) (§6.2), and A B^T.
  Definition: Lemma lem:transp; Low.
- field.py: Legendre, Tonelli-Shanks, Alg. alg:sosmodp, Prop. lem:lemsqrt.
- alg1.py (O2): Alg. alg:MIAHMM and Alg. alg:2M
  re-derived step by step in numpy.
- closed_forms.py: Vandermonde geometric-sum closed forms for full-size sampled checks.

Pins (tests/test_oracle_*.py, ``-m "not gpu"``): brute force on tiny fields, exhaustive
enumeration of GF(3)^{2x4} / GF(5)^{2x2}, worked values from SPEC.md, closed forms,
float64 BLAS (exact since k (p-1)^2 < 2^53), invariants.  Parity is pinned for every
function here; none is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_LIB = None


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so with plain gcc + OpenMP."""
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O3", "-march=native", "-fopenmp", "-shared", "-fPIC",
                               "-Wall", src, "-o", _SO])
    return _SO


def _lib():
    global _LIB
    if _LIB is None:
        build()
        lib = ctypes.CDLL(_SO)
        i64, u32, vp = ctypes.c_int64, ctypes.c_uint32, ctypes.c_void_p
        lib.oracle_syrk_t_rows.argtypes = [i64, i64, u32, vp, i64, vp, i64, i64, i64]
        lib.oracle_syrk_h_rows.argtypes = [i64, i64, u32, vp, i64, vp, i64, i64, i64]
        lib.oracle_gemm_nt.argtypes = [i64, i64, i64, u32, vp, i64, vp, i64, vp, i64]
        lib.oracle_syrk_q_rows.argtypes = [i64, i64, u32, vp, i64, vp, i64, i64, i64]
        for f in (lib.oracle_syrk_t_rows, lib.oracle_syrk_h_rows, lib.oracle_gemm_nt, lib.oracle_syrk_q_rows):
            f.restype = ctypes.c_int
        lib.oracle_num_threads.restype = ctypes.c_int
        _LIB = lib
    return _LIB


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def syrk_t(A: np.ndarray, p: int, rows=None) -> np.ndarray:
    """Low(A A^T) mod p as an m x m uint32 array (upper strictly = 0).  rows=(r0, r1) limits
    the computed rows (entries outside stay 0)."""
    A = np.ascontiguousarray(A, dtype=np.uint32)
    m, k = A.shape
    C = np.zeros((m, m), dtype=np.uint32)
    r0, r1 = (0, m) if rows is None else rows
    rc = _lib().oracle_syrk_t_rows(m, k, p, _ptr(A), k, _ptr(C), m, r0, r1)
    if rc:
        raise RuntimeError(f"oracle_syrk_t_rows rc={rc}")
    return C


def syrk_h(A: np.ndarray, p: int, rows=None) -> np.ndarray:
    """Low(A A^H) over GF(p)[i]/(i^2+1); A: (m, k, 2) interleaved (re, im); returns (m, m, 2)."""
    A = np.ascontiguousarray(A, dtype=np.uint32)
    m, k, _ = A.shape
    C = np.zeros((m, m, 2), dtype=np.uint32)
    r0, r1 = (0, m) if rows is None else rows
    rc = _lib().oracle_syrk_h_rows(m, k, p, _ptr(A), k, _ptr(C), m, r0, r1)
    if rc:
        raise RuntimeError(f"oracle_syrk_h_rows rc={rc}")
    return C


def syrk_q(M: np.ndarray, p: int, rows=None) -> np.ndarray:
    """Low(M M^H) over the quaternions H_GF(p) (§6.2); M: (m, k, 4) interleaved
    (x1, x2, x3, x4) = x1 + x2 i + x3 j + x4 k; returns (m, m, 4)."""
    M = np.ascontiguousarray(M, dtype=np.uint32)
    m, k, _ = M.shape
    C = np.zeros((m, m, 4), dtype=np.uint32)
    r0, r1 = (0, m) if rows is None else rows
    rc = _lib().oracle_syrk_q_rows(m, k, p, _ptr(M), k, _ptr(C), m, r0, r1)
    if rc:
        raise RuntimeError(f"oracle_syrk_q_rows rc={rc}")
    return C


def gemm_nt(A: np.ndarray, B: np.ndarray, p: int) -> np.ndarray:
    """A B^T mod p (full)."""
    A = np.ascontiguousarray(A, dtype=np.uint32)
    B = np.ascontiguousarray(B, dtype=np.uint32)
    m, k = A.shape
    n, k2 = B.shape
    assert k == k2
    C = np.zeros((m, n), dtype=np.uint32)
    rc = _lib().oracle_gemm_nt(m, n, k, p, _ptr(A), k, _ptr(B), k, _ptr(C), n)
    if rc:
        raise RuntimeError(f"oracle_gemm_nt rc={rc}")
    return C


def num_threads() -> int:
    return int(_lib().oracle_num_threads())


def syrk_update(A: np.ndarray, C: np.ndarray, p: int, alpha: int, beta: int, phi: str = "T") -> np.ndarray:
    """SYRK / HERK form (Table tab:schedule:AATpC): returns C' with
    Low(C') = alpha Low(A phi(A)) + beta Low(C) mod p and Up(C') = Up(C) (old values kept).
    Composed from the O1 definition; alpha, beta in GF(p) scale every component alike for
    phi = H (re, im) and phi = Q (the four quaternion components)."""
    base = {"T": syrk_t, "H": syrk_h, "Q": syrk_q}[phi](A, p)
    out = C.copy()
    m = C.shape[0]
    mask = np.tril(np.ones((m, m), dtype=bool))
    if C.ndim == 3:
        mask = mask[:, :, None] & np.ones((1, 1, C.shape[2]), dtype=bool)
    new = (int(alpha) % p * base.astype(np.int64) + int(beta) % p * (C.astype(np.int64) % p)) % p
    out[mask] = new[mask].astype(np.uint32)
    return out
