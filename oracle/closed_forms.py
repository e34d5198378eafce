"""Closed forms that pin the oracle and the GPU path at full size (TEST INFRASTRUCTURE ONLY).

Geometric-sum closed form of a Vandermonde product (SURVEY.md §8(c) pin 4): with
A[i][t] = x_i^t (t = 0..k-1),

    (A A^T)_{ij} = sum_t (x_i x_j)^t = (r^k - 1) / (r - 1),  r = x_i x_j  (r != 1),   = k  (r = 1)

and over GF(p^2) = GF(p)[i]/(i^2+1) with A[i][t] = z_i^t and phi = conjugate transpose,

    (A A^H)_{ij} = sum_t (z_i conj(z_j))^t   (same geometric sum in GF(p^2)).

Costs O(log k) per entry, no O(k) work, so it checks sampled entries of 32768-wide outputs.
"""
from __future__ import annotations

import numpy as np


def _powmod_vec(base, e: int, p: int):
    base = np.asarray(base, dtype=np.int64) % p
    result = np.ones_like(base)
    while e:
        if e & 1:
            result = result * base % p
        base = base * base % p
        e >>= 1
    return result


def _inv_vec(x, p: int):
    return _powmod_vec(x, p - 2, p)


def vandermonde_syrk_entries(x, rows, k: int, p: int):
    """For each i in rows, the vector C[i][0..i] of Low(A A^T), A[i][t] = x_i^t mod p."""
    x = np.asarray(x, dtype=np.int64) % p
    out = []
    for i in rows:
        r = x[i] * x[: i + 1] % p
        num = (_powmod_vec(r, k, p) - 1) % p
        den = (r - 1) % p
        one = den == 0
        val = num * _inv_vec(np.where(one, 1, den), p) % p
        out.append(np.where(one, k % p, val).astype(np.int64))
    return out


# --- GF(p^2) = GF(p)[i]/(i^2+1), elements as (re, im) int64 pairs -------------------------

def _cmul(ar, ai, br, bi, p):
    return (ar * br - ai * bi) % p, (ar * bi + ai * br) % p


def _cpow(ar, ai, e: int, p: int):
    rr, ri = np.ones_like(ar), np.zeros_like(ai)
    while e:
        if e & 1:
            rr, ri = _cmul(rr, ri, ar, ai, p)
        ar, ai = _cmul(ar, ai, ar, ai, p)
        e >>= 1
    return rr, ri


def _cinv(ar, ai, p):
    n = (ar * ar + ai * ai) % p            # norm; nonzero for z != 0 when p = 3 mod 4
    ninv = _inv_vec(n, p)
    return ar * ninv % p, (-ai) * ninv % p


def vandermonde_herk_entries(z, rows, k: int, p: int):
    """Rows of Low(A A^H) for A[i][t] = z_i^t in GF(p^2); z: (m, 2).  Returns (re, im) per row."""
    z = np.asarray(z, dtype=np.int64) % p
    out = []
    for i in rows:
        cr, ci = z[: i + 1, 0], (-z[: i + 1, 1]) % p          # conj(z_j)
        rr, ri = _cmul(z[i, 0], z[i, 1], cr, ci, p)            # r = z_i conj(z_j)
        pr, pi = _cpow(rr, ri, k, p)
        nr, ni = (pr - 1) % p, pi % p                           # r^k - 1
        dr, di = (rr - 1) % p, ri % p                           # r - 1
        one = (dr == 0) & (di == 0)
        ir, ii = _cinv(np.where(one, 1, dr), np.where(one, 0, di), p)
        vr, vi = _cmul(nr, ni, ir, ii, p)
        out.append((np.where(one, k % p, vr), np.where(one, 0, vi)))
    return out
