"""Whole-output checks of Low(C) = Low(A phi(A)) mod p for the -m gpu full-size parity tests
(tests/test_gpu_fullsize_exact.py), device-agnostic and pinned on the CPU against the oracle
(tests/test_fullsize_check.py).  Test infrastructure: no method arithmetic of the CUDA path.

- freivalds_low: C r == A (phi(A) r) mod p on the host in the ring's own arithmetic (GF(p),
  GF(p)[i]/(i^2+1) with phi = conjugate transpose, the quaternions over GF(p) with phi =
  conjugate transpose; quaternion table), C's upper triangle completed by
  Lemma lem:uplow.  float64, exact while sums stay below 2^53.
- exact_low_mismatches: every lower entry against sum_t A_it phi(A_jt) mod p evaluated as float64
  matrix products with torch (cuBLAS on the GPU), exact since k (p-1)^2 < 2^53 (SURVEY.md
  §8(c)-6, the paper's "dsyrk + mod p" route).
"""
import numpy as np

EXACT_F64 = 2.0 ** 53


def _matvec(X, v, w, conj_left=False, transpose=False, rows=1024):
    """sum over the contracted index of X[i, t] * v[t] (or conj(X[t, i]) * v[t] with transpose),
    X (m, k, w), v (k, w) / (m, w): the ring product written per component with float64 BLAS
    matvecs over blocks of `rows` rows of X (bounded host memory); exact while every sum stays
    below 2^53."""
    m = X.shape[0]
    if transpose:
        out = None
        for r0 in range(0, m, rows):
            part = _matvec_block(X[r0:r0 + rows], v[r0:r0 + rows], w, conj_left, True)
            out = part if out is None else out + part
        return out
    return np.concatenate([_matvec_block(X[r0:r0 + rows], v, w, conj_left, False) for r0 in range(0, m, rows)])


def _matvec_block(X, v, w, conj_left, transpose):
    comps = [np.ascontiguousarray(X[..., q], dtype=np.float64) for q in range(w)]
    if w == 1:
        M = comps[0].T if transpose else comps[0]
        return (M @ v[:, 0])[:, None]

    def mv(q, vec):
        M = comps[q].T if transpose else comps[q]
        return M @ vec
    sgn = -1.0 if conj_left else 1.0
    if w == 2:   # (xr + i xi)(vr + i vi), xi -> -xi when conjugated
        xr_vr, xr_vi = mv(0, v[:, 0]), mv(0, v[:, 1])
        xi_vr, xi_vi = sgn * mv(1, v[:, 0]), sgn * mv(1, v[:, 1])
        return np.stack([xr_vr - xi_vi, xr_vi + xi_vr], axis=-1)
    prods = [[(sgn if q else 1.0) * mv(q, v[:, r]) for r in range(4)] for q in range(4)]   # x_q v_r
    a, b, c, d = prods
    return np.stack([a[0] - b[1] - c[2] - d[3], a[1] + b[0] + c[3] - d[2],
                     a[2] - b[3] + c[0] + d[1], a[3] + b[2] - c[1] + d[0]], axis=-1)


def freivalds_low(Ah, Cl, p, w, nvec=2, seed=0, block=2048):
    """C r == A (phi(A) r) mod p, C completed from Low(C) by Up(C) = phi(Low(C)).
    Ah (m, k, w) residues, Cl (m, m, w) residues (only the lower triangle is read)."""
    m = Ah.shape[0]
    rng = np.random.default_rng(seed)
    for _ in range(nvec):
        r = rng.integers(0, p, size=(m, w)).astype(np.float64)
        t = np.mod(_matvec(Ah, r, w, conj_left=True, transpose=True), p)   # phi(A) r
        rhs = np.mod(_matvec(Ah, t, w), p)                                   # A (phi(A) r)
        lhs = np.zeros((m, w))
        for r0 in range(0, m, block):
            r1 = min(m, r0 + block)
            blk = Cl[r0:r1, :r1].astype(np.float64)                  # rows r0..r1, cols < r1
            ii = np.arange(r0, r1)[:, None]
            jj = np.arange(r1)[None, :]
            lower = (jj <= ii)[..., None]
            strict = (jj < ii)[..., None]
            L = np.where(lower, blk, 0.0)
            lhs[r0:r1] += _matvec(L, r[:r1], w)                      # sum_{j <= i} C_ij r_j
            # upper entries C_ji = phi(C_ij) for j < i contribute to rows j < r1
            U = np.where(strict, blk, 0.0)
            lhs[:r1] += _matvec(U, r[r0:r1], w, conj_left=True, transpose=True)
        if not np.array_equal(np.mod(lhs, p), rhs):
            return False
    return True


# ----------------------------------------------------------------------------- GPU float64 product
def exact_low_mismatches(torch, A, C, p, w, block=2048):
    """Number of lower-triangle entries of C that differ from the definition
    sum_t A_it phi(A_jt) mod p, evaluated as float64 products on the GPU (exact: k (p-1)^2 < 2^53)."""
    m, k = A.shape[0], A.shape[1]
    assert k * 4.0 * (p - 1) ** 2 < EXACT_F64
    comps = [A[..., q].to(torch.float64) for q in range(w)]
    bad = 0
    for r0 in range(0, m, block):
        r1 = min(m, r0 + block)
        mm = lambda x, y: x[r0:r1] @ y[:r1].T                       # noqa: E731
        if w == 1:
            refs = [mm(comps[0], comps[0])]
        elif w == 2:      # (x_i + i y_i)(x_j - i y_j)
            x, y = comps
            refs = [mm(x, x) + mm(y, y), mm(y, x) - mm(x, y)]
        else:             # M_i conj(M_j), M = a + b i + c j + d k
            a, b, c, d = comps
            refs = [mm(a, a) + mm(b, b) + mm(c, c) + mm(d, d),
                    mm(b, a) - mm(a, b) + mm(d, c) - mm(c, d),
                    mm(c, a) - mm(a, c) + mm(b, d) - mm(d, b),
                    mm(d, a) - mm(a, d) + mm(c, b) - mm(b, c)]
        ii = torch.arange(r0, r1, device=A.device)[:, None]
        jj = torch.arange(r1, device=A.device)[None, :]
        lower = jj <= ii
        for q, ref in enumerate(refs):
            ref = torch.remainder(ref, p).to(torch.int32)
            got = C[r0:r1, :r1, q]
            bad += int(((ref != got) & lower).sum().item())
        del refs
    return bad
