"""O2 -- CPU re-derivation of the paper's algorithms (TEST INFRASTRUCTURE ONLY).

Step by step in the paper's order and notation, on numpy int64 residues mod p (values < p
<= 2^16 so every product fits; numpy matmul is the only library primitive used, as the
"general matrix multiplication" of the paper).  Arrays may carry leading batch axes so the
exhaustive pins can run thousands of tiny matrices at once.

- syrk_def(A, p)                 Low(A A^T): the plain definition (Lemma lem:transp)
- apply_Y(X, Y, p)               X Y for Y = i I or Y = [[a,b],[-b,a]] (x) I
                                 (Prop. lem:pigeonhole): [X1 X2] -> [aX1 - bX2, bX1 + aX2]
- alg1(A, p, Y, depth)           Alg. alg:MIAHMM recursing on P1, P2, P5 (the algorithm box,
                                 PAPER.md:308; the proof's "P7" at PAPER.md:343 is read as P5)
- herk_def(X, Y, p)              (X+iY)(X+iY)^H over GF(p)[i]/(i^2+1) by definition
- alg2m(X, Y, p, ...)            Alg. alg:2M with phi = conjugate transpose
Odd dimensions are zero-padded, which leaves A A^T unchanged.
"""
from __future__ import annotations

import numpy as np


class MulCounter:
    """Counts base-ring multiplications in leaf/general products (SPEC.md:348 count law)."""

    def __init__(self):
        self.mults = 0


def _T(X):
    return np.swapaxes(X, -1, -2)


def low(X):
    """Low(X): keep i >= j, zero elsewhere."""
    m, n = X.shape[-2:]
    return np.where(np.tril(np.ones((m, n), dtype=bool)), X, 0)


def syrk_def(A, p, counter: MulCounter | None = None):
    """Low(A A^T) mod p, classical (the oracle definition)."""
    A = np.asarray(A, dtype=np.int64) % p
    if counter is not None:
        m, n = A.shape[-2:]
        counter.mults += m * (m + 1) // 2 * n * int(np.prod(A.shape[:-2], dtype=np.int64))
    return low((A @ _T(A)) % p)


def gemm_def(A, B, p, counter: MulCounter | None = None):
    """A B^T mod p (a general product A phi(B) over GF(p))."""
    A = np.asarray(A, dtype=np.int64) % p
    B = np.asarray(B, dtype=np.int64) % p
    if counter is not None:
        counter.mults += A.shape[-2] * B.shape[-2] * A.shape[-1] * int(
            np.prod(A.shape[:-2], dtype=np.int64))
    return (A @ _T(B)) % p


def apply_Y(X, Y, p):
    """X Y mod p without materialising Y.  Y = ('scalar', i, 0) or ('rot2', a, b)."""
    kind, a, b = Y
    if kind == "scalar":
        return (X * a) % p
    n = X.shape[-1]
    assert n % 2 == 0, "Rot2 needs an even dimension"
    X1, X2 = X[..., : n // 2], X[..., n // 2:]
    return np.concatenate([(a * X1 - b * X2) % p, (b * X1 + a * X2) % p], axis=-1)


def materialize_Y(Y, n, p):
    """Explicit n x n matrix of Y (for the skew-unitary pin Y Y^T = -I)."""
    return apply_Y(np.eye(n, dtype=np.int64), Y, p)


def _pad(A, m2, n2):
    m, n = A.shape[-2:]
    if (m, n) == (m2, n2):
        return A
    out = np.zeros(A.shape[:-2] + (m2, n2), dtype=np.int64)
    out[..., :m, :n] = A
    return out


def alg1(A, p, Y, depth: int, counter: MulCounter | None = None):
    """Alg. alg:MIAHMM: returns Low(A phi(A)) (phi = transpose over GF(p)), as a full array with
    zeros strictly above the diagonal.  depth = number of recursive levels (0 = classical)."""
    A = np.asarray(A, dtype=np.int64) % p
    m, n = A.shape[-2:]
    if depth == 0 or m < 2 or n < 2:
        return syrk_def(A, p, counter)
    # zero padding to even m and even inner halves (Rot2 needs n/2 even)
    step = 4 if Y[0] == "rot2" else 2
    m2 = m + (m % 2)
    n2 = -(-n // step) * step
    A = _pad(A, m2, n2)
    h, q = m2 // 2, n2 // 2
    # Split A = [[A11, A12], [A21, A22]], A11 in R^{m/2 x n/2}
    A11, A12 = A[..., :h, :q], A[..., :h, q:]
    A21, A22 = A[..., h:, :q], A[..., h:, q:]
    # 4 additions and 2 multiplications by Y
    S1 = apply_Y((A21 - A11) % p, Y, p)
    S2 = (A22 - apply_Y(A21, Y, p)) % p
    S3 = (S1 - A22) % p
    S4 = (S3 + A12) % p
    # 3 recursive (P1, P2, P5) and 2 general products (P3, P4)
    P1 = alg1(A11, p, Y, depth - 1, counter)
    P2 = alg1(A12, p, Y, depth - 1, counter)
    P3 = gemm_def(A22, S4, p, counter)            # A22 phi(S4)
    P4 = gemm_def(S1, S2, p, counter)             # S1 phi(S2)
    P5 = alg1(S3, p, Y, depth - 1, counter)
    # 3 half additions and 2 complete additions
    U1 = (P1 + P5) % p                            # Low(U1) <- Low(P1) + Low(P5)
    U3 = (P1 + P2) % p                            # Low(U3) <- Low(P1) + Low(P2)
    U1 = (U1 + _T(U1) - U1 * np.eye(h, dtype=np.int64)) % p   # Up(U1) <- phi(Low(U1))
    U2 = (U1 + P4) % p
    U4 = (U2 + P3) % p
    U5 = low((U2 + _T(P4)) % p)                   # Low(U5) <- Low(U2) + Low(phi(P4))
    out = np.zeros(A.shape[:-2] + (m2, m2), dtype=np.int64)
    out[..., :h, :h] = low(U3)
    out[..., h:, :h] = U4
    out[..., h:, h:] = U5
    return out[..., :m, :m]


def herk_def(X, Yim, p):
    """(X + iY)(X + iY)^H over GF(p)[i]/(i^2+1) by definition; returns (Re, Im), lower only."""
    X = np.asarray(X, dtype=np.int64) % p
    Yim = np.asarray(Yim, dtype=np.int64) % p
    re = (X @ _T(X) + Yim @ _T(Yim)) % p
    im = (Yim @ _T(X) - X @ _T(Yim)) % p
    return low(re), low(im)


def alg2m(X, Yim, p, syrk=None):
    """Alg. alg:2M over K = GF(p), E = GF(p)[i]/(i^2+1), phi = conjugate
    transpose.  i commutes with K; phi(i) = conj(i) = -i; eps = i phi(i) = -i^2 = 1 in K.
    M = (G - eps H - phi(H)) + H phi(i) + i phi(H), with H = A phi(B), G = (A+B) phi(A + eps B)
    where A = X (real part), B = Yim (imaginary part); on K, phi acts as the transpose.
    ``syrk`` computes Low(Z Z^T) for G (default: definition; pass alg1 to compose).
    Returns (Re, Im) of Low(M)."""
    X = np.asarray(X, dtype=np.int64) % p
    Yim = np.asarray(Yim, dtype=np.int64) % p
    eps = 1
    H = gemm_def(X, Yim, p)                                   # H = A phi(B)
    T = (X + Yim) % p
    assert np.array_equal(T, (X + eps * Yim) % p)             # A + B == A + eps B since eps = 1
    G = syrk_def(T, p) if syrk is None else syrk(T)           # G = (A+B) phi(A + eps B), Low
    m = X.shape[-2]
    G = (G + _T(G) - G * np.eye(m, dtype=np.int64)) % p       # full symmetric G (Lemma lem:uplow)
    re = (G - eps * H - _T(H)) % p                            # G - eps H - phi(H)
    # H phi(i) + i phi(H) = H (-i) + i H^T = i (H^T - H)
    im = (_T(H) - H) % p
    return low(re), low(im)


# ----------------------------------------------------------------------------- GF(p^2) Alg. 1
def _cmul_conjT(Xr, Xi, Yr, Yi, p):
    """X phi(Y) = X Y^H over GF(p)[i]/(i^2+1) by definition: (Xr + i Xi)(Yr^T - i Yi^T)."""
    re = (Xr @ _T(Yr) + Xi @ _T(Yi)) % p
    im = (Xi @ _T(Yr) - Xr @ _T(Yi)) % p
    return re, im


def alg1_herk(X, Yim, p, y, depth: int = 1):
    """Alg. alg:MIAHMM directly over E = GF(p)[i]/(i^2+1), p = 3 mod 4, with
    phi = conjugate transpose and the skew-unitary Y = (a + ib) I, a^2 + b^2 = -1 (PAPER.md
    §4.4, 750-758: conj(a + ib) = a - ib, so Y Y^H = (a^2 + b^2) I = -I).  A = X + i Yim.
    Returns (Re, Im) of Low(A A^H); recursion on P1, P2, P5 down to `depth` levels, the
    recursion leaves and P3, P4 by definition."""
    a, b = y
    Xr = np.asarray(X, dtype=np.int64) % p
    Xi = np.asarray(Yim, dtype=np.int64) % p
    m, n = Xr.shape[-2:]
    if depth == 0 or m < 2 or n < 2:
        re, im = _cmul_conjT(Xr, Xi, Xr, Xi, p)
        return low(re), low(im)
    m2, n2 = m + (m % 2), n + (n % 2)
    Xr, Xi = _pad(Xr, m2, n2), _pad(Xi, m2, n2)
    h, q = m2 // 2, n2 // 2
    blk = lambda Z: (Z[..., :h, :q], Z[..., :h, q:], Z[..., h:, :q], Z[..., h:, q:])
    A11r, A12r, A21r, A22r = blk(Xr)
    A11i, A12i, A21i, A22i = blk(Xi)

    def ymul(Zr, Zi):   # Z Y = (a + ib) Z
        return (a * Zr - b * Zi) % p, (b * Zr + a * Zi) % p

    # 4 additions and 2 multiplications by Y
    S1r, S1i = ymul((A21r - A11r) % p, (A21i - A11i) % p)
    tr, ti = ymul(A21r, A21i)
    S2r, S2i = (A22r - tr) % p, (A22i - ti) % p
    S3r, S3i = (S1r - A22r) % p, (S1i - A22i) % p
    S4r, S4i = (S3r + A12r) % p, (S3i + A12i) % p
    # 3 recursive (P1, P2, P5) and 2 general products (P3, P4)
    P1 = alg1_herk(A11r, A11i, p, y, depth - 1)
    P2 = alg1_herk(A12r, A12i, p, y, depth - 1)
    P3 = _cmul_conjT(A22r, A22i, S4r, S4i, p)     # A22 phi(S4)
    P4 = _cmul_conjT(S1r, S1i, S2r, S2i, p)       # S1 phi(S2)
    P5 = alg1_herk(S3r, S3i, p, y, depth - 1)
    # 3 half additions and 2 complete additions
    U1r, U1i = (P1[0] + P5[0]) % p, (P1[1] + P5[1]) % p      # Low(U1)
    U3r, U3i = (P1[0] + P2[0]) % p, (P1[1] + P2[1]) % p      # Low(U3)
    eye = np.eye(h, dtype=np.int64)
    U1r = (U1r + _T(U1r) - U1r * eye) % p                     # Up(U1) <- phi(Low(U1)) = conj(Low(U1))^T
    U1i = (U1i - _T(U1i) - U1i * eye) % p
    U2r, U2i = (U1r + P4[0]) % p, (U1i + P4[1]) % p
    U4r, U4i = (U2r + P3[0]) % p, (U2i + P3[1]) % p
    U5r, U5i = low((U2r + _T(P4[0])) % p), low((U2i - _T(P4[1])) % p)   # Low(U2) + Low(phi(P4))
    re = np.zeros(Xr.shape[:-2] + (m2, m2), dtype=np.int64)
    im = np.zeros_like(re)
    re[..., :h, :h], im[..., :h, :h] = low(U3r), low(U3i)
    re[..., h:, :h], im[..., h:, :h] = U4r, U4i
    re[..., h:, h:], im[..., h:, h:] = U5r, U5i
    return re[..., :m, :m], im[..., :m, :m]


# ----------------------------------------------------------------------------- quaternions
def quat_def(A, B, C, D, p):
    """M M^H for M = A + B i + C j + D k over H_GF(p), by the expansion of PAPER.md:1925-1945:
    H1 = AA^T + BB^T + CC^T + DD^T, H2 = (BA^T - AB^T) + (DC^T - CD^T),
    H3 = (CA^T - AC^T) + (BD^T - DB^T), H4 = (DA^T - AD^T) + (CB^T - BC^T).  Returns Low of each."""
    A, B, C, D = (np.asarray(Z, dtype=np.int64) % p for Z in (A, B, C, D))
    mm = lambda X, Y: X @ _T(Y)
    H1 = (mm(A, A) + mm(B, B) + mm(C, C) + mm(D, D)) % p
    H2 = (mm(B, A) - mm(A, B) + mm(D, C) - mm(C, D)) % p
    H3 = (mm(C, A) - mm(A, C) + mm(B, D) - mm(D, B)) % p
    H4 = (mm(D, A) - mm(A, D) + mm(C, B) - mm(B, C)) % p
    return low(H1), low(H2), low(H3), low(H4)


def alg2m3m(A, B, C, D, p, syrk=None):
    """Alg. alg:2M3M: M M^H for M = A + B i + C j + D k with 6
    multiplications, one of them (Q6) a product of a matrix by its transpose (``syrk``, default
    the definition; pass alg1 to run Q6 through Alg. alg:MIAHMM).  Returns Low(H1..H4)."""
    A, B, C, D = (np.asarray(Z, dtype=np.int64) % p for Z in (A, B, C, D))
    m = A.shape[-2]
    U1 = (A + B) % p
    U2 = (C + D) % p
    Q1 = gemm_def(C, A, p)                                   # C A^T
    Q2 = gemm_def(D, B, p)                                   # D B^T
    Q3 = gemm_def(U2, U1, p)                                 # U2 U1^T
    Q4 = gemm_def(A, B, p)                                   # A B^T
    Q5 = gemm_def(C, D, p)                                   # C D^T
    W = (U1 + U2) % p
    Q6 = syrk_def(W, p) if syrk is None else syrk(W)         # (U1 + U2)(U1^T + U2^T), Low
    Q6 = (Q6 + _T(Q6) - Q6 * np.eye(m, dtype=np.int64)) % p
    T1 = (Q1 - Q2) % p
    T2 = (Q4 + Q5) % p
    T3 = (Q1 + Q2 - Q3) % p
    H1 = low((Q6 - (_T(Q3) + Q3) - (_T(T2) + T2)) % p)
    H2 = low((_T(T2) - T2) % p)
    H3 = low((T1 - _T(T1)) % p)
    H4 = low((_T(T3) - T3) % p)
    return H1, H2, H3, H4
