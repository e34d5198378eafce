"""Pins for the O1 oracle (oracle/oracle.c) against things other than itself:
worked values (tests/golden), pure-Python brute force, float64 BLAS (exact here), closed
forms and invariants.  CPU only."""
import itertools

import numpy as np
import pytest

import oracle
from oracle import closed_forms as cf
from inputs import (uniform_matrix, uniform_matrix_ext, vandermonde_points, vandermonde_matrix,
                    constant_matrix)

PRIMES = [2, 3, 7, 97, 8191, 65521, 2147483647]


def brute_syrk(A, p):
    m, k = len(A), len(A[0]) if len(A) else 0
    C = [[0] * m for _ in range(m)]
    for i in range(m):
        for j in range(i + 1):
            C[i][j] = sum(int(A[i][t]) * int(A[j][t]) for t in range(k)) % p
    return np.array(C, dtype=np.uint32).reshape(m, m)


def brute_herk(A, p):
    """(x + iy)(x' - iy') summed over t, by hand complex arithmetic with i^2 = -1."""
    m, k = A.shape[0], A.shape[1]
    C = np.zeros((m, m, 2), dtype=np.uint32)
    for i in range(m):
        for j in range(i + 1):
            re = im = 0
            for t in range(k):
                x, y = int(A[i, t, 0]), int(A[i, t, 1])
                xp, yp = int(A[j, t, 0]), int(-int(A[j, t, 1]))
                re += x * xp - y * yp
                im += x * yp + y * xp
            C[i, j] = (re % p, im % p)
    return C


def test_worked_syrk_gemm(golden):
    for e in golden["syrk"]:
        C = oracle.syrk_t(np.array(e["A"], dtype=np.uint32), e["p"])
        assert C.tolist() == e["low"], e["cite"]
    for e in golden["gemm"]:
        C = oracle.gemm_nt(np.array(e["A"]), np.array(e["B"]), e["p"])
        assert C.tolist() == e["C"], e["cite"]


@pytest.mark.parametrize("p", PRIMES)
def test_o1_vs_bruteforce(p):
    rng = np.random.default_rng(p)
    for m, k in [(1, 1), (1, 5), (3, 1), (4, 7), (7, 3), (6, 6), (5, 0)]:
        A = rng.integers(0, p, size=(m, k), dtype=np.uint64).astype(np.uint32)
        assert np.array_equal(oracle.syrk_t(A, p), brute_syrk(A.tolist(), p)), (m, k)


def test_o1_noncanonical_inputs_reduced():
    p = 97
    rng = np.random.default_rng(1)
    A = rng.integers(0, 2**32, size=(9, 13), dtype=np.uint64).astype(np.uint32)
    assert np.array_equal(oracle.syrk_t(A, p), brute_syrk((A % p).tolist(), p))


@pytest.mark.parametrize("p", [97, 8191, 65521])
def test_o1_vs_float64_blas(p):
    """Paper's own classical route (dsyrk + mod p) is exact here since
    k (p-1)^2 < 2^53; numpy float64 matmul is an independent library computation."""
    A = uniform_matrix(150, 700, seed=11, p=p)
    assert 700 * (p - 1) ** 2 < 2**53
    F = A.astype(np.float64) @ A.astype(np.float64).T
    ref = np.tril(np.mod(F, p)).astype(np.uint32)
    assert np.array_equal(oracle.syrk_t(A, p), ref)


def test_o1_gemm_vs_bruteforce_and_identity():
    p = 65521
    rng = np.random.default_rng(3)
    A = rng.integers(0, p, size=(5, 9)).astype(np.uint32)
    B = rng.integers(0, p, size=(4, 9)).astype(np.uint32)
    ref = np.array([[sum(int(A[i, t]) * int(B[j, t]) for t in range(9)) % p for j in range(4)]
                    for i in range(5)], dtype=np.uint32)
    assert np.array_equal(oracle.gemm_nt(A, B, p), ref)
    I = np.eye(9, dtype=np.uint32)
    assert np.array_equal(oracle.gemm_nt(A, I, p), A)          # A I^T = A


@pytest.mark.parametrize("p", [97, 8191, 65521])
def test_o1_closed_forms(p):
    m, k = 64, 300
    # Vandermonde geometric sums
    x = vandermonde_points(m, 5, p)
    A = vandermonde_matrix(x, k, p)
    C = oracle.syrk_t(A, p)
    rows = list(range(m))
    ref = cf.vandermonde_syrk_entries(x, rows, k, p)
    for i in rows:
        assert np.array_equal(C[i, : i + 1], ref[i]), i
    # identity -> identity (lower), all ones -> k mod p
    assert np.array_equal(oracle.syrk_t(np.eye(m, dtype=np.uint32), p), np.eye(m, dtype=np.uint32))
    ones = oracle.syrk_t(np.ones((m, k), dtype=np.uint32), p)
    assert np.array_equal(ones, np.tril(np.full((m, m), k % p, dtype=np.uint32)))
    # constant c -> k c^2 mod p
    c = p - 3
    Cc = oracle.syrk_t(constant_matrix(m, k, c, p), p)
    assert np.array_equal(Cc, np.tril(np.full((m, m), k * c * c % p, dtype=np.uint32)))
    # rank one: A = u v^T -> C = (v.v) u u^T
    rng = np.random.default_rng(p)
    u = rng.integers(0, p, m).astype(np.int64)
    v = rng.integers(0, p, k).astype(np.int64)
    A1 = (u[:, None] * v[None, :] % p).astype(np.uint32)
    vv = int((v * v % p).sum() % p)
    ref1 = np.tril(np.outer(u, u) % p * vv % p).astype(np.uint32)
    assert np.array_equal(oracle.syrk_t(A1, p), ref1)


def test_o1_trace_and_rows_subset():
    p = 8191
    A = uniform_matrix(80, 123, seed=2, p=p)
    C = oracle.syrk_t(A, p)
    a = A.astype(np.int64)
    assert int(np.trace(C.astype(np.int64)) % p) == int((a * a).sum() % p)   # trace(AA^T)=sum a^2
    part = oracle.syrk_t(A, p, rows=(40, 80))
    assert np.array_equal(part[40:], C[40:]) and not part[:40].any()


@pytest.mark.parametrize("p", [3, 7, 8191, 131071, 2147483647])
def test_o1_herk_bruteforce(p):
    A = uniform_matrix_ext(6, 5, seed=9, p=p)
    assert np.array_equal(oracle.syrk_h(A, p), brute_herk(A, p))


def test_o1_herk_closed_form_and_invariants():
    p = 8191
    m, k = 40, 257
    rng = np.random.default_rng(4)
    z = rng.integers(1, p, size=(m, 2))
    A = vandermonde_matrix(z, k, p)
    C = oracle.syrk_h(A, p)
    ref = cf.vandermonde_herk_entries(z, range(m), k, p)
    for i in range(m):
        assert np.array_equal(C[i, : i + 1, 0], ref[i][0]) and np.array_equal(C[i, : i + 1, 1], ref[i][1])
    # Hermitian: diagonal imaginary part is 0; diag real = sum x^2 + y^2
    U = uniform_matrix_ext(30, 50, seed=1, p=p).astype(np.int64)
    H = oracle.syrk_h(U.astype(np.uint32), p)
    assert not H[np.arange(30), np.arange(30), 1].any()
    assert np.array_equal(H[np.arange(30), np.arange(30), 0], (U ** 2).sum(axis=(1, 2)) % p)
    # 2M scalar worked value: (2+3i)(2-3i) = 13
    s = oracle.syrk_h(np.array([[[2, 3]]], dtype=np.uint32), p)
    assert s[0, 0].tolist() == [13, 0]


def test_o1_herk_equals_real_embedding():
    """Over GF(p)[i]/(i^2+1), Re and Im of A A^H are the base-field products
    X X^T + Y Y^T and Y X^T - X Y^T: checked with the *transpose* oracle on stacked blocks,
    a different code path of O1."""
    p = 8191
    A = uniform_matrix_ext(20, 33, seed=5, p=p)
    X, Y = A[..., 0], A[..., 1]
    H = oracle.syrk_h(A, p)
    Z = np.concatenate([X, Y], axis=1)                 # [X Y] [X Y]^T = X X^T + Y Y^T
    assert np.array_equal(H[..., 0], oracle.syrk_t(Z, p))
    im_full = (oracle.gemm_nt(Y, X, p).astype(np.int64) - oracle.gemm_nt(X, Y, p)) % p
    assert np.array_equal(H[..., 1], np.tril(im_full).astype(np.uint32))


def test_inputs_generator_known_values():
    """The counter-based generator is pinned to a direct big-integer evaluation of its formula."""
    from inputs.gen import splitmix64
    M = (1 << 64) - 1

    def sm(z):
        z = (z + 0x9E3779B97F4A7C15) & M
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        return z ^ (z >> 31)
    seed, p = 1, 8191
    r = uniform_matrix(3, 4, seed, p).ravel()
    for j in range(12):
        assert int(r[j]) == (sm(sm(seed) ^ j) * p) >> 64
    assert splitmix64(0) == sm(0)
    # uniform-ish: all residues in range, mean near (p-1)/2
    big = uniform_matrix(512, 512, 3, 65521)
    assert big.max() < 65521 and abs(big.mean() - 32760) < 200


def test_freivalds_helper_has_teeth():
    """The full-size GPU check (tests/gpu_util.freivalds) accepts the oracle's Low(C) and
    rejects it after any single-entry corruption (upper-triangle completion included)."""
    from gpu_util import freivalds
    p = 8191
    A = uniform_matrix(300, 150, seed=3, p=p)
    C = oracle.syrk_t(A, p)
    assert freivalds(A, C, p)
    for (i, j) in [(0, 0), (299, 0), (150, 149), (299, 299)]:
        bad = C.copy()
        bad[i, j] = (bad[i, j] + 1) % p
        assert not freivalds(A, bad, p), (i, j)


def test_syrk_update_special_cases(golden):
    """alpha = 1, beta = 0 is the plain product; alpha = 0, beta = 1 keeps Low(C) (reduced);
    the upper triangle is never touched (SPEC.md:354-356 examples)."""
    p = 13
    A = uniform_matrix(9, 7, seed=2, p=p)
    rng = np.random.default_rng(0)
    C = rng.integers(0, 2**31, size=(9, 9)).astype(np.uint32)
    one = oracle.syrk_update(A, C, p, 1, 0)
    assert np.array_equal(np.tril(one), oracle.syrk_t(A, p))
    keep = oracle.syrk_update(A, C, p, 0, 1)
    assert np.array_equal(np.tril(keep), np.tril(C % p))
    both = oracle.syrk_update(A, C, p, 3, 5)
    assert np.array_equal(np.triu(both, 1), np.triu(C, 1))
    ref = (3 * brute_syrk(A.tolist(), p).astype(np.int64) + 5 * (C.astype(np.int64) % p)) % p
    assert np.array_equal(np.tril(both), np.tril(ref).astype(np.uint32))


@pytest.mark.parametrize("alpha,beta", [(1, 0), (0, 1), (3, 5), (10, 10)])
def test_syrk_update_hermitian_branch(alpha, beta):
    """The phi = H branch of syrk_update (HERK form, Table tab:schedule:AATpC)
    against pure-Python brute force over GF(11)[i]/(i^2+1): Low(C') = alpha Low(A A^H) +
    beta Low(C) with alpha, beta in GF(p) scaling re and im alike, on both components of the
    lower triangle (diagonal included), and Up(C') = Up(C) untouched in both components."""
    p = 11
    rng = np.random.default_rng(alpha * 7 + beta)
    m, k = 6, 5
    A = rng.integers(0, p, size=(m, k, 2)).astype(np.uint32)
    C = rng.integers(0, 3 * p, size=(m, m, 2)).astype(np.uint32)     # non-canonical old values too
    got = oracle.syrk_update(A, C, p, alpha, beta, phi="H")
    herk = brute_herk(A, p)
    for i in range(m):
        for j in range(m):
            for q in range(2):
                if j <= i:
                    want = (alpha * int(herk[i, j, q]) + beta * (int(C[i, j, q]) % p)) % p
                else:
                    want = int(C[i, j, q])
                assert int(got[i, j, q]) == want, (i, j, q)


@pytest.mark.parametrize("alpha,beta", [(1, 0), (0, 1), (4, 9)])
def test_syrk_update_quaternion_branch(alpha, beta):
    """The phi = Q branch of syrk_update against pure-Python quaternion arithmetic over GF(7):
    C_ij = sum_t M_it conj(M_jt) with the table i^2 = j^2 = k^2 = ijk = -1,
    written out per component; Low scaled, Up untouched."""
    p = 7
    rng = np.random.default_rng(alpha + 10 * beta)
    m, k = 5, 4
    M = rng.integers(0, p, size=(m, k, 4)).astype(np.uint32)
    C = rng.integers(0, 3 * p, size=(m, m, 4)).astype(np.uint32)
    got = oracle.syrk_update(M, C, p, alpha, beta, phi="Q")

    def qmul(x, y):
        a, b, c, d = x
        e, f, g, h = y
        return (a * e - b * f - c * g - d * h, a * f + b * e + c * h - d * g,
                a * g - b * h + c * e + d * f, a * h + b * g - c * f + d * e)
    for i in range(m):
        for j in range(m):
            if j <= i:
                acc = [0, 0, 0, 0]
                for t in range(k):
                    x = [int(v) for v in M[i, t]]
                    y = [int(M[j, t, 0])] + [-int(v) for v in M[j, t, 1:]]
                    acc = [u + v for u, v in zip(acc, qmul(x, y))]
                want = [(alpha * acc[q] + beta * (int(C[i, j, q]) % p)) % p for q in range(4)]
            else:
                want = [int(v) for v in C[i, j]]
            assert [int(v) for v in got[i, j]] == want, (i, j)
