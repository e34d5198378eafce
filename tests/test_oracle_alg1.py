"""Pins for O2 (oracle/alg1.py, the paper's Alg. 1 and Alg. 2M re-derived) and oracle/field.py:
exhaustive enumeration over tiny fields, worked values, identities, and agreement with O1."""
import itertools

import numpy as np
import pytest

import oracle
from oracle import alg1 as A1
from oracle import field as F
from inputs import uniform_matrix, uniform_matrix_ext


def test_field_worked_values(golden):
    for e in golden["legendre"]:
        assert F.legendre(e["a"], e["p"]) == e["value"], e["cite"]
    for e in golden["mod_sqrt"]:
        assert F.mod_sqrt(e["a"], e["p"]) == e["value"], e["cite"]
    for e in golden["sos"]:
        assert list(F.sos(e["k"], e["p"])) == e["value"], e["cite"]
    for e in golden["sqrt_minus_one"]:
        assert F.sqrt_minus_one(e["p"]) == e["value"], e["cite"]
    for e in golden["skew_unitary"]:
        assert F.skew_unitary(e["p"]) == (e["kind"], e["a"], e["b"]), e["cite"]


def test_field_properties():
    primes = [q for q in range(3, 1000) if F.is_prime(q)]
    for q in primes:
        a, b = F.sos(q - 1, q)                      # Prop. lem:pigeonhole existence
        assert (a * a + b * b) % q == q - 1
        for k in (1, 2, 3, 5, q - 2):
            a, b = F.sos(k, q)
            assert (a * a + b * b - k) % q == 0
        squares = {x * x % q for x in range(1, q)}
        for x in range(1, min(q, 60)):
            assert F.legendre(x, q) == (1 if x in squares else -1)
            r = F.mod_sqrt(x * x % q, q)
            assert r in (x, q - x) and r <= q - r
        if q % 4 == 1:
            i = F.sqrt_minus_one(q)
            assert i * i % q == q - 1
        else:
            assert F.sqrt_minus_one(q) is None and (q - 1) not in squares


@pytest.mark.parametrize("p,expect", [(97, ("scalar", 22, 0)), (65521, ("scalar", 24297, 0)),
                                      (8191, ("rot2", 2670, 5929))])
def test_skew_unitary_identity(p, expect):
    """Y phi(Y) = -I (Eq. eq:skewu), on the materialised Y."""
    Y = F.skew_unitary(p)
    assert Y == expect
    for n in (2, 4, 8):
        M = A1.materialize_Y(Y, n, p)
        assert np.array_equal((M @ M.T) % p, (-np.eye(n, dtype=np.int64)) % p)
    kind, a, b = Y
    assert ((a * a + b * b) % p == p - 1) if kind == "rot2" else (a * a % p == p - 1)


def _all_matrices(p, m, n):
    vals = np.array(list(itertools.product(range(p), repeat=m * n)), dtype=np.int64)
    return vals.reshape(-1, m, n)


@pytest.mark.parametrize("p,m,n,Y", [(3, 2, 4, ("rot2", 1, 1)), (5, 2, 2, ("scalar", 2, 0))])
def test_alg1_exhaustive_tiny_fields(p, m, n, Y):
    """Every A in GF(p)^{m x n}: Alg. 1 (depth 1) = Low(A A^T) (SURVEY.md 'facts verified')."""
    As = _all_matrices(p, m, n)
    got = A1.alg1(As, p, Y, depth=1)
    ref = A1.syrk_def(As, p)
    assert np.array_equal(got, ref)


def test_alg1_gf7_rot2_sample():
    p, Y = 7, ("rot2", 3, 2)
    rng = np.random.default_rng(0)
    As = rng.integers(0, p, size=(50000, 2, 4))
    assert np.array_equal(A1.alg1(As, p, Y, 1), A1.syrk_def(As, p))


@pytest.mark.parametrize("p", [97, 8191, 65521, 13, 7])
@pytest.mark.parametrize("depth", [1, 2, 3])
def test_alg1_vs_o1(p, depth):
    Y = F.skew_unitary(p)
    for (m, k) in [(16, 16), (24, 40), (33, 17), (9, 50), (50, 9)]:
        A = uniform_matrix(m, k, seed=m * 100 + k, p=p)
        got = A1.alg1(A, p, Y, depth)
        assert np.array_equal(got.astype(np.uint32), oracle.syrk_t(A, p)), (m, k)


def test_alg1_any_valid_Y_same_result():
    """C is identical for any valid skew-unitary Y (both sqrt(-1) choices; all (a,b))."""
    p = 13
    A = uniform_matrix(12, 20, seed=7, p=p)
    ref = oracle.syrk_t(A, p)
    for i in (5, 8):
        assert np.array_equal(A1.alg1(A, p, ("scalar", i, 0), 2).astype(np.uint32), ref)
    p = 7
    A = uniform_matrix(12, 20, seed=8, p=p)
    ref = oracle.syrk_t(A, p)
    pairs = [(a, b) for a in range(p) for b in range(p) if (a * a + b * b) % p == p - 1]
    assert len(pairs) > 2
    for a, b in pairs:
        assert np.array_equal(A1.alg1(A, p, ("rot2", a, b), 2).astype(np.uint32), ref)


def test_alg1_invalid_Y_breaks():
    """Negative control: a Y that is NOT skew-unitary gives a wrong C (the pin has teeth)."""
    p = 13
    A = uniform_matrix(8, 8, seed=1, p=p)
    assert not np.array_equal(A1.alg1(A, p, ("scalar", 3, 0), 1).astype(np.uint32),
                              oracle.syrk_t(A, p))


def test_count_law(golden):
    for e in golden["count_law"]:
        c = A1.MulCounter()
        n, p = e["n"], e["p"]
        A = uniform_matrix(n, n, seed=1, p=p)
        d = int(np.log2(n))
        A1.alg1(A, p, F.skew_unitary(p), depth=d, counter=c)
        assert c.mults == e["mults"], e["cite"]


def test_alg1_leading_ratio():
    """Table tab:ffcomplex: multiplication count / classical count -> 2/5 as
    depth grows (ring MACs R_d = 3 R_{d-1}(m/2,k/2) + 2 (m/2)^2 (k/2))."""
    for n, d, expect in [(64, 1, 7 / 16), (64, 2, 53 / 128)]:
        c = A1.MulCounter()
        A1.alg1(uniform_matrix(n, n, 1, 13), 13, F.skew_unitary(13), d, counter=c)
        classical = n * (n + 1) // 2 * n
        lead = c.mults / n ** 3
        assert abs(lead - expect) < 2.0 / n, (d, lead, expect)   # lower-order diagonal terms
        assert c.mults < classical


def test_2m_scalar_worked_value(golden):
    for e in golden["twom_scalar"]:
        re, im = A1.alg2m(np.array(e["X"]), np.array(e["Y"]), e["p"])
        assert int(re[0, 0]) == e["re"] and int(im[0, 0]) == e["im"], e["cite"]


@pytest.mark.parametrize("p", [3, 7, 8191])
def test_2m_vs_definition_and_o1(p):
    A = uniform_matrix_ext(21, 14, seed=p, p=p)
    X, Y = A[..., 0], A[..., 1]
    re, im = A1.alg2m(X, Y, p)
    dre, dim = A1.herk_def(X, Y, p)
    assert np.array_equal(re, dre) and np.array_equal(im, dim)
    O = oracle.syrk_h(A, p)
    assert np.array_equal(re.astype(np.uint32), O[..., 0]) and np.array_equal(im.astype(np.uint32), O[..., 1])
    # G through Alg. 1 (composition used by the GPU path) gives the same result
    Yk = F.skew_unitary(p)
    re2, im2 = A1.alg2m(X, Y, p, syrk=lambda T: A1.alg1(T, p, Yk, 2))
    assert np.array_equal(re2, dre) and np.array_equal(im2, dim)


def test_2m_exhaustive_gf3():
    """All 2x2 matrices over GF(9) = GF(3)[i]/(i^2+1) (3^8 = 6561 cases)."""
    p = 3
    allm = _all_matrices(p, 2, 4)
    X, Y = allm[:, :, :2], allm[:, :, 2:]
    re, im = A1.alg2m(X, Y, p)
    dre, dim = A1.herk_def(X, Y, p)
    assert np.array_equal(re, dre) and np.array_equal(im, dim)


# ---------------------------------------------------------------- Alg. 1 over GF(p^2)
def _sos_minus1(p):
    a, b = F.sos(p - 1, p)
    assert (a * a + b * b) % p == p - 1
    return a, b


def test_alg1_herk_exhaustive_gf9():
    """Every 2x2 matrix over GF(9) = GF(3)[i]/(i^2+1): one level of Alg. 1 with Y = (a+ib) I,
    a^2 + b^2 = -1 (§4.4), equals the definition (X+iY)(X+iY)^H."""
    p = 3
    allm = _all_matrices(p, 2, 4)
    X, Y = allm[:, :, :2], allm[:, :, 2:]
    re, im = A1.alg1_herk(X, Y, p, _sos_minus1(p), 1)
    dre, dim = A1.herk_def(X, Y, p)
    assert np.array_equal(re, dre) and np.array_equal(im, dim)


@pytest.mark.parametrize("p", [7, 11, 8191, 131071])
@pytest.mark.parametrize("depth", [1, 2])
def test_alg1_herk_vs_definition_and_o1(p, depth):
    A = uniform_matrix_ext(23, 18, seed=p + depth, p=p)
    re, im = A1.alg1_herk(A[..., 0], A[..., 1], p, _sos_minus1(p), depth)
    O = oracle.syrk_h(A, p)
    assert np.array_equal(re.astype(np.uint32), O[..., 0]) and np.array_equal(im.astype(np.uint32), O[..., 1])


def test_alg1_herk_non_skew_unitary_breaks():
    """Negative control: y with y conj(y) != -1 gives a wrong product (the pin can fail)."""
    p = 8191
    A = uniform_matrix_ext(10, 8, seed=3, p=p)
    dre, dim = A1.herk_def(A[..., 0], A[..., 1], p)
    re, im = A1.alg1_herk(A[..., 0], A[..., 1], p, (1, 1), 1)    # 1 + 1 = 2 != -1
    assert not (np.array_equal(re, dre) and np.array_equal(im, dim))
