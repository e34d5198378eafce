"""Pins of the quaternion oracle: O1 oracle_syrk_q (C, Hamilton product by
definition) and O2 quat_def / alg2m3m (numpy, §6.2) against values the paper's
multiplication table fixes, a pure-Python brute force, the complex special case (pinned
independently) and exhaustive enumeration over GF(3)."""
import itertools

import numpy as np
import pytest

import oracle
from oracle import alg1 as A1
from oracle import field as F
from inputs import uniform_matrix_ext, uniform_matrix_quat


def qmul(x, y, p):
    """Quaternion product by the table of PAPER.md:1553-1558."""
    x1, x2, x3, x4 = x
    y1, y2, y3, y4 = y
    return ((x1 * y1 - x2 * y2 - x3 * y3 - x4 * y4) % p,
            (x1 * y2 + x2 * y1 + x3 * y4 - x4 * y3) % p,
            (x1 * y3 - x2 * y4 + x3 * y1 + x4 * y2) % p,
            (x1 * y4 + x2 * y3 - x3 * y2 + x4 * y1) % p)


def qconj(x, p):
    return (x[0] % p, -x[1] % p, -x[2] % p, -x[3] % p)


def brute(M, p, order="left"):
    m, k, _ = M.shape
    out = np.zeros((m, m, 4), dtype=np.int64)
    for i in range(m):
        for j in range(i + 1):
            s = [0, 0, 0, 0]
            for t in range(k):
                a, b = [int(v) for v in M[i, t]], qconj([int(v) for v in M[j, t]], p)
                w = qmul(a, b, p) if order == "left" else qmul(b, a, p)
                s = [(s[c] + w[c]) % p for c in range(4)]
            out[i, j] = s
    return out


def test_quaternion_table_identities():
    """ij = k, jk = i, ki = j, ji = -k, i^2 = j^2 = k^2 = ijk = -1."""
    p = 7
    one, i, j, k = (1, 0, 0, 0), (0, 1, 0, 0), (0, 0, 1, 0), (0, 0, 0, 1)
    neg = lambda q: tuple(-c % p for c in q)
    assert qmul(i, j, p) == k and qmul(j, k, p) == i and qmul(k, i, p) == j
    assert qmul(j, i, p) == neg(k)
    for q in (i, j, k):
        assert qmul(q, q, p) == neg(one)
    assert qmul(qmul(i, j, p), k, p) == neg(one)


def test_quaternion_worked_values(golden):
    for e in golden["quaternion"]:
        M = np.array(e["M"], dtype=np.uint32)
        got = oracle.syrk_q(M, e["p"])
        for r, row in enumerate(e["low"]):
            for c, q in enumerate(row):
                assert tuple(int(v) for v in got[r, c]) == tuple(v % e["p"] for v in q), e["cite"]


@pytest.mark.parametrize("p", [3, 7, 97, 8191, 131071])
def test_o1_quat_vs_brute_force(p):
    M = uniform_matrix_quat(6, 5, seed=p, p=p)
    assert np.array_equal(oracle.syrk_q(M, p).astype(np.int64), brute(M, p))


def test_product_order_matters():
    """Negative control: the reversed order conj(M_jt) M_it is a different (wrong) result."""
    p = 8191
    M = uniform_matrix_quat(5, 4, seed=1, p=p)
    assert not np.array_equal(oracle.syrk_q(M, p).astype(np.int64), brute(M, p, order="right"))


@pytest.mark.parametrize("p", [7, 8191])
def test_o1_quat_reduces_to_complex_case(p):
    """C = D = 0: M = A + B i lies in GF(p)[i], so (H1, H2) = Low(A A^H) of the (independently
    pinned) GF(p^2) oracle and H3 = H4 = 0."""
    X = uniform_matrix_ext(20, 13, seed=p, p=p)
    M = np.zeros((20, 13, 4), dtype=np.uint32)
    M[..., :2] = X
    Q = oracle.syrk_q(M, p)
    Hc = oracle.syrk_h(X, p)
    assert np.array_equal(Q[..., :2], Hc)
    assert not Q[..., 2:].any()


@pytest.mark.parametrize("p", [97, 65521])
def test_o1_quat_invariants(p):
    M = uniform_matrix_quat(17, 11, seed=3, p=p)
    Q = oracle.syrk_q(M, p)
    d = np.arange(17)
    assert not Q[d, d, 1:].any()                                   # q conj(q) is real
    norms = (M.astype(np.int64) ** 2).sum(axis=(1, 2)) % p
    assert np.array_equal(Q[d, d, 0].astype(np.int64), norms)


@pytest.mark.parametrize("p", [7, 8191, 131071])
def test_o2_quat_def_and_2m3m_vs_o1(p):
    M = uniform_matrix_quat(19, 14, seed=p + 1, p=p)
    parts = [M[..., c] for c in range(4)]
    O = oracle.syrk_q(M, p)
    D = A1.quat_def(*parts, p)
    for c in range(4):
        assert np.array_equal(D[c].astype(np.uint32), O[..., c])
    H = A1.alg2m3m(*parts, p)
    for c in range(4):
        assert np.array_equal(H[c].astype(np.uint32), O[..., c])
    # Q6 through Alg. 1 (the composition the GPU path uses) gives the same result
    Yk = F.skew_unitary(p)
    H2 = A1.alg2m3m(*parts, p, syrk=lambda W: A1.alg1(W, p, Yk, 2))
    for c in range(4):
        assert np.array_equal(H2[c], H[c])


def test_o2_2m3m_exhaustive_gf3():
    """Every 2 x 1 quaternion matrix over GF(3) (3^8 = 6561 cases): alg:2M3M = definition."""
    p = 3
    vals = np.array(list(itertools.product(range(p), repeat=8)), dtype=np.int64).reshape(-1, 2, 1, 4)
    parts = [vals[..., c] for c in range(4)]
    H = A1.alg2m3m(*parts, p)
    D = A1.quat_def(*parts, p)
    for c in range(4):
        assert np.array_equal(H[c], D[c])
