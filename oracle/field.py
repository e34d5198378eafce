"""Oracle-side prime-field number theory (TEST INFRASTRUCTURE ONLY; independent of the CUDA
path's own host constants in paper_2101_01025_b200/csrc).

- legendre(a, p)            Euler's criterion a^((p-1)/2)                     (Alg. alg:sosmodp line 1)
- mod_sqrt(a, p)            Tonelli-Shanks, tie-break min(r, p-r)             (Remark alg:FFSoS, PAPER.md:716-721;
                                                                                tie-break reading: SPEC.md:56)
- sos(k, p)                 Alg. alg:sosmodp (SoS), step by step
- sqrt_minus_one(p)         Prop. lem:lemsqrt
- skew_unitary(p, phi)      the Y the path uses: i*I when p = 1 mod 4,
                            Rot2 [[a,b],[-b,a]] (x) I with a^2+b^2 = -1 when p = 3 mod 4
                            (Prop. lem:pigeonhole, (a,b) from Alg. 2)
"""
from __future__ import annotations


def is_prime(n: int) -> bool:
    if n < 2:
        return False
    if n % 2 == 0:
        return n == 2
    d = 3
    while d * d <= n:
        if n % d == 0:
            return False
        d += 2
    return True


def legendre(a: int, p: int) -> int:
    """Legendre symbol via Euler's criterion; p an odd prime."""
    if p == 2 or not is_prime(p):
        raise ValueError("legendre needs an odd prime")
    a %= p
    if a == 0:
        return 0
    return 1 if pow(a, (p - 1) // 2, p) == 1 else -1


def mod_sqrt(a: int, p: int) -> int:
    """Tonelli-Shanks square root of a quadratic residue; returns min(r, p-r)."""
    a %= p
    if a == 0:
        return 0
    if legendre(a, p) != 1:
        raise ValueError(f"{a} is not a square mod {p}")
    q, s = p - 1, 0
    while q % 2 == 0:
        q //= 2
        s += 1
    z = 2
    while legendre(z, p) != -1:
        z += 1
    m, c, t, r = s, pow(z, q, p), pow(a, q, p), pow(a, (q + 1) // 2, p)
    while t != 1:
        i, t2 = 0, t
        while t2 != 1:
            t2 = t2 * t2 % p
            i += 1
        b = pow(c, 1 << (m - i - 1), p)
        m, c, t, r = i, b * b % p, t * b * b % p, r * b % p
    return min(r, p - r)


def lowest_qnr(p: int) -> int:
    """Alg. 2: s <- 2; while (s/p) == 1: s <- s+1."""
    s = 2
    while legendre(s, p) == 1:
        s += 1
    return s


def sos(k: int, p: int):
    """Alg. alg:sosmodp: (a, b) with a^2 + b^2 = k mod p."""
    k %= p
    if legendre(k, p) == 1 or k == 0:          # k is a square mod p -> (sqrt(k), 0)
        return mod_sqrt(k, p), 0
    s = lowest_qnr(p)                           # smallest quadratic non-residue
    c = mod_sqrt(s - 1, p)                      # s-1 must be a square
    r = k * pow(s, -1, p) % p                   # r <- k s^-1 mod p
    a = mod_sqrt(r, p)                          # k = a^2 s = a^2 (1 + c^2)
    return a, a * c % p


def sqrt_minus_one(p: int):
    """Prop. lem:lemsqrt: sqrt(-1) exists in GF(p) iff p = 2 or p = 1 mod 4; None otherwise."""
    if p == 2:
        return 1
    if p % 4 == 1:
        return mod_sqrt(p - 1, p)
    return None


def skew_unitary(p: int):
    """('scalar', i, 0) with Y = i I, or ('rot2', a, b) with Y = [[a,b],[-b,a]] (x) I."""
    i = sqrt_minus_one(p)
    if i is not None:
        return ("scalar", i, 0)
    a, b = sos(p - 1, p)
    return ("rot2", a, b)
