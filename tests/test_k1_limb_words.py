"""Host model of the fused K1's packed limb words (preadd.cu: limb_words_u).

The kernel packs two offset residues u = c + (p-1)/2 per 32-bit word and forms the int8 limb
bytes with whole-word adds, shifts, masks and byte permutes.  This test replays exactly those
32-bit operations (wrapping) for every residue of the scheme boundary primes and compares the
bytes with the limb split the leaf contract defines (DESIGN.md §3 table):
  scheme 1 (p <= 16763): hi = floor((c + 64) / 128), lo = c - 128 hi, mid = hi + lo (s8 each)
  scheme 2 (p <= 65521): hi = floor(c / 256) (s8), lo = c - 256 hi (u8)
A carry between the two 16-bit lanes, a wrong offset or a wrong byte selector fails it.
"""
import numpy as np
import pytest

M32 = 0xFFFFFFFF


def byte_perm(a, b, sel):
    """__byte_perm(a, b, sel): bytes 0-3 of a, 4-7 of b, selector nibbles pick the result bytes"""
    src = [(a >> (8 * i)) & 0xFF for i in range(4)] + [(b >> (8 * i)) & 0xFF for i in range(4)]
    return sum(src[(sel >> (4 * i)) & 7] << (8 * i) for i in range(4))


def words_scheme1(u, koff):
    K = ((koff + 32768 - 128 * 66) * 0x10001) & M32
    v01 = (u[0] + (u[1] << 16) + K) & M32
    v23 = (u[2] + (u[3] << 16) + K) & M32
    h01, h23 = (v01 >> 7) & 0x00FF00FF, (v23 >> 7) & 0x00FF00FF
    l01, l23 = ((v01 & 0x007F007F) + 0x00C000C0) & M32, ((v23 & 0x007F007F) + 0x00C000C0) & M32
    return (byte_perm(h01, h23, 0x6420), byte_perm(l01, l23, 0x6420),
            byte_perm((h01 + l01) & M32, (h23 + l23) & M32, 0x6420))


def words_scheme2(u, koff):
    K = ((0x8000 - koff) * 0x10001) & M32
    v01 = (u[0] + (u[1] << 16) + K) & M32
    v23 = (u[2] + (u[3] << 16) + K) & M32
    return (byte_perm(v01, v23, 0x7531) ^ 0x80808080, byte_perm(v01, v23, 0x6420))


def limbs_contract(c, scheme):
    if scheme == 1:
        hi = (c + 64) >> 7
        lo = c - 128 * hi
        return [hi & 0xFF, lo & 0xFF, (hi + lo) & 0xFF]
    hi = c >> 8
    lo = c - 256 * hi
    return [hi & 0xFF, lo & 0xFF]


@pytest.mark.parametrize("p,scheme", [(257, 1), (4099, 1), (8191, 1), (12289, 1), (16763, 1),
                                      (16787, 2), (40009, 2), (65519, 2), (65521, 2)])
def test_fused_k1_limb_words_every_residue(p, scheme):
    h = (p - 1) // 2
    # koff as k1_core passes it: 64 + 128 * 66 - h (scheme 1), h (scheme 2)
    koff = 64 + 128 * 66 - h if scheme == 1 else h
    xs = np.arange(p, dtype=np.int64)
    rng = np.random.default_rng(p)
    # every residue once in each of the four lanes (rolled copies), plus random groups
    groups = [np.roll(xs, s) for s in range(4)]
    lanes = np.stack(groups, axis=1)
    lanes = np.concatenate([lanes, rng.integers(0, p, size=(4096, 4))])
    fn = words_scheme1 if scheme == 1 else words_scheme2
    for g in lanes:
        cs = [int(x) if x <= h else int(x) - p for x in g]
        us = [c + h for c in cs]
        words = fn(us, koff)
        for pl, w in enumerate(words):
            got = [(w >> (8 * e)) & 0xFF for e in range(4)]
            want = [limbs_contract(c, scheme)[pl] for c in cs]
            assert got == want, (p, g, pl)
