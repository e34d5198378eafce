"""Host-compiled checks of the CUDA path's device arithmetic helpers (csrc/modp.cuh is
__host__ __device__): the Shoup-fused epilogue step acc_mulred(x, w, part) = (part + x w) mod p
used by the leaf kernel, against exact Python integers, for every int32 extreme and random
inputs at the limb-scheme boundary primes."""
import os
import random
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2101_01025_b200", "csrc")

PRIMES = [3, 5, 97, 251, 257, 8191, 16763, 16787, 65521, 65537, 131041, 131071, 262139]

PROG = r"""
#include <cstdio>
#include <cstdlib>
#include "modp.cuh"
using namespace adj;
int main() {
  unsigned p, w, part; long long x;
  while (scanf("%u %u %lld %u", &p, &w, &x, &part) == 4) {
    ShoupW s = make_shoup(w, p);
    printf("%u\n", acc_mulred((int32_t)x, s.wc, s.wq, part, p));
  }
  return 0;
}
"""


@pytest.fixture(scope="module")
def prog(tmp_path_factory):
    d = tmp_path_factory.mktemp("modp")
    src, exe = d / "t.cpp", d / "t"
    src.write_text(PROG)
    subprocess.run(["g++", "-O2", "-std=c++17", "-I", CSRC, str(src), "-o", str(exe)], check=True)
    return str(exe)


def test_acc_mulred_exact(prog):
    rng = random.Random(7)
    cases = []
    xs_fixed = [-2**31, -2**31 + 1, -1, 0, 1, 2**31 - 1, 2**31 - 2, -2**30, 2**30]
    for p in PRIMES:
        ws = sorted({0, 1, 2, p - 1, p - 2, (p - 1) // 2, (p + 1) // 2} | {rng.randrange(p) for _ in range(20)})
        for w in ws:
            for x in xs_fixed + [rng.randrange(-2**31, 2**31) for _ in range(20)]:
                for part in (0, p - 1, rng.randrange(p)):
                    cases.append((p, w, x, part))
    inp = "".join(f"{p} {w} {x} {part}\n" for p, w, x, part in cases)
    out = subprocess.run([prog], input=inp, capture_output=True, text=True, check=True).stdout.split()
    assert len(out) == len(cases)
    for (p, w, x, part), got in zip(cases, out):
        assert int(got) == (part + x * w) % p, (p, w, x, part, got)


PROG2 = r"""
#include <cstdio>
#include "modp.cuh"
using namespace adj;
int main() {
  unsigned p, a, b, x;
  while (scanf("%u %u %u %u", &p, &a, &b, &x) == 4) {
    ModP m = make_modp(p);
    printf("%u %u %u %u\n", addmod(a, b, m), submod(a, b, m), mod_u32(x, m), mulmod_any(a, b, m));
  }
  return 0;
}
"""


def test_add_sub_mod_exact(tmp_path):
    """addmod / submod / mod_u32 / mulmod_any (unsigned-min forms) against exact integers: residue
    extremes, every 32-bit extreme for the reduction, random values, at the limb-scheme primes."""
    src, exe = tmp_path / "t2.cpp", tmp_path / "t2"
    src.write_text(PROG2)
    subprocess.run(["g++", "-O2", "-std=c++17", "-I", CSRC, str(src), "-o", str(exe)], check=True)
    rng = random.Random(11)
    cases = []
    for p in PRIMES:
        res = sorted({0, 1, p - 1, p - 2, (p - 1) // 2, (p + 1) // 2} | {rng.randrange(p) for _ in range(12)})
        xs = [0, 1, p - 1, p, p + 1, 2 * p - 1, 2 * p, 2**32 - 1, 2**32 - p, 2**31] + [rng.randrange(2**32) for _ in range(8)]
        for a in res:
            for b in res:
                cases.append((p, a, b, xs[(a + b) % len(xs)]))
    inp = "".join(f"{p} {a} {b} {x}\n" for p, a, b, x in cases)
    out = subprocess.run([str(exe)], input=inp, capture_output=True, text=True, check=True).stdout.split("\n")
    for (p, a, b, x), line in zip(cases, out):
        assert list(map(int, line.split())) == [(a + b) % p, (a - b) % p, x % p, a * b % p], (p, a, b, x, line)


PROG3 = r"""
#include <cstdio>
#include <vector>
#include "modp.cuh"
using namespace adj;
// stdin: records of 11 uint32 (p, yk, x11a, x11b, x21a, x21b, x22a, x22b, ya, yb, pad)
// stdout: 4 uint32 per record (S1a, S1b, S2a, S2b offset residues)
int main() {
  uint32_t r[11];
  std::vector<uint32_t> out;
  while (fread(r, 4, 11, stdin) == 11) {
    const uint32_t p = r[0];
    uint32_t s[4];
    const K1Const kc = make_k1const(p, r[8], r[9]);
    const bool wide = p > 16763;
    if (r[1] == 0) {
      if (wide) k1_s1_s2<true, 0>(r[2], r[3], r[4], r[5], r[6], r[7], kc, s[0], s[1], s[2], s[3]);
      else k1_s1_s2<false, 0>(r[2], r[3], r[4], r[5], r[6], r[7], kc, s[0], s[1], s[2], s[3]);
    } else {
      if (wide) k1_s1_s2<true, 1>(r[2], r[3], r[4], r[5], r[6], r[7], kc, s[0], s[1], s[2], s[3]);
      else k1_s1_s2<false, 1>(r[2], r[3], r[4], r[5], r[6], r[7], kc, s[0], s[1], s[2], s[3]);
    }
    out.insert(out.end(), s, s + 4);
  }
  fwrite(out.data(), 4, out.size(), stdout);
  return 0;
}
"""

LAZY_PRIMES = [3, 5, 97, 251, 257, 8191, 16763, 16787, 32749, 65519, 65521, 65537, 131041, 131071, 199999, 262139]


def test_k1_s1_s2_reductions(tmp_path):
    """K1's reduction of the Y products (modp.cuh k1_s1_s2, used by preadd.cu): S1 = (A21 - A11) Y
    and S2 = A22 - A21 Y for Y = i I and Y = Rot2(a, b), as
    offset residues (v + (p-1)/2) mod p, against exact integers -- the exact int32 + Barrett
    path (p <= 16763), the Shoup path (p > 16763, Y = i I) and the float quotient estimate
    (p > 16763, Rot2).  Every combination of extreme residues {0, 1, h, h+1, p-2, p-1} of the six
    inputs, with extreme and actual skew-unitary Y coefficients, plus random inputs, at primes
    of every limb scheme (1 plane, K7, s8/u8, 6-plane)."""
    import itertools
    import numpy as np
    src, exe = tmp_path / "t3.cpp", tmp_path / "t3"
    src.write_text(PROG3)
    subprocess.run(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-I", CSRC, str(src), "-o", str(exe)], check=True)
    import oracle.field as of
    recs = []
    rng = np.random.default_rng(5)
    for p in LAZY_PRIMES:
        h = (p - 1) // 2
        ext = np.array([0, 1, h, h + 1, p - 2, p - 1], dtype=np.uint64)
        xs = np.array(list(itertools.product(range(6), repeat=6)), dtype=np.int64)
        X = ext[xs]                                                     # (46656, 6)
        if p % 4 == 1:
            yset = [(of.mod_sqrt(p - 1, p), 0)]
        elif p > 3:
            yset = [tuple(of.sos(p - 1, p))]
        else:
            yset = [(1, 1)]
        yset += [(p - 1, p - 1), (p - 1, 1), (h, h + 1), (1, p - 1)]
        for yk in (0, 1):
            for ya, yb in yset:
                n = X.shape[0]
                R = np.zeros((n, 11), dtype=np.uint64)
                R[:, 0], R[:, 1], R[:, 2:8], R[:, 8], R[:, 9] = p, yk, X, ya, yb
                recs.append(R)
            n = 60000
            R = np.zeros((n, 11), dtype=np.uint64)
            R[:, 0], R[:, 1] = p, yk
            R[:, 2:10] = rng.integers(0, p, size=(n, 8))
            recs.append(R)
    R = np.concatenate(recs).astype(np.uint32)
    out = subprocess.run([str(exe)], input=R.tobytes(), capture_output=True, check=True).stdout
    got = np.frombuffer(out, dtype=np.uint32).reshape(-1, 4).astype(np.int64)
    assert got.shape[0] == R.shape[0]
    Ri = R.astype(np.int64)
    p, yk = Ri[:, 0], Ri[:, 1]
    x11a, x11b, x21a, x21b, x22a, x22b, ya, yb = (Ri[:, c] for c in range(2, 10))
    h = (p - 1) // 2
    d1, d2 = x21a - x11a, x21b - x11b
    s1a = np.where(yk == 0, ya * d1, ya * d1 - yb * d2)
    s1b = np.where(yk == 0, ya * d2, yb * d1 + ya * d2)
    s2a = np.where(yk == 0, x22a - ya * x21a, x22a - (ya * x21a - yb * x21b))
    s2b = np.where(yk == 0, x22b - ya * x21b, x22b - (yb * x21a + ya * x21b))
    want = np.stack([(v + h) % p for v in (s1a, s1b, s2a, s2b)], axis=1)
    bad = np.nonzero((got != want).any(axis=1))[0]
    assert bad.size == 0, (bad.size, R[bad[:5]].tolist(), got[bad[:5]].tolist(), want[bad[:5]].tolist())


PROG_LAZY3 = r"""
#include <cstdio>
#include "modp.cuh"
using namespace adj;
int main() {
  unsigned p, w; long long x;
  while (scanf("%u %u %lld", &p, &w, &x) == 3) {
    ShoupW s = make_shoup(w, p);
    printf("%u\n", mulred_lazy3((int32_t)x, s.wc, s.wq, p));
  }
  return 0;
}
"""


def test_mulred_lazy3_range_and_residue(tmp_path):
    """The wide leaf's intermediate Horner step (modp.cuh mulred_lazy3): x w mod p + {0, p, 2p},
    always in [0, 3p), for every int32 extreme and random x at the scheme boundary primes."""
    src, exe = tmp_path / "tl.cpp", tmp_path / "tl"
    src.write_text(PROG_LAZY3)
    subprocess.run(["g++", "-O2", "-std=c++17", "-I", CSRC, str(src), "-o", str(exe)], check=True)
    rng = random.Random(11)
    cases = []
    xs_fixed = [-2**31, -2**31 + 1, -1, 0, 1, 2**31 - 1, 2**31 - 2, -2**30, 2**30]
    for p in PRIMES:
        ws = sorted({0, 1, 2, p - 1, p - 2, (p - 1) // 2, (p + 1) // 2} | {rng.randrange(p) for _ in range(20)})
        for w in ws:
            for x in xs_fixed + [rng.randrange(-2**31, 2**31) for _ in range(30)]:
                cases.append((p, w, x))
    inp = "".join(f"{p} {w} {x}\n" for p, w, x in cases)
    out = subprocess.run([str(exe)], input=inp, capture_output=True, text=True, check=True).stdout.split()
    assert len(out) == len(cases)
    for (p, w, x), got in zip(cases, out):
        g = int(got)
        assert 0 <= g < 3 * p and g % p == (x * w) % p, (p, w, x, g)
