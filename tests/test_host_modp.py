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
