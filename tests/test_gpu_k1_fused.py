"""GPU parity of the fused K1 of levels 1 + 2 (preadd.cu preadd2_kernel: one read of A, level-1
S3 kept in registers for the level-2 nodes; Alg. alg:MIAHMM pre-additions).
It runs for phi = T at depth >= 2 with uint16 input when m and k are multiples of 512; these
shapes, every limb scheme below 2^16 and both skew-unitary forms of Y (p = 1 and 3 mod 4) are
compared with the oracle element by element, bit-exact."""
import numpy as np
import pytest

import oracle
from inputs import uniform_matrix
from gpu_util import to_dev

pytestmark = pytest.mark.gpu

# scheme 0 (p <= 255), 1 (K7, p <= 16763), 2 (s8/u8, p <= 65521); Y = sqrt(-1) I or Rot2
PRIMES = [97, 251, 7681, 8191, 65521, 65519]


@pytest.fixture(scope="module")
def adj():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    import paper_2101_01025_b200 as adj
    adj.lib()
    return adj


def _run16(adj, A, p, depth, flags=0, noncanon=None):
    import torch
    m, k = A.shape
    Ad = to_dev(A).to(torch.int16) if noncanon is None else torch.from_numpy(noncanon.view(np.int16)).cuda()
    C = torch.full((m, m), -1, dtype=torch.int16, device="cuda")
    adj.adjprod_modp_ex(m, k, p, 0, Ad, k, C, m, depth=depth, flags=flags | adj.ADJ_IN_U16 | adj.ADJ_OUT_U16)
    torch.cuda.synchronize()
    return C.cpu().numpy().view(np.uint16).astype(np.uint32)


@pytest.mark.parametrize("p", PRIMES)
@pytest.mark.parametrize("depth", [2, 3])
@pytest.mark.parametrize("m,k", [(512, 512), (1024, 1536), (1536, 1024)])
def test_fused_k1_vs_oracle(adj, p, depth, m, k):
    A = uniform_matrix(m, k, seed=m + 3 * k + depth + p, p=p)
    got = _run16(adj, A, p, depth)
    ref = oracle.syrk_t(A, p)
    lo = np.tril(np.ones((m, m), dtype=bool))
    assert np.array_equal(got[lo], ref[lo]), (p, depth, m, k)
    assert np.all(got[~lo] == 0xFFFF)


@pytest.mark.parametrize("p", [251, 8191, 65521])
def test_fused_k1_noncanonical_input(adj, p):
    """uint16 values >= p are read mod p (the reducing path of the fused kernel)."""
    m, k = 1024, 512
    A = uniform_matrix(m, k, seed=99, p=p)
    rng = np.random.default_rng(7)
    raw = A.astype(np.uint64) + p * rng.integers(0, (65536 - A.astype(np.int64)) // p + 1, size=A.shape).astype(np.uint64)
    raw = np.minimum(raw, 65535).astype(np.uint16)
    raw[raw % p != A % p] = A[raw % p != A % p]     # keep each value congruent to A
    assert np.array_equal(raw.astype(np.uint32) % p, A % p) and (raw >= p).any()
    got = _run16(adj, A, p, 2, noncanon=np.ascontiguousarray(raw))
    assert np.array_equal(np.tril(got), np.tril(oracle.syrk_t(A, p)))


def test_fused_k1_inside_lowmem_children(adj):
    """ADJ_LOW_MEM at depth 3: the children (1024 x 1024 at depth 2, the S3 child from workspace
    residues) take the fused K1."""
    p = 65521
    A = uniform_matrix(2048, 2048, seed=5, p=p)
    got = _run16(adj, A, p, 3, flags=adj.ADJ_LOW_MEM)
    assert np.array_equal(np.tril(got), np.tril(oracle.syrk_t(A, p)))
