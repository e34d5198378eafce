"""Seeded random combinations of the φ = T path's options against the O1 oracle, bit-exact:
shape (ragged, 1..700), prime from every limb scheme, depth 0..3, uint32 / uint16 input and
output, strided views, the SYRK form with random alpha / beta, ADJ_FILL_UPPER."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

PRIMES = [3, 97, 251, 257, 4099, 8191, 16763, 16787, 40009, 65521, 65537, 131071, 262139]


@pytest.fixture(scope="module")
def adj():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    import paper_2101_01025_b200 as adj
    adj.lib()
    return adj


@pytest.mark.parametrize("case", range(160))
def test_fuzz_phi_t(adj, case):
    import torch
    rng = np.random.default_rng(1000 + case)
    p = int(rng.choice(PRIMES))
    m, k = int(rng.integers(1, 700)), int(rng.integers(1, 700))
    depth = int(rng.integers(0, 4))
    pad_a, pad_c = int(rng.integers(0, 9)), int(rng.integers(0, 9))
    in16 = p < 65536 and rng.random() < 0.4
    mode = rng.choice(["plain", "syrk", "fill"]) if not in16 else rng.choice(["plain", "out16"])
    lda, ldc = k + pad_a, m + pad_c
    if in16:
        Araw = rng.integers(0, 1 << 16, size=(m, lda), dtype=np.uint16)
        A = (Araw[:, :k].astype(np.uint32) % p).astype(np.uint32)
        dA = torch.from_numpy(Araw.view(np.int16)).cuda()
    else:
        Araw = rng.integers(0, 1 << 32, size=(m, lda), dtype=np.uint64).astype(np.uint32)
        A = (Araw[:, :k] % p).astype(np.uint32)
        dA = torch.from_numpy(Araw.view(np.int32)).cuda()
    flags = adj.ADJ_IN_U16 if in16 else 0
    ref = oracle.syrk_t(A, p)
    lo = np.tril(np.ones((m, m), dtype=bool))
    if mode == "out16":
        C = torch.full((m, ldc), -1, dtype=torch.int16, device="cuda")
        adj.adjprod_modp_ex(m, k, p, 0, dA, lda, C, ldc, depth=depth, flags=flags | adj.ADJ_OUT_U16)
        torch.cuda.synchronize()
        got = C.cpu().numpy().view(np.uint16)[:, :m].astype(np.uint32)
        assert np.array_equal(got[lo], ref[lo]), (p, m, k, depth)
        assert np.all(got[~lo] == 0xFFFF)
        return
    C0 = rng.integers(0, 1 << 32, size=(m, ldc), dtype=np.uint64).astype(np.uint32)
    C = torch.from_numpy(C0.view(np.int32).copy()).cuda()
    if mode == "syrk":
        alpha, beta = int(rng.integers(0, p)), int(rng.integers(0, p))
        adj.adjprod_modp_syrk(m, k, p, 0, alpha, dA, lda, beta, C, ldc, depth=depth, flags=flags)
        exp = oracle.syrk_update(A, C0[:, :m].copy(), p, alpha, beta)
    else:
        adj.adjprod_modp_ex(m, k, p, 0, dA, lda, C, ldc, depth=depth,
                            flags=flags | (adj.ADJ_FILL_UPPER if mode == "fill" else 0))
        exp = np.where(lo, ref, (ref.T if mode == "fill" else C0[:, :m]))
    torch.cuda.synchronize()
    got = C.cpu().numpy().view(np.uint32)
    assert np.array_equal(got[:, :m], exp), (p, m, k, depth, mode, in16)
    assert np.array_equal(got[:, m:], C0[:, m:]), (p, m, k, depth, mode)   # columns past m untouched
