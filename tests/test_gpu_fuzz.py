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


PRIMES_3MOD4 = [3, 251, 8191, 16763, 16787, 65519, 131071, 262139]


@pytest.mark.parametrize("case", range(80))
def test_fuzz_phi_h_and_q(adj, case):
    """phi = H (2M, or one level of Alg. 1 over GF(p^2)) and phi = Q (6M): random ragged shapes,
    depths, strides, plain / FILL_UPPER."""
    import torch
    rng = np.random.default_rng(5000 + case)
    phi = "H" if case % 2 == 0 else "Q"
    p = int(rng.choice(PRIMES_3MOD4)) if phi == "H" else int(rng.choice(PRIMES))
    w = 2 if phi == "H" else 4
    m, k = int(rng.integers(1, 300)), int(rng.integers(1, 300))
    depth = int(rng.integers(0, 3))
    lda, ldc = k + int(rng.integers(0, 5)), m + int(rng.integers(0, 5))
    alg1 = phi == "H" and rng.random() < 0.5
    fill = rng.random() < 0.3
    in16 = p < 65536 and rng.random() < 0.4
    out16 = in16 and not (alg1 or fill) and rng.random() < 0.7
    if in16:
        Araw = rng.integers(0, 1 << 16, size=(m, lda, w), dtype=np.uint16)
        dA = torch.from_numpy(Araw.reshape(m, lda * w).view(np.int16)).cuda()
    else:
        Araw = rng.integers(0, 1 << 32, size=(m, lda, w), dtype=np.uint64).astype(np.uint32)
        dA = torch.from_numpy(Araw.reshape(m, lda * w).view(np.int32)).cuda()
    A = (Araw[:, :k].astype(np.uint32) % p).astype(np.uint32)
    ref = oracle.syrk_h(A, p) if phi == "H" else oracle.syrk_q(A, p)
    if out16:
        C0 = rng.integers(0, 1 << 16, size=(m, ldc, w), dtype=np.uint64).astype(np.uint32)
        C = torch.from_numpy(C0.astype(np.uint16).reshape(m, ldc * w).view(np.int16).copy()).cuda()
    else:
        C0 = rng.integers(0, 1 << 32, size=(m, ldc, w), dtype=np.uint64).astype(np.uint32)
        C = torch.from_numpy(C0.reshape(m, ldc * w).view(np.int32).copy()).cuda()
    flags = ((adj.ADJ_HERK_ALG1 if alg1 else 0) | (adj.ADJ_FILL_UPPER if fill else 0)
             | (adj.ADJ_IN_U16 if in16 else 0) | (adj.ADJ_OUT_U16 if out16 else 0))
    adj.adjprod_modp_ex(m, k, p, adj.ADJ_PHI_H if phi == "H" else adj.ADJ_PHI_Q, dA, lda, C, ldc,
                        depth=1 if alg1 else depth, flags=flags)
    torch.cuda.synchronize()
    got = C.cpu().numpy().view(np.uint16 if out16 else np.uint32).astype(np.uint32).reshape(m, ldc, w)
    lo = np.tril(np.ones((m, m), dtype=bool))
    assert np.array_equal(got[:, :m][lo], ref[lo]), (phi, p, m, k, depth, alg1)
    if fill:   # Up(C) = phi(Low(C)): conjugation negates the imaginary components
        up = ~lo
        conj = ref.transpose(1, 0, 2).astype(np.int64)
        conj[..., 1:] = (-conj[..., 1:]) % p
        assert np.array_equal(got[:, :m][up], conj.astype(np.uint32)[up]), (phi, p, m, k, depth)
    else:
        assert np.array_equal(got[:, :m][~lo], C0[:, :m][~lo])
    assert np.array_equal(got[:, m:], C0[:, m:])


@pytest.mark.parametrize("case", range(40))
def test_fuzz_gemm(adj, case):
    import torch
    rng = np.random.default_rng(9000 + case)
    p = int(rng.choice(PRIMES))
    m, n, k = (int(x) for x in rng.integers(1, 600, size=3))
    lda, ldb, ldc = k + int(rng.integers(0, 5)), k + int(rng.integers(0, 5)), n + int(rng.integers(0, 5))
    Ar = rng.integers(0, 1 << 32, size=(m, lda), dtype=np.uint64).astype(np.uint32)
    Br = rng.integers(0, 1 << 32, size=(n, ldb), dtype=np.uint64).astype(np.uint32)
    C = torch.zeros((m, ldc), dtype=torch.int32, device="cuda")
    adj.gemm_modp(m, n, k, p, torch.from_numpy(Ar.view(np.int32)).cuda(), lda,
                  torch.from_numpy(Br.view(np.int32)).cuda(), ldb, C, ldc)
    torch.cuda.synchronize()
    ref = oracle.gemm_nt((Ar[:, :k] % p).astype(np.uint32), (Br[:, :k] % p).astype(np.uint32), p)
    assert np.array_equal(C.cpu().numpy().view(np.uint32)[:, :n], ref), (p, m, n, k)
