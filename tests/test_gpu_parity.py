"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element,
bit-exact (all arithmetic is exact mod p).  Sizes span several 128-row tiles and ragged tails."""
import numpy as np
import pytest

import oracle
from inputs import uniform_matrix, uniform_matrix_ext, constant_matrix
from gpu_util import low, to_dev, to_host

pytestmark = pytest.mark.gpu

PRIMES = [3, 97, 251, 257, 8191, 16741, 16763, 16787, 65521]
# p > 2^16: three balanced base-64 digits + pair sums, 3-way Karatsuba; the
# paper's own moduli 131071 and 131041 and the largest supported prime
WIDE_PRIMES = [65537, 131041, 131071, 262139]


@pytest.fixture(scope="module")
def adj():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    import paper_2101_01025_b200 as adj
    adj.lib()
    return adj


def test_input_generator_gpu_matches_cpu(adj):
    import torch
    from inputs.gpu import uniform_residues_cuda
    from inputs import uniform_residues
    t = torch.empty(1 << 20, dtype=torch.int32, device="cuda")
    for seed, p in [(1, 97), (2, 8191), (3, 65521)]:
        uniform_residues_cuda(t, seed, p)
        assert np.array_equal(to_host(t), uniform_residues(1 << 20, seed, p))


@pytest.mark.parametrize("p", PRIMES + WIDE_PRIMES)
def test_limb_split_exhaustive_all_residues(adj, p):
    """Every residue x of GF(p) through split -> int8 MMA -> recombine: x * c for several c,
    including the limb extremes (SURVEY.md §8(c) pin 1)."""
    xs = np.arange(p, dtype=np.uint32).reshape(p, 1)
    cs = np.array([[1], [p - 1], [2], [(p - 1) // 2], [(p + 1) // 2], [p // 3 + 1]], dtype=np.uint32) % p
    C = adj.gemm(to_dev(xs), to_dev(cs), p)
    ref = (xs.astype(np.int64) * cs.astype(np.int64).T) % p
    assert np.array_equal(to_host(C), ref.astype(np.uint32))


@pytest.mark.parametrize("p", PRIMES + WIDE_PRIMES)
@pytest.mark.parametrize("m,n,k", [(1, 1, 1), (128, 128, 128), (200, 300, 257), (130, 129, 1000), (256, 512, 64)])
def test_gemm_vs_oracle(adj, p, m, n, k):
    A = uniform_matrix(m, k, seed=m + k, p=p)
    B = uniform_matrix(n, k, seed=n + 3 * k, p=p)
    C = adj.gemm(to_dev(A), to_dev(B), p)
    assert np.array_equal(to_host(C), oracle.gemm_nt(A, B, p))


@pytest.mark.parametrize("p", PRIMES)
@pytest.mark.parametrize("depth", [0, 1, 2, 3])
@pytest.mark.parametrize("m,k", [(1, 5), (7, 3), (129, 200), (300, 300), (513, 1100)])
def test_adjprod_T_vs_oracle(adj, p, depth, m, k):
    A = uniform_matrix(m, k, seed=7 * m + k + depth, p=p)
    C = adj.adjprod(to_dev(A), p, depth=depth)
    got = to_host(C)
    assert np.array_equal(got, oracle.syrk_t(A, p)), (p, depth, m, k)


@pytest.mark.parametrize("p", WIDE_PRIMES)
@pytest.mark.parametrize("depth", [0, 1, 2, 3])
@pytest.mark.parametrize("m,k", [(1, 5), (129, 200), (513, 1100)])
def test_adjprod_T_wide_vs_oracle(adj, p, depth, m, k):
    A = uniform_matrix(m, k, seed=11 * m + k + depth, p=p)
    got = to_host(adj.adjprod(to_dev(A), p, depth=depth))
    assert np.array_equal(got, oracle.syrk_t(A, p)), (p, depth, m, k)


@pytest.mark.parametrize("p", [8191, 131071])
@pytest.mark.parametrize("depth", [0, 1, 2])
@pytest.mark.parametrize("m,k", [(1, 1), (33, 17), (260, 300), (700, 513)])
def test_adjprod_H_vs_oracle(adj, p, depth, m, k):
    A = uniform_matrix_ext(m, k, seed=m * 31 + k, p=p)
    C = adj.adjprod(to_dev(A), p, phi="H", depth=depth)
    assert np.array_equal(to_host(C), oracle.syrk_h(A, p))


@pytest.mark.parametrize("p", [97, 8191, 65521])
def test_noncanonical_inputs_and_strided_views(adj, p):
    import torch
    rng = np.random.default_rng(p)
    m, k, lda, ldc = 150, 333, 345, 161
    full = rng.integers(0, 2**32, size=(m, lda), dtype=np.uint64).astype(np.uint32)
    A = full[:, :k]
    dA = to_dev(full)
    C = torch.full((m, ldc), -1, dtype=torch.int32, device="cuda")
    adj.adjprod_modp_ex(m, k, p, 0, dA, lda, C, ldc, depth=1)
    got = to_host(C)
    assert np.array_equal(low(got[:, :m]), oracle.syrk_t(A % p, p))
    # strict upper triangle and padding columns untouched
    untouched = ~np.tril(np.ones((m, ldc), dtype=bool))
    assert (got[untouched] == 0xFFFFFFFF).all()


@pytest.mark.parametrize("phi", ["T", "H"])
def test_fill_upper(adj, phi):
    p = 8191
    if phi == "T":
        A = uniform_matrix(200, 300, seed=1, p=p)
    else:
        A = uniform_matrix_ext(200, 300, seed=1, p=p)
    C = to_host(adj.adjprod(to_dev(A), p, phi=phi, depth=1, fill_upper=True))
    if phi == "T":
        assert np.array_equal(C, C.T)
    else:
        assert np.array_equal(C[..., 0], C[..., 0].T)
        assert np.array_equal(C[..., 1], (p - C[..., 1].T.astype(np.int64)) % p)


def test_k_zero_and_m_zero(adj):
    import torch
    C = torch.full((5, 5), 7, dtype=torch.int32, device="cuda")
    A = torch.zeros((5, 1), dtype=torch.int32, device="cuda")
    adj.adjprod_modp(5, 0, 97, 0, A, 1, C, 5)
    got = to_host(C)
    assert (np.tril(got) == 0).all() and (got[np.triu_indices(5, 1)] == 7).all()


@pytest.mark.parametrize("p,c,k,depth", [
    (65521, 65521 - 32513, 32768, 0),   # lo = 255, hi = -128: u8*u8 and cross at the int32 bound
    (8191, 8191 - 64, 32768, 0),        # lo = -64
    (8191, 8191 - 4032, 65536, 0),      # mid extreme
    (97, 48, 4096, 0),
    (65521, 65521 - 32513, 32768, 1),
    (262139, 262139 - 131069, 32768, 0),   # wide scheme: c = -(p-1)/2
    (131071, 131071 - 2080, 524288, 0),    # c = -2080: digits (0, -32, -32), d1 + d0 = -64: every
                                           # product 4096, k past the 2^31 / 4096 bound (2 segments)
])
def test_overflow_stress_constant(adj, p, c, k, depth):
    """Constant A = c: C = k c^2 mod p everywhere (SURVEY.md §8(c) pin 4, overflow stress)."""
    m = 256
    A = constant_matrix(m, k, c, p)
    got = to_host(adj.adjprod(to_dev(A), p, depth=depth))
    exp = k * c * c % p
    assert (got[np.tril_indices(m)] == exp).all()
    B = constant_matrix(130, k, c, p)
    G = to_host(adj.gemm(to_dev(A), to_dev(B), p))
    assert (G == exp).all()


@pytest.mark.parametrize("c", [65521 - 32513, 32760])   # (hi, lo) = (-128, 255) and (127, 248)
def test_overflow_stress_constant_wide_leaf(adj, c):
    """Constant A = c on the wide-N leaf with K segmentation: 8192 x 65536 over GF(65521) at depth
    0 is 272 wide jobs (the 256 x 512 leaf by the makespan rule) whose K = 512 k-blocks run as two
    segments per accumulator, each starting from the lazy Horner value < 3p the previous unit left
    in TMEM (modp.cuh mulred_lazy3, field.cpp limb_kmax_from_residue) and accumulating 32768
    extreme products: C = k c^2 mod p everywhere (SURVEY.md §8(c) pin 4)."""
    import torch
    p, m, k = 65521, 8192, 65536
    assert adj.adjprod_modp_leaf_tile(m, k, p, 0, 0, adj.ADJ_IN_U16 | adj.ADJ_OUT_U16) == 512
    A = torch.full((m, k), c if c < 32768 else c - 65536, dtype=torch.int16, device="cuda")   # uint16 bits
    C = adj.adjprod(A, p, depth=0, out16=True)
    got = (C.to(torch.int32) & 0xFFFF)
    lo = torch.tril(torch.ones((m, m), dtype=torch.bool, device="cuda"))
    assert bool((got[lo] == k * c * c % p).all())


def test_depth_invariance(adj):
    p = 65521
    A = uniform_matrix(1000, 1500, seed=3, p=p)
    dA = to_dev(A)
    ref = to_host(adj.adjprod(dA, p, depth=0))
    for d in (1, 2, 3):
        assert np.array_equal(to_host(adj.adjprod(dA, p, depth=d)), ref)


def test_dist_single_rank(adj):
    """adjprod_modp_dist through NCCL with one rank equals the single-GPU call."""
    import torch
    p = 8191
    A = uniform_matrix(300, 500, seed=4, p=p)
    dA = to_dev(A)
    uid = adj.adj_comm_get_unique_id()
    comm = adj.adj_comm_init(1, uid, 0)
    C = torch.zeros((300, 300), dtype=torch.int32, device="cuda")
    adj.adjprod_modp_dist(300, 500, p, 0, dA, 500, C, 300, 0, comm)
    assert np.array_equal(to_host(C), oracle.syrk_t(A, p))
    adj.adj_comm_destroy(comm)


def test_errors_on_device(adj):
    import torch
    A = torch.zeros((4, 4), dtype=torch.int32, device="cuda")
    with pytest.raises(adj.AdjError):
        adj.adjprod_modp_ex(4, 4, 97, 0, A, 4, A, 4)   # overlap
    ws = torch.zeros(16, dtype=torch.uint8, device="cuda")
    C = torch.zeros((300, 300), dtype=torch.int32, device="cuda")
    B = torch.zeros((300, 300), dtype=torch.int32, device="cuda")
    with pytest.raises(adj.AdjError) as e:
        adj.adjprod_modp_ex(300, 300, 97, 0, B, 300, C, 300, depth=1, workspace=ws, workspace_bytes=16)
    assert e.value.status == 3


@pytest.mark.parametrize("p,k,m", [(65521, 40000, 300), (65521, 70000, 130), (97, 140000, 64), (8191, 240000, 64),
                                   (131071, 600000, 40)])
def test_k_segmentation_beyond_int32_bound(adj, p, k, m):
    """Inner dimension above the limb scheme's int32 bound: the leaf splits K
    into segments, each reduced mod p and summed (depth 0 and gemm_modp)."""
    A = uniform_matrix(m, k, seed=k + m, p=p)
    dA = to_dev(A)
    got = to_host(adj.adjprod(dA, p, depth=0))
    assert np.array_equal(got, oracle.syrk_t(A, p))
    B = uniform_matrix(70, k, seed=k + 1, p=p)
    G = to_host(adj.gemm(dA, to_dev(B), p))
    assert np.array_equal(G, oracle.gemm_nt(A, B, p))


def test_k_segmentation_overflow_stress(adj):
    p, c, k = 65521, 65521 - 32513, 70000          # lo = 255, hi = -128, 3 segments
    A = constant_matrix(256, k, c, p)
    got = to_host(adj.adjprod(to_dev(A), p, depth=0))
    assert (got[np.tril_indices(256)] == k * c * c % p).all()


@pytest.mark.parametrize("p", [8191, 131071])
@pytest.mark.parametrize("phi", ["T", "H"])
@pytest.mark.parametrize("depth", [0, 1, 2])
@pytest.mark.parametrize("alpha,beta", [(1, 0), (0, 1), (3, 5), (8190, 8190), (12345, 0), (1, 1)])
def test_syrk_form_alpha_beta(adj, p, phi, depth, alpha, beta):
    """Low(C) <- alpha Low(A phi(A)) + beta Low(C), fused into the final writes."""
    import torch
    m, k = 300, 260
    A = uniform_matrix(m, k, seed=5, p=p) if phi == "T" else uniform_matrix_ext(m, k, seed=5, p=p)
    rng = np.random.default_rng(depth * 31 + alpha)
    shape = (m, m) if phi == "T" else (m, m, 2)
    C0 = rng.integers(0, 2**32, size=shape, dtype=np.uint64).astype(np.uint32)
    dC = to_dev(C0)
    adj.adjprod_modp_syrk(m, k, p, 0 if phi == "T" else 1, alpha, to_dev(A), k, beta, dC, m, depth=depth)
    assert np.array_equal(to_host(dC), oracle.syrk_update(A, C0, p, alpha, beta, phi))


def test_syrk_form_k0_and_gemm_unaffected(adj):
    import torch
    p = 97
    C0 = np.arange(25, dtype=np.uint32).reshape(5, 5) * 1000
    dC = to_dev(C0)
    adj.adjprod_modp_syrk(5, 0, p, 0, 7, torch.zeros((5, 1), dtype=torch.int32, device="cuda"), 1, 3, dC, 5)
    ref = C0.copy()
    ref[np.tril_indices(5)] = (3 * (C0[np.tril_indices(5)].astype(np.int64) % p)) % p
    assert np.array_equal(to_host(dC), ref)


# ---------------------------------------------------------------- SURVEY.md §8(f)-2
# phi = H by one level of Alg. alg:MIAHMM directly over GF(p^2), Y = (a + ib) I (PAPER.md
# §4.4, 750-758), 2M Hermitian leaves and 3M general leaves (ADJ_HERK_ALG1): the same Low(C).
HERK_PRIMES = [3, 7, 251, 8191, 16763, 65519, 131071]


@pytest.mark.parametrize("p", HERK_PRIMES)
@pytest.mark.parametrize("m,k", [(1, 1), (2, 2), (33, 17), (129, 200), (260, 300), (700, 513)])
def test_herk_alg1_vs_oracle(adj, p, m, k):
    A = uniform_matrix_ext(m, k, seed=m * 7 + k, p=p)
    C = adj.adjprod(to_dev(A), p, phi="H", herk="alg1")
    assert np.array_equal(to_host(C), oracle.syrk_h(A, p))


def test_herk_alg1_fill_upper_and_untouched(adj):
    import torch
    p, m, k = 8191, 300, 260
    A = uniform_matrix_ext(m, k, seed=9, p=p)
    C = torch.full((m, m, 2), -1, dtype=torch.int32, device="cuda")
    adj.adjprod(to_dev(A), p, phi="H", herk="alg1", out=C)
    got = to_host(C)
    ref = oracle.syrk_h(A, p)
    lo = np.tril(np.ones((m, m), dtype=bool))
    assert np.array_equal(got[lo], ref[lo])
    assert (got[~lo] == 0xFFFFFFFF).all()
    F = to_host(adj.adjprod(to_dev(A), p, phi="H", herk="alg1", fill_upper=True))
    assert np.array_equal(F[..., 0], F[..., 0].T)
    assert np.array_equal(F[..., 1], (p - F[..., 1].T.astype(np.int64)) % p)
    assert np.array_equal(F[lo], ref[lo])


@pytest.mark.parametrize("alpha,beta", [(1, 0), (0, 1), (3, 5), (8190, 8190)])
def test_herk_alg1_syrk_form(adj, alpha, beta):
    p, m, k = 8191, 300, 260
    A = uniform_matrix_ext(m, k, seed=5, p=p)
    rng = np.random.default_rng(alpha + 7 * beta)
    C0 = rng.integers(0, 2**32, size=(m, m, 2), dtype=np.uint64).astype(np.uint32)
    dC = to_dev(C0)
    adj.adjprod_modp_syrk(m, k, p, 1, alpha, to_dev(A), k, beta, dC, m, flags=adj.ADJ_HERK_ALG1)
    assert np.array_equal(to_host(dC), oracle.syrk_update(A, C0, p, alpha, beta, "H"))


def test_herk_alg1_strided_and_noncanonical(adj):
    import torch
    p, m, k, lda, ldc = 8191, 150, 333, 341, 157
    rng = np.random.default_rng(3)
    full = rng.integers(0, 2**32, size=(m, lda, 2), dtype=np.uint64).astype(np.uint32)
    C = torch.zeros((m, ldc, 2), dtype=torch.int32, device="cuda")
    adj.adjprod_modp_ex(m, k, p, 1, to_dev(full), lda, C, ldc, flags=adj.ADJ_HERK_ALG1)
    got = to_host(C)[:, :m]
    ref = oracle.syrk_h(full[:, :k] % p, p)
    lo = np.tril(np.ones((m, m), dtype=bool))
    assert np.array_equal(got[lo], ref[lo])


def test_herk_alg1_depth_must_be_one(adj):
    import torch
    A = torch.zeros((8, 8, 2), dtype=torch.int32, device="cuda")
    C = torch.zeros((8, 8, 2), dtype=torch.int32, device="cuda")
    with pytest.raises(adj.AdjError):
        adj.adjprod_modp_ex(8, 8, 8191, 1, A, 8, C, 8, depth=2, flags=adj.ADJ_HERK_ALG1)


# ---------------------------------------------------------------- SURVEY.md §8(f)-4
# phi = quaternion conjugate transpose (ADJ_PHI_Q), Alg. alg:2M3M (6M) with
# Q6 through Alg. alg:MIAHMM at the requested depth, against the Hamilton-product oracle.
QUAT_PRIMES = [3, 97, 251, 257, 8191, 16787, 65521, 131071]


@pytest.mark.parametrize("p", QUAT_PRIMES)
@pytest.mark.parametrize("depth", [0, 1, 2])
@pytest.mark.parametrize("m,k", [(1, 1), (2, 3), (33, 17), (129, 200), (260, 300)])
def test_quat_vs_oracle(adj, p, depth, m, k):
    from inputs import uniform_matrix_quat
    M = uniform_matrix_quat(m, k, seed=m * 13 + k + depth, p=p)
    C = adj.adjprod(to_dev(M), p, phi="Q", depth=depth)
    assert np.array_equal(to_host(C), oracle.syrk_q(M, p))


def test_quat_fill_upper_untouched_and_strided(adj):
    import torch
    from inputs import uniform_matrix_quat
    p, m, k, ldm, ldc = 8191, 150, 210, 223, 161
    rng = np.random.default_rng(11)
    full = rng.integers(0, 2**32, size=(m, ldm, 4), dtype=np.uint64).astype(np.uint32)
    C = torch.full((m, ldc, 4), -1, dtype=torch.int32, device="cuda")
    adj.adjprod_modp_ex(m, k, p, adj.ADJ_PHI_Q, to_dev(full), ldm, C, ldc, depth=1)
    got = to_host(C)
    ref = oracle.syrk_q(full[:, :k] % p, p)
    lo = np.tril(np.ones((m, m), dtype=bool))
    assert np.array_equal(got[:, :m][lo], ref[lo])
    assert (got[:, :m][~lo] == 0xFFFFFFFF).all() and (got[:, m:] == 0xFFFFFFFF).all()
    M = uniform_matrix_quat(200, 120, seed=4, p=p)
    F = to_host(adj.adjprod(to_dev(M), p, phi="Q", fill_upper=True))
    assert np.array_equal(F[..., 0], F[..., 0].T)                       # H(j,i) = conj(H(i,j))
    for c in (1, 2, 3):
        assert np.array_equal(F[..., c], (p - F[..., c].T.astype(np.int64)) % p)


@pytest.mark.parametrize("alpha,beta", [(1, 0), (0, 1), (3, 5), (8190, 8190)])
def test_quat_syrk_form(adj, alpha, beta):
    from inputs import uniform_matrix_quat
    p, m, k = 8191, 200, 150
    M = uniform_matrix_quat(m, k, seed=6, p=p)
    rng = np.random.default_rng(alpha * 3 + beta)
    C0 = rng.integers(0, 2**32, size=(m, m, 4), dtype=np.uint64).astype(np.uint32)
    dC = to_dev(C0)
    adj.adjprod_modp_syrk(m, k, p, adj.ADJ_PHI_Q, alpha, to_dev(M), k, beta, dC, m)
    assert np.array_equal(to_host(dC), oracle.syrk_update(M, C0, p, alpha, beta, phi="Q"))


def test_quat_overflow_stress_constant(adj):
    """Constant quaternion matrix at the int32 accumulation bound of each Q product (limb
    extremes, k beyond one K segment)."""
    from inputs import constant_matrix
    p, m, k = 8191, 128, 240000
    M = np.stack([constant_matrix(m, k, c, p) for c in (p - 64, p - 4032, 4032, 64)], axis=-1)
    got = to_host(adj.adjprod(to_dev(M), p, phi="Q", depth=0))
    ref = oracle.syrk_q(M[:2], p)
    assert (got[np.tril_indices(m)] == ref[1, 0]).all()


# ---------------------------------------------------------------- SURVEY.md §8(e)-2
# Output-tile sharding: every rank's share (adjprod_modp_shard) run one after the other on this
# device into one C must give all of Low(C); one share writes only its own regions.
@pytest.mark.parametrize("p", [97, 8191, 65521, 131071])
@pytest.mark.parametrize("depth", [0, 1])
@pytest.mark.parametrize("m,k", [(5, 3), (300, 200), (1030, 520)])
@pytest.mark.parametrize("nranks", [1, 2, 3, 5])
def test_shard_all_ranks_give_low_c(adj, p, depth, m, k, nranks):
    import torch
    A = uniform_matrix(m, k, seed=m + nranks, p=p)
    dA = to_dev(A)
    C = torch.full((m, m), -1, dtype=torch.int32, device="cuda")
    for r in range(nranks):
        adj.adjprod_modp_shard(m, k, p, 0, dA, k, C, m, r, nranks, depth=depth)
    got = to_host(C)
    lo = np.tril(np.ones((m, m), dtype=bool))
    assert np.array_equal(got[lo], oracle.syrk_t(A, p)[lo])
    assert (got[~lo] == 0xFFFFFFFF).all()


def test_shard_writes_only_its_regions(adj):
    import torch
    p, m, k, n = 8191, 1030, 300, 3
    A = uniform_matrix(m, k, seed=2, p=p)
    ref = oracle.syrk_t(A, p)
    for depth in (0, 1):
        for r in range(n):
            C = torch.full((m, m), -1, dtype=torch.int32, device="cuda")
            adj.adjprod_modp_shard(m, k, p, 0, to_dev(A), k, C, m, r, n, depth=depth)
            got = to_host(C)
            mine = np.zeros((m, m), dtype=bool)
            for (r0, c0, rows, cols, lower) in adj.adj_shard_layout(m, k, p, r, n, depth=depth):
                ii, jj = np.meshgrid(np.arange(rows) + r0, np.arange(cols) + c0, indexing="ij")
                mine[r0:r0 + rows, c0:c0 + cols] = (jj <= ii) if lower else True
            assert np.array_equal(got[mine], ref[mine])
            assert (got[~mine] == 0xFFFFFFFF).all()


def test_dist_tiles_single_rank(adj):
    """ADJ_DIST_TILES through the NCCL entry point with one rank (the multi-rank gather is covered
    by tests/test_dist_gloo.py)."""
    import torch
    p, m, k = 8191, 700, 300
    A = uniform_matrix(m, k, seed=8, p=p)
    comm = adj.adj_comm_init(1, adj.adj_comm_get_unique_id(), 0)
    try:
        C = torch.zeros((m, m), dtype=torch.int32, device="cuda")
        adj.adjprod_modp_dist(m, k, p, 0, to_dev(A), k, C, m, 0, comm, depth=1, flags=adj.ADJ_DIST_TILES)
        assert np.array_equal(low(to_host(C)), oracle.syrk_t(A, p))
    finally:
        adj.adj_comm_destroy(comm)


@pytest.mark.parametrize("p", [97, 8191, 65521, 131071])
def test_tail_column_half_jobs(adj, p):
    """Last-wave tiles split into two N = 128 column halves (74 clusters, 19..37 tail tiles):
    gemm 2560^2 (100 tiles, tail 26) and a depth-0 SYRK of m = 4608 (171 lower tiles, tail 23)."""
    A = uniform_matrix(2560, 300, seed=3, p=p)
    B = uniform_matrix(2560, 300, seed=4, p=p)
    C = adj.gemm(to_dev(A), to_dev(B), p)
    assert np.array_equal(to_host(C), oracle.gemm_nt(A, B, p))
    A = uniform_matrix(4608, 200, seed=5, p=p)
    C = to_host(adj.adjprod(to_dev(A), p, depth=0))
    rows = [0, 1, 2047, 2048, 4350, 4607]
    ref = oracle.syrk_t(A, p)
    for r in rows:
        assert np.array_equal(C[r, : r + 1], ref[r, : r + 1]), r
    assert np.array_equal(low(C), ref)


# ---------------------------------------------------------------- split-K building blocks
@pytest.mark.parametrize("p", [97, 8191, 65521, 131071])
@pytest.mark.parametrize("depth", [0, 1])
@pytest.mark.parametrize("G", [1, 2, 3, 5])
def test_partials_of_column_slices_sum_to_low_c(adj, p, depth, G):
    """adjprod_modp_partial on every rank's column slice (adj_dist_kslice) into G narrow residue
    buffers, then adj_sum_partials: the split-K exchange path of adjprod_modp_dist, ranks run one
    after the other on this device."""
    import torch
    m, k = 300, 700
    A = uniform_matrix(m, k, seed=G * 7 + depth, p=p)
    dA = to_dev(A)
    dt = torch.int16 if p < 65536 else torch.int32
    R = torch.zeros((G, m, m), dtype=dt, device="cuda")
    for r in range(G):
        k0, k1 = adj.adj_dist_kslice(k, G, r)
        adj.adjprod_modp_partial(m, k1 - k0, p, 0, dA[:, k0:], k, R[r], m, depth=depth)
    C = torch.full((m, m), -1, dtype=torch.int32, device="cuda")
    adj.adj_sum_partials(m, p, R, m, m * m, G, C, m)
    got = to_host(C)
    lo = np.tril(np.ones((m, m), dtype=bool))
    assert np.array_equal(got[lo], oracle.syrk_t(A, p)[lo])
    assert (got[~lo] == 0xFFFFFFFF).all()


@pytest.mark.parametrize("depth", [0, 1, 2])
def test_cuda_graph_capture_and_replay(adj, depth):
    """One call is a fixed stream-ordered launch sequence with no host synchronisation: it can be
    captured into a CUDA graph (after a first call builds the cached plan) and replayed."""
    import torch
    p, m, k = 8191, 600, 520
    A = uniform_matrix(m, k, seed=21, p=p)
    dA = to_dev(A)
    ws_bytes = adj.adjprod_modp_workspace_size(m, k, p, 0, depth)
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device="cuda")
    C = torch.zeros((m, m), dtype=torch.int32, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        adj.adjprod_modp_ex(m, k, p, 0, dA, k, C, m, depth=depth, workspace=ws, workspace_bytes=ws_bytes, stream=s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        adj.adjprod_modp_ex(m, k, p, 0, dA, k, C, m, depth=depth, workspace=ws, workspace_bytes=ws_bytes, stream=s)
    ref = oracle.syrk_t(A, p)
    for _ in range(3):
        C.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert np.array_equal(low(to_host(C)), ref)


@pytest.mark.parametrize("p", [8191, 131071])
@pytest.mark.parametrize("depth", [0, 1])
def test_shard_pack_unpack_round_trip(adj, p, depth):
    """The gather step of ADJ_DIST_TILES on one device: each rank's regions packed from C into a
    contiguous buffer (uint16 residues for p < 2^16) and unpacked into a fresh C land exactly on
    that rank's regions."""
    import torch
    m, k, G = 1030, 300, 3
    A = uniform_matrix(m, k, seed=4, p=p)
    C = to_dev(oracle.syrk_t(A, p))
    for r in range(G):
        rects = adj.adj_shard_layout(m, k, p, r, G, depth=depth)
        n = sum(rows * cols for (_, _, rows, cols, _) in rects)
        buf = torch.empty(max(n, 1), dtype=torch.int16 if p < 65536 else torch.int32, device="cuda")
        adj.adj_shard_pack(m, k, p, r, G, C, m, buf, unpack=False, depth=depth)
        C2 = torch.full((m, m), -1, dtype=torch.int32, device="cuda")
        adj.adj_shard_pack(m, k, p, r, G, C2, m, buf, unpack=True, depth=depth)
        got, ref = to_host(C2), to_host(C)
        mine = np.zeros((m, m), dtype=bool)
        for (r0, c0, rows, cols, lower) in rects:
            ii, jj = np.meshgrid(np.arange(rows) + r0, np.arange(cols) + c0, indexing="ij")
            mine[r0:r0 + rows, c0:c0 + cols] = (jj <= ii) if lower else True
        assert np.array_equal(got[mine], ref[mine])
        assert (got[~mine] == 0xFFFFFFFF).all()


def test_dynamic_job_scheduler_forced_small_shapes():
    """The dynamic (atomic-counter) leaf job scheduler is chosen for long launches only; force it
    (ADJ_LEAF_DYNAMIC, read once per process) on small shapes of every path in a subprocess."""
    import os
    import subprocess
    import sys
    code = r'''
import numpy as np, torch, oracle, paper_2101_01025_b200 as adj
from inputs import uniform_matrix, uniform_matrix_ext, uniform_matrix_quat
def dev(a): return torch.from_numpy(np.ascontiguousarray(a).view(np.int32)).cuda()
def host(t): return t.cpu().numpy().view(np.uint32)
bad = 0
for p, m, k, d in [(97, 300, 200, 0), (8191, 700, 513, 1), (65521, 513, 1100, 2), (131071, 400, 300, 1)]:
    A = uniform_matrix(m, k, seed=m, p=p)
    bad += not np.array_equal(np.tril(host(adj.adjprod(dev(A), p, depth=d))), oracle.syrk_t(A, p))
A = uniform_matrix(1000, 300, seed=1, p=8191); B = uniform_matrix(777, 300, seed=2, p=8191)
bad += not np.array_equal(host(adj.gemm(dev(A), dev(B), 8191)), oracle.gemm_nt(A, B, 8191))
H = uniform_matrix_ext(300, 200, seed=3, p=8191)
bad += not np.array_equal(host(adj.adjprod(dev(H), 8191, phi="H")), oracle.syrk_h(H, 8191))
Q = uniform_matrix_quat(200, 150, seed=4, p=8191)
bad += not np.array_equal(host(adj.adjprod(dev(Q), 8191, phi="Q")), oracle.syrk_q(Q, 8191))
print("BAD", bad)
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, ADJ_LEAF_DYNAMIC="1", PYTHONPATH=root)
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600, cwd=root)
    assert "BAD 0" in out.stdout, out.stdout + out.stderr


@pytest.mark.parametrize("p", [3, 251, 257, 8191, 16763, 16787, 65521])
@pytest.mark.parametrize("depth", [0, 1, 2])
@pytest.mark.parametrize("m,k", [(1, 3), (129, 200), (300, 300), (513, 1100)])
def test_adjprod_T_compact_io(adj, p, depth, m, k):
    """ADJ_IN_U16 / ADJ_OUT_U16: uint16 A (any value 0..65535, read mod p) and uint16 Low(C),
    every combination, against the oracle on A mod p."""
    import torch
    rng = np.random.default_rng(m * 7 + k + p)
    A16 = rng.integers(0, 1 << 16, size=(m, k), dtype=np.uint16)
    A16[0, 0] = 65535
    ref = oracle.syrk_t((A16.astype(np.uint32) % p).astype(np.uint32), p)
    dA16 = torch.from_numpy(A16.view(np.int16)).cuda()
    dA32 = to_dev((A16.astype(np.uint32) % p).astype(np.uint32))
    for dA in (dA16, dA32):
        for out16 in (False, True):
            C = adj.adjprod(dA, p, depth=depth, out16=out16)
            torch.cuda.synchronize()
            got = C.cpu().numpy().view(np.uint16 if out16 else np.uint32).astype(np.uint32)
            assert np.array_equal(got, ref), (p, depth, m, k, dA.element_size(), out16)


def test_adjprod_T_compact_io_strided_and_errors(adj):
    import torch
    p, m, k = 8191, 300, 260
    rng = np.random.default_rng(5)
    A16 = rng.integers(0, 1 << 16, size=(m, k + 12), dtype=np.uint16)
    ref = oracle.syrk_t((A16[:, :k].astype(np.uint32) % p).astype(np.uint32), p)
    dA = torch.from_numpy(A16.view(np.int16)).cuda()
    out = torch.full((m, m + 20), -1, dtype=torch.int16, device="cuda")
    adj.adjprod_modp_ex(m, k, p, adj.ADJ_PHI_T, dA, k + 12, out, m + 20, depth=1,
                        flags=adj.ADJ_IN_U16 | adj.ADJ_OUT_U16)
    torch.cuda.synchronize()
    got = out.cpu().numpy().view(np.uint16)
    assert np.array_equal(low(got[:, :m].astype(np.uint32)), ref)
    assert np.all(np.triu(got[:, :m], 1)[np.triu_indices(m, 1)] == 0xFFFF)   # Up(C) untouched
    assert np.all(got[:, m:] == 0xFFFF)
    # a 2-byte-aligned view with an odd leading dimension: the scalar-load paths, every depth
    for depth in (0, 1, 2):
        for mm, kk in ((1, 3), (129, 200), (513, 1100)):
            B16 = rng.integers(0, 1 << 16, size=(mm, kk + 3), dtype=np.uint16)
            dB = torch.from_numpy(B16.view(np.int16)).cuda()[:, 1:kk + 1]
            refb = oracle.syrk_t((B16[:, 1:kk + 1].astype(np.uint32) % p).astype(np.uint32), p)
            Cb = adj.adjprod(dB, p, depth=depth, out16=True)
            torch.cuda.synchronize()
            assert np.array_equal(Cb.cpu().numpy().view(np.uint16).astype(np.uint32), refb), (depth, mm, kk)
    # odd ldc and a 2-byte-offset output: the scalar-store paths
    for depth in (0, 1):
        big = torch.full((m, m + 4), -1, dtype=torch.int16, device="cuda")
        adj.adjprod_modp_ex(m, k, p, adj.ADJ_PHI_T, dA, k + 12, big[:, 1:], m + 4, depth=depth,
                            flags=adj.ADJ_IN_U16 | adj.ADJ_OUT_U16)
        torch.cuda.synchronize()
        g2 = big.cpu().numpy().view(np.uint16)[:, 1:m + 1].astype(np.uint32)
        assert np.array_equal(low(g2), ref), depth
        assert np.all(big.cpu().numpy()[:, 0] == -1)
    # k = 0: Low(C) = 0 in uint16
    out0 = torch.full((4, 4), -1, dtype=torch.int16, device="cuda")
    adj.adjprod_modp_ex(4, 0, p, adj.ADJ_PHI_T, dA, 1, out0, 4, flags=adj.ADJ_OUT_U16)
    torch.cuda.synchronize()
    g0 = out0.cpu().numpy().view(np.uint16)
    assert np.all(g0[np.tril_indices(4)] == 0) and np.all(g0[np.triu_indices(4, 1)] == 0xFFFF)
    C32 = torch.zeros((m, m), dtype=torch.int32, device="cuda")
    bad = [dict(p=131071, flags=adj.ADJ_IN_U16), dict(p=8191, flags=adj.ADJ_OUT_U16 | adj.ADJ_FILL_UPPER)]
    for b in bad:
        with pytest.raises(adj.AdjError):
            adj.adjprod_modp_ex(m, k, b["p"], adj.ADJ_PHI_T, dA, k + 12, C32, m, flags=b["flags"])
    with pytest.raises(adj.AdjError):   # phi = Q with p > 2^16
        adj.adjprod_modp_ex(m // 2, k // 4, 65537, adj.ADJ_PHI_Q, dA, (k + 12) // 4, C32, m // 4, flags=adj.ADJ_IN_U16)
    with pytest.raises(adj.AdjError):   # SYRK form with a uint16 Low(C)
        adj.adjprod_modp_syrk(m, k, p, adj.ADJ_PHI_T, 3, dA, k + 12, 1, out, m + 20, flags=adj.ADJ_OUT_U16)


# ---------------------------------------------------------------- ADJ_IN_U16 on the multi-GPU paths
@pytest.mark.parametrize("p", [251, 8191, 65521])
@pytest.mark.parametrize("depth", [0, 1])
def test_compact_input_shards_and_partials(adj, p, depth):
    """uint16 A (any value, read mod p) through adjprod_modp_shard (3 ranks' shares into one C)
    and adjprod_modp_partial on the k-slices (+ adj_sum_partials), each rank after the other."""
    import torch
    m, k = 700, 900
    rng = np.random.default_rng(p + depth)
    A16 = rng.integers(0, 1 << 16, size=(m, k), dtype=np.uint16)
    ref = oracle.syrk_t((A16.astype(np.uint32) % p).astype(np.uint32), p)
    dA = torch.from_numpy(A16.view(np.int16)).cuda()
    C = torch.zeros((m, m), dtype=torch.int32, device="cuda")
    for r in range(3):
        adj.adjprod_modp_shard(m, k, p, 0, dA, k, C, m, r, 3, depth=depth, flags=adj.ADJ_IN_U16)
    assert np.array_equal(low(to_host(C)), ref)
    G = 3
    R = torch.zeros((G, m, m), dtype=torch.int16, device="cuda")
    for r in range(G):
        k0, k1 = adj.adj_dist_kslice(k, G, r)
        adj.adjprod_modp_partial(m, k1 - k0, p, 0, dA[:, k0:], k, R[r], m, depth=depth, flags=adj.ADJ_IN_U16)
    C2 = torch.zeros((m, m), dtype=torch.int32, device="cuda")
    adj.adj_sum_partials(m, p, R, m, m * m, G, C2, m)
    assert np.array_equal(low(to_host(C2)), ref)


@pytest.mark.parametrize("flags_name", ["", "ADJ_DIST_TILES", "ADJ_DIST_P2P"])
def test_compact_input_dist_single_rank(adj, flags_name):
    import torch
    p, m, k = 8191, 600, 500
    rng = np.random.default_rng(3)
    A16 = rng.integers(0, 1 << 16, size=(m, k), dtype=np.uint16)
    ref = oracle.syrk_t((A16.astype(np.uint32) % p).astype(np.uint32), p)
    comm = adj.adj_comm_init(1, adj.adj_comm_get_unique_id(), 0)
    try:
        C = torch.zeros((m, m), dtype=torch.int32, device="cuda")
        flags = adj.ADJ_IN_U16 | (getattr(adj, flags_name) if flags_name else 0)
        adj.adjprod_modp_dist(m, k, p, 0, torch.from_numpy(A16.view(np.int16)).cuda(), k, C, m, 0, comm,
                              depth=1, flags=flags)
        assert np.array_equal(low(to_host(C)), ref)
        with pytest.raises(adj.AdjError):
            adj.adjprod_modp_dist(m, k, p, 0, torch.from_numpy(A16.view(np.int16)).cuda(), k, C, m, 0, comm,
                                  depth=1, flags=adj.ADJ_OUT_U16)
    finally:
        adj.adj_comm_destroy(comm)


@pytest.mark.parametrize("p", [251, 8191, 16763, 65519])
@pytest.mark.parametrize("depth", [0, 1, 2])
@pytest.mark.parametrize("m,k", [(1, 3), (129, 200), (300, 257)])
def test_adjprod_H_compact_io(adj, p, depth, m, k):
    """ADJ_IN_U16 / ADJ_OUT_U16 for phi = H (2M): (re, im) uint16 pairs in (any value, read mod
    p) and out, every combination, strided; one level of Alg. 1 over GF(p^2) reads uint16 too."""
    import torch
    rng = np.random.default_rng(m * 5 + k + p + depth)
    lda = k + 3
    A16 = rng.integers(0, 1 << 16, size=(m, lda, 2), dtype=np.uint16)
    Ared = (A16[:, :k].astype(np.uint32) % p).astype(np.uint32)
    ref = oracle.syrk_h(Ared, p)
    dA16 = torch.from_numpy(A16.reshape(m, lda * 2).view(np.int16)).cuda()
    dA32 = torch.from_numpy(np.ascontiguousarray(Ared).reshape(m, k * 2).view(np.int32)).cuda()
    lo = np.tril(np.ones((m, m), dtype=bool))
    for dA, ld in ((dA16, lda), (dA32, k)):
        for out16 in (False, True):
            C = torch.zeros((m, m * 2), dtype=torch.int16 if out16 else torch.int32, device="cuda")
            flags = (adj.ADJ_IN_U16 if dA.element_size() == 2 else 0) | (adj.ADJ_OUT_U16 if out16 else 0)
            adj.adjprod_modp_ex(m, k, p, adj.ADJ_PHI_H, dA, ld, C, m, depth=depth, flags=flags)
            torch.cuda.synchronize()
            got = C.cpu().numpy().view(np.uint16 if out16 else np.uint32).astype(np.uint32).reshape(m, m, 2)
            assert np.array_equal(got[lo], ref[lo]), (p, depth, m, k, dA.element_size(), out16)
    if depth == 1:   # Alg. 1 over GF(p^2) with uint16 input
        C = torch.zeros((m, m * 2), dtype=torch.int32, device="cuda")
        adj.adjprod_modp_ex(m, k, p, adj.ADJ_PHI_H, dA16, lda, C, m, depth=1,
                            flags=adj.ADJ_IN_U16 | adj.ADJ_HERK_ALG1)
        torch.cuda.synchronize()
        got = C.cpu().numpy().view(np.uint32).reshape(m, m, 2)
        assert np.array_equal(got[lo], ref[lo]), (p, m, k, "alg1")


@pytest.mark.parametrize("p", [251, 8191, 65521])
@pytest.mark.parametrize("depth", [0, 1])
@pytest.mark.parametrize("m,k", [(1, 3), (129, 200), (260, 131)])
def test_adjprod_Q_compact_io(adj, p, depth, m, k):
    """ADJ_IN_U16 / ADJ_OUT_U16 for phi = Q (6M): 4 uint16 components in (any value, read mod p)
    and out, every combination, strided."""
    import torch
    rng = np.random.default_rng(m * 3 + k + p + depth)
    lda = k + 2
    M16 = rng.integers(0, 1 << 16, size=(m, lda, 4), dtype=np.uint16)
    Mred = (M16[:, :k].astype(np.uint32) % p).astype(np.uint32)
    ref = oracle.syrk_q(Mred, p)
    dM16 = torch.from_numpy(M16.reshape(m, lda * 4).view(np.int16)).cuda()
    dM32 = torch.from_numpy(np.ascontiguousarray(Mred).reshape(m, k * 4).view(np.int32)).cuda()
    lo = np.tril(np.ones((m, m), dtype=bool))
    for dM, ld in ((dM16, lda), (dM32, k)):
        for out16 in (False, True):
            C = torch.zeros((m, m * 4), dtype=torch.int16 if out16 else torch.int32, device="cuda")
            flags = (adj.ADJ_IN_U16 if dM.element_size() == 2 else 0) | (adj.ADJ_OUT_U16 if out16 else 0)
            adj.adjprod_modp_ex(m, k, p, adj.ADJ_PHI_Q, dM, ld, C, m, depth=depth, flags=flags)
            torch.cuda.synchronize()
            got = C.cpu().numpy().view(np.uint16 if out16 else np.uint32).astype(np.uint32).reshape(m, m, 4)
            assert np.array_equal(got[lo], ref[lo]), (p, depth, m, k, dM.element_size(), out16)


# ---------------------------------------------------------------- multi-GPU building blocks, round 2
@pytest.mark.parametrize("p", [8191, 65521])
@pytest.mark.parametrize("depth,m,k", [(1, 3000, 700), (0, 4100, 300), (1, 1030, 520)])
@pytest.mark.parametrize("nranks", [3, 8])
def test_shard_rank_local_preadd_with_garbage_workspace(adj, p, depth, m, k, nranks):
    """Each rank's share pre-adds only the rows of the tile bands its tiles read (adj_shard_rows);
    with a caller workspace filled with garbage before every rank's call, no rank may read a row
    it did not write: all shares into one C give Low(C) bit-exactly, Up(C) untouched."""
    import torch
    A = uniform_matrix(m, k, seed=m + nranks + depth, p=p)
    dA = to_dev(A)
    ws_bytes = adj.adjprod_modp_workspace_size(m, k, p, 0, depth)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
    C = torch.full((m, m), -1, dtype=torch.int32, device="cuda")
    for r in range(nranks):
        ws.fill_(0x5A + 13 * r)
        adj.adjprod_modp_shard(m, k, p, 0, dA, k, C, m, r, nranks, depth=depth, workspace=ws, workspace_bytes=ws_bytes)
    got = to_host(C)
    lo = np.tril(np.ones((m, m), dtype=bool))
    assert np.array_equal(got[lo], oracle.syrk_t(A, p)[lo])
    assert (got[~lo] == 0xFFFFFFFF).all()


@pytest.mark.parametrize("phi", ["T", "H", "Q"])
@pytest.mark.parametrize("in16", [False, True])
@pytest.mark.parametrize("G", [2, 3, 8])
def test_dist_partial_pointer_per_rank(adj, phi, in16, G):
    """adjprod_modp_dist_partial -- the per-rank computation of the split-K path, with the exact
    k-slice pointer adjprod_modp_dist builds (k0 x adj_elem_bytes(phi, flags) bytes into each
    row) -- for phi = T / H / Q and uint16 / uint32 input: the ranks' partials summed mod p give
    the oracle's Low(C)."""
    import torch
    from inputs import uniform_matrix_quat
    p, m, k = 8191, 130, 333
    w = {"T": 1, "H": 2, "Q": 4}[phi]
    gen = {"T": uniform_matrix, "H": uniform_matrix_ext, "Q": uniform_matrix_quat}[phi]
    ref = {"T": oracle.syrk_t, "H": oracle.syrk_h, "Q": oracle.syrk_q}[phi]
    A = gen(m, k, G + 5, p)
    want = ref(A, p).reshape(m, m, w).astype(np.int64)
    code = {"T": adj.ADJ_PHI_T, "H": adj.ADJ_PHI_H, "Q": adj.ADJ_PHI_Q}[phi]
    flags = adj.ADJ_IN_U16 if in16 else 0
    assert adj.adj_elem_bytes(code, flags) == (2 if in16 else 4) * w
    dA = torch.from_numpy(A.reshape(m, k * w).astype(np.uint16).view(np.int16)).cuda() if in16 else to_dev(A.reshape(m, k * w))
    acc = np.zeros((m, m, w), dtype=np.int64)
    for r in range(G):
        R = torch.full((m, m * w), -1, dtype=torch.int32, device="cuda")
        adj.adjprod_modp_dist_partial(m, k, p, code, dA, k, R, m, r, G, flags=flags)
        part = to_host(R).reshape(m, m, w)
        acc += np.where(np.tril(np.ones((m, m), dtype=bool))[:, :, None], part, 0)
        assert (part[~np.tril(np.ones((m, m), dtype=bool))] == 0xFFFFFFFF).all()
    lo = np.tril(np.ones((m, m), dtype=bool))
    assert np.array_equal((acc % p)[lo], want[lo])
