"""Full-size parity at every BASELINE config, in the launch configuration bench.py times
(same depth choice, same seeded device-generated inputs): sampled rows against the O1 oracle
(bit-exact), Vandermonde closed forms on sampled rows, and a Freivalds check of the whole
lower triangle (C r = A (A^T r) mod p, exact in float64 here)."""
import numpy as np
import pytest

import oracle
from oracle import closed_forms as cf
from inputs import vandermonde_points, vandermonde_matrix
from gpu_util import freivalds as _freivalds

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch
    assert torch.cuda.is_available()
    import paper_2101_01025_b200 as adj
    import bench
    return torch, adj, bench


def _run(env, cfg, A_dev, io16=None):
    """The bench's launch: its depth, and (io16=None) its residue storage -- uint16 A and Low(C)
    (ADJ_IN_U16 | ADJ_OUT_U16) for phi = T, p < 2^16, else uint32.  Returns Low(C) as uint32."""
    torch, adj, bench = env
    m, k, p = cfg["m"], cfg["k"], cfg["p"]
    phi = adj.ADJ_PHI_H if cfg["phi"] == "H" else adj.ADJ_PHI_T
    depth = cfg["depth"] if cfg["depth"] is not None else adj.adjprod_modp_auto_depth(m, k, p, phi)
    w = 2 if phi else 1
    if io16 is None:
        io16 = cfg["phi"] in ("T", "H") and p < 65536
    if io16:
        A16 = A_dev.to(torch.int16)
        C = torch.zeros((m, m * w), dtype=torch.int16, device="cuda")
        adj.adjprod_modp_ex(m, k, p, phi, A16, k, C, m, depth=depth, flags=adj.ADJ_IN_U16 | adj.ADJ_OUT_U16)
        del A16
        torch.cuda.synchronize()
        return C.to(torch.int32) & 0xFFFF, depth
    C = torch.zeros((m, m * w), dtype=torch.int32, device="cuda")
    adj.adjprod_modp_ex(m, k, p, phi, A_dev, k, C, m, depth=depth)
    torch.cuda.synchronize()
    return C, depth


@pytest.mark.parametrize("name,io16", [("c1", None), ("c2", None), ("c2", False), ("c5", None), ("c4", None),
                                       ("c3", None)])
def test_config_sampled_rows_and_freivalds(env, name, io16):
    torch, adj, bench = env
    from inputs.gpu import uniform_residues_cuda
    cfg = bench.CONFIGS[name]
    m, k, p = cfg["m"], cfg["k"], cfg["p"]
    w = 2 if cfg["phi"] == "H" else 1
    A = torch.empty((m, k * w), dtype=torch.int32, device="cuda")
    uniform_residues_cuda(A, seed=1, p=p)
    C, depth = _run(env, cfg, A, io16)
    Ah = A.cpu().numpy().view(np.uint32).reshape((m, k, 2) if w == 2 else (m, k))
    Ch = C.cpu().numpy().view(np.uint32).reshape((m, m, 2) if w == 2 else (m, m))
    del C
    rng = np.random.default_rng(7)
    rows = sorted({0, 1, m // 2, m - 2, m - 1} | set(int(x) for x in rng.integers(0, m, 3)))
    f = oracle.syrk_h if w == 2 else oracle.syrk_t
    for r in rows:
        ref = f(Ah, p, rows=(r, r + 1))
        assert np.array_equal(Ch[r, : r + 1], ref[r, : r + 1]), (name, depth, r)
    if w == 1 and m * k <= 8192 * 8192:
        assert _freivalds(Ah, Ch, p), (name, depth)


@pytest.mark.parametrize("name", ["c2", "c3"])
def test_config_vandermonde_closed_form(env, name):
    """A[i][t] = x_i^t: every entry of Low(C) is a geometric sum; check 64 random full rows."""
    torch, adj, bench = env
    cfg = dict(bench.CONFIGS[name])
    m, k, p = cfg["m"], cfg["k"], cfg["p"]
    if name == "c3":                     # keep host generation bounded: 32768 x 8192 slice of k
        k = cfg["k"] = 8192
    x = vandermonde_points(m, 3, p)
    Ah = vandermonde_matrix(x, k, p)
    A = torch.from_numpy(Ah.view(np.int32)).cuda()
    C, depth = _run(env, cfg, A)
    Ch = C.cpu().numpy().view(np.uint32)
    rng = np.random.default_rng(1)
    rows = sorted(set(int(r) for r in rng.integers(0, m, 64)) | {m - 1})
    ref = cf.vandermonde_syrk_entries(x, rows, k, p)
    for r, rr in zip(rows, ref):
        assert np.array_equal(Ch[r, : r + 1].astype(np.int64), rr), (name, depth, r)


def test_c5_vandermonde_hermitian(env):
    torch, adj, bench = env
    cfg = bench.CONFIGS["c5"]
    m, k, p = cfg["m"], 2048, cfg["p"]
    rng = np.random.default_rng(5)
    z = rng.integers(1, p, size=(m, 2))
    Ah = vandermonde_matrix(z, k, p)
    A = torch.from_numpy(Ah.reshape(m, 2 * k).view(np.int32)).cuda()
    cfg2 = dict(cfg, k=k)
    C, depth = _run(env, cfg2, A)
    Ch = C.cpu().numpy().view(np.uint32).reshape(m, m, 2)
    rows = sorted(set(int(r) for r in rng.integers(0, m, 32)) | {m - 1})
    ref = cf.vandermonde_herk_entries(z, rows, k, p)
    for r, (re, im) in zip(rows, ref):
        assert np.array_equal(Ch[r, : r + 1, 0].astype(np.int64), re) and \
            np.array_equal(Ch[r, : r + 1, 1].astype(np.int64), im), r


@pytest.mark.parametrize("io16", [True, False])
def test_q5_quaternion_sampled_rows(env, io16):
    """SURVEY §8(f)-4 at the bench's q5 size (8192^2 over H_GF(8191), Alg. 2M3M), in the bench's
    uint16 storage and in uint32."""
    torch, adj, bench = env
    from inputs.gpu import uniform_residues_cuda
    cfg = bench.CONFIGS["q5"]
    m, k, p = cfg["m"], cfg["k"], cfg["p"]
    A = torch.empty((m, k * 4), dtype=torch.int32, device="cuda")
    uniform_residues_cuda(A, seed=1, p=p)
    if io16:
        C16 = torch.zeros((m, m * 4), dtype=torch.int16, device="cuda")
        adj.adjprod_modp_ex(m, k, p, adj.ADJ_PHI_Q, A.to(torch.int16), k, C16, m,
                            flags=adj.ADJ_IN_U16 | adj.ADJ_OUT_U16)
        C = C16.to(torch.int32) & 0xFFFF
        del C16
    else:
        C = torch.zeros((m, m * 4), dtype=torch.int32, device="cuda")
        adj.adjprod_modp_ex(m, k, p, adj.ADJ_PHI_Q, A, k, C, m)
    torch.cuda.synchronize()
    Ah = A.cpu().numpy().view(np.uint32).reshape(m, k, 4)
    Ch = C.cpu().numpy().view(np.uint32).reshape(m, m, 4)
    for r in (0, 4097, m - 1):
        ref = oracle.syrk_q(Ah, p, rows=(r, r + 1))
        assert np.array_equal(Ch[r, : r + 1], ref[r, : r + 1]), r


def test_c5_herk_alg1_sampled_rows(env):
    """SURVEY §8(f)-2 at c5 size: one level of Alg. 1 over GF(8191^2) (ADJ_HERK_ALG1)."""
    torch, adj, bench = env
    from inputs.gpu import uniform_residues_cuda
    cfg = bench.CONFIGS["c5"]
    m, k, p = cfg["m"], cfg["k"], cfg["p"]
    A = torch.empty((m, k * 2), dtype=torch.int32, device="cuda")
    uniform_residues_cuda(A, seed=1, p=p)
    C = torch.zeros((m, m * 2), dtype=torch.int32, device="cuda")
    adj.adjprod_modp_ex(m, k, p, adj.ADJ_PHI_H, A, k, C, m, flags=adj.ADJ_HERK_ALG1)
    torch.cuda.synchronize()
    Ah = A.cpu().numpy().view(np.uint32).reshape(m, k, 2)
    Ch = C.cpu().numpy().view(np.uint32).reshape(m, m, 2)
    for r in (0, 1, 4095, 4096, m - 1):
        ref = oracle.syrk_h(Ah, p, rows=(r, r + 1))
        assert np.array_equal(Ch[r, : r + 1], ref[r, : r + 1]), r


@pytest.mark.parametrize("depth", [0, 1])
def test_c2_output_tile_shards(env, depth):
    """SURVEY §8(e)-2 at c2 size: the 8 ranks' shares run one after the other into one C give
    Low(C) (sampled rows + Freivalds over the whole lower triangle)."""
    torch, adj, bench = env
    from inputs.gpu import uniform_residues_cuda
    cfg = bench.CONFIGS["c2"]
    m, k, p = cfg["m"], cfg["k"], cfg["p"]
    A = torch.empty((m, k), dtype=torch.int32, device="cuda")
    uniform_residues_cuda(A, seed=1, p=p)
    C = torch.zeros((m, m), dtype=torch.int32, device="cuda")
    for r in range(8):
        adj.adjprod_modp_shard(m, k, p, 0, A, k, C, m, r, 8, depth=depth)
    torch.cuda.synchronize()
    Ah = A.cpu().numpy().view(np.uint32)
    Ch = C.cpu().numpy().view(np.uint32)
    for r in (0, 300, 4095, 4096, m - 1):
        ref = oracle.syrk_t(Ah, p, rows=(r, r + 1))
        assert np.array_equal(Ch[r, : r + 1], ref[r, : r + 1]), r
    assert _freivalds(Ah, Ch, p)


@pytest.mark.parametrize("m,k,p,depth", [(5001, 4099, 8191, 2), (3001, 70001, 65521, -1), (2999, 3001, 131071, 1),
                                         (4097, 257, 97, 3)])
def test_ragged_medium_sampled_rows(env, m, k, p, depth):
    """Ragged shapes well past one tile wave at several depths, including a k past the int32
    accumulation bound of the 65521 scheme (K segments) and the wide scheme: sampled rows plus
    Freivalds over the whole lower triangle."""
    torch, adj, bench = env
    from inputs.gpu import uniform_residues_cuda
    A = torch.empty((m, k), dtype=torch.int32, device="cuda")
    uniform_residues_cuda(A, seed=m + k, p=p)
    C = torch.zeros((m, m), dtype=torch.int32, device="cuda")
    adj.adjprod_modp_ex(m, k, p, 0, A, k, C, m, depth=depth)
    torch.cuda.synchronize()
    Ah = A.cpu().numpy().view(np.uint32)
    Ch = C.cpu().numpy().view(np.uint32)
    for r in sorted({0, 1, m // 3, m // 2, m // 2 + 1, m - 2, m - 1}):
        ref = oracle.syrk_t(Ah, p, rows=(r, r + 1))
        assert np.array_equal(Ch[r, : r + 1], ref[r, : r + 1]), (m, k, p, depth, r)
    assert _freivalds(Ah, Ch, p)
