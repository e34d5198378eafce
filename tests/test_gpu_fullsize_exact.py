"""Whole-output parity at the BASELINE configs, in the launch configuration bench.py times
(same depth choice, same residue storage, same seeded device-generated inputs).

Every entry of Low(C) is checked, two independent ways:

1. Freivalds over the whole lower triangle on the host, in the field's own arithmetic
   (GF(p), GF(p)[i]/(i^2+1), the quaternions over GF(p)): C r = A (phi(A) r) mod p for two seeded
   vectors r, computed in float64, which is exact because every partial sum stays below 2^53
   (m (p-1)^2 < 2^47 at c3).  Lemma lem:transp defines C; C's strict upper
   triangle is completed as phi(Low(C)) by Lemma lem:uplow.  A wrong entry
   survives one vector with probability <= 1/p.
2. Entry by entry against the plain definition evaluated as a float64 product on the GPU (the
   library special case of SURVEY.md §8(c)-6: "dsyrk + mod p"), exact since
   k (p-1)^2 < 2^53 at every config (c3: 1.4e14, c4: 8.8e12), reduced mod p and compared with
   every lower-triangle entry.  The float64 product is cuBLAS, not this repo's kernels.

Plus BASELINE configs[1]'s "full symmetric check": c2 with ADJ_FILL_UPPER gives C = C^T.
"""
import numpy as np
import pytest

from fullsize_check import exact_low_mismatches, freivalds_low

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch
    assert torch.cuda.is_available()
    import paper_2101_01025_b200 as adj
    import bench
    return torch, adj, bench


def _bench_run(env, name, depth=None, seed=1):
    """The bench's launch for config `name`: its depth and residue storage (uint16 A and Low(C)
    with ADJ_IN_U16 | ADJ_OUT_U16 when p < 2^16).  Returns (A residues int32 on the device,
    Low(C) as int32 on the device (m x m x w), depth)."""
    torch, adj, bench = env
    from inputs.gpu import uniform_residues_cuda
    cfg = bench.CONFIGS[name]
    m, k, p = cfg["m"], cfg["k"], cfg["p"]
    phi = {"T": adj.ADJ_PHI_T, "H": adj.ADJ_PHI_H, "Q": adj.ADJ_PHI_Q}[cfg["phi"]]
    w = {"T": 1, "H": 2, "Q": 4}[cfg["phi"]]
    if depth is None:
        depth = cfg["depth"] if cfg["depth"] is not None else adj.adjprod_modp_auto_depth(m, k, p, phi)
    A = torch.empty((m, k * w), dtype=torch.int32, device="cuda")
    uniform_residues_cuda(A, seed=seed, p=p)
    assert p < 65536
    A16 = A.to(torch.int16)
    C16 = torch.zeros((m, m * w), dtype=torch.int16, device="cuda")
    ws = adj.adjprod_modp_workspace_size(m, k, p, phi, depth, adj.ADJ_IN_U16 | adj.ADJ_OUT_U16)
    W = torch.empty(max(ws, 1), dtype=torch.uint8, device="cuda")
    adj.adjprod_modp_ex(m, k, p, phi, A16, k, C16, m, depth=depth, flags=adj.ADJ_IN_U16 | adj.ADJ_OUT_U16,
                        workspace=W, workspace_bytes=ws)
    torch.cuda.synchronize()
    del A16, W
    C = (C16.to(torch.int32) & 0xFFFF).view(m, m, w)
    del C16
    return A.view(m, k, w), C, depth


@pytest.mark.parametrize("name", ["c2", "c2@1", "c3", "c4", "c5", "q5"])
def test_whole_low_c_bench_launch(env, name):
    """Every entry of Low(C) at the config, in the bench's launch configuration (depth, uint16
    residues), against the float64 product on the GPU and by Freivalds on the host.  c2@1: c2
    through one level of Alg. 1 (the bench's depth1_alg1 comparator; its automatic depth is 0)."""
    torch, adj, bench = env
    name, _, d = name.partition("@")
    cfg = bench.CONFIGS[name]
    p = cfg["p"]
    A, C, depth = _bench_run(env, name, int(d) if d else None)
    w = A.shape[2]
    if name == "c3":
        assert depth == 2          # the depth-2 tree the N = 1 headline times
    if name in ("c3", "c4"):       # ... on the wide-N leaf (256 x 512 tiles, Horner in TMEM)
        assert adj.adjprod_modp_leaf_tile(A.shape[0], A.shape[1], p, 0, depth,
                                          adj.ADJ_IN_U16 | adj.ADJ_OUT_U16) == 512
    assert exact_low_mismatches(torch, A, C, p, w) == 0, (name, depth)
    Ah = A.cpu().numpy().view(np.uint32)
    Ch = C.cpu().numpy().view(np.uint32)
    del A, C
    torch.cuda.empty_cache()
    assert freivalds_low(Ah, Ch, p, w), (name, depth)


@pytest.mark.parametrize("seed", [2, 3])
@pytest.mark.parametrize("name", ["c2", "c3", "c4", "c5", "q5"])
def test_whole_low_c_other_seeds(env, name, seed):
    """parity on seeds {1, 2, 3}.  Seeds 2 and 3 at every BASELINE config in the
    bench's launch configuration: every entry of Low(C) against the float64 product on the GPU
    (the Freivalds pass runs on seed 1 above)."""
    torch, adj, bench = env
    A, C, depth = _bench_run(env, name, None, seed)
    assert exact_low_mismatches(torch, A, C, bench.CONFIGS[name]["p"], A.shape[2]) == 0, (name, seed, depth)
    del A, C
    torch.cuda.empty_cache()


def test_c2_fill_upper_full_symmetric(env):
    """BASELINE configs[1]: lower triangle + full symmetric check.  ADJ_FILL_UPPER writes
    Up(C) = Low(C)^T (Lemma lem:uplow), so C == C^T over the whole 8192^2 matrix, and every
    entry equals the float64 product mod p."""
    torch, adj, bench = env
    from inputs.gpu import uniform_residues_cuda
    cfg = bench.CONFIGS["c2"]
    m, k, p = cfg["m"], cfg["k"], cfg["p"]
    A = torch.empty((m, k), dtype=torch.int32, device="cuda")
    uniform_residues_cuda(A, seed=1, p=p)
    C = torch.full((m, m), -1, dtype=torch.int32, device="cuda")
    adj.adjprod_modp_ex(m, k, p, adj.ADJ_PHI_T, A, k, C, m, depth=1, flags=adj.ADJ_FILL_UPPER)   # through Alg. 1
    torch.cuda.synchronize()
    assert torch.equal(C, C.T)
    Af = A.to(torch.float64)
    for r0 in range(0, m, 2048):
        ref = torch.remainder(Af[r0:r0 + 2048] @ Af.T, p).to(torch.int32)
        assert torch.equal(ref, C[r0:r0 + 2048]), r0
