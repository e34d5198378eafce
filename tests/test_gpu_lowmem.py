"""GPU parity of the low-memory temporary schedule (ADJ_LOW_MEM; the GPU
counterpart of the in-place schedules of Table tab:schedule:AAT): the root
level's P1, P3, P5 formed in C's own blocks, the root arena reused by the children, K4 in
place.  Compared with the oracle element by element, bit-exact, and with Up(C) untouched."""
import numpy as np
import pytest

import oracle
from inputs import uniform_matrix
from gpu_util import to_dev, to_host

pytestmark = pytest.mark.gpu

SENT = 0xFFFFFFFF


@pytest.fixture(scope="module")
def adj():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    import paper_2101_01025_b200 as adj
    adj.lib()
    return adj


def _run(adj, A, p, depth, ldc_extra=0, io16=False):
    import torch
    m, k = A.shape
    ldc = m + ldc_extra
    dt = torch.int16 if io16 else torch.int32
    Cbuf = torch.full((m, ldc), -1, dtype=dt, device="cuda")
    Ad = to_dev(A)
    if io16:
        Ad = Ad.to(torch.int16)
    flags = adj.ADJ_LOW_MEM | ((adj.ADJ_IN_U16 | adj.ADJ_OUT_U16) if io16 else 0)
    adj.adjprod_modp_ex(m, k, p, 0, Ad, k, Cbuf, ldc, depth=depth, flags=flags)
    torch.cuda.synchronize()
    got = Cbuf.cpu().numpy()
    got = (got.view(np.uint16).astype(np.uint32) if io16 else got.view(np.uint32))[:, :m]
    sent = 0xFFFF if io16 else SENT
    return got, sent


@pytest.mark.parametrize("p", [97, 8191, 65521, 131071])
@pytest.mark.parametrize("depth", [1, 2, 3])
@pytest.mark.parametrize("m,k", [(128, 200), (512, 700), (1088, 1001)])
def test_lowmem_vs_oracle(adj, p, depth, m, k):
    A = uniform_matrix(m, k, seed=13 * m + k + depth, p=p)
    got, sent = _run(adj, A, p, depth)
    ref = oracle.syrk_t(A, p)
    lo = np.tril(np.ones((m, m), dtype=bool))
    assert np.array_equal(got[lo], ref[lo]), (p, depth, m, k)
    assert np.all(got[~lo] == sent), "Up(C) must stay untouched"


@pytest.mark.parametrize("p", [8191, 65521])
@pytest.mark.parametrize("depth", [1, 2])
def test_lowmem_u16_io_and_strided_c(adj, p, depth):
    m, k = 1024, 1536
    A = uniform_matrix(m, k, seed=5 + depth, p=p)
    ref = oracle.syrk_t(A, p)
    lo = np.tril(np.ones((m, m), dtype=bool))
    for io16, extra in [(True, 0), (True, 8), (False, 8)]:
        got, sent = _run(adj, A, p, depth, ldc_extra=extra, io16=io16)
        assert np.array_equal(got[lo], ref[lo]), (p, depth, io16, extra)
        assert np.all(got[~lo] == sent)


def test_lowmem_same_as_grouped_schedule(adj):
    """Both schedules give the identical Low(C) at a size spanning many 256-tiles."""
    import torch
    m, k, p = 2048, 2048, 65521
    A = to_dev(uniform_matrix(m, k, seed=77, p=p))
    C1 = adj.adjprod(A, p, depth=2)
    C2 = adj.adjprod(A, p, depth=2, low_mem=True)
    torch.cuda.synchronize()
    assert torch.equal(torch.tril(C1), torch.tril(C2))


def test_lowmem_workspace_smaller_and_caller_workspace(adj):
    import torch
    m, k, p = 2048, 3000, 8191
    w_def = adj.adjprod_modp_workspace_size(m, k, p, 0, depth=2)
    w_lm = adj.adjprod_modp_workspace_size(m, k, p, 0, depth=2, flags=adj.ADJ_LOW_MEM)
    assert w_lm < w_def
    A = uniform_matrix(m, k, seed=3, p=p)
    ws = torch.empty(w_lm, dtype=torch.uint8, device="cuda")
    C = torch.zeros((m, m), dtype=torch.int32, device="cuda")
    adj.adjprod_modp_ex(m, k, p, 0, to_dev(A), k, C, m, depth=2, flags=adj.ADJ_LOW_MEM, workspace=ws,
                        workspace_bytes=w_lm)
    got = to_host(C)
    assert np.array_equal(np.tril(got), np.tril(oracle.syrk_t(A, p)))
    with pytest.raises(adj.AdjError):   # one byte short
        adj.adjprod_modp_ex(m, k, p, 0, to_dev(A), k, C, m, depth=2, flags=adj.ADJ_LOW_MEM, workspace=ws,
                            workspace_bytes=w_lm - 1)


def test_lowmem_misaligned_c_rejected(adj):
    import torch
    m, k, p = 256, 300, 97
    A = to_dev(uniform_matrix(m, k, seed=1, p=p))
    C = torch.zeros((m, m + 4), dtype=torch.int32, device="cuda")
    with pytest.raises(adj.AdjError):
        adj.adjprod_modp_ex(m, k, p, 0, A, k, C, m + 4, depth=1, flags=adj.ADJ_LOW_MEM)


def test_lowmem_ignored_where_it_does_not_apply(adj):
    """m % 64 != 0, depth 0 or the SYRK form: the flag is ignored and the result is the same."""
    import torch
    p = 8191
    for m, k, depth in [(200, 300, 1), (256, 300, 0)]:
        A = uniform_matrix(m, k, seed=m, p=p)
        got = to_host(adj.adjprod(to_dev(A), p, depth=depth, low_mem=True))
        assert np.array_equal(np.tril(got), np.tril(oracle.syrk_t(A, p)))
        assert adj.adjprod_modp_workspace_size(m, k, p, 0, depth=depth, flags=adj.ADJ_LOW_MEM) == \
            adj.adjprod_modp_workspace_size(m, k, p, 0, depth=depth)
    m, k = 256, 300
    A = uniform_matrix(m, k, seed=9, p=p)
    C0 = uniform_matrix(m, m, seed=10, p=p)
    C = to_dev(C0)
    adj.adjprod_modp_syrk(m, k, p, 0, 3, to_dev(A), k, 5, C, m, depth=1, flags=adj.ADJ_LOW_MEM)
    ref = oracle.syrk_update(A, C0, p, 3, 5)
    assert np.array_equal(np.tril(to_host(C)), np.tril(ref))


def test_small_caller_workspace_falls_back_to_lowmem(adj):
    """Without ADJ_LOW_MEM, a caller workspace below the grouped schedule's size but at least the
    low-memory size runs the low-memory schedule (same Low(C)); below that it is refused."""
    import torch
    m, k, p = 1024, 1200, 65521
    w_def = adj.adjprod_modp_workspace_size(m, k, p, 0, depth=2)
    w_lm = adj.adjprod_modp_workspace_size(m, k, p, 0, depth=2, flags=adj.ADJ_LOW_MEM)
    assert w_lm < w_def
    A = uniform_matrix(m, k, seed=21, p=p)
    ws = torch.empty(w_lm, dtype=torch.uint8, device="cuda")
    C = torch.zeros((m, m), dtype=torch.int32, device="cuda")
    adj.adjprod_modp_ex(m, k, p, 0, to_dev(A), k, C, m, depth=2, workspace=ws, workspace_bytes=w_lm)
    assert np.array_equal(np.tril(to_host(C)), np.tril(oracle.syrk_t(A, p)))
    with pytest.raises(adj.AdjError):
        adj.adjprod_modp_ex(m, k, p, 0, to_dev(A), k, C, m, depth=2, workspace=ws, workspace_bytes=w_lm - 256)


@pytest.mark.parametrize("low_mem", [False, True])
def test_graph_capture_fused_k1_and_lowmem(adj, low_mem):
    """The fused K1 (uint16, m, k multiples of 512, depth 2) and the low-memory schedule (its
    child calls and in-place K4) are fixed stream-ordered launch sequences: captured into a CUDA
    graph and replayed, they reproduce the oracle's Low(C)."""
    import torch
    p, m, k, depth = 65521, 1024, 1536, 2
    A = uniform_matrix(m, k, seed=31, p=p)
    dA = to_dev(A).to(torch.int16)
    flags = adj.ADJ_IN_U16 | adj.ADJ_OUT_U16 | (adj.ADJ_LOW_MEM if low_mem else 0)
    ws_bytes = adj.adjprod_modp_workspace_size(m, k, p, 0, depth, flags=flags)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
    C = torch.zeros((m, m), dtype=torch.int16, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        adj.adjprod_modp_ex(m, k, p, 0, dA, k, C, m, depth=depth, flags=flags, workspace=ws, workspace_bytes=ws_bytes,
                            stream=s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        adj.adjprod_modp_ex(m, k, p, 0, dA, k, C, m, depth=depth, flags=flags, workspace=ws, workspace_bytes=ws_bytes,
                            stream=s)
    ref = np.tril(oracle.syrk_t(A, p))
    for _ in range(2):
        C.zero_()
        g.replay()
        torch.cuda.synchronize()
        got = C.cpu().numpy().view(np.uint16).astype(np.uint32)
        assert np.array_equal(np.tril(got), ref)


def test_lowmem_fill_upper(adj):
    """ADJ_LOW_MEM with ADJ_FILL_UPPER: Up(C) = Low(C)^T is written after the in-place K4."""
    import torch
    m, k, p = 1024, 700, 8191
    A = uniform_matrix(m, k, seed=41, p=p)
    C = torch.full((m, m), -1, dtype=torch.int32, device="cuda")
    adj.adjprod_modp_ex(m, k, p, 0, to_dev(A), k, C, m, depth=2, flags=adj.ADJ_LOW_MEM | adj.ADJ_FILL_UPPER)
    got = to_host(C)
    ref = oracle.syrk_t(A, p)
    lo = np.tril(np.ones((m, m), dtype=bool))
    assert np.array_equal(got[lo], ref[lo])
    assert np.array_equal(got, got.T)
