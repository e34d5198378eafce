"""The building blocks of ADJ_DIST_TILES | ADJ_DIST_P2P (output-tile sharding with the gather
fused into the final kernel) on one GPU: the root exports its C (a torch
allocation, at an offset inside it) with adj_ipc_export, other processes map it with
adj_ipc_open and run their share (adjprod_modp_shard) with the mapped pointer as the output, so
their final kernel -- the leaf epilogue at depth 0, K4 at depth 1 -- stores the owned regions
straight into the root's C.  The root's Low(C) must then equal the oracle bit-exactly and its
strict upper triangle (and the bytes around C) must be untouched.  Here every process uses
device 0 (CUDA IPC between processes on one device); on a multi-GPU node the same calls map the
root's C over NVLink (tests/test_gpu_multi.py drives the collective)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _peer(rank, nranks, case, rec, q_done):
    import torch
    torch.cuda.set_device(0)
    import paper_2101_01025_b200 as adj
    from inputs import uniform_matrix
    m, k, p, depth, in16, ldc = case
    A = uniform_matrix(m, k, 31, p)
    dA = torch.from_numpy(A.astype(np.uint16).view(np.int16) if in16 else A.view(np.int32)).cuda()
    ptr = adj.adj_ipc_open(rec)
    try:
        adj.adjprod_modp_shard(m, k, p, adj.ADJ_PHI_T, dA, k, ptr, ldc, rank, nranks, depth=depth,
                               flags=adj.ADJ_IN_U16 if in16 else 0)
        torch.cuda.synchronize()
    finally:
        adj.adj_ipc_close(ptr)
    q_done.put(rank)


@pytest.mark.parametrize("case,nranks", [((1030, 700, 8191, 1, False, 1030), 2),
                                         ((1030, 700, 8191, 0, True, 1040), 3),
                                         ((777, 520, 65521, 1, True, 800), 3),
                                         ((600, 333, 131071, 1, False, 600), 2)])
def test_shard_stores_into_a_peer_mapped_c(case, nranks):
    import torch
    import torch.multiprocessing as mp
    import oracle
    import paper_2101_01025_b200 as adj
    from inputs import uniform_matrix
    m, k, p, depth, in16, ldc = case
    A = uniform_matrix(m, k, 31, p)
    off = 4099                                       # C starts inside the allocation, unaligned to it
    big = torch.full((off + m * ldc + 64,), -1, dtype=torch.int32, device="cuda")
    C = big[off:off + m * ldc]
    torch.cuda.synchronize()
    rec = adj.adj_ipc_export(C)
    assert int.from_bytes(rec[64:72], "little") % 4 == 0 and len(rec) == 72
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_peer, args=(r, nranks, case, rec, q)) for r in range(1, nranks)]
    for pr in procs:
        pr.start()
    dA = torch.from_numpy(A.astype(np.uint16).view(np.int16) if in16 else A.view(np.int32)).cuda()
    adj.adjprod_modp_shard(m, k, p, adj.ADJ_PHI_T, dA, k, C, ldc, 0, nranks, depth=depth,
                           flags=adj.ADJ_IN_U16 if in16 else 0)
    done = sorted(q.get(timeout=300) for _ in procs)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert done == list(range(1, nranks))
    torch.cuda.synchronize()
    allv = big.cpu().numpy().view(np.uint32)
    got = allv[off:off + m * ldc].reshape(m, ldc)
    ref = oracle.syrk_t(A, p)
    lo = np.tril(np.ones((m, m), dtype=bool))
    assert np.array_equal(got[:, :m][lo], ref[lo])
    assert (got[:, :m][~lo] == 0xFFFFFFFF).all()                     # Up(C) untouched
    assert (got[:, m:] == 0xFFFFFFFF).all()                          # padding columns untouched
    assert (allv[:off] == 0xFFFFFFFF).all() and (allv[off + m * ldc:] == 0xFFFFFFFF).all()


def test_ipc_export_offsets():
    """The record names the allocation's base and the byte offset of the pointer inside it."""
    import torch
    import paper_2101_01025_b200 as adj
    big = torch.empty(1 << 20, dtype=torch.int32, device="cuda")
    r0 = adj.adj_ipc_export(big)
    for off in (1, 777, 4096):
        r = adj.adj_ipc_export(big[off:])
        assert r[:64] == r0[:64]
        assert int.from_bytes(r[64:], "little") - int.from_bytes(r0[64:], "little") == 4 * off
