"""adjprod_modp_dist with N > 1 ranks, one process per GPU over NCCL: every mode
(split-K with the packed uint32 reduce, output-tile sharding with the rank-local pre-addition and
the gather of result tiles, split-K with peer stores into the root's window, output-tile sharding with peer stores into the
root's C) against the oracle,
bit-exactly, on the root.  Needs N devices: skipped when fewer are visible (the round's GPU box
has one; the driver's 8-GPU step runs it)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _ndev():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, cases, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import paper_2101_01025_b200 as adj
    from inputs import uniform_matrix, uniform_matrix_ext, uniform_matrix_quat
    uid = [adj.adj_comm_get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = adj.adj_comm_init(world, uid[0], rank)
    try:
        for (m, k, p, phi, mode, depth, in16) in cases:
            w = {"T": 1, "H": 2, "Q": 4}[phi]
            gen = {"T": uniform_matrix, "H": uniform_matrix_ext, "Q": uniform_matrix_quat}[phi]
            A = gen(m, k, 17, p).reshape(m, k * w)
            code = {"T": adj.ADJ_PHI_T, "H": adj.ADJ_PHI_H, "Q": adj.ADJ_PHI_Q}[phi]
            flags = {"splitk": 0, "tiles": adj.ADJ_DIST_TILES, "p2p": adj.ADJ_DIST_P2P,
                     "tiles-p2p": adj.ADJ_DIST_TILES | adj.ADJ_DIST_P2P}[mode]
            if in16:
                flags |= adj.ADJ_IN_U16
                dA = torch.from_numpy(A.astype(np.uint16).view(np.int16)).cuda()
            else:
                dA = torch.from_numpy(A.view(np.int32)).cuda()
            C = torch.full((m, m * w), -1, dtype=torch.int32, device="cuda")
            adj.adjprod_modp_dist(m, k, p, code, dA, k, C, m, 0, comm, depth=depth, flags=flags)
            torch.cuda.synchronize()
            if rank == 0:
                got = C.cpu().numpy().view(np.uint32).reshape(m, m, w)
                ref = {"T": oracle.syrk_t, "H": oracle.syrk_h, "Q": oracle.syrk_q}[phi](
                    A.reshape(m, k, w) if w > 1 else A, p).reshape(m, m, w)
                lo = np.tril(np.ones((m, m), dtype=bool))
                ok = np.array_equal(got[lo], ref[lo]) and bool((got[~lo] == 0xFFFFFFFF).all())
                q.put(((m, k, p, phi, mode, depth, in16), ok))
            dist.barrier()
    finally:
        adj.adj_comm_destroy(comm)
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_dist_all_modes_n_ranks(world):
    if _ndev() < world:
        pytest.skip(f"needs {world} GPUs ({_ndev()} visible)")
    import torch.multiprocessing as mp
    cases = [(1030, 700, 8191, "T", "splitk", -1, False), (1030, 700, 8191, "T", "tiles", 1, False),
             (1030, 700, 8191, "T", "tiles", 0, True), (1030, 700, 8191, "T", "p2p", -1, True),
             (600, 900, 65521, "T", "splitk", 2, True), (300, 257, 8191, "H", "splitk", 1, False),
             (200, 130, 8191, "Q", "splitk", 0, True), (700, 500, 131071, "T", "tiles", 1, False),
             (1030, 700, 8191, "T", "tiles-p2p", 1, False), (1030, 700, 8191, "T", "tiles-p2p", 0, True),
             (777, 520, 65521, "T", "tiles-p2p", 1, True), (600, 333, 131071, "T", "tiles-p2p", 1, False)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cases, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=600) for _ in cases]
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    assert all(ok for _, ok in res), res
