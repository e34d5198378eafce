"""Multi-rank host logic of the split-K path (adjprod_modp_dist) on CPU:
world_size-2 gloo process groups.  Each rank takes the column slice the C ABI assigns it
(adj_dist_kslice), computes its residue partial Low(A_r A_r^T) mod p with the oracle, the
partials are summed exactly by a collective reduce and reduced mod p on the root -- the same
arithmetic the NCCL path performs -- and the result must equal the single-process oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, cases, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import paper_2101_01025_b200 as adj
    from inputs import uniform_matrix, uniform_matrix_ext
    try:
        for (m, k, p, phi) in cases:
            k0, k1 = adj.adj_dist_kslice(k, world, rank)
            if phi == "T":
                A = uniform_matrix(m, k, seed=11, p=p)
                part = oracle.syrk_t(np.ascontiguousarray(A[:, k0:k1]), p)
            else:
                A = uniform_matrix_ext(m, k, seed=11, p=p)
                part = oracle.syrk_h(np.ascontiguousarray(A[:, k0:k1]), p)
            t = torch.from_numpy(part.astype(np.int64))
            # residues summed exactly: each entry < world * p < 2^32 (uint32 in the NCCL path)
            dist.reduce(t, dst=0, op=dist.ReduceOp.SUM)
            if rank == 0:
                assert int(t.max()) < world * p < 2**32
                got = (t.numpy() % p).astype(np.uint32)
                ref = oracle.syrk_t(A, p) if phi == "T" else oracle.syrk_h(A, p)
                out_q.put((m, k, p, phi, bool(np.array_equal(got, ref))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 4])
def test_split_k_reduce_gloo(world):
    cases = [(37, 100, 8191, "T"), (64, 7, 65521, "T"), (20, 33, 8191, "H"), (5, 1, 97, "T")]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cases, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    results = [q.get(timeout=5) for _ in cases]
    assert all(ok for *_, ok in results), results


def test_kslice_partition():
    import paper_2101_01025_b200 as adj
    for k in [0, 1, 7, 8, 9, 100, 8192, 131072, 131071]:
        for G in [1, 2, 3, 4, 8]:
            sl = [adj.adj_dist_kslice(k, G, r) for r in range(G)]
            cover = []
            for k0, k1 in sl:
                assert 0 <= k0 <= k1 <= k and (k0 % 8 == 0 or k0 == k)
                cover.extend(range(k0, k1))
            assert cover == list(range(k)), (k, G)


def _tiles_worker(rank, world, port, cases, out_q):
    """Output-tile sharding (ADJ_DIST_TILES): every rank computes the regions of Low(C) it owns
    (adj_shard_layout, here with the oracle on the full A), packs them row by row in region order
    -- the layout dist_tiles' pack kernel uses -- and the root receives and unpacks them."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import paper_2101_01025_b200 as adj
    from inputs import uniform_matrix
    try:
        for (m, k, p, depth) in cases:
            A = uniform_matrix(m, k, seed=5, p=p)
            full = oracle.syrk_t(A, p)
            mine = adj.adj_shard_layout(m, k, p, rank, world, depth=depth)
            buf = np.concatenate([full[r0:r0 + rows, c0:c0 + cols].reshape(-1) for (r0, c0, rows, cols, _) in mine]
                                 or [np.zeros(0, dtype=np.uint32)]).astype(np.int64)
            n = torch.tensor([buf.size])
            sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
            dist.all_gather(sizes, n)
            if rank == 0:
                C = np.zeros((m, m), dtype=np.uint32)
                parts = {0: buf}
                for q in range(1, world):
                    t = torch.zeros(int(sizes[q]), dtype=torch.int64)
                    dist.recv(t, src=q)
                    parts[q] = t.numpy()
                for q in range(world):
                    off = 0
                    for (r0, c0, rows, cols, lower) in adj.adj_shard_layout(m, k, p, q, world, depth=depth):
                        blk = parts[q][off:off + rows * cols].reshape(rows, cols)
                        off += rows * cols
                        for i in range(rows):
                            ncol = min(cols, r0 + i - c0 + 1) if lower else cols
                            C[r0 + i, c0:c0 + ncol] = blk[i, :ncol]
                out_q.put((m, k, p, depth, bool(np.array_equal(C, full))))
            else:
                dist.send(torch.from_numpy(buf), dst=0)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 4])
def test_tile_sharding_gather_gloo(world):
    cases = [(300, 40, 8191, 0), (700, 33, 97, 1), (5, 3, 65521, 0), (1030, 16, 8191, 1)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_tiles_worker, args=(r, world, port, cases, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in cases]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert all(ok for (*_, ok) in res), res
