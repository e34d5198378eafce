"""Multi-rank host logic of adjprod_modp_dist on CPU: world_size 2-4 gloo
process groups, every rank using the C ABI's own host functions (libadjprod.so loads without a
GPU): adj_dist_kslice for its column slice, adj_elem_bytes for the byte offset of that slice in
a row of A (the pointer adjprod_modp_dist_partial reads, for phi = T / H / Q and uint16 / uint32
storage), adj_shard_layout / adj_shard_rows for the output-tile shares.  The per-rank arithmetic
is the oracle's; the exchange is the one the NCCL path performs (the lower triangle packed row
by row as uint32 words, summed exactly by a reduce, reduced mod p on the root; the result
regions gathered to the root)."""
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


def _pack_lower(C):
    """Low(C) row by row (row i: i + 1 elements of w words at element offset i (i + 1) / 2)."""
    m = C.shape[0]
    return np.concatenate([C[i, : i + 1].reshape(-1) for i in range(m)]) if m else np.zeros(0, C.dtype)


def _slice_by_bytes(A_rows_bytes, lda_bytes, off, k_slice, elem, dtype, w):
    """the rank's slice read the way the C ABI reads it: k_slice elements of `elem` bytes starting
    at byte offset `off` of every row (row pitch lda_bytes)"""
    m = A_rows_bytes.shape[0]
    raw = A_rows_bytes[:, off: off + k_slice * elem]
    return np.ascontiguousarray(raw).view(dtype).reshape(m, k_slice, w)


def _worker(rank, world, port, cases, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import paper_2101_01025_b200 as adj
    from inputs import uniform_matrix, uniform_matrix_ext, uniform_matrix_quat
    try:
        for (m, k, p, phi, in16) in cases:
            w = {"T": 1, "H": 2, "Q": 4}[phi]
            A = {"T": uniform_matrix, "H": uniform_matrix_ext, "Q": uniform_matrix_quat}[phi](m, k, 11, p)
            A = A.reshape(m, k, w)
            dtype = np.uint16 if in16 else np.uint32
            code = {"T": adj.ADJ_PHI_T, "H": adj.ADJ_PHI_H, "Q": adj.ADJ_PHI_Q}[phi]
            elem = adj.adj_elem_bytes(code, adj.ADJ_IN_U16 if in16 else 0)
            assert elem == np.dtype(dtype).itemsize * w
            rows = np.ascontiguousarray(A.astype(dtype)).view(np.uint8).reshape(m, -1)   # the caller's buffer
            k0, k1 = adj.adj_dist_kslice(k, world, rank)
            Ar = _slice_by_bytes(rows, rows.shape[1], k0 * elem, k1 - k0, elem, dtype, w).astype(np.uint32)
            f = {"T": lambda X: oracle.syrk_t(X[..., 0], p), "H": lambda X: oracle.syrk_h(X, p),
                 "Q": lambda X: oracle.syrk_q(X, p)}[phi]
            part = f(Ar).reshape(m, m, w)
            t = torch.from_numpy(_pack_lower(part).astype(np.int64))
            # residues summed exactly: each word < world * p < 2^32 (uint32 in the NCCL path)
            dist.reduce(t, dst=0, op=dist.ReduceOp.SUM)
            if rank == 0:
                assert (int(t.max()) if t.numel() else 0) < world * p < 2**32
                got = (t.numpy() % p).astype(np.uint32)
                ref = f(A).reshape(m, m, w)
                out_q.put((m, k, p, phi, in16, bool(np.array_equal(got, _pack_lower(ref)))))
    except Exception as e:   # report instead of leaving the parent waiting on the queue
        out_q.put(("error", rank, repr(e), False))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 4])
def test_split_k_reduce_gloo(world):
    cases = [(37, 100, 8191, "T", False), (64, 7, 65521, "T", True), (20, 33, 8191, "H", False),
             (21, 45, 8191, "H", True), (9, 17, 8191, "Q", True), (5, 1, 97, "T", False)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cases, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    results = []
    for _ in cases:
        results.append(q.get(timeout=300))
        assert results[-1][0] != "error", results[-1]
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
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
            # the rows this rank pre-adds cover both tile bands of every pair it owns
            ranges = adj.adj_shard_rows(m, k, p, rank, world, depth=depth)
            mh = -(-m // 2) if depth == 1 else m
            for (r0, c0, _, _, _) in mine:
                if r0 < mh and c0 < mh:
                    for b in (r0 // 256, c0 // 256):
                        assert any(lo <= 256 * b < hi for lo, hi in ranges), (rank, b, ranges)
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
