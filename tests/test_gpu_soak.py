"""Race detection by repetition (compute-sanitizer is not available on the GPU pool): all
arithmetic is exact mod p, so whatever order the persistent leaf claims its jobs in, whatever the
claim-wave gate and the K4 / K5 passes overlap with, every call must return the same bits.  A
missing barrier, a stage released too early, a job claimed twice or a read of workspace bytes no
kernel of this call wrote shows up as a run that differs from the first one (or from the
oracle).  Each repetition starts from a poisoned output and a poisoned caller workspace.

The contract of include/adjprod.h ("concurrent calls on different streams with different
workspaces") is exercised the same way: two problems interleaved on two streams."""
import numpy as np
import pytest

import oracle
from inputs import uniform_matrix, uniform_matrix_ext, uniform_matrix_quat
from gpu_util import to_dev, to_host

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def adj():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    import paper_2101_01025_b200 as adj
    adj.lib()
    return adj


def _gen(phi, m, k, seed, p):
    return {"T": uniform_matrix, "H": uniform_matrix_ext, "Q": uniform_matrix_quat}[phi](m, k, seed=seed, p=p)


def _oracle_rows(phi, A, p, rows):
    return {"T": oracle.syrk_t, "H": oracle.syrk_h, "Q": oracle.syrk_q}[phi](A, p, rows=rows)


# (phi, p, m, k, depth, repetitions, leaf tile width): launches of several waves on 74 CTA pairs,
# a ragged one, the 3-limb scheme, 2M and 6M.  The last column is adjprod_modp_leaf_tile's answer
# (asserted below, so the list keeps covering both leaf kernels): 512 = the wide-N leaf with
# dynamic claiming and the claim-wave gate, 256 = the 256 x 256 leaf with its K-split tail
CASES = [
    ("T", 65521, 8192, 8192, 0, 12, 512),
    ("T", 65521, 8192, 8192, 1, 12, 512),
    ("T", 8191, 6144, 4096, 2, 12, 512),
    ("T", 65521, 5000, 3001, 2, 12, 256),
    ("T", 131071, 4096, 2048, 1, 8, 256),
    ("H", 8191, 3072, 2048, 1, 8, 512),
    ("Q", 8191, 2048, 1024, 0, 8, 256),
]


@pytest.mark.parametrize("phi,p,m,k,depth,reps,tile", CASES)
def test_repeated_calls_bit_identical_poisoned_workspace(adj, phi, p, m, k, depth, reps, tile):
    import torch
    ph = {"T": 0, "H": 1, "Q": 2}[phi]
    assert adj.adjprod_modp_leaf_tile(m, k, p, ph, depth) == tile
    w = {"T": 1, "H": 2, "Q": 4}[phi]
    A = _gen(phi, m, k, seed=7 * m + depth, p=p)
    dA = to_dev(A)
    ws_bytes = adj.adjprod_modp_workspace_size(m, k, p, ph, depth)
    ws = torch.empty(max(ws_bytes, 16), dtype=torch.uint8, device="cuda")
    shape = (m, m) if w == 1 else (m, m, w)
    first = None
    for r in range(reps):
        ws.fill_((0x5A + 37 * r) & 0xFF)                     # stale products of another call
        C = torch.full(shape, -1, dtype=torch.int32, device="cuda")
        adj.adjprod_modp_ex(m, k, p, ph, dA, k, C, m, depth=depth, workspace=ws, workspace_bytes=ws_bytes)
        torch.cuda.synchronize()
        if first is None:
            first = C
            rows = sorted({0, 1, 255, 256, m // 2 - 1, m // 2, m // 2 + 257, m - 2, m - 1})
            got = to_host(C)
            for i in rows:                                   # Low(C) rows vs the oracle, Up(C) untouched
                ref = _oracle_rows(phi, A, p, (i, i + 1))
                assert np.array_equal(got[i, : i + 1], ref[i, : i + 1]), (phi, p, m, k, depth, i)
                assert (got[i, i + 1:] == 0xFFFFFFFF).all(), (phi, p, m, k, depth, i)
        else:
            assert torch.equal(C, first), f"run {r} differs from run 0: {(C != first).sum().item()} words"


# small launches on the 256 x 256 leaf; then two long launches of the wide-N leaf, whose persistent
# grids (one CTA pair per SM pair each) share the SMs, so the claim-wave gate of either may wait on
# a job whose CTA is not resident: its wait is bounded and the launch degrades to ungated
@pytest.mark.parametrize("PROBS", [[(65521, 4096, 4096, 2), (8191, 3000, 5000, 1)],
                                   [(65521, 8192, 8192, 1), (8191, 6144, 4096, 2)]])
def test_two_streams_two_workspaces_interleaved(adj, PROBS):
    """Two different problems issued alternately on two streams, each with its own workspace and
    output (include/adjprod.h: concurrent calls on different streams with different workspaces):
    every result equals the one the same call gives alone."""
    import torch
    probs = PROBS
    state = []
    for p, m, k, depth in probs:
        A = uniform_matrix(m, k, seed=m + k, p=p)
        dA = to_dev(A)
        nb = adj.adjprod_modp_workspace_size(m, k, p, 0, depth)
        ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
        alone = torch.zeros((m, m), dtype=torch.int32, device="cuda")
        adj.adjprod_modp_ex(m, k, p, 0, dA, k, alone, m, depth=depth, workspace=ws, workspace_bytes=nb)
        torch.cuda.synchronize()
        rows = [0, 255, 256, m // 2, m - 1]
        got = to_host(alone)
        for i in rows:
            ref = oracle.syrk_t(A, p, rows=(i, i + 1))
            assert np.array_equal(got[i, : i + 1], ref[i, : i + 1])
        state.append((p, m, k, depth, dA, ws, nb, alone, torch.cuda.Stream()))
    outs = [[], []]
    for r in range(6):
        for j, (p, m, k, depth, dA, ws, nb, alone, s) in enumerate(state):
            C = torch.zeros((m, m), dtype=torch.int32, device="cuda")
            s.wait_stream(torch.cuda.current_stream())       # C's zero fill
            adj.adjprod_modp_ex(m, k, p, 0, dA, k, C, m, depth=depth, workspace=ws, workspace_bytes=nb, stream=s)
            outs[j].append(C)
    torch.cuda.synchronize()
    for j, st in enumerate(state):
        for r, C in enumerate(outs[j]):
            assert torch.equal(C, st[7]), f"problem {j}, round {r}: differs from the call run alone"


@pytest.mark.parametrize("name,reps", [("c3", 6), ("c4", 6)])
def test_full_size_bench_launch_repeats_bit_identical(adj, name, reps):
    """The metric's configurations in the launch bench.py times (depth 2, uint16 residues, the
    wide-N leaf with 1840+ jobs claimed dynamically behind the claim-wave gate, board at its power
    cap): back-to-back calls, each from a poisoned Low(C) and a poisoned workspace, return the same
    bits.  The first run's values are checked entry by entry in test_gpu_fullsize_exact.py."""
    import torch
    import bench
    from inputs.gpu import uniform_residues_cuda
    cfg = bench.CONFIGS[name]
    m, k, p = cfg["m"], cfg["k"], cfg["p"]
    fl = adj.ADJ_IN_U16 | adj.ADJ_OUT_U16
    depth = adj.adjprod_modp_auto_depth(m, k, p, 0)
    assert depth == 2 and adj.adjprod_modp_leaf_tile(m, k, p, 0, depth, fl) == 512
    A = torch.empty((m, k), dtype=torch.int32, device="cuda")
    uniform_residues_cuda(A, seed=1, p=p)
    A16 = A.to(torch.int16)
    del A
    nb = adj.adjprod_modp_workspace_size(m, k, p, 0, depth, fl)
    W = torch.empty(nb, dtype=torch.uint8, device="cuda")
    first = None
    for r in range(reps):
        W.fill_((0xC3 + 29 * r) & 0xFF)
        C16 = torch.full((m, m), -1, dtype=torch.int16, device="cuda")
        adj.adjprod_modp_ex(m, k, p, 0, A16, k, C16, m, depth=depth, flags=fl, workspace=W, workspace_bytes=nb)
        if first is None:
            first = C16
        else:
            assert torch.equal(C16, first), f"{name}: run {r} differs from run 0"
    i = m - 1                                   # last row: Low(C) row complete, nothing above the diagonal
    j = 5
    assert (first[j, j + 1:] == -1).all()       # Up(C) untouched
    assert int(first[i].to(torch.int32).bitwise_and(0xFFFF).max()) < p


@pytest.mark.parametrize("p,m,k,depth,io16", [(65521, 8192, 8192, 2, True), (8191, 6144, 4096, 2, False),
                                              (65521, 4608, 3000, 3, True)])
def test_low_memory_schedule_repeats_bit_identical(adj, p, m, k, depth, io16):
    """ADJ_LOW_MEM: the root's products are formed in C's own blocks and K4 runs in place (every
    thread overwrites only positions it has read itself), arenas are reused across
    children.  Repeated from poisoned C and workspace it must return, every time, the grouped
    schedule's Low(C) bit for bit (which the first loop of this file ties to the oracle)."""
    import torch
    A = uniform_matrix(m, k, seed=3 * m + depth, p=p)
    dt = torch.int16 if io16 else torch.int32
    dA = torch.from_numpy(A.astype(np.uint16).view(np.int16)).cuda() if io16 else to_dev(A)
    io = (adj.ADJ_IN_U16 | adj.ADJ_OUT_U16) if io16 else 0
    ref = torch.full((m, m), -1, dtype=dt, device="cuda")
    adj.adjprod_modp_ex(m, k, p, 0, dA, k, ref, m, depth=depth, flags=io)
    torch.cuda.synchronize()
    got = ref.cpu().numpy().view(np.uint16 if io16 else np.uint32)
    for i in (0, 255, 256, m // 2 + 1, m - 1):
        want = oracle.syrk_t(A, p, rows=(i, i + 1))
        assert np.array_equal(got[i, : i + 1].astype(np.uint32), want[i, : i + 1]), (p, m, k, depth, i)
    fl = io | adj.ADJ_LOW_MEM
    nb = adj.adjprod_modp_workspace_size(m, k, p, 0, depth, fl)
    assert nb < adj.adjprod_modp_workspace_size(m, k, p, 0, depth, io)     # the low-memory schedule applies
    W = torch.empty(nb, dtype=torch.uint8, device="cuda")
    for r in range(8):
        W.fill_((0x3C + 41 * r) & 0xFF)
        C = torch.full((m, m), -1, dtype=dt, device="cuda")
        adj.adjprod_modp_ex(m, k, p, 0, dA, k, C, m, depth=depth, flags=fl, workspace=W, workspace_bytes=nb)
        assert torch.equal(C, ref), f"low-memory run {r}: {(C != ref).sum().item()} entries differ from the grouped schedule"


def test_host_threads_call_concurrently(adj):
    """include/adjprod.h: calls may come from several host threads (different streams, different
    workspaces); the plan cache and the workspace pool are locked.  Four threads (ctypes drops the
    GIL inside the call), each with its own stream and two shapes of its own - so plans are built
    and inserted while other threads launch - repeat their calls; every result equals the one the
    same call gave alone on the main thread (tied to the oracle on sampled rows)."""
    import threading
    import torch
    jobs = [(65521, 2304, 1536, 2), (8191, 2000, 3000, 1), (97, 1500, 700, 1), (131071, 1280, 1024, 1),
            (65521, 1111, 999, 1), (8191, 2560, 2560, 2), (251, 900, 2100, 0), (16763, 1792, 512, 1)]
    items = []
    for p, m, k, depth in jobs:
        A = uniform_matrix(m, k, seed=p + m, p=p)
        dA = to_dev(A)
        alone = torch.zeros((m, m), dtype=torch.int32, device="cuda")
        adj.adjprod_modp_ex(m, k, p, 0, dA, k, alone, m, depth=depth)
        got = to_host(alone)
        for i in (0, m // 2, m - 1):
            ref = oracle.syrk_t(A, p, rows=(i, i + 1))
            assert np.array_equal(got[i, : i + 1], ref[i, : i + 1]), (p, m, k, depth, i)
        items.append((p, m, k, depth, dA, alone))
    torch.cuda.synchronize()
    errors = []

    def worker(t):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            mine = items[2 * t: 2 * t + 2]
            # new shapes per thread as well: their plans are built under the lock while others launch
            for r in range(10):
                for p, m, k, depth, dA, alone in mine:
                    with torch.cuda.stream(s):
                        C = torch.zeros((m, m), dtype=torch.int32, device="cuda")
                        adj.adjprod_modp_ex(m, k, p, 0, dA, k, C, m, depth=depth, stream=s)
                        mm = m - 128 * (1 + (r + t) % 3)           # a shape only this thread uses
                        C2 = torch.zeros((mm, mm), dtype=torch.int32, device="cuda")
                        adj.adjprod_modp_ex(mm, k, p, 0, dA, k, C2, mm, depth=depth, stream=s)
                    s.synchronize()
                    if not torch.equal(C, alone):
                        errors.append(f"thread {t} round {r}: {(p, m, k, depth)} differs")
                    if not torch.equal(C2, alone[:mm, :mm]):      # leading rows of A give the leading block
                        errors.append(f"thread {t} round {r}: {(p, mm, k, depth)} differs")
        except Exception as e:                                     # noqa: BLE001
            errors.append(f"thread {t}: {type(e).__name__}: {e}")

    threads = [threading.Thread(target=worker, args=(t,)) for t in range(4)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert not errors, errors[:5]


def test_plan_cache_eviction_over_many_shapes(adj):
    """More distinct shapes than the plan cache holds (64, LRU over the plans no call is using):
    plans are evicted, their device tile lists freed and rebuilt on the next use; every call,
    before and after its plan's eviction, matches the oracle on the whole Low(C)."""
    p = 8191
    shapes = [(130 + 3 * i, 64 + (i % 5) * 32, i % 2) for i in range(80)]
    As = {}
    for rnd in range(2):
        for m, k, depth in shapes + shapes[:10]:
            if (m, k) not in As:
                A = uniform_matrix(m, k, seed=m * 1000 + k, p=p)
                As[(m, k)] = (to_dev(A), oracle.syrk_t(A, p))
            dA, ref = As[(m, k)]
            C = adj.adjprod(dA, p, depth=depth)
            assert np.array_equal(to_host(C), ref), (rnd, m, k, depth)
