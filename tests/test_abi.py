"""C-ABI checks that need no GPU: the library loads, exports every symbol include/adjprod.h
declares, host-side constants, workspace sizing and synchronous argument validation."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2101_01025_b200 as adj
from paper_2101_01025_b200 import _lib
from oracle import field as F

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "adjprod.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(adj\w*|gemm_modp)\s*\(", src)) - {"adj_stream_t"})


def test_library_exports_every_declared_symbol():
    L = adj.lib()
    names = header_functions()
    assert len(names) >= 16
    for n in names:
        assert hasattr(L, n), n
    assert sorted(_lib.EXPORTS) == names


def test_status_strings():
    L = adj.lib()
    for code, name in _lib.STATUS.items():
        assert L.adj_status_string(code).decode() == name


@pytest.mark.parametrize("p", [3, 5, 7, 13, 97, 251, 257, 8191, 16763, 16787, 65521, 65537, 131041, 131071,
                               262139])
def test_skew_unitary_matches_paper_construction(p):
    """Host constants of the CUDA path vs the oracle's independent field code; Y phi(Y) = -I."""
    kind, a, b = adj.adj_skew_unitary(p)
    okind, oa, ob = F.skew_unitary(p)
    assert (kind, a, b) == ({"scalar": 0, "rot2": 1}[okind], oa, ob)
    if kind == 0:
        assert a * a % p == p - 1
    else:
        assert (a * a + b * b) % p == p - 1


def test_sos_worked_values(golden):
    for e in golden["sos"]:
        assert list(adj.adj_sos(e["p"], e["k"])) == e["value"], e["cite"]
    for q in [q for q in range(3, 400) if F.is_prime(q)]:
        a, b = adj.adj_sos(q, q - 1)
        assert (a * a + b * b) % q == q - 1


def test_validation_is_synchronous_and_needs_no_gpu():
    with pytest.raises(adj.AdjError) as e:
        adj.adjprod_modp(4, 4, 91, 0, 1, 4, 2, 4, stream=0)             # 91 = 7 * 13 not prime
    assert e.value.status == 2
    with pytest.raises(adj.AdjError) as e:
        adj.adjprod_modp(4, 4, 262147, 0, 1, 4, 2, 4, stream=0)         # > 262139 = largest prime < 2^18
    assert e.value.status == 2
    with pytest.raises(adj.AdjError) as e:
        adj.adjprod_modp(4, 4, 97, 1, 1, 4, 2, 4, stream=0)             # phi = H needs p = 3 mod 4
    assert e.value.status == 2
    with pytest.raises(adj.AdjError) as e:
        adj.adjprod_modp(-1, 4, 97, 0, 1, 4, 2, 4, stream=0)
    assert e.value.status == 1
    with pytest.raises(adj.AdjError) as e:
        adj.adjprod_modp(4, 4, 97, 0, 4096, 3, 8192, 4, stream=0)       # lda < k
    assert e.value.status == 1
    with pytest.raises(adj.AdjError) as e:
        adj.adjprod_modp(4, 4, 97, 0, 4096, 4, 4100, 4, stream=0)       # A and C overlap
    assert e.value.status == 1
    adj.adjprod_modp(0, 4, 97, 0, 0, 4, 0, 0, stream=0)      # m = 0 is a no-op


def test_header_flag_values_match_binding():
    import re
    text = open(os.path.join(ROOT, "include", "adjprod.h")).read()
    for name in ("ADJ_FILL_UPPER", "ADJ_HERK_ALG1", "ADJ_DIST_TILES", "ADJ_DIST_P2P", "ADJ_IN_U16", "ADJ_OUT_U16"):
        mt = re.search(name + r" = (\d+)u", text)
        assert mt and int(mt.group(1)) == getattr(adj, name), name


def test_compact_io_validation_needs_no_gpu():
    I16, O16 = adj.ADJ_IN_U16, adj.ADJ_OUT_U16
    for args, flags in [((4, 4, 131071, 0), I16),                 # p > 2^16: residues need 32 bits
                        ((4, 4, 8191, 0), O16 | adj.ADJ_FILL_UPPER),
                        ((4, 4, 8191, 1), O16 | adj.ADJ_HERK_ALG1),   # phi = H: 2M output only
                        ((4, 4, 65537, 2), I16)]:                 # phi = Q, p > 2^16
        with pytest.raises(adj.AdjError) as e:
            adj.adjprod_modp_ex(*args, 4096, 4, 8192, 4, flags=flags, stream=0)
        assert e.value.status == 1, (args, flags)
    with pytest.raises(adj.AdjError) as e:                        # SYRK form into a uint16 Low(C)
        adj.adjprod_modp_syrk(4, 4, 8191, 0, 3, 4096, 4, 1, 8192, 4, flags=O16, stream=0)
    assert e.value.status == 1
    # the overlap check counts 2-byte elements: A (16 uint16) ends where C starts
    with pytest.raises(adj.AdjError) as e:
        adj.adjprod_modp_ex(4, 4, 8191, 0, 4096, 4, 4096 + 32, 4, flags=I16 | O16, stream=0)
    assert e.value.status != 1                                     # passes validation, then no device
    with pytest.raises(adj.AdjError) as e:
        adj.adjprod_modp_ex(4, 4, 8191, 0, 4096, 4, 4096 + 32, 4, stream=0)
    assert e.value.status == 1                                     # 4-byte A overlaps


def test_workspace_and_depth_planning():
    assert adj.adjprod_modp_auto_depth(64, 64, 97, 0) == 0
    # measured B200 crossovers (R13): recurse while (m/2)^2 (k/2) >= 2^38 per level
    assert adj.adjprod_modp_auto_depth(8192, 8192, 8191, 0) == 0        # c2: classical 8% faster
    assert adj.adjprod_modp_auto_depth(16384, 16384, 8191, 0) == 1
    assert adj.adjprod_modp_auto_depth(16384, 131072, 8191, 0) == 2     # c4
    assert adj.adjprod_modp_auto_depth(32768, 32768, 65521, 0) == 2     # c3
    assert adj.adjprod_modp_auto_depth(8192, 8192, 8191, 1) == 0        # c5 (2M)
    assert adj.adjprod_modp_auto_depth(8192, 8192, 8191, 2) == 0        # q5 (6M)
    # inner dimension above the int32 bound at depth 0 forces recursion (65521: k_max = 32896)
    assert adj.adjprod_modp_auto_depth(1000, 100000, 65521, 0) >= 2
    w0 = adj.adjprod_modp_workspace_size(8192, 8192, 8191, 0, depth=0)
    w1 = adj.adjprod_modp_workspace_size(8192, 8192, 8191, 0, depth=1)
    w2 = adj.adjprod_modp_workspace_size(8192, 8192, 8191, 0, depth=2)
    # depth 0: 3 int8 planes of 8192 x 8192; depth 1: 7 operands x 3 planes at 4096^2 + 5 P buffers;
    # plus 256x256 u16 fixup slots for the K-split tail tiles, reserved for the worst case (one per
    # cluster pair: 148 / 2 = 74, independent of the tile list) and the 256-byte job counter of the
    # dynamic scheduler (after rounding to 256 bytes)
    def tail(w, base):
        extra = w - base - 256
        slot = 256 * 256 * 2
        return extra >= 0 and extra % slot < 256 and extra // slot == 74
    assert tail(w0, 3 * 8192 * 8192)
    assert tail(w1, 7 * 3 * 4096 * 4096 + 5 * 4096 * 4096 * 2)
    assert w2 > 0
    # k above the int32 bound of the limb scheme is handled by K segmentation (no error)
    assert tail(adj.adjprod_modp_workspace_size(256, 40000, 65521, 0, depth=0), 2 * 256 * 40064)
    # a shard's plan (filtered tile list) fits the same workspace as the full plan
    assert adj.adjprod_modp_workspace_size(8192, 8192, 8191, 0, depth=1) == w1


def test_herk_alg1_workspace_planning():
    """ADJ_HERK_ALG1: 21 limb operands of (m/2) x (k/2) plus 12 product
    buffers of (m/2)^2 residues; depth other than 1 is refused synchronously (no GPU needed)."""
    m, k, p = 8192, 8192, 8191
    w = adj.adjprod_modp_workspace_size(m, k, p, 1, depth=-1, flags=adj.ADJ_HERK_ALG1)
    arena = 21 * 3 * 4096 * 4096
    bufs = 12 * 4096 * 4096 * 2
    assert arena + bufs <= w <= arena + bufs + 64 * 65536 * 2 * 64 + 4096
    with pytest.raises(adj.AdjError):
        adj.adjprod_modp_workspace_size(m, k, p, 1, depth=2, flags=adj.ADJ_HERK_ALG1)
    # ignored for phi = T
    assert adj.adjprod_modp_workspace_size(m, k, p, 0, depth=1, flags=adj.ADJ_HERK_ALG1) == \
        adj.adjprod_modp_workspace_size(m, k, p, 0, depth=1)


@pytest.mark.parametrize("m,k,depth", [(1, 5, 0), (100, 64, 0), (1000, 500, 0), (1000, 700, 1), (3000, 256, 1),
                                       (4097, 1000, 1)])
@pytest.mark.parametrize("nranks", [1, 2, 3, 5, 8])
def test_shard_layout_partitions_low_c(m, k, depth, nranks):
    """Output-tile sharding: the regions adj_shard_layout gives the ranks
    cover every element of Low(C) exactly once and nothing above the diagonal."""
    import numpy as np
    cover = np.zeros((m, m), dtype=np.int32)
    for r in range(nranks):
        for (r0, c0, rows, cols, lower) in adj.adj_shard_layout(m, k, 8191, r, nranks, depth=depth):
            assert 0 <= r0 and r0 + rows <= m and 0 <= c0 and c0 + cols <= m
            blk = np.ones((rows, cols), dtype=np.int32)
            if lower:
                ii, jj = np.meshgrid(np.arange(rows) + r0, np.arange(cols) + c0, indexing="ij")
                blk = (jj <= ii).astype(np.int32)
            cover[r0:r0 + rows, c0:c0 + cols] += blk
    assert np.array_equal(cover, np.tril(np.ones((m, m), dtype=np.int32)))


def test_shard_layout_balanced():
    """The deterministic block deal keeps the ranks' shares of Low(C) within 10% of the mean
    (whole blocks of band groups are dealt; the planner trades a few % of leaf balance for
    pre-adding only the rows a rank reads)."""
    for m in (8192, 32768):
        for depth in (0, 1):
            for n in (2, 4, 8):
                sizes = []
                for r in range(n):
                    rects = adj.adj_shard_layout(m, m, 8191, r, n, depth=depth)
                    sizes.append(sum(rows * cols for (_, _, rows, cols, _) in rects))
                assert max(sizes) <= 1.10 * (sum(sizes) / n), (m, depth, n, sizes)


@pytest.mark.parametrize("m,depth,nranks", [(32768, 1, 8), (32768, 1, 4), (32768, 1, 3), (8192, 1, 8), (8192, 0, 8),
                                            (1030, 1, 3), (700, 0, 2), (32768, 1, 1)])
def test_shard_rows_cover_every_band_the_tiles_read(m, depth, nranks):
    """A rank's pre-addition rows (adj_shard_rows) cover the operand rows of every tile pair it
    owns -- bands I and J of each owned pair (I, J), read off its C11 regions (depth 1) or its C
    regions (depth 0) -- and, at 8 ranks of c3, only half of all rows (the blocked deal)."""
    mh = -(-m // 2) if depth == 1 else m
    rows_pad = -(-mh // 128) * 128
    total = []
    for r in range(nranks):
        ranges = adj.adj_shard_rows(m, m, 8191, r, nranks, depth=depth)
        covered = np.zeros(rows_pad + 256, dtype=bool)
        for lo, hi in ranges:
            assert 0 <= lo < hi <= rows_pad
            covered[lo:hi] = True
        for (r0, c0, rows, cols, _) in adj.adj_shard_layout(m, m, 8191, r, nranks, depth=depth):
            if r0 < mh and c0 < mh:     # C11 (depth 1) / C (depth 0): tile pair (r0 / 256, c0 / 256)
                for b in (r0 // 256, c0 // 256):
                    assert covered[256 * b: min(256 * b + 256, rows_pad)].all(), (r, b)
        total.append(int(covered.sum()))
    if (m, depth, nranks) == (32768, 1, 8):
        assert max(total) <= rows_pad // 2, total


def test_maximum_sizes_are_planned_or_refused():
    """The packed tile descriptor holds 12-bit tile indices: a leaf operand of 4096 x 256 rows or
    more is refused with ADJ_ERR_INVALID_VALUE at planning time (never a silent wrap); one level
    of Alg. 1 halves it back into range."""
    m = 4096 * 256
    with pytest.raises(adj.AdjError) as e:
        adj.adjprod_modp_workspace_size(m, 256, 8191, 0, 0)
    assert e.value.status == 1
    with pytest.raises(adj.AdjError) as e:
        adj.adjprod_modp_workspace_size(m + 1000, 64, 97, 0, 0)
    assert e.value.status == 1
    # largest single-tile-index-range leaf still planned (m = 4095 x 256 at depth 0)
    assert adj.adjprod_modp_workspace_size(4095 * 256, 32, 97, 0, 0) > 0


def test_lowmem_workspace_within_twice_a_at_bench_sizes():
    """ADJ_LOW_MEM: at c3 (32768^2, depth 2) and c4 (16384 x 131072, depth
    2) the workspace is at most twice the uint16 A, and below the grouped schedule's."""
    import paper_2101_01025_b200 as adj
    for m, k, p in [(32768, 32768, 65521), (16384, 131072, 8191)]:
        w_def = adj.adjprod_modp_workspace_size(m, k, p, 0, depth=2)
        w_lm = adj.adjprod_modp_workspace_size(m, k, p, 0, depth=2, flags=adj.ADJ_LOW_MEM)
        a16 = 2 * m * k
        assert w_lm <= 2 * a16 < w_def, (m, k, w_lm / a16, w_def / a16)


def test_lowmem_workspace_layout():
    """The low-memory workspace is [S3 | P2 | P4 | max(root arena, child workspace)] (plan.cpp
    build_lowmem_plan), recomputed here from the level sizes: S3 is mh x kh
    residues, P2 / P4 rows_pad^2 residues, the root arena 4 operands x planes x rows_pad x kpad
    int8 (plus the tail's fixup slots and the job counter), the children ordinary calls of
    shape mh x kh one level shallower."""
    import paper_2101_01025_b200 as adj
    rup = lambda x, a: -(-x // a) * a
    for m, k, p, d in [(32768, 32768, 65521, 2), (16384, 131072, 8191, 2), (2048, 3000, 8191, 2), (1024, 1001, 97, 1)]:
        planes = 1 if p <= 255 else (3 if p <= 16763 else 2)
        res = 2
        mh, kh = m // 2, 8 * -(-k // 16)
        rp, kp = rup(mh, 128), max(128, rup(kh, 128))
        head = rup(mh * kh * res, 256) + 2 * rup(rp * rp * res, 256)
        arena = rup(4 * planes * rp * kp, 256)
        child = adj.adjprod_modp_workspace_size(mh, kh, p, 0, depth=d - 1)
        w = adj.adjprod_modp_workspace_size(m, k, p, 0, depth=d, flags=adj.ADJ_LOW_MEM)
        fixup_and_counter = 74 * 256 * 256 * res + 256   # worst-case tail slots (num_sms / 2) + job counter
        assert w == rup(head + max(arena + fixup_and_counter, child), 256), (m, k, p, d)


def test_ipc_validation_needs_no_gpu():
    """adj_ipc_export / adj_ipc_open / adj_ipc_close (the building blocks of ADJ_DIST_TILES |
    ADJ_DIST_P2P) reject null pointers and unknown mappings before touching CUDA."""
    import re
    text = open(os.path.join(ROOT, "include", "adjprod.h")).read()
    assert int(re.search(r"#define ADJ_IPC_RECORD_BYTES (\d+)", text).group(1)) == adj._lib.ADJ_IPC_RECORD_BYTES
    with pytest.raises(adj.AdjError) as e:
        adj.adj_ipc_export(0)
    assert e.value.status == 1
    L = adj.lib()
    out = ctypes.c_void_p(0)
    assert L.adj_ipc_open(None, ctypes.byref(out)) == 1
    rec = bytes(64) + (-8).to_bytes(8, "little", signed=True)       # negative offset
    assert L.adj_ipc_open(rec, ctypes.byref(out)) == 1
    with pytest.raises(adj.AdjError) as e:
        adj.adj_ipc_close(0x1000)                                     # never opened
    assert e.value.status == 1


def test_leaf_tile_query():
    """The wide-N leaf (256 x 512 tiles) serves long launches (c3 / c4, the metric's configs) and
    shorter ones whose whole waves of wide jobs beat the narrow tail-balanced makespan (c2 and the
    6-plane x131071: 4 waves x 1.74 < 7.1); the smallest configs keep 256 x 256 tiles."""
    assert adj.adjprod_modp_leaf_tile(32768, 32768, 65521, 0) == 512       # c3, depth 2
    assert adj.adjprod_modp_leaf_tile(16384, 131072, 8191, 0) == 512      # c4, depth 2
    assert adj.adjprod_modp_leaf_tile(8192, 8192, 8191, 0) == 512         # c2
    assert adj.adjprod_modp_leaf_tile(8192, 8192, 131071, 0) == 512       # x131071
    assert adj.adjprod_modp_leaf_tile(2048, 2048, 8191, 0) == 256         # one short wave
    assert adj.adjprod_modp_leaf_tile(256, 256, 97, 0, depth=1) == 256     # c1
    assert adj.adjprod_modp_leaf_tile(0, 5, 97, 0) == 256
    with pytest.raises(adj.AdjError) as e:
        adj.adjprod_modp_leaf_tile(4, 4, 91, 0)
    assert e.value.status == 2
