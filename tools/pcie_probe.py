"""Dev tool: host <-> device copy rates of the e2e pipeline's buffers (c3: 2 GiB uint16 A in,
1.06 GiB of Low(C) row blocks out), alone, chunked, on two streams, with the opposite direction
running, and beside the c3 compute.  One JSON line per case (GB/s = bytes / device time)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

GB = 1e9
nA = 32768 * 32768          # uint16 residues of c3's A
nC = 32768 * 32768 // 2     # about the lower-triangle row blocks of Low(C)
hA = torch.empty(nA, dtype=torch.int16, pin_memory=True)
hC = torch.empty(nC, dtype=torch.int16, pin_memory=True)
dA = torch.empty(nA, dtype=torch.int16, device="cuda")
dC = torch.empty(nC, dtype=torch.int16, device="cuda")
hA.fill_(1)
s1, s2, s3 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=3):
    best = None
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        cur = torch.cuda.current_stream()
        e0.record(cur)
        fn(cur, e0)
        for s in (s1, s2, s3):
            cur.wait_stream(s)
        e1.record(cur)
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) * 1e-3
        best = t if best is None else min(best, t)
    return best


def h2d_one(cur, e0):
    s1.wait_event(e0)
    with torch.cuda.stream(s1):
        dA.copy_(hA, non_blocking=True)


def h2d_chunks(n, nstreams):
    def f(cur, e0):
        ch = nA // n
        ss = [s1, s2, s3][:nstreams]
        for s in ss:
            s.wait_event(e0)
        for i in range(n):
            with torch.cuda.stream(ss[i % nstreams]):
                dA[i * ch:(i + 1) * ch].copy_(hA[i * ch:(i + 1) * ch], non_blocking=True)
    return f


def d2h_one(cur, e0):
    s2.wait_event(e0)
    with torch.cuda.stream(s2):
        hC.copy_(dC, non_blocking=True)


def both(cur, e0):
    h2d_one(cur, e0)
    d2h_one(cur, e0)


cases = [("h2d_2GiB_one_copy", h2d_one, nA * 2), ("h2d_8_chunks_1_stream", h2d_chunks(8, 1), nA * 2),
         ("h2d_8_chunks_2_streams", h2d_chunks(8, 2), nA * 2), ("h2d_16_chunks_3_streams", h2d_chunks(16, 3), nA * 2),
         ("d2h_1GiB_one_copy", d2h_one, nC * 2)]
for name, fn, nbytes in cases:
    t = timed(fn)
    print(json.dumps({"case": name, "bytes": nbytes, "s": round(t, 5), "GBps": round(nbytes / t / GB, 2)}))
t = timed(both)
print(json.dumps({"case": "h2d_2GiB_and_d2h_1GiB_concurrent", "s": round(t, 5),
                  "h2d_GBps_if_limiting": round(nA * 2 / t / GB, 2)}))

# beside the c3 compute (power-capped SMs): H2D on a side stream while adjprod runs back to back
if "--compute" in sys.argv:
    import paper_2101_01025_b200 as adj
    from inputs.gpu import uniform_residues_cuda
    m = k = 32768
    p = 65521
    A32 = torch.empty((m, k), dtype=torch.int32, device="cuda")
    uniform_residues_cuda(A32, 1, p)
    A = A32.to(torch.int16)
    del A32
    C = torch.zeros((m, m), dtype=torch.int16, device="cuda")
    fl = adj.ADJ_IN_U16 | adj.ADJ_OUT_U16
    d = adj.adjprod_modp_auto_depth(m, k, p, 0)
    wsb = adj.adjprod_modp_workspace_size(m, k, p, 0, d, flags=fl)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    for rep in range(3):
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record(s3)
        with torch.cuda.stream(s3):
            for _ in range(2):
                adj.adjprod_modp_ex(m, k, p, 0, A, k, C, m, depth=d, flags=fl, workspace=ws, workspace_bytes=wsb,
                                    stream=s3)
        ev[1].record(s3)
        s1.wait_event(ev[0])
        ev[2].record(s1)
        with torch.cuda.stream(s1):
            dA.copy_(hA, non_blocking=True)
        ev[3].record(s1)
        torch.cuda.synchronize()
        print(json.dumps({"case": "h2d_2GiB_beside_c3_compute", "compute_ms_2_calls": round(ev[0].elapsed_time(ev[1]), 2),
                          "h2d_ms": round(ev[2].elapsed_time(ev[3]), 2),
                          "GBps": round(nA * 2 / (ev[2].elapsed_time(ev[3]) * 1e-3) / GB, 2)}))
