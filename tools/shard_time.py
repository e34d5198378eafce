"""Dev tool: device time of each rank's output-tile share (adjprod_modp_shard) for G ranks, run one
after the other on one device, to project multi-GPU strong scaling (the gather is not included).
Env: N (m = k), P (prime), DEPTHS (e.g. "1"), GS (e.g. "1 2 4 8"); A as uint16 (ADJ_IN_U16) like
bench.py when p < 2^16."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2101_01025_b200 as adj  # noqa: E402
from inputs.gpu import uniform_residues_cuda  # noqa: E402

m = k = int(os.environ.get("N", "8192"))
p = int(os.environ.get("P", "8191"))
A = torch.empty((m, k), dtype=torch.int32, device="cuda")
uniform_residues_cuda(A, 1, p)
flags = 0
if p < 65536:
    A = A.to(torch.int16)
    flags = adj.ADJ_IN_U16
C = torch.zeros((m, m), dtype=torch.int32, device="cuda")
for depth in [int(x) for x in os.environ.get("DEPTHS", "0 1").split()]:
    for G in [int(x) for x in os.environ.get("GS", "1 2 4 8").split()]:
        for _ in range(2):
            adj.adjprod_modp_shard(m, k, p, 0, A, k, C, m, 0, G, depth=depth, flags=flags)
        torch.cuda.synchronize()
        ts = []
        for r in range(G):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(3):
                adj.adjprod_modp_shard(m, k, p, 0, A, k, C, m, r, G, depth=depth, flags=flags)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) / 3)
        print(f"m={m} p={p} depth {depth} G={G}: per-rank share ms max {max(ts):.3f} min {min(ts):.3f} "
              f"(sum {sum(ts):.2f})", flush=True)
