"""Dev tool: device time of one rank's output-tile share (adjprod_modp_shard) for G ranks, to project
multi-GPU strong scaling on one device (the gather is not included)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2101_01025_b200 as adj  # noqa: E402
from inputs.gpu import uniform_residues_cuda  # noqa: E402

m = k = int(os.environ.get("N", "8192"))
p = 8191
A = torch.empty((m, k), dtype=torch.int32, device="cuda")
uniform_residues_cuda(A, 1, p)
C = torch.zeros((m, m), dtype=torch.int32, device="cuda")
for depth in (0, 1):
    for G in (1, 2, 4, 8):
        for _ in range(3):
            adj.adjprod_modp_shard(m, k, p, 0, A, k, C, m, 0, G, depth=depth)
        torch.cuda.synchronize()
        ts = []
        for r in range(G):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(5):
                adj.adjprod_modp_shard(m, k, p, 0, A, k, C, m, r, G, depth=depth)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) / 5)
        print(f"m={m} depth {depth} G={G}: per-rank share ms max {max(ts):.4f} min {min(ts):.4f}")
