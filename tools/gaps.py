"""Dev tool: per-class kernel time (library events around each launch) vs the whole-step time."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2101_01025_b200 as adj  # noqa: E402
from inputs.gpu import uniform_residues_cuda  # noqa: E402

m = k = int(os.environ.get("N", "8192"))
p = int(os.environ.get("P", "8191"))
for depth in (0, 1):
    A = torch.empty((m, k), dtype=torch.int32, device="cuda")
    uniform_residues_cuda(A, 1, p)
    C = torch.zeros((m, m), dtype=torch.int32, device="cuda")
    wsb = adj.adjprod_modp_workspace_size(m, k, p, 0, depth)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream()
    for _ in range(5):
        adj.adjprod_modp_ex(m, k, p, 0, A, k, C, m, depth=depth, workspace=ws, workspace_bytes=wsb, stream=s)
    torch.cuda.synchronize()
    reps = 20
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    adj.adj_profile_enable(False)
    a.record(s)
    for _ in range(reps):
        adj.adjprod_modp_ex(m, k, p, 0, A, k, C, m, depth=depth, workspace=ws, workspace_bytes=wsb, stream=s)
    b.record(s)
    torch.cuda.synchronize()
    t_noprof = a.elapsed_time(b) / reps
    adj.adj_profile_enable(True)
    adj.adj_profile_read()
    a.record(s)
    for _ in range(reps):
        adj.adjprod_modp_ex(m, k, p, 0, A, k, C, m, depth=depth, workspace=ws, workspace_bytes=wsb, stream=s)
    b.record(s)
    torch.cuda.synchronize()
    prof = adj.adj_profile_read()
    adj.adj_profile_enable(False)
    tot = sum(v[0] for v in prof.values()) / reps
    print(f"depth {depth}: back-to-back step {t_noprof:.4f} ms (no events), with events {a.elapsed_time(b) / reps:.4f}; "
          f"kernels {tot:.4f} ms: " + ", ".join(f"{c} {v[0] / reps:.4f} ({v[1] // reps})" for c, v in prof.items()))
