"""Dev tool: leaf-kernel time of gemm_modp (m x n x k, one GEMM product) and adjprod (depth d)
via the library's profiling events; prints int8 TOP/s of the leaf launch (algorithmic ops).
ADJ_LEAF_DEBUG switches apply (diagnostics only; results are then garbage)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2101_01025_b200 as adj  # noqa: E402
from bench import limb_mmas  # noqa: E402
from inputs.gpu import uniform_residues_cuda  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=8192)
ap.add_argument("--n", type=int, default=8192)
ap.add_argument("--k", type=int, default=8192)
ap.add_argument("--p", type=int, default=8191)
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
A = torch.empty((a.m, a.k), dtype=torch.int32, device="cuda")
B = torch.empty((a.n, a.k), dtype=torch.int32, device="cuda")
uniform_residues_cuda(A, 1, a.p)
uniform_residues_cuda(B, 2, a.p)
C = torch.zeros((a.m, a.n), dtype=torch.int32, device="cuda")
for _ in range(3):
    adj.gemm_modp(a.m, a.n, a.k, a.p, A, a.k, B, a.k, C, a.n)
torch.cuda.synchronize()
adj.adj_profile_enable(True)
adj.adj_profile_read()
for _ in range(a.reps):
    adj.gemm_modp(a.m, a.n, a.k, a.p, A, a.k, B, a.k, C, a.n)
torch.cuda.synchronize()
prof = adj.adj_profile_read()
adj.adj_profile_enable(False)
ms = prof["leaf"][0] / a.reps
ops = 2.0 * a.m * a.n * a.k * limb_mmas(a.p)
print(f"gemm {a.m}x{a.n}x{a.k} p={a.p}: leaf {ms:.4f} ms/launch, {ops / ms * 1e-9:.1f} int8 TOP/s "
      f"(ADJ_LEAF_DEBUG={os.environ.get('ADJ_LEAF_DEBUG', '0')}) split+other {prof['preadd'][0] / a.reps:.4f} ms")
