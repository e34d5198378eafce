"""Dev tool: run one adjprod call of a bench config several times (for ncu / compute-sanitizer)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2101_01025_b200 as adj  # noqa: E402
from bench import CONFIGS  # noqa: E402
from inputs.gpu import uniform_residues_cuda  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--depth", type=int, default=None)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--gemm", action="store_true", help="run gemm_modp m x m x k instead")
ap.add_argument("--io16", action="store_true", help="uint16 A and Low(C) (ADJ_IN_U16 | ADJ_OUT_U16)")
ap.add_argument("--m", type=int, default=None, help="override the config's m")
ap.add_argument("--k", type=int, default=None, help="override the config's k")
a = ap.parse_args()
cfg = CONFIGS[a.config]
m, k, p = a.m or cfg["m"], a.k or cfg["k"], cfg["p"]
w = 2 if cfg["phi"] == "H" else 1
phi = 1 if w == 2 else 0
A = torch.empty((m, k * w), dtype=torch.int32, device="cuda")
uniform_residues_cuda(A, 1, p)
C = torch.zeros((m, m * w), dtype=torch.int32, device="cuda")
flags = 0
if a.io16:
    A, C = A.to(torch.int16), C.to(torch.int16)
    flags = adj.ADJ_IN_U16 | adj.ADJ_OUT_U16
d = a.depth if a.depth is not None else (cfg["depth"] if cfg["depth"] is not None else adj.adjprod_modp_auto_depth(m, k, p, phi))
for _ in range(a.reps):
    if a.gemm:
        adj.gemm_modp(m, m, k, p, A, k, A, k, C, m)
    else:
        adj.adjprod_modp_ex(m, k, p, phi, A, k, C, m, depth=d, flags=flags)
torch.cuda.synchronize()
print("ok", a.config, "depth", d)
