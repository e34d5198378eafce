import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2101_01025_b200 as adj, oracle
from inputs import uniform_matrix
for (m, k, p, d) in [(512, 256, 97, 0), (1030, 700, 8191, 0), (1030, 700, 8191, 1), (777, 1300, 65521, 1), (600, 520, 131071, 0), (2048, 2048, 65521, 2)]:
    A = uniform_matrix(m, k, 5, p)
    C = adj.adjprod(torch.from_numpy(A.view(np.int32)).cuda(), p, depth=d)
    torch.cuda.synchronize()
    got = C.cpu().numpy().view(np.uint32); ref = oracle.syrk_t(A, p)
    lo = np.tril(np.ones((m, m), dtype=bool))
    print(m, k, p, d, "OK" if np.array_equal(got[lo], ref[lo]) else f"MISMATCH {(got[lo]!=ref[lo]).sum()}", flush=True)
