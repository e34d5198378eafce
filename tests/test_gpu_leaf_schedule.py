"""The leaf's job-scheduling variants change only when jobs start and in which K order a job's
units load their k-blocks, never the result (claim-wave gate, K-direction
alternation, accumulator order).  A 16384² problem at depth 1 is a launch of 1840 wide-N jobs
(> 16 waves: dynamic claiming, the gate on); each variant runs in its own process (the switches
are read once per process) and must return the same Low(C) bit for bit, and the default's
sampled rows (the last rows of every 256-row band and the ragged end) must equal the oracle's
(Lemma lem:transp)."""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
from inputs import uniform_matrix

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
M = K = 16384
PRIMES = (65521, 8191)   # s8 / u8 scheme (alternation on by default) and K7 (off)

CHILD = r"""
import hashlib, json, sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_2101_01025_b200 as adj
from inputs import uniform_matrix
m = k = int(sys.argv[2])
rows = [int(x) for x in sys.argv[5].split(",")]
out = {}
for p in (int(x) for x in sys.argv[4].split(",")):
    A = torch.from_numpy(uniform_matrix(m, k, seed=5, p=p).astype(np.int32)).cuda().to(torch.int16)
    C = torch.zeros((m, m), dtype=torch.int16, device="cuda")
    adj.adjprod_modp_ex(m, k, p, 0, A, k, C, m, depth=1, flags=adj.ADJ_IN_U16 | adj.ADJ_OUT_U16)
    torch.cuda.synchronize()
    L = torch.tril(C).cpu().numpy()
    out[p] = hashlib.sha256(L.tobytes()).hexdigest()
    np.save(f"{sys.argv[3]}_{p}.npy", L[rows])
json.dump(out, open(sys.argv[3] + ".json", "w"))
"""

VARIANTS = {
    "default": {},
    "no_gate_claim_ahead": {"ADJ_LEAF_GATE": "0"},
    "claim_at_start_no_gate": {"ADJ_LEAF_GATE": "-1"},
    "hard_gate": {"ADJ_LEAF_GATE_PRE": "0"},
    "kalt_every_scheme_other_order": {"ADJ_LEAF_KALT": "2", "ADJ_ACC_ORDER": "0"},
    "leaf2_gated": {"ADJ_LEAF_WIDE": "0"},
}
ROWS = [255, 256, 4095, 8191, 8192, 12543, M - 2, M - 1]


@pytest.fixture(scope="module")
def results(tmp_path_factory):
    import json
    d = tmp_path_factory.mktemp("sched")
    out = {}
    for name, env in VARIANTS.items():
        e = dict(os.environ)
        e.update(env)
        stem = str(d / name)
        r = subprocess.run([sys.executable, "-c", CHILD, ROOT, str(M), stem, ",".join(map(str, PRIMES)),
                            ",".join(map(str, ROWS))], env=e, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, (name, r.stderr[-2000:])
        h = json.load(open(stem + ".json"))
        out[name] = {p: (h[str(p)], np.load(f"{stem}_{p}.npy")) for p in PRIMES}
    return out


@pytest.mark.parametrize("p", PRIMES)
@pytest.mark.parametrize("name", [v for v in VARIANTS if v != "default"])
def test_schedule_variant_same_result(results, name, p):
    """sha256 of the whole Low(C) (uint16) equals the default's"""
    assert results[name][p][0] == results["default"][p][0], name


@pytest.mark.parametrize("p", PRIMES)
def test_schedule_default_sampled_rows_vs_oracle(results, p):
    A = uniform_matrix(M, K, seed=5, p=p)
    got = results["default"][p][1].view(np.uint16).astype(np.uint32)
    for i, r in enumerate(ROWS):
        ref = oracle.syrk_t(A[: r + 1], p, rows=(r, r + 1))   # row r of Low(C) needs rows 0..r of A
        assert np.array_equal(got[i, : r + 1], ref[r, : r + 1]), (p, r)
