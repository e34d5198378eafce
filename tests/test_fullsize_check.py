"""Pins of the whole-output checks used by the full-size GPU parity tests (tests/fullsize_check.py)
against the O1 oracle on small inputs, in all three rings: each accepts the oracle's Low(C) and
rejects it after a single entry is changed by one (CPU only)."""
import numpy as np
import pytest
import torch

import oracle
from fullsize_check import exact_low_mismatches, freivalds_low
from inputs import uniform_matrix, uniform_matrix_ext, uniform_matrix_quat

CASES = [(1, uniform_matrix, oracle.syrk_t), (2, uniform_matrix_ext, oracle.syrk_h), (4, uniform_matrix_quat, oracle.syrk_q)]


@pytest.mark.parametrize("w,gen,f", CASES, ids=["T", "H", "Q"])
@pytest.mark.parametrize("p", [7, 8191, 65519])
def test_checks_accept_oracle_and_reject_one_wrong_entry(w, gen, f, p):
    if w > 1 and p % 4 != 3:
        pytest.skip("GF(p)[i]/(i^2+1) needs p = 3 mod 4")
    m, k = 300, 170
    A = gen(m, k, 3, p).reshape(m, k, w)
    C = f(A if w > 1 else A[..., 0], p).reshape(m, m, w)
    At = torch.from_numpy(A.view(np.int32))
    assert freivalds_low(A, C, p, w, block=128)
    assert exact_low_mismatches(torch, At, torch.from_numpy(C.view(np.int32)), p, w, block=128) == 0
    for (i, j) in ((211, 97), (299, 299), (5, 0)):
        for q in range(w):
            C2 = C.copy()
            C2[i, j, q] = (C2[i, j, q] + 1) % p
            assert not freivalds_low(A, C2, p, w, block=128), (i, j, q)
            assert exact_low_mismatches(torch, At, torch.from_numpy(C2.view(np.int32)), p, w, block=128) == 1
    # the strict upper triangle is never read
    C3 = C.copy()
    C3[3, 200] = 1
    assert freivalds_low(A, C3, p, w, block=128)
