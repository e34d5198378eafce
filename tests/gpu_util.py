"""Helpers for the -m gpu parity tests: host<->device marshalling only (no method arithmetic)."""
import numpy as np


def to_dev(a: np.ndarray):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int32)).cuda()


def to_host(t) -> np.ndarray:
    import torch
    torch.cuda.synchronize()
    return t.cpu().numpy().view(np.uint32)


def low(C: np.ndarray) -> np.ndarray:
    m = C.shape[0]
    mask = np.tril(np.ones((m, m), dtype=bool))
    if C.ndim == 3:
        mask = mask[:, :, None]
    return np.where(mask, C, 0)


def freivalds(Ah, Cl, p, nvec=2, seed=0):
    """Low(C) symmetric completion times r vs A (A^T r), all mod p, exact in float64."""
    rng = np.random.default_rng(seed)
    m = Cl.shape[0]
    Af = Ah.astype(np.float64)
    for _ in range(nvec):
        r = rng.integers(0, p, size=m).astype(np.float64)
        t = np.mod(Af.T @ r, p)
        rhs = np.mod(Af @ t, p)
        lhs = np.zeros(m)
        for r0 in range(0, m, 4096):                     # C r from Low(C), blocked rows
            r1 = min(m, r0 + 4096)
            L = np.tril(Cl[r0:r1].astype(np.float64), k=r0)   # entries j <= i of rows r0..r1
            lhs[r0:r1] += L @ r
            # upper part: C[i][j] for j > i equals Low(C)[j][i]
            lhs += np.tril(Cl[r0:r1].astype(np.float64), k=r0 - 1).T @ r[r0:r1]
        if not np.array_equal(np.mod(lhs, p), rhs):
            return False
    return True


