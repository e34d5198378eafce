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
