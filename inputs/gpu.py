"""Device-side twin of inputs.gen.uniform_residues (loads inputs/_gen.so built by build())."""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "_gen.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run __graft_entry__.build()")
        lib = ctypes.CDLL(path)
        lib.adjgen_uniform.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64,
                                       ctypes.c_uint32, ctypes.c_uint64, ctypes.c_void_p]
        lib.adjgen_uniform.restype = ctypes.c_int
        _LIB = lib
    return _LIB


def uniform_residues_cuda(out, seed: int, p: int, start: int = 0):
    """Fill a contiguous CUDA uint32/int32 torch tensor with the seeded residues."""
    import torch
    assert out.is_cuda and out.is_contiguous() and out.element_size() == 4
    stream = torch.cuda.current_stream(out.device).cuda_stream
    rc = _lib().adjgen_uniform(out.data_ptr(), out.numel(), seed & ((1 << 64) - 1), p,
                               start, stream)
    if rc != 0:
        raise RuntimeError(f"adjgen_uniform failed: {rc}")
    return out
