"""Thin ctypes binding of include/adjprod.h (argument marshalling only).

Every step of the hot path runs in libadjprod.so's sm_100a kernels; there is no CPU or
PyTorch fallback.  If the library is missing, every call raises.
"""
from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libadjprod.so")

ADJ_PHI_T = 0
ADJ_PHI_H = 1
ADJ_PHI_Q = 2
ADJ_FILL_UPPER = 1
ADJ_HERK_ALG1 = 2
ADJ_DIST_TILES = 4
ADJ_DIST_P2P = 8
ADJ_IN_U16 = 16
ADJ_OUT_U16 = 32
ADJ_LOW_MEM = 64
ADJ_IPC_RECORD_BYTES = 72
STATUS = {0: "ADJ_OK", 1: "ADJ_ERR_INVALID_VALUE", 2: "ADJ_ERR_UNSUPPORTED_MODULUS", 3: "ADJ_ERR_WORKSPACE",
          4: "ADJ_ERR_CUDA", 5: "ADJ_ERR_NCCL", 6: "ADJ_ERR_ARCH"}

# every symbol include/adjprod.h declares (checked by tests/test_abi.py)
EXPORTS = ["adjprod_modp", "adjprod_modp_ex", "adjprod_modp_syrk", "adjprod_modp_workspace_size", "adjprod_modp_auto_depth", "adjprod_modp_leaf_tile",
           "gemm_modp", "adj_skew_unitary", "adj_sos", "adj_mod_lower", "adj_comm_get_unique_id",
           "adj_comm_init", "adj_comm_destroy", "adjprod_modp_dist", "adj_dist_kslice", "adj_elem_bytes", "adjprod_modp_dist_partial", "adjprod_modp_shard", "adj_shard_layout", "adj_shard_rows", "adjprod_modp_partial", "adj_sum_partials", "adj_shard_pack", "adj_ipc_export", "adj_ipc_open", "adj_ipc_close", "adj_status_string", "adj_last_error",
           "adj_launch_count", "adj_launch_count_reset", "adj_profile_enable", "adj_profile_read"]


class AdjError(RuntimeError):
    def __init__(self, status: int, fn: str, detail: str):
        self.status = status
        super().__init__(f"{fn}: {STATUS.get(status, status)}: {detail}")


class adj_opts_t(ctypes.Structure):
    _fields_ = [("depth", ctypes.c_int), ("flags", ctypes.c_uint32), ("workspace", ctypes.c_void_p),
                ("workspace_bytes", ctypes.c_size_t)]


_LIB = None


def lib() -> ctypes.CDLL:
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
        L = ctypes.CDLL(LIB_PATH)
        i64, u32, vp, ci = ctypes.c_int64, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_int
        sig = {
            "adjprod_modp": [i64, i64, u32, ci, vp, i64, vp, i64, vp],
            "adjprod_modp_ex": [i64, i64, u32, ci, vp, i64, vp, i64, ctypes.POINTER(adj_opts_t), vp],
            "adjprod_modp_syrk": [i64, i64, u32, ci, u32, vp, i64, u32, vp, i64, ctypes.POINTER(adj_opts_t), vp],
            "adjprod_modp_workspace_size": [i64, i64, u32, ci, ctypes.POINTER(adj_opts_t),
                                            ctypes.POINTER(ctypes.c_size_t)],
            "adjprod_modp_auto_depth": [i64, i64, u32, ci, ctypes.POINTER(ci)],
            "adjprod_modp_leaf_tile": [i64, i64, u32, ci, ctypes.POINTER(adj_opts_t), ctypes.POINTER(ci)],
            "gemm_modp": [i64, i64, i64, u32, vp, i64, vp, i64, vp, i64, vp],
            "adj_skew_unitary": [u32, ci, ctypes.POINTER(ci), ctypes.POINTER(u32), ctypes.POINTER(u32)],
            "adj_sos": [u32, u32, ctypes.POINTER(u32), ctypes.POINTER(u32)],
            "adj_mod_lower": [i64, u32, ci, vp, i64, vp],
            "adj_comm_get_unique_id": [ctypes.c_char_p],
            "adj_comm_init": [ci, ctypes.c_char_p, ci, ctypes.POINTER(vp)],
            "adj_comm_destroy": [vp],
            "adjprod_modp_dist": [i64, i64, u32, ci, vp, i64, vp, i64, ci, vp, ctypes.POINTER(adj_opts_t), vp],
            "adj_dist_kslice": [i64, ci, ci, ctypes.POINTER(i64), ctypes.POINTER(i64)],
            "adj_elem_bytes": [ci, u32, ctypes.POINTER(i64)],
            "adjprod_modp_dist_partial": [i64, i64, u32, ci, vp, i64, vp, i64, ci, ci, ctypes.POINTER(adj_opts_t), vp],
            "adj_shard_rows": [i64, i64, u32, ci, ci, ci, ctypes.POINTER(i64), i64, ctypes.POINTER(i64)],
            "adjprod_modp_shard": [i64, i64, u32, ci, vp, i64, vp, i64, ci, ci, ctypes.POINTER(adj_opts_t), vp],
            "adjprod_modp_partial": [i64, i64, u32, ci, vp, i64, vp, i64, ctypes.POINTER(adj_opts_t), vp],
            "adj_sum_partials": [i64, u32, vp, i64, i64, ci, vp, i64, vp],
            "adj_shard_pack": [i64, i64, u32, ci, ci, ci, vp, i64, vp, ci, vp],
            "adj_ipc_export": [vp, ctypes.c_char_p],
            "adj_ipc_open": [ctypes.c_char_p, ctypes.POINTER(vp)],
            "adj_ipc_close": [vp],
            "adj_shard_layout": [i64, i64, u32, ci, ci, ci, ctypes.POINTER(i64), i64, ctypes.POINTER(i64),
                                 ctypes.POINTER(i64)],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = ci
        L.adj_status_string.argtypes = [ci]
        L.adj_status_string.restype = ctypes.c_char_p
        L.adj_last_error.restype = ctypes.c_char_p
        L.adj_launch_count.restype = ctypes.c_uint64
        L.adj_profile_enable.argtypes = [ci]
        L.adj_profile_enable.restype = None
        L.adj_profile_read.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_uint64)]
        L.adj_profile_read.restype = ci
        _LIB = L
    return _LIB


def _check(status: int, fn: str):
    if status != 0:
        raise AdjError(status, fn, lib().adj_last_error().decode())


def _ptr(x):
    if x is None:
        return None
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    return int(x)


def _stream(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if hasattr(stream, "cuda_stream"):
        return stream.cuda_stream
    return int(stream)


def _opts(depth=-1, flags=0, workspace=None, workspace_bytes=0):
    return adj_opts_t(depth, flags, _ptr(workspace), workspace_bytes)


# ---------------------------------------------------------------------- C ABI, same names
def adjprod_modp(m, k, p, phi, A, lda, C, ldc, stream=None):
    _check(lib().adjprod_modp(m, k, p, phi, _ptr(A), lda, _ptr(C), ldc, _stream(stream)), "adjprod_modp")


def adjprod_modp_ex(m, k, p, phi, A, lda, C, ldc, depth=-1, flags=0, workspace=None, workspace_bytes=0,
                    stream=None):
    o = _opts(depth, flags, workspace, workspace_bytes)
    _check(lib().adjprod_modp_ex(m, k, p, phi, _ptr(A), lda, _ptr(C), ldc, ctypes.byref(o), _stream(stream)),
           "adjprod_modp_ex")


def adjprod_modp_syrk(m, k, p, phi, alpha, A, lda, beta, C, ldc, depth=-1, flags=0, workspace=None,
                      workspace_bytes=0, stream=None):
    o = _opts(depth, flags, workspace, workspace_bytes)
    _check(lib().adjprod_modp_syrk(m, k, p, phi, alpha % p, _ptr(A), lda, beta % p, _ptr(C), ldc, ctypes.byref(o),
                                   _stream(stream)), "adjprod_modp_syrk")


def adjprod_modp_workspace_size(m, k, p, phi, depth=-1, flags=0) -> int:
    o = _opts(depth, flags)
    n = ctypes.c_size_t(0)
    _check(lib().adjprod_modp_workspace_size(m, k, p, phi, ctypes.byref(o), ctypes.byref(n)),
           "adjprod_modp_workspace_size")
    return n.value


def adjprod_modp_auto_depth(m, k, p, phi) -> int:
    d = ctypes.c_int(0)
    _check(lib().adjprod_modp_auto_depth(m, k, p, phi, ctypes.byref(d)), "adjprod_modp_auto_depth")
    return d.value


def adjprod_modp_leaf_tile(m, k, p, phi, depth=-1, flags=0) -> int:
    o = _opts(depth, flags)
    t = ctypes.c_int(0)
    _check(lib().adjprod_modp_leaf_tile(m, k, p, phi, ctypes.byref(o), ctypes.byref(t)), "adjprod_modp_leaf_tile")
    return t.value


def gemm_modp(m, n, k, p, A, lda, B, ldb, C, ldc, stream=None):
    _check(lib().gemm_modp(m, n, k, p, _ptr(A), lda, _ptr(B), ldb, _ptr(C), ldc, _stream(stream)), "gemm_modp")


def adj_skew_unitary(p, phi=ADJ_PHI_T):
    kind, a, b = ctypes.c_int(0), ctypes.c_uint32(0), ctypes.c_uint32(0)
    _check(lib().adj_skew_unitary(p, phi, ctypes.byref(kind), ctypes.byref(a), ctypes.byref(b)), "adj_skew_unitary")
    return kind.value, a.value, b.value


def adj_sos(p, k):
    a, b = ctypes.c_uint32(0), ctypes.c_uint32(0)
    _check(lib().adj_sos(p, k, ctypes.byref(a), ctypes.byref(b)), "adj_sos")
    return a.value, b.value


def adj_mod_lower(m, p, phi, X, ldx, stream=None):
    _check(lib().adj_mod_lower(m, p, phi, _ptr(X), ldx, _stream(stream)), "adj_mod_lower")


def adj_comm_get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().adj_comm_get_unique_id(buf), "adj_comm_get_unique_id")
    return buf.raw


def adj_comm_init(nranks: int, uid: bytes, rank: int):
    c = ctypes.c_void_p(0)
    _check(lib().adj_comm_init(nranks, uid, rank, ctypes.byref(c)), "adj_comm_init")
    return c.value


def adj_comm_destroy(comm):
    _check(lib().adj_comm_destroy(comm), "adj_comm_destroy")


def adj_ipc_export(ptr) -> bytes:
    buf = ctypes.create_string_buffer(ADJ_IPC_RECORD_BYTES)
    _check(lib().adj_ipc_export(_ptr(ptr), buf), "adj_ipc_export")
    return buf.raw


def adj_ipc_open(rec: bytes) -> int:
    out = ctypes.c_void_p(0)
    _check(lib().adj_ipc_open(rec, ctypes.byref(out)), "adj_ipc_open")
    return out.value


def adj_ipc_close(ptr):
    _check(lib().adj_ipc_close(_ptr(ptr)), "adj_ipc_close")


def adjprod_modp_dist(m, k, p, phi, A, lda, C, ldc, root, comm, depth=-1, flags=0, stream=None):
    o = _opts(depth, flags)
    _check(lib().adjprod_modp_dist(m, k, p, phi, _ptr(A), lda, _ptr(C), ldc, root, comm, ctypes.byref(o),
                                   _stream(stream)), "adjprod_modp_dist")


def adjprod_modp_shard(m, k, p, phi, A, lda, C, ldc, rank, nranks, depth=-1, workspace=None, workspace_bytes=0,
                       stream=None, flags=0):
    o = _opts(depth, flags, workspace, workspace_bytes)
    _check(lib().adjprod_modp_shard(m, k, p, phi, _ptr(A), lda, _ptr(C), ldc, rank, nranks, ctypes.byref(o),
                                    _stream(stream)), "adjprod_modp_shard")


def adjprod_modp_partial(m, k, p, phi, A, lda, R, ldr, depth=-1, stream=None, flags=0):
    o = _opts(depth, flags)
    _check(lib().adjprod_modp_partial(m, k, p, phi, _ptr(A), lda, _ptr(R), ldr, ctypes.byref(o), _stream(stream)),
           "adjprod_modp_partial")


def adj_sum_partials(m, p, R, ldr, stride, n, C, ldc, stream=None):
    _check(lib().adj_sum_partials(m, p, _ptr(R), ldr, stride, n, _ptr(C), ldc, _stream(stream)), "adj_sum_partials")


def adj_shard_pack(m, k, p, rank, nranks, C, ldc, buf, unpack=False, depth=-1, stream=None):
    _check(lib().adj_shard_pack(m, k, p, depth, rank, nranks, _ptr(C), ldc, _ptr(buf), 1 if unpack else 0,
                                _stream(stream)), "adj_shard_pack")


def adj_shard_layout(m, k, p, rank, nranks, depth=-1):
    """[(row0, col0, rows, cols, lower), ...] of the regions of C that `rank` writes (host)."""
    n, e = ctypes.c_int64(0), ctypes.c_int64(0)
    _check(lib().adj_shard_layout(m, k, p, depth, rank, nranks, None, 0, ctypes.byref(n), ctypes.byref(e)),
           "adj_shard_layout")
    buf = (ctypes.c_int64 * max(1, 5 * n.value))()
    _check(lib().adj_shard_layout(m, k, p, depth, rank, nranks, buf, n.value, ctypes.byref(n), ctypes.byref(e)),
           "adj_shard_layout")
    return [tuple(buf[5 * i: 5 * i + 5]) for i in range(n.value)]


def adj_shard_rows(m, k, p, rank, nranks, depth=-1):
    """[(lo, hi), ...] rows of the top-level operands `rank` pre-adds in adjprod_modp_shard (host)."""
    n = ctypes.c_int64(0)
    _check(lib().adj_shard_rows(m, k, p, depth, rank, nranks, None, 0, ctypes.byref(n)), "adj_shard_rows")
    buf = (ctypes.c_int64 * max(1, 2 * n.value))()
    _check(lib().adj_shard_rows(m, k, p, depth, rank, nranks, buf, n.value, ctypes.byref(n)), "adj_shard_rows")
    return [(buf[2 * i], buf[2 * i + 1]) for i in range(n.value)]


def adjprod_modp_dist_partial(m, k, p, phi, A, lda, R, ldr, rank, nranks, depth=-1, flags=0, stream=None):
    o = _opts(depth, flags)
    _check(lib().adjprod_modp_dist_partial(m, k, p, phi, _ptr(A), lda, _ptr(R), ldr, rank, nranks, ctypes.byref(o),
                                           _stream(stream)), "adjprod_modp_dist_partial")


def adj_dist_kslice(k, nranks, rank):
    k0, k1 = ctypes.c_int64(0), ctypes.c_int64(0)
    _check(lib().adj_dist_kslice(k, nranks, rank, ctypes.byref(k0), ctypes.byref(k1)), "adj_dist_kslice")
    return k0.value, k1.value


def adj_elem_bytes(phi, flags=0) -> int:
    """bytes of one element of A as the entry points read it (rank r's k-slice offset = k0 x this)"""
    b = ctypes.c_int64(0)
    _check(lib().adj_elem_bytes(phi, flags, ctypes.byref(b)), "adj_elem_bytes")
    return b.value


def adj_launch_count() -> int:
    return int(lib().adj_launch_count())


def adj_launch_count_reset():
    lib().adj_launch_count_reset()


def adj_profile_enable(on: bool = True):
    lib().adj_profile_enable(1 if on else 0)


PROFILE_CLASSES = ("leaf", "preadd", "combine", "other")


def adj_profile_read():
    """{class: (ms, launches)} since the last read (synchronises on the recorded events)."""
    ms = (ctypes.c_double * 4)()
    n = (ctypes.c_uint64 * 4)()
    _check(lib().adj_profile_read(ms, n), "adj_profile_read")
    return {PROFILE_CLASSES[i]: (ms[i], int(n[i])) for i in range(4)}
