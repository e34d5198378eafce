"""B200-native C = A phi(A) mod p (arXiv 2101.01025, Alg. alg:MIAHMM + Alg. alg:2M).

The product path is libadjprod.so (include/adjprod.h); this package is its thin binding
(``_lib``: the C ABI under the same names) plus torch-tensor conveniences that only allocate
output memory and marshal pointers.  There is no CPU fallback: without the built library or
without an sm_100 GPU every call raises.
"""
from __future__ import annotations

from ._lib import (ADJ_IN_U16, ADJ_OUT_U16, ADJ_LOW_MEM, ADJ_DIST_P2P, ADJ_DIST_TILES, ADJ_FILL_UPPER, ADJ_HERK_ALG1, ADJ_PHI_H, ADJ_PHI_Q, ADJ_PHI_T, AdjError, adj_comm_destroy, adj_comm_get_unique_id,
                   adj_comm_init, adj_launch_count, adj_launch_count_reset, adj_mod_lower, adj_profile_enable, adj_profile_read, adj_skew_unitary, adj_sos,
                   adj_dist_kslice, adj_elem_bytes, adj_shard_layout, adj_shard_rows, adjprod_modp_dist_partial, adj_shard_pack, adj_ipc_export, adj_ipc_open, adj_ipc_close, adj_sum_partials, adjprod_modp, adjprod_modp_partial, adjprod_modp_shard, adjprod_modp_auto_depth, adjprod_modp_leaf_tile, adjprod_modp_dist, adjprod_modp_ex, adjprod_modp_syrk,
                   adjprod_modp_workspace_size, gemm_modp, lib)

__all__ = ["ADJ_IN_U16", "ADJ_OUT_U16", "ADJ_LOW_MEM", "adj_shard_pack", "adj_ipc_export", "adj_ipc_open", "adj_ipc_close", "ADJ_DIST_P2P", "adjprod_modp_partial", "adj_sum_partials", "ADJ_DIST_TILES", "adjprod_modp_shard", "adj_shard_layout", "ADJ_PHI_T", "ADJ_PHI_H", "ADJ_PHI_Q", "ADJ_FILL_UPPER", "ADJ_HERK_ALG1", "AdjError", "adjprod_modp", "adjprod_modp_ex", "adjprod_modp_syrk", "adjprod_modp_leaf_tile",
           "adjprod_modp_workspace_size", "adjprod_modp_auto_depth", "gemm_modp", "adj_skew_unitary", "adj_sos",
           "adj_mod_lower", "adj_dist_kslice", "adj_elem_bytes", "adj_shard_rows", "adjprod_modp_dist_partial", "adj_comm_get_unique_id", "adj_comm_init", "adj_comm_destroy", "adjprod_modp_dist",
           "adj_launch_count", "adj_launch_count_reset", "adj_profile_enable", "adj_profile_read", "lib", "adjprod", "gemm"]


def adjprod(A, p: int, phi: str = "T", depth: int = -1, fill_upper: bool = False, out=None, workspace=None,
            stream=None, herk: str = "2m", out16: bool = False, low_mem: bool = False):
    """Low(A phi(A)) mod p for a CUDA int32/uint32 tensor A (m x k; m x k x 2 for phi='H', GF(p^2);
    m x k x 4 for phi='Q', quaternions over GF(p)).

    Returns an m x m (x 2) int32 tensor holding uint32 residues; its strict upper triangle is
    whatever `out` held (zeros for a fresh output) unless fill_upper.  For phi='H', herk='alg1'
    selects one level of Alg. alg:MIAHMM directly over GF(p^2) (ADJ_HERK_ALG1) instead of 2M.
    Compact residues (phi='T', p < 2^16): a 2-byte A (int16/uint16 tensor) is read as uint16
    (ADJ_IN_U16); out16 (or a 2-byte `out`) writes Low(C) as uint16 (ADJ_OUT_U16).  low_mem
    selects the low-memory temporary schedule where it applies (ADJ_LOW_MEM)."""
    import torch
    assert A.is_cuda and A.element_size() in (2, 4)
    ph = {"T": ADJ_PHI_T, "H": ADJ_PHI_H, "Q": ADJ_PHI_Q}[phi.upper()]
    w = {ADJ_PHI_T: 1, ADJ_PHI_H: 2, ADJ_PHI_Q: 4}[ph]
    m, k = A.shape[0], A.shape[1]
    lda = A.stride(0) // w
    out16 = out16 or (out is not None and out.element_size() == 2)
    if out is None:
        shape = (m, m) if w == 1 else (m, m, w)
        out = torch.zeros(shape, dtype=torch.int16 if out16 else torch.int32, device=A.device)
    ldc = out.stride(0) // w
    nbytes = workspace.numel() * workspace.element_size() if workspace is not None else 0
    flags = ((ADJ_FILL_UPPER if fill_upper else 0) | (ADJ_HERK_ALG1 if herk == "alg1" else 0)
             | (ADJ_IN_U16 if A.element_size() == 2 else 0) | (ADJ_OUT_U16 if out16 else 0)
             | (ADJ_LOW_MEM if low_mem else 0))
    adjprod_modp_ex(m, k, p, ph, A, lda, out, ldc, depth=depth, flags=flags,
                    workspace=workspace, workspace_bytes=nbytes, stream=stream)
    return out


def gemm(A, B, p: int, out=None, stream=None):
    """A B^T mod p for CUDA int32/uint32 tensors A (m x k), B (n x k)."""
    import torch
    m, k = A.shape
    n = B.shape[0]
    if out is None:
        out = torch.empty((m, n), dtype=torch.int32, device=A.device)
    gemm_modp(m, n, k, p, A, A.stride(0), B, B.stride(0), out, out.stride(0), stream=stream)
    return out
