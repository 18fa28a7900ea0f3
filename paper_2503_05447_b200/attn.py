"""Softmax attention over the C-ABI (host mirror of attention.hpp / parallel.hpp).

  softmax_attention_parallel(q, k, v, causal, row_offset)   attention.hpp:18-38
  sp_attention_rank(comm, q_loc, k_loc, v_loc, n_total)     parallel.hpp:380-387
Batched device layout [B, N, H, D] bf16 (D = 128); a single head is (N, d) like the reference.
"""
import ctypes

import torch

from . import _lib
from .lsm import _DTYPES, _workspace


def _bind():
    L = _lib.lib()
    if getattr(L, "_attn_bound", False):
        return L
    vp, sz, i = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int
    L.lmoe_attn_fwd.restype = i
    L.lmoe_attn_fwd.argtypes = [i, i, i, i, i, i, vp, vp, vp, vp, i, vp]
    L.lmoe_sp_attn_workspace_size.restype = sz
    L.lmoe_sp_attn_workspace_size.argtypes = [i, i, i, i, i, i]
    L.lmoe_sp_attn_fwd.restype = i
    L.lmoe_sp_attn_fwd.argtypes = [i, i, i, i, i, vp, vp, vp, vp, vp, i, i, vp, sz, vp]
    L.lmoe_sp_attn_last_gather_elements.restype = ctypes.c_longlong
    L._attn_bound = True
    return L


def softmax_attention_parallel(q, k, v, causal=True, row_offset=0, out=None, stream=None):
    """O = softmax(Q K^T / sqrt(d), mask j <= i + row_offset) V for [B, Nq|Nk, H, D] bf16."""
    L = _bind()
    if q.dim() == 2:  # one head, (N, d) as in the reference
        return softmax_attention_parallel(q[None, :, None], k[None, :, None], v[None, :, None], causal,
                                          row_offset)[0, :, 0]
    B, Nq, H, D = q.shape
    Nk = k.shape[1]
    if k.shape != v.shape or k.shape[0] != B or k.shape[2:] != q.shape[2:]:
        raise RuntimeError("shape mismatch in softmax_attention_parallel: %s vs %s"
                           % (tuple(q.shape), tuple(k.shape)))
    q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
    o = out if out is not None else torch.empty_like(q)
    st = stream if stream is not None else torch.cuda.current_stream(q.device).cuda_stream
    off = int(row_offset) if causal else Nk
    _lib.check(L.lmoe_attn_fwd(B, Nq, Nk, H, D, _DTYPES[q.dtype], _lib.ptr(q), _lib.ptr(k), _lib.ptr(v),
                               _lib.ptr(o), off, ctypes.c_void_p(st)))
    return o


def sp_attention_rank(comm, q_loc, k_loc, v_loc, n_total, out=None, stream=None):
    """This rank's causal attention output for its chunk_range slice of an n_total sequence."""
    L = _bind()
    B, N, H, D = q_loc.shape
    dt = _DTYPES[q_loc.dtype]
    ws = _workspace(L.lmoe_sp_attn_workspace_size(B, n_total, H, D, dt, comm.world), q_loc.device)
    o = out if out is not None else torch.empty_like(q_loc)
    st = stream if stream is not None else torch.cuda.current_stream(q_loc.device).cuda_stream
    _lib.check(L.lmoe_sp_attn_fwd(B, n_total, H, D, dt, _lib.ptr(q_loc), _lib.ptr(k_loc), _lib.ptr(v_loc),
                                  _lib.ptr(o), comm.handle, comm.rank, comm.world, _lib.ptr(ws), ws.numel(),
                                  ctypes.c_void_p(st)))
    return o


def last_gather_elements():
    return _bind().lmoe_sp_attn_last_gather_elements()
