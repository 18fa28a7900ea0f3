"""Host mirror of the reference LSM interface (lsm.hpp) over the C-ABI.

Names, argument meaning and error texts follow /root/reference/proj/include/lmoe/lsm.hpp:
  LsmInstance / FeatureMap / LsmSpec.make / LsmGates / MemoryState  (lsm.hpp:30-273)
  lsm_forward_chunked(q, k, v, gates, spec, chunk_size, final_state) (lsm.hpp:668-708)
Tensors are torch CUDA tensors (torch is plumbing for device memory and streams only).
A single head is (N, d) exactly like the reference; the batched device layout is
[B, N, H, d] (per batch row, the reference's (N x H*d) projection, model.hpp:234-243).
"""
import ctypes
import dataclasses
import math
from typing import Optional

import torch

from . import _lib

INSTANCES = ["bla", "lightning", "retnet", "gla", "deltanet", "gated_deltanet", "rebased",
             "gfw", "gateloop", "ttt", "titans", "s4", "mamba", "mamba2", "hgrn2", "rwkv6",
             "rwkv7"]


class LsmInstance:
    BLA, LIGHTNING, RETNET, GLA, REBASED, MAMBA2, HGRN2, RWKV6 = 0, 1, 2, 3, 6, 13, 14, 15
    # no chunk-parallel form (lsm_forward_recurrent)
    DELTANET, GATED_DELTANET, GFW, GATELOOP, TTT, TITANS, S4, MAMBA, RWKV7 = 4, 5, 7, 8, 9, 10, 11, 12, 16
    RECURRENT = (4, 5, 7, 8, 9, 10, 11, 12, 16)


class FeatureMap:
    IDENTITY, ELU_PLUS_ONE, SQUARED = 0, 1, 2


@dataclasses.dataclass
class LsmSpec:
    """lmoe::LsmSpec (lsm.hpp:126-204).  mamba2_a_raw is per head ([H] tensor or float)."""
    instance: int = LsmInstance.BLA
    feature_map: int = FeatureMap.IDENTITY
    use_normalizer: bool = False
    d_k: int = 0
    d_v: int = 0
    scalar_decay: float = 1.0
    mamba2_a_raw: Optional[torch.Tensor] = None
    # static parameters of S4 / Mamba (LsmSpec::make, lsm.hpp:166-177), per head:
    # s4_delta_raw, s4_b [H, d_k]; s4_A_raw, mamba_A_raw [H, d_k, d_v] (fp32)
    s4_delta_raw: Optional[torch.Tensor] = None
    s4_b: Optional[torch.Tensor] = None
    s4_A_raw: Optional[torch.Tensor] = None
    mamba_A_raw: Optional[torch.Tensor] = None

    @staticmethod
    def make(instance, d_k, d_v=None):
        """Defaults of LsmSpec::make (lsm.hpp:146-165)."""
        if isinstance(instance, str):
            instance = INSTANCES.index(instance)
        s = LsmSpec(instance=instance, d_k=d_k, d_v=d_v or d_k)
        if instance == LsmInstance.BLA:
            s.feature_map, s.use_normalizer = FeatureMap.ELU_PLUS_ONE, True
        elif instance == LsmInstance.REBASED:
            s.feature_map, s.use_normalizer = FeatureMap.SQUARED, True
        elif instance == LsmInstance.LIGHTNING:
            s.scalar_decay = 0.95
        elif instance == LsmInstance.RETNET:
            s.scalar_decay = 1.0 - 1.0 / 32.0
        return s

    def name(self):
        return INSTANCES[self.instance]


@dataclasses.dataclass
class LsmGates:
    """lmoe::LsmGates (lsm.hpp:206-247): a_pre [.., N, d_k] (TokenVector, RWKV7, Mamba) or
    [.., N] (DeltaNet, GatedDeltaNet, Titans); b_pre [.., N]; alpha_pre [.., N, d_k] and
    beta_pre [.., N, d_v] (GFW, GateLoop)."""
    a_pre: Optional[torch.Tensor] = None
    b_pre: Optional[torch.Tensor] = None
    alpha_pre: Optional[torch.Tensor] = None
    beta_pre: Optional[torch.Tensor] = None


@dataclasses.dataclass
class MemoryState:
    """lmoe::MemoryState (lsm.hpp:264-281): M (d_k x d_v) fp32, z (d_k) fp32 or None."""
    M: Optional[torch.Tensor] = None
    z: Optional[torch.Tensor] = None
    step: int = 0


_DTYPES = {torch.bfloat16: 1, torch.float32: 0}
_ws_cache = {}


def _workspace(nbytes, device):
    key = (device, nbytes)
    ws = _ws_cache.get(key)
    if ws is None:
        _ws_cache.clear()
        ws = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
        _ws_cache[key] = ws
    return ws


# TEST ONLY: set to True to make the scalar-decay kernels shift the within-chunk cumulative
# decay by one token (the reference's kern::chunk_decay_fault(), lsm.hpp:310-317)
TEST_DECAY_FAULT = False


def make_desc(spec, chunk_size, check=True, timing=False):
    d = _lib.LsmDesc()
    d.instance = int(spec.instance)
    d.feature_map = int(spec.feature_map)
    d.use_normalizer = int(bool(spec.use_normalizer))
    d.scalar_decay = float(spec.scalar_decay)
    d.chunk_size = int(chunk_size)
    d.flags = (1 if check else 0) | (2 if timing else 0) | (4 if TEST_DECAY_FAULT else 0)
    return d


def lsm_forward_batched(q, k, v, gates, spec, chunk_size=64, initial_state=None,
                        final_state=None, out=None, check=True, stream=None, timing=False):
    """[B,N,H,D] forward for all heads.  final_state (MemoryState) receives [B,H,D,D] / [B,H,D]."""
    B, N, H, D = q.shape
    for t in (k, v):
        if t.shape != q.shape or t.dtype != q.dtype:
            raise RuntimeError("shape mismatch in lsm_forward_chunked: %s vs %s"
                               % (tuple(q.shape), tuple(t.shape)))
    if q.dtype not in _DTYPES:
        raise RuntimeError("lsm_forward_chunked: dtype must be bf16 or fp32")
    q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
    o = out if out is not None else torch.empty_like(q)
    a_raw = None
    if spec.instance == LsmInstance.MAMBA2:
        ar = spec.mamba2_a_raw
        if ar is None:
            raise RuntimeError("LsmSpec: mamba2_a_raw required for mamba2")
        a_raw = torch.as_tensor(ar, dtype=torch.float32, device=q.device).reshape(-1).expand(H).contiguous()
    b_pre = None
    if gates is not None and gates.b_pre is not None:
        b_pre = gates.b_pre.to(torch.float32).contiguous()
    a_pre = None
    if gates is not None and gates.a_pre is not None:
        a_pre = gates.a_pre.to(q.dtype).contiguous()
    M0 = z0 = None
    if initial_state is not None:
        M0 = initial_state.M.to(torch.float32).contiguous()
        if initial_state.z is not None:
            z0 = initial_state.z.to(torch.float32).contiguous()
    M_out = z_out = None
    if final_state is not None:
        M_out = torch.empty(B, H, D, D, dtype=torch.float32, device=q.device)
        z_out = torch.empty(B, H, D, dtype=torch.float32, device=q.device) if spec.use_normalizer else None
    desc = make_desc(spec, chunk_size, check, timing)
    L = _lib.lib()
    dt = _DTYPES[q.dtype]
    nbytes = L.lmoe_lsm_fwd_workspace_size(ctypes.byref(desc), B, N, H, D, dt)
    ws = _workspace(nbytes, q.device)
    st = stream if stream is not None else torch.cuda.current_stream(q.device).cuda_stream
    rc = L.lmoe_lsm_fwd(ctypes.byref(desc), B, N, H, D, dt, _lib.ptr(q), _lib.ptr(k), _lib.ptr(v),
                        _lib.ptr(a_pre), _lib.ptr(b_pre), _lib.ptr(a_raw), _lib.ptr(M0),
                        _lib.ptr(z0), _lib.ptr(o), _lib.ptr(M_out), _lib.ptr(z_out),
                        _lib.ptr(ws), ws.numel(), ctypes.c_void_p(st))
    _lib.check(rc)
    if final_state is not None:
        final_state.M, final_state.z, final_state.step = M_out, z_out, N
    return o


def forward_plan(spec, B, N, H, D, dtype=torch.bfloat16):
    """lmoe_lsm_fwd_plan: {"fused": single-read persistent kernel?, "local": local-state output
    pass + combine + correction (no state pass)?, "segments", "seg_len", "ctas_per_head"} for a
    [B, N, H, D] forward of this spec."""
    info = (ctypes.c_int * 4)()
    desc = make_desc(spec, 64)
    _lib.check(_lib.lib().lmoe_lsm_fwd_plan(ctypes.byref(desc), B, N, H, D, _DTYPES[dtype], info))
    return {"fused": info[0] == 1, "local": info[0] == 2, "segments": info[1], "seg_len": info[2],
            "ctas_per_head": info[3]}


def lsm_forward_chunked(q, k, v, gates, spec, chunk_size, final_state=None):
    """lsm_forward_chunked (lsm.hpp:668-708) for one head: q, k (N, d_k), v (N, d_v)."""
    if q.dim() != 2:
        raise RuntimeError("lsm_forward_chunked: expects (N, d) per-head matrices")
    g = None
    if gates is not None:
        g = LsmGates(a_pre=None if gates.a_pre is None else gates.a_pre[None, :, None, :],
                     b_pre=None if gates.b_pre is None else gates.b_pre[None, :, None])
    fs = MemoryState() if final_state is not None else None
    o = lsm_forward_batched(q[None, :, None, :], k[None, :, None, :], v[None, :, None, :], g,
                            spec, chunk_size, final_state=fs)
    if final_state is not None:
        final_state.M = fs.M[0, 0]
        final_state.z = None if fs.z is None else fs.z[0, 0]
        final_state.step = q.shape[0]
    return o[0, :, 0, :]


@dataclasses.dataclass
class LsmGrads:
    """Gradients of lsm_forward_chunked w.r.t. its inputs (the reference tape's results)."""
    dq: torch.Tensor
    dk: torch.Tensor
    dv: torch.Tensor
    da_pre: Optional[torch.Tensor] = None
    db_pre: Optional[torch.Tensor] = None
    da_raw: Optional[torch.Tensor] = None
    dM0: Optional[torch.Tensor] = None
    # recurrent kinds (lsm_backward_recurrent): GFW / GateLoop gates, S4 / Mamba static parameters
    dalpha_pre: Optional[torch.Tensor] = None
    dbeta_pre: Optional[torch.Tensor] = None
    ds4_delta_raw: Optional[torch.Tensor] = None
    ds4_b: Optional[torch.Tensor] = None
    ds4_A_raw: Optional[torch.Tensor] = None
    dmamba_A_raw: Optional[torch.Tensor] = None


def _mamba_a_raw(spec, H, device):
    if spec.instance != LsmInstance.MAMBA2:
        return None
    if spec.mamba2_a_raw is None:
        raise RuntimeError("LsmSpec: mamba2_a_raw required for mamba2")
    return torch.as_tensor(spec.mamba2_a_raw, dtype=torch.float32, device=device).reshape(-1).expand(H).contiguous()


def lsm_backward_batched(q, k, v, gates, spec, dO, initial_state=None, dM_final=None,
                         chunk_size=64, check=True, stream=None, timing=False):
    """VJP of lsm_forward_batched: [B,N,H,D] q, k, v, dO (+ optional dM_final [B,H,D,D]).

    Returns LsmGrads (dq, dk, dv in the input dtype; db_pre [B,N,H] and da_raw [H] fp32 for
    Mamba2; dM0 [B,H,D,D] fp32).  Runs on the device only (lmoe_lsm_bwd)."""
    B, N, H, D = q.shape
    for t in (k, v, dO):
        if t.shape != q.shape or t.dtype != q.dtype:
            raise RuntimeError("shape mismatch in lsm backward: %s vs %s" % (tuple(q.shape), tuple(t.shape)))
    q, k, v, dO = q.contiguous(), k.contiguous(), v.contiguous(), dO.contiguous()
    dev = q.device
    a_raw = _mamba_a_raw(spec, H, dev)
    b_pre = None
    if gates is not None and gates.b_pre is not None:
        b_pre = gates.b_pre.to(torch.float32).contiguous()
    a_pre = None
    if gates is not None and gates.a_pre is not None:
        a_pre = gates.a_pre.to(q.dtype).contiguous()
    M0 = None
    if initial_state is not None and initial_state.M is not None:
        M0 = initial_state.M.to(torch.float32).contiguous()
    if spec.use_normalizer and initial_state is not None and initial_state.z is not None:
        # lmoe_lsm_bwd differentiates the forward with z_in = 0 (its C-ABI carries no z0)
        raise RuntimeError("lsm_backward_batched: a carried-in normaliser state z is not supported")
    dMf = None if dM_final is None else dM_final.to(torch.float32).contiguous()
    g = LsmGrads(dq=torch.empty_like(q), dk=torch.empty_like(k), dv=torch.empty_like(v))
    g.dM0 = torch.empty(B, H, D, D, dtype=torch.float32, device=dev)
    if spec.instance == LsmInstance.MAMBA2:
        g.db_pre = torch.empty(B, N, H, dtype=torch.float32, device=dev)
        g.da_raw = torch.empty(H, dtype=torch.float32, device=dev)
    if a_pre is not None:
        g.da_pre = torch.empty_like(a_pre)
    desc = make_desc(spec, chunk_size, check, timing)
    L = _lib.lib()
    dt = _DTYPES[q.dtype]
    nbytes = L.lmoe_lsm_bwd_workspace_size(ctypes.byref(desc), B, N, H, D, dt)
    ws = _workspace(nbytes, dev)
    st = stream if stream is not None else torch.cuda.current_stream(dev).cuda_stream
    P = _lib.ptr
    rc = L.lmoe_lsm_bwd(ctypes.byref(desc), B, N, H, D, dt, P(q), P(k), P(v), P(a_pre), P(b_pre),
                        P(a_raw), P(M0), P(dO), P(dMf), P(g.dq), P(g.dk), P(g.dv), P(g.da_pre),
                        P(g.db_pre), P(g.da_raw), P(g.dM0), P(ws), ws.numel(), ctypes.c_void_p(st))
    _lib.check(rc)
    return g


class LsmFunction(torch.autograd.Function):
    """Autograd binding: forward = lmoe_lsm_fwd, backward = lmoe_lsm_bwd (device only).

    LsmFunction.apply(q, k, v, b_pre, spec, chunk_size[, a_pre, a_raw]): the gate tensors are
    autograd inputs -- b_pre [B,N,H] (Mamba2), a_pre [B,N,H,D] (GLA / HGRN2 / RWKV6) and a_raw
    [H] (the Mamba2 decay parameter; defaults to spec.mamba2_a_raw, whose gradient is then
    dropped, as for any non-input)."""

    @staticmethod
    def forward(ctx, q, k, v, b_pre, spec, chunk_size, *extra):
        import copy
        a_pre = extra[0] if len(extra) > 0 else None
        a_raw = extra[1] if len(extra) > 1 else None
        sp = spec
        if a_raw is not None:
            sp = copy.copy(spec)
            sp.mamba2_a_raw = a_raw.detach()
        gates = LsmGates(b_pre=b_pre, a_pre=a_pre) if (b_pre is not None or a_pre is not None) else None
        o = lsm_forward_batched(q, k, v, gates, sp, chunk_size, check=False)
        ctx.save_for_backward(q, k, v, b_pre, a_pre)
        ctx.spec, ctx.chunk = sp, chunk_size
        ctx.n_in = 6 + len(extra)
        return o

    @staticmethod
    def backward(ctx, dO):
        q, k, v, b_pre, a_pre = ctx.saved_tensors
        gates = LsmGates(b_pre=b_pre, a_pre=a_pre) if (b_pre is not None or a_pre is not None) else None
        g = lsm_backward_batched(q, k, v, gates, ctx.spec, dO.to(q.dtype), chunk_size=ctx.chunk, check=False)
        return (g.dq, g.dk, g.dv, g.db_pre, None, None, g.da_pre, g.da_raw)[:ctx.n_in]


def _cu_array(cu_seqlens):
    """Host int32 array of PackedBatch::boundaries (model.hpp:86-121)."""
    import numpy as np
    arr = np.ascontiguousarray(np.asarray(list(cu_seqlens), dtype=np.int32))
    return arr, arr.ctypes.data_as(ctypes.c_void_p), len(arr) - 1


def lsm_forward_varlen(q, k, v, gates, spec, cu_seqlens, chunk_size=64, final_states=False, check=True,
                       stream=None):
    """Packed documents: q, k, v [1, T, H, D]; document i = rows [cu[i], cu[i+1]); the state is
    zero at every boundary (model_forward runs the mixer per document, model.hpp:374-405).
    Returns o (and [n_docs, H, D, D] final states when final_states)."""
    _, T, H, D = q.shape
    q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
    cu, cu_p, n_docs = _cu_array(cu_seqlens)
    a_raw = None
    if spec.instance == LsmInstance.MAMBA2:
        a_raw = torch.as_tensor(spec.mamba2_a_raw, dtype=torch.float32, device=q.device).reshape(-1).expand(H).contiguous()
    b_pre = gates.b_pre.to(torch.float32).contiguous() if gates is not None and gates.b_pre is not None else None
    a_pre = gates.a_pre.to(q.dtype).contiguous() if gates is not None and gates.a_pre is not None else None
    o = torch.empty_like(q)
    M = torch.empty(n_docs, H, D, D, dtype=torch.float32, device=q.device) if final_states else None
    desc = make_desc(spec, chunk_size, check)
    L = _lib.lib()
    dt = _DTYPES[q.dtype]
    ws = _workspace(L.lmoe_lsm_varlen_workspace_size(ctypes.byref(desc), T, cu_p, n_docs, H, D, dt, 0), q.device)
    st = stream if stream is not None else torch.cuda.current_stream(q.device).cuda_stream
    P = _lib.ptr
    _lib.check(L.lmoe_lsm_fwd_varlen(ctypes.byref(desc), T, cu_p, n_docs, H, D, dt, P(q), P(k), P(v), P(a_pre),
                                     P(b_pre), P(a_raw), P(o), P(M), P(ws), ws.numel(), ctypes.c_void_p(st)))
    return (o, M) if final_states else o


def lsm_backward_varlen(q, k, v, gates, spec, dO, cu_seqlens, chunk_size=64, check=True, stream=None):
    """VJP of lsm_forward_varlen; da_raw sums over documents."""
    _, T, H, D = q.shape
    q, k, v, dO = q.contiguous(), k.contiguous(), v.contiguous(), dO.contiguous()
    cu, cu_p, n_docs = _cu_array(cu_seqlens)
    a_raw = None
    if spec.instance == LsmInstance.MAMBA2:
        a_raw = torch.as_tensor(spec.mamba2_a_raw, dtype=torch.float32, device=q.device).reshape(-1).expand(H).contiguous()
    b_pre = gates.b_pre.to(torch.float32).contiguous() if gates is not None and gates.b_pre is not None else None
    a_pre = gates.a_pre.to(q.dtype).contiguous() if gates is not None and gates.a_pre is not None else None
    g = LsmGrads(dq=torch.empty_like(q), dk=torch.empty_like(q), dv=torch.empty_like(q))
    if spec.instance == LsmInstance.MAMBA2:
        g.db_pre = torch.empty(1, T, H, dtype=torch.float32, device=q.device)
        g.da_raw = torch.empty(H, dtype=torch.float32, device=q.device)
    if a_pre is not None:
        g.da_pre = torch.empty_like(a_pre)
    desc = make_desc(spec, chunk_size, check)
    L = _lib.lib()
    dt = _DTYPES[q.dtype]
    need = L.lmoe_lsm_varlen_workspace_size(ctypes.byref(desc), T, cu_p, n_docs, H, D, dt, 1)
    ws = _workspace(need + 256 + 4 * H, q.device)
    st = stream if stream is not None else torch.cuda.current_stream(q.device).cuda_stream
    P = _lib.ptr
    _lib.check(L.lmoe_lsm_bwd_varlen(ctypes.byref(desc), T, cu_p, n_docs, H, D, dt, P(q), P(k), P(v), P(a_pre),
                                     P(b_pre), P(a_raw), P(dO), P(g.dq), P(g.dk), P(g.dv), P(g.da_pre), P(g.db_pre),
                                     P(g.da_raw), P(ws), ws.numel(), ctypes.c_void_p(st)))
    return g


class _RecInputs(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in ("a_vec", "a_scal", "b_pre", "alpha_pre", "beta_pre", "s4_delta_raw",
                                                "s4_b", "s4_A_raw", "mamba_A_raw")]


def lsm_forward_recurrent(q, k, v, gates, spec, initial_state=None, final_state=None, check=True, stream=None):
    """The kinds without a chunk-parallel form (DeltaNet, GatedDeltaNet, GFW, GateLoop, TTT,
    Titans, RWKV7, S4, Mamba): recurrent_step (lsm.hpp:335-441) token by token on the device
    (lmoe_lsm_fwd_recurrent).  q, k, v [B, N, H, D]; gates / static params as LsmGates / LsmSpec."""
    B, N, H, D = q.shape
    q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
    L = _lib.lib()
    if not getattr(L, "_rec_bound", False):
        L.lmoe_lsm_fwd_recurrent.restype = ctypes.c_int
        L.lmoe_lsm_fwd_recurrent.argtypes = ([ctypes.POINTER(_lib.LsmDesc)] + [ctypes.c_int] * 5 + [ctypes.c_void_p] * 8
                                             + [ctypes.c_size_t, ctypes.c_void_p])
        L._rec_bound = True
    keep = []

    def ptr(t, dtype=None):
        if t is None:
            return None
        t = t.to(dtype or t.dtype).contiguous()
        keep.append(t)
        return t.data_ptr()

    g = gates or LsmGates()
    vec_a = spec.instance in (LsmInstance.RWKV7, LsmInstance.MAMBA)
    rin = _RecInputs(a_vec=ptr(g.a_pre, q.dtype) if vec_a else None,
                     a_scal=None if vec_a else ptr(g.a_pre, torch.float32),
                     b_pre=ptr(g.b_pre, torch.float32), alpha_pre=ptr(g.alpha_pre, q.dtype),
                     beta_pre=ptr(g.beta_pre, q.dtype), s4_delta_raw=ptr(spec.s4_delta_raw, torch.float32),
                     s4_b=ptr(spec.s4_b, torch.float32), s4_A_raw=ptr(spec.s4_A_raw, torch.float32),
                     mamba_A_raw=ptr(spec.mamba_A_raw, torch.float32))
    M0 = None if initial_state is None else ptr(initial_state.M, torch.float32)
    o = torch.empty_like(q)
    M_out = torch.empty(B, H, D, D, dtype=torch.float32, device=q.device) if final_state is not None else None
    desc = make_desc(spec, 64, check)
    ws = _workspace(256, q.device)  # the device error flag
    st = stream if stream is not None else torch.cuda.current_stream(q.device).cuda_stream
    _lib.check(L.lmoe_lsm_fwd_recurrent(ctypes.byref(desc), B, N, H, D, _DTYPES[q.dtype], q.data_ptr(),
                                        k.data_ptr(), v.data_ptr(), ctypes.byref(rin), M0, o.data_ptr(),
                                        None if M_out is None else M_out.data_ptr(), ws.data_ptr(), ws.numel(),
                                        ctypes.c_void_p(st)))
    if final_state is not None:
        final_state.M, final_state.z, final_state.step = M_out, None, N
    return o


class _RecGrads(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in ("da_vec", "da_scal", "db_pre", "dalpha_pre", "dbeta_pre",
                                                "ds4_delta_raw", "ds4_b", "ds4_A_raw", "dmamba_A_raw")]


def lsm_backward_recurrent(q, k, v, gates, spec, dO, initial_state=None, dM_final=None, check=True, stream=None):
    """Gradients of lsm_forward_recurrent (the reference tape over recurrent_step, lsm.hpp:335-441)
    for DeltaNet, GatedDeltaNet, GFW, GateLoop, TTT, Titans, RWKV7, S4, Mamba
    (lmoe_lsm_bwd_recurrent).  Returns LsmGrads: dq, dk, dv, the gate gradients that apply
    (da_pre, db_pre, dalpha_pre, dbeta_pre), the static ones (ds4_*, dmamba_A_raw; summed over
    the batch) and dM0."""
    B, N, H, D = q.shape
    q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
    L = _lib.lib()
    if not getattr(L, "_recb_bound", False):
        L.lmoe_lsm_bwd_recurrent_workspace_size.restype = ctypes.c_size_t
        L.lmoe_lsm_bwd_recurrent_workspace_size.argtypes = [ctypes.POINTER(_lib.LsmDesc)] + [ctypes.c_int] * 5
        L.lmoe_lsm_bwd_recurrent.restype = ctypes.c_int
        L.lmoe_lsm_bwd_recurrent.argtypes = ([ctypes.POINTER(_lib.LsmDesc)] + [ctypes.c_int] * 5
                                             + [ctypes.c_void_p] * 13 + [ctypes.c_size_t, ctypes.c_void_p])
        L._recb_bound = True
    keep = []

    def ptr(t, dtype=None):
        if t is None:
            return None
        t = t.to(dtype or t.dtype).contiguous()
        keep.append(t)
        return t.data_ptr()

    dev = q.device
    g = gates or LsmGates()
    inst = spec.instance
    vec_a = inst in (LsmInstance.RWKV7, LsmInstance.MAMBA)
    rin = _RecInputs(a_vec=ptr(g.a_pre, q.dtype) if vec_a else None,
                     a_scal=None if vec_a else ptr(g.a_pre, torch.float32),
                     b_pre=ptr(g.b_pre, torch.float32), alpha_pre=ptr(g.alpha_pre, q.dtype),
                     beta_pre=ptr(g.beta_pre, q.dtype), s4_delta_raw=ptr(spec.s4_delta_raw, torch.float32),
                     s4_b=ptr(spec.s4_b, torch.float32), s4_A_raw=ptr(spec.s4_A_raw, torch.float32),
                     mamba_A_raw=ptr(spec.mamba_A_raw, torch.float32))
    gr = LsmGrads(dq=torch.empty_like(q), dk=torch.empty_like(k), dv=torch.empty_like(v))
    gr.dM0 = torch.empty(B, H, D, D, dtype=torch.float32, device=dev)
    if g.a_pre is not None:
        gr.da_pre = torch.empty(g.a_pre.shape, dtype=q.dtype if vec_a else torch.float32, device=dev)
    if g.b_pre is not None:
        gr.db_pre = torch.empty(g.b_pre.shape, dtype=torch.float32, device=dev)
    if g.alpha_pre is not None:
        gr.dalpha_pre = torch.empty(g.alpha_pre.shape, dtype=q.dtype, device=dev)
        gr.dbeta_pre = torch.empty(g.beta_pre.shape, dtype=q.dtype, device=dev)
    for name in ("s4_delta_raw", "s4_b", "s4_A_raw", "mamba_A_raw"):
        t = getattr(spec, name)
        if t is not None:
            setattr(gr, "d" + name, torch.empty(t.shape, dtype=torch.float32, device=dev))
    P = lambda t: None if t is None else t.data_ptr()
    rg = _RecGrads(da_vec=P(gr.da_pre) if vec_a else None, da_scal=None if vec_a else P(gr.da_pre),
                   db_pre=P(gr.db_pre), dalpha_pre=P(gr.dalpha_pre), dbeta_pre=P(gr.dbeta_pre),
                   ds4_delta_raw=P(gr.ds4_delta_raw), ds4_b=P(gr.ds4_b), ds4_A_raw=P(gr.ds4_A_raw),
                   dmamba_A_raw=P(gr.dmamba_A_raw))
    M0 = None if initial_state is None else ptr(initial_state.M, torch.float32)
    dMf = None if dM_final is None else ptr(dM_final, torch.float32)
    desc = make_desc(spec, 64, check)
    ws = _workspace(L.lmoe_lsm_bwd_recurrent_workspace_size(ctypes.byref(desc), B, N, H, D, _DTYPES[q.dtype]), dev)
    st = stream if stream is not None else torch.cuda.current_stream(dev).cuda_stream
    _lib.check(L.lmoe_lsm_bwd_recurrent(ctypes.byref(desc), B, N, H, D, _DTYPES[q.dtype], q.data_ptr(), k.data_ptr(),
                                        v.data_ptr(), ctypes.byref(rin), M0, ptr(dO, q.dtype), dMf,
                                        gr.dq.data_ptr(), gr.dk.data_ptr(), gr.dv.data_ptr(), ctypes.byref(rg),
                                        gr.dM0.data_ptr(), ws.data_ptr(), ws.numel(), ctypes.c_void_p(st)))
    return gr
