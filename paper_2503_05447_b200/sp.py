"""LSM sequence parallelism (host mirror of parallel.hpp) over the C-ABI.

  chunk_range(n, t, rank)                    parallel.hpp:192-197
  NcclComm                                   replaces the thread-simulated RankGroup
                                             (parallel.hpp:39-178): one process per GPU,
                                             an NCCL communicator owned by liblmoe_cuda
  sp_lsm_masked_rank(comm, q_loc, ...)       parallel.hpp:303-376 -- ONE ncclAllGather of the
                                             all-heads state payload per call
  sp_forward_masked_loopback(q, ..., world)  the same algorithm with `world` virtual ranks on
                                             one device (device copies as the gather)
  sp_lsm_nomask_rank / sp_forward_nomask_loopback   parallel.hpp:282-297, 391-403 (Alg. 1)
torch.distributed is used only to ship the 128-byte NCCL unique id (bootstrap).
"""
import ctypes

import torch

from . import _lib
from .lsm import LsmGrads, LsmInstance, _DTYPES, _workspace, make_desc


def chunk_range(n, t, rank):
    """Balanced contiguous split; sizes differ by at most one, rank order (parallel.hpp:192)."""
    if n < t:
        raise RuntimeError("chunk_range: need at least one row per rank")
    base, rem = divmod(n, t)
    r0 = rank * base + min(rank, rem)
    return r0, r0 + base + (1 if rank < rem else 0)


def _bind():
    L = _lib.lib()
    if getattr(L, "_sp_bound", False):
        return L
    vp, sz, i = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int
    P = ctypes.POINTER(_lib.LsmDesc)
    L.lmoe_sp_payload_floats.restype = sz
    L.lmoe_sp_payload_floats.argtypes = [P, i, i, i]
    L.lmoe_sp_lsm_fwd_workspace_size.restype = sz
    L.lmoe_sp_lsm_fwd_workspace_size.argtypes = [P, i, i, i, i, i, i]
    L.lmoe_sp_lsm_fwd.restype = i
    L.lmoe_sp_lsm_fwd.argtypes = [P, i, i, i, i, i, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, i, i,
                                  vp, sz, vp]
    L.lmoe_sp_lsm_fwd_loopback_workspace_size.restype = sz
    L.lmoe_sp_lsm_fwd_loopback_workspace_size.argtypes = [P, i, i, i, i, i, i]
    L.lmoe_sp_lsm_fwd_loopback.restype = i
    L.lmoe_sp_lsm_fwd_loopback.argtypes = [P, i, i, i, i, i, vp, vp, vp, vp, vp, vp, vp, vp, vp,
                                           i, vp, sz, vp]
    L.lmoe_sp_lsm_nomask_workspace_size.restype = sz
    L.lmoe_sp_lsm_nomask_workspace_size.argtypes = [P, i, i, i, i, i, i]
    L.lmoe_sp_lsm_nomask_fwd.restype = i
    L.lmoe_sp_lsm_nomask_fwd.argtypes = [P, i, i, i, i, i, vp, vp, vp, vp, vp, i, i, vp, sz, vp]
    L.lmoe_sp_lsm_nomask_fwd_loopback.restype = i
    L.lmoe_sp_lsm_nomask_fwd_loopback.argtypes = [P, i, i, i, i, i, vp, vp, vp, vp, i, vp, sz, vp]
    L.lmoe_sp_lsm_bwd_workspace_size.restype = sz
    L.lmoe_sp_lsm_bwd_workspace_size.argtypes = [P, i, i, i, i, i, i]
    L.lmoe_sp_lsm_bwd.restype = i
    L.lmoe_sp_lsm_bwd.argtypes = [P, i, i, i, i, i] + [vp] * 15 + [i, i, vp, sz, vp]
    L.lmoe_sp_lsm_bwd_loopback_workspace_size.restype = sz
    L.lmoe_sp_lsm_bwd_loopback_workspace_size.argtypes = [P, i, i, i, i, i, i]
    L.lmoe_sp_lsm_bwd_loopback.restype = i
    L.lmoe_sp_lsm_bwd_loopback.argtypes = [P, i, i, i, i, i] + [vp] * 14 + [i, vp, sz, vp]
    L.lmoe_sp_last_gather_elements.restype = ctypes.c_longlong
    L.lmoe_nccl_unique_id.argtypes = [vp]
    L.lmoe_nccl_comm_init.argtypes = [ctypes.POINTER(vp), i, i, vp]
    L.lmoe_nccl_comm_destroy.argtypes = [vp]
    L._sp_bound = True
    return L


class NcclComm:
    """NCCL communicator of the library.  Bootstrap: rank 0 creates the unique id, the
    process group (gloo or nccl) broadcasts it; every rank calls ncclCommInitRank.

    world == 1: no communicator by default (the entry points then run the local pass, a
    gather over one rank being the identity).  single_rank_nccl=True creates a real 1-rank
    NCCL communicator instead, so the SP phase structure runs with its ncclAllGather on one
    GPU (used by the GPU tests to execute the NCCL path)."""

    def __init__(self, rank, world, device=None, single_rank_nccl=False):
        L = _bind()
        self.rank, self.world = rank, world
        self.handle = ctypes.c_void_p(None)
        if world == 1:
            if single_rank_nccl:
                buf = (ctypes.c_uint8 * 128)()
                _lib.check(L.lmoe_nccl_unique_id(ctypes.cast(buf, ctypes.c_void_p)))
                _lib.check(L.lmoe_nccl_comm_init(ctypes.byref(self.handle), 1, 0,
                                                 ctypes.cast(buf, ctypes.c_void_p)))
            return
        import torch.distributed as dist
        buf = (ctypes.c_uint8 * 128)()
        if rank == 0:
            _lib.check(L.lmoe_nccl_unique_id(ctypes.cast(buf, ctypes.c_void_p)))
        t = torch.tensor(list(buf), dtype=torch.uint8)
        if dist.get_backend() == "nccl":
            t = t.to(device or torch.device("cuda", torch.cuda.current_device()))
        dist.broadcast(t, 0)
        ids = bytes(t.cpu().tolist())
        idbuf = (ctypes.c_uint8 * 128).from_buffer_copy(ids)
        _lib.check(L.lmoe_nccl_comm_init(ctypes.byref(self.handle), world, rank,
                                         ctypes.cast(idbuf, ctypes.c_void_p)))

    def close(self):
        if self.handle.value:
            _bind().lmoe_nccl_comm_destroy(self.handle)
            self.handle = ctypes.c_void_p(None)


def _common(q, gates, spec):
    B, N, H, D = q.shape
    a_raw = None
    if spec.instance == LsmInstance.MAMBA2:
        a_raw = torch.as_tensor(spec.mamba2_a_raw, dtype=torch.float32,
                                device=q.device).reshape(-1).expand(H).contiguous()
    b_pre = None
    if gates is not None and gates.b_pre is not None:
        b_pre = gates.b_pre.to(torch.float32).contiguous()
    return B, N, H, D, a_raw, b_pre


def _a_pre(q, gates):
    """TokenVector gate pre-activations in the input dtype, or None."""
    if gates is None or gates.a_pre is None:
        return None
    return gates.a_pre.to(q.dtype).contiguous()


def _grads_like(q, gates, spec):
    B, N, H, D = q.shape
    g = LsmGrads(dq=torch.empty_like(q), dk=torch.empty_like(q), dv=torch.empty_like(q))
    g.dM0 = torch.zeros(B, H, D, D, dtype=torch.float32, device=q.device)
    if spec.instance == LsmInstance.MAMBA2:
        g.db_pre = torch.empty(B, N, H, dtype=torch.float32, device=q.device)
        g.da_raw = torch.empty(H, dtype=torch.float32, device=q.device)
    if gates is not None and gates.a_pre is not None:
        g.da_pre = torch.empty_like(q)
    return g


def sp_lsm_masked_rank(comm, q_loc, k_loc, v_loc, gates_loc, spec, chunk_size=64,
                       final_state=None, out=None, check=True, timing=False, stream=None):
    """This rank's output for its contiguous slice [B, N_loc, H, D] (parallel.hpp:303-376)."""
    L = _bind()
    B, N, H, D, a_raw, b_pre = _common(q_loc, gates_loc, spec)
    o = out if out is not None else torch.empty_like(q_loc)
    desc = make_desc(spec, chunk_size, check, timing)
    dt = _DTYPES[q_loc.dtype]
    nbytes = L.lmoe_sp_lsm_fwd_workspace_size(ctypes.byref(desc), B, N, H, D, dt, comm.world)
    ws = _workspace(nbytes, q_loc.device)
    M_out = z_out = None
    if final_state is not None:
        M_out = torch.empty(B, H, D, D, dtype=torch.float32, device=q_loc.device)
        if spec.use_normalizer:
            z_out = torch.empty(B, H, D, dtype=torch.float32, device=q_loc.device)
    st = stream if stream is not None else torch.cuda.current_stream(q_loc.device).cuda_stream
    rc = L.lmoe_sp_lsm_fwd(ctypes.byref(desc), B, N, H, D, dt, _lib.ptr(q_loc), _lib.ptr(k_loc),
                           _lib.ptr(v_loc), _lib.ptr(_a_pre(q_loc, gates_loc)), _lib.ptr(b_pre), _lib.ptr(a_raw), _lib.ptr(o),
                           _lib.ptr(M_out), _lib.ptr(z_out), comm.handle, comm.rank, comm.world,
                           _lib.ptr(ws), ws.numel(), ctypes.c_void_p(st))
    _lib.check(rc)
    if final_state is not None:
        final_state.M, final_state.z = M_out, z_out
    return o


def sp_forward_masked_loopback(q, k, v, gates, spec, world, chunk_size=64, final_state=None,
                               check=True):
    """sp_forward_masked (parallel.hpp:405-418) with `world` virtual ranks on one device."""
    L = _bind()
    B, N, H, D, a_raw, b_pre = _common(q, gates, spec)
    o = torch.empty_like(q)
    desc = make_desc(spec, chunk_size, check)
    dt = _DTYPES[q.dtype]
    nbytes = L.lmoe_sp_lsm_fwd_loopback_workspace_size(ctypes.byref(desc), B, N, H, D, dt, world)
    ws = _workspace(nbytes, q.device)
    M_out = z_out = None
    if final_state is not None:
        M_out = torch.empty(B, H, D, D, dtype=torch.float32, device=q.device)
        if spec.use_normalizer:
            z_out = torch.empty(B, H, D, dtype=torch.float32, device=q.device)
    st = torch.cuda.current_stream(q.device).cuda_stream
    rc = L.lmoe_sp_lsm_fwd_loopback(ctypes.byref(desc), B, N, H, D, dt, _lib.ptr(q), _lib.ptr(k),
                                    _lib.ptr(v), _lib.ptr(_a_pre(q, gates)), _lib.ptr(b_pre), _lib.ptr(a_raw),
                                    _lib.ptr(o), _lib.ptr(M_out), _lib.ptr(z_out), world,
                                    _lib.ptr(ws), ws.numel(), ctypes.c_void_p(st))
    _lib.check(rc)
    if final_state is not None:
        final_state.M, final_state.z = M_out, z_out
    return o


def sp_lsm_backward_rank(comm, q_loc, k_loc, v_loc, gates_loc, spec, dO_loc, chunk_size=64, check=True,
                         stream=None):
    """VJP of sp_lsm_masked_rank for this rank's slice (lmoe_sp_lsm_bwd): two all-gathers
    (forward payload, reverse-time payload), then the exact local backward.  Returns LsmGrads;
    da_raw is this rank's contribution (sum over ranks = the full gradient)."""
    L = _bind()
    B, N, H, D, a_raw, b_pre = _common(q_loc, gates_loc, spec)
    g = _grads_like(q_loc, gates_loc, spec)
    desc = make_desc(spec, chunk_size, check)
    dt = _DTYPES[q_loc.dtype]
    nbytes = L.lmoe_sp_lsm_bwd_workspace_size(ctypes.byref(desc), B, N, H, D, dt, comm.world)
    ws = _workspace(nbytes, q_loc.device)
    st = stream if stream is not None else torch.cuda.current_stream(q_loc.device).cuda_stream
    P = _lib.ptr
    rc = L.lmoe_sp_lsm_bwd(ctypes.byref(desc), B, N, H, D, dt, P(q_loc), P(k_loc), P(v_loc),
                           P(_a_pre(q_loc, gates_loc)), P(b_pre), P(a_raw), P(dO_loc.contiguous()), P(g.dq),
                           P(g.dk), P(g.dv), P(g.da_pre), P(g.db_pre), P(g.da_raw), P(g.dM0), comm.handle,
                           comm.rank, comm.world, P(ws), ws.numel(), ctypes.c_void_p(st))
    _lib.check(rc)
    return g


def sp_backward_masked_loopback(q, k, v, gates, spec, dO, world, chunk_size=64, check=True):
    """The SP backward with `world` virtual ranks on one device over the full sequence (B == 1)."""
    L = _bind()
    B, N, H, D, a_raw, b_pre = _common(q, gates, spec)
    g = _grads_like(q, gates, spec)
    desc = make_desc(spec, chunk_size, check)
    dt = _DTYPES[q.dtype]
    nbytes = L.lmoe_sp_lsm_bwd_loopback_workspace_size(ctypes.byref(desc), B, N, H, D, dt, world)
    ws = _workspace(nbytes, q.device)
    st = torch.cuda.current_stream(q.device).cuda_stream
    P = _lib.ptr
    rc = L.lmoe_sp_lsm_bwd_loopback(ctypes.byref(desc), B, N, H, D, dt, P(q), P(k), P(v), P(_a_pre(q, gates)),
                                    P(b_pre), P(a_raw), P(dO.contiguous()), P(g.dq), P(g.dk), P(g.dv),
                                    P(g.da_pre), P(g.db_pre), P(g.da_raw), P(g.dM0), world, P(ws), ws.numel(),
                                    ctypes.c_void_p(st))
    _lib.check(rc)
    return g


def last_gather_elements():
    """Elements moved by the last SP all-gather (RankGroup::comm_log, parallel.hpp:87-93)."""
    return int(_bind().lmoe_sp_last_gather_elements())


def payload_floats(spec, B, H, D):
    desc = make_desc(spec, 64)
    return int(_bind().lmoe_sp_payload_floats(ctypes.byref(desc), B, H, D))


def sp_lsm_nomask_rank(comm, q_loc, k_loc, v_loc, spec, out=None, check=True, stream=None):
    """Unmasked SP (parallel.hpp:282-297): O = phi(Q_loc) . sum over ALL ranks of phi(K)^T V."""
    L = _bind()
    B, N, H, D = q_loc.shape
    o = out if out is not None else torch.empty_like(q_loc)
    desc = make_desc(spec, 64, check)
    dt = _DTYPES[q_loc.dtype]
    ws = _workspace(L.lmoe_sp_lsm_nomask_workspace_size(ctypes.byref(desc), B, N, H, D, dt, comm.world),
                    q_loc.device)
    st = stream if stream is not None else torch.cuda.current_stream(q_loc.device).cuda_stream
    _lib.check(L.lmoe_sp_lsm_nomask_fwd(ctypes.byref(desc), B, N, H, D, dt, _lib.ptr(q_loc), _lib.ptr(k_loc),
                                        _lib.ptr(v_loc), _lib.ptr(o), comm.handle, comm.rank, comm.world,
                                        _lib.ptr(ws), ws.numel(), ctypes.c_void_p(st)))
    return o


def sp_forward_nomask_loopback(q, k, v, spec, world, check=True):
    """sp_forward_nomask (parallel.hpp:391-403) with `world` virtual ranks on one device."""
    L = _bind()
    B, N, H, D = q.shape
    q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
    o = torch.empty_like(q)
    desc = make_desc(spec, 64, check)
    dt = _DTYPES[q.dtype]
    nb = L.lmoe_sp_lsm_fwd_loopback_workspace_size(ctypes.byref(desc), B, N, H, D, dt, world)
    ws = _workspace(nb, q.device)
    st = torch.cuda.current_stream(q.device).cuda_stream
    _lib.check(L.lmoe_sp_lsm_nomask_fwd_loopback(ctypes.byref(desc), B, N, H, D, dt, _lib.ptr(q), _lib.ptr(k),
                                                 _lib.ptr(v), _lib.ptr(o), world, _lib.ptr(ws), ws.numel(),
                                                 ctypes.c_void_p(st)))
    return o
