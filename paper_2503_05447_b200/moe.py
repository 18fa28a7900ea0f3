"""Host mirror of the reference MoE interface (moe.hpp) over the C-ABI.

  MoeConfig (moe.hpp:15-27), route (:58-85), load_balance_loss (:90-103),
  MoeLayer.init / forward (:106-149).  The device computes in bf16 with fp32 accumulation;
  weights keep the reference layouts: router (hidden, E), w_gate / w_up (E, hidden, ffn),
  w_down (E, ffn, hidden).
"""
import ctypes
import dataclasses
import math

import torch

from . import _lib

_ws = {}


def _workspace(nbytes, device):
    key = (device, nbytes)
    if key not in _ws:
        _ws.clear()
        _ws[key] = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
    return _ws[key]


def _bind():
    L = _lib.lib()
    if getattr(L, "_moe_bound", False):
        return L
    vp, sz, i = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int
    L.lmoe_moe_workspace_size.restype = sz
    L.lmoe_moe_workspace_size.argtypes = [i, i, i, i, i]
    L.lmoe_moe_route.restype = i
    L.lmoe_moe_route.argtypes = [vp, i, i, i, vp, vp, vp, vp, vp, vp, sz, vp]
    L.lmoe_moe_forward.restype = i
    L.lmoe_moe_forward.argtypes = [i, i, i, i, i, vp, vp, vp, vp, vp, vp, i, vp, vp, vp, vp, vp, sz, vp]
    L.lmoe_moe_dispatch_read.restype = i
    L.lmoe_moe_dispatch_read.argtypes = [i, i, i, i, i, vp, vp, vp, vp, vp]
    L._moe_bound = True
    return L


@dataclasses.dataclass
class MoeConfig:
    """moe.hpp:15-27."""
    num_experts: int = 1
    top_k: int = 1
    hidden: int = 0
    ffn_dim: int = 0
    aux_loss_weight: float = 0.01

    def validate(self):
        if self.num_experts < 1 or self.top_k < 1 or self.top_k > self.num_experts:
            raise RuntimeError("MoeConfig: need 1 <= top_k <= num_experts")
        if self.hidden <= 0 or self.ffn_dim <= 0:
            raise RuntimeError("MoeConfig: nonpositive dims")


@dataclasses.dataclass
class RoutingDecision:
    """moe.hpp:52-56.  expert_ids (T, k) int32, ascending per token; gates_topk (T, k) the
    renormalised gates of those ids; full_probs (T, E) or None.  `gates` gives the
    reference's dense (T, E) form (zeros outside the selection)."""
    expert_ids: torch.Tensor
    gates_topk: torch.Tensor
    full_probs: torch.Tensor = None
    counts: torch.Tensor = None
    aux: torch.Tensor = None

    @property
    def gates(self):
        T, k = self.expert_ids.shape
        E = self.full_probs.shape[1] if self.full_probs is not None else int(self.expert_ids.max()) + 1
        dense = torch.zeros(T, E, dtype=torch.float32, device=self.expert_ids.device)
        dense.scatter_(1, self.expert_ids.long(), self.gates_topk)
        return dense


def route(router_logits, top_k, stream=None):
    """route (moe.hpp:58-85) on fp32 logits (T, E); aux = load_balance_loss (moe.hpp:90)."""
    L = _bind()
    logits = router_logits.to(torch.float32).contiguous()
    T, E = logits.shape
    dev = logits.device
    ids = torch.empty(T, top_k, dtype=torch.int32, device=dev)
    gates = torch.empty(T, top_k, dtype=torch.float32, device=dev)
    probs = torch.empty(T, E, dtype=torch.float32, device=dev)
    counts = torch.empty(E, dtype=torch.int32, device=dev)
    aux = torch.empty(1, dtype=torch.float32, device=dev)
    nbytes = L.lmoe_moe_workspace_size(T, 64, 64, E, max(top_k, 1))
    ws = _workspace(nbytes, dev)
    st = stream if stream is not None else torch.cuda.current_stream(dev).cuda_stream
    _lib.check(L.lmoe_moe_route(_lib.ptr(logits), T, E, top_k, _lib.ptr(ids), _lib.ptr(gates),
                                _lib.ptr(probs), _lib.ptr(counts), _lib.ptr(aux), _lib.ptr(ws),
                                ws.numel(), ctypes.c_void_p(st)))
    return RoutingDecision(ids, gates, probs, counts, aux)


def load_balance_loss(dec):
    """moe.hpp:90-103 (computed on device by route)."""
    return dec.aux


@dataclasses.dataclass
class MoeLayer:
    """MoeLayer (moe.hpp:106-149) with bf16 device weights."""
    config: MoeConfig
    router: torch.Tensor   # (hidden, E)
    w_gate: torch.Tensor   # (E, hidden, ffn)
    w_up: torch.Tensor     # (E, hidden, ffn)
    w_down: torch.Tensor   # (E, ffn, hidden)

    @staticmethod
    def init(cfg, generator=None, device="cuda", dtype=torch.bfloat16):
        """Reference init (moe.hpp:37-41, 114-115): N(0, 1/hidden) router and gate/up,
        N(0, 1/ffn) down projections."""
        cfg.validate()
        g = generator
        E, h, f = cfg.num_experts, cfg.hidden, cfg.ffn_dim

        def rn(*shape, std):
            return (torch.randn(*shape, device=device, generator=g) * std).to(dtype)
        return MoeLayer(cfg, rn(h, E, std=1 / math.sqrt(h)), rn(E, h, f, std=1 / math.sqrt(h)),
                        rn(E, h, f, std=1 / math.sqrt(h)), rn(E, f, h, std=1 / math.sqrt(f)))

    def forward(self, x, y_f32=False, return_routing=False, stream=None, out=None):
        """(y, aux) for x (T, hidden) bf16 -- moe.hpp:133-149."""
        self.config.validate()
        L = _bind()
        cfg = self.config
        x = x.to(torch.bfloat16).contiguous()
        T = x.shape[0]
        dev = x.device
        y = out if out is not None else torch.empty(T, cfg.hidden, dtype=torch.float32 if y_f32 else torch.bfloat16, device=dev)
        aux = torch.empty(1, dtype=torch.float32, device=dev)
        logits = ids = gates = None
        if return_routing:
            logits = torch.empty(T, cfg.num_experts, dtype=torch.float32, device=dev)
            ids = torch.empty(T, cfg.top_k, dtype=torch.int32, device=dev)
            gates = torch.empty(T, cfg.top_k, dtype=torch.float32, device=dev)
        nbytes = L.lmoe_moe_workspace_size(T, cfg.hidden, cfg.ffn_dim, cfg.num_experts, cfg.top_k)
        ws = _workspace(nbytes, dev)
        st = stream if stream is not None else torch.cuda.current_stream(dev).cuda_stream
        _lib.check(L.lmoe_moe_forward(T, cfg.hidden, cfg.ffn_dim, cfg.num_experts, cfg.top_k,
                                      _lib.ptr(x), _lib.ptr(self.router), _lib.ptr(self.w_gate),
                                      _lib.ptr(self.w_up), _lib.ptr(self.w_down), _lib.ptr(y),
                                      int(y_f32), _lib.ptr(aux), _lib.ptr(logits), _lib.ptr(ids),
                                      _lib.ptr(gates), _lib.ptr(ws), ws.numel(), ctypes.c_void_p(st)))
        self._last_ws = ws
        if return_routing:
            return y, aux, RoutingDecision(ids, gates), logits
        return y, aux

    def dispatch(self, T):
        """slot positions (T, k), token of each permuted row (T*k,), expert offsets (E+1,) of
        the last forward (the stable permutation of moe.hpp:137-139)."""
        L = _bind()
        cfg = self.config
        dev = self._last_ws.device
        sp = torch.empty(T, cfg.top_k, dtype=torch.int32, device=dev)
        pt = torch.empty(T * cfg.top_k, dtype=torch.int32, device=dev)
        off = torch.empty(cfg.num_experts + 1, dtype=torch.int32, device=dev)
        st = torch.cuda.current_stream(dev).cuda_stream
        _lib.check(L.lmoe_moe_dispatch_read(T, cfg.hidden, cfg.ffn_dim, cfg.num_experts, cfg.top_k,
                                            _lib.ptr(self._last_ws), _lib.ptr(sp), _lib.ptr(pt),
                                            _lib.ptr(off), ctypes.c_void_p(st)))
        return sp, pt, off
