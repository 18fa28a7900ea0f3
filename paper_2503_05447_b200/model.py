"""Host mirror of the reference model assembly over the C-ABI block executor.

  ModelConfig                       model.hpp:18-40 (fields the device path uses)
  Model.init(cfg, seed)             build_model (model.hpp:336-362): same shapes and init scales
  Model.from_arrays(arrays)         load parameters (e.g. the reference's own, tests/golden)
  Model.forward(tokens)             model_forward (model.hpp:374-405) for equal-length docs
  Model.forward_packed(tokens, b)   model_forward over a PackedBatch (model.hpp:86-121):
                                    positions restart and the mixer runs per document
  Model.forward(tokens, comm, n)    hybrid_sp_forward (parallel.hpp:477-506): this rank's
                                    chunk_range slice of ONE document; L blocks use masked
                                    state SP, N blocks the K/V all-gather
Every block is one lmoe_block_fwd call (csrc/block.cu); torch holds device memory only.
"""
import ctypes
import dataclasses
import math
from typing import List, Optional

import torch

from . import _lib
from .lsm import LsmInstance, LsmSpec, _workspace, make_desc

BF16 = torch.bfloat16


class _BlockDesc(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("hidden", ctypes.c_int), ("heads", ctypes.c_int),
                ("num_experts", ctypes.c_int), ("top_k", ctypes.c_int), ("ffn_dim", ctypes.c_int),
                ("norm_eps", ctypes.c_float), ("lsm", _lib.LsmDesc)]


class _BlockWeights(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in ("norm_mixer", "norm_moe", "w_qkv", "w_gate_b", "a_raw", "wo",
                                                "router", "w_gate", "w_up", "w_down")]


def _bind():
    L = _lib.lib()
    if getattr(L, "_model_bound", False):
        return L
    vp, sz, i = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int
    L.lmoe_block_workspace_size.restype = sz
    L.lmoe_block_workspace_size.argtypes = [ctypes.POINTER(_BlockDesc), i, i, i, i]
    L.lmoe_block_fwd.restype = i
    L.lmoe_block_fwd.argtypes = [ctypes.POINTER(_BlockDesc), ctypes.POINTER(_BlockWeights), i, i, i, vp, vp, vp,
                                 i, i, vp, sz, vp]
    L.lmoe_block_varlen_workspace_size.restype = sz
    L.lmoe_block_varlen_workspace_size.argtypes = [ctypes.POINTER(_BlockDesc), i, vp, i]
    L.lmoe_block_fwd_varlen.restype = i
    L.lmoe_block_fwd_varlen.argtypes = [ctypes.POINTER(_BlockDesc), ctypes.POINTER(_BlockWeights), i, vp, i, vp,
                                        vp, vp, sz, vp]
    L.lmoe_embed.restype = i
    L.lmoe_embed.argtypes = [vp, i, i, i, i, vp, vp, vp, vp]
    L.lmoe_rmsnorm.restype = i
    L.lmoe_rmsnorm.argtypes = [vp, i, i, vp, ctypes.c_float, vp, vp]
    L.lmoe_gemm_workspace_size.restype = sz
    L.lmoe_gemm_workspace_size.argtypes = [i]
    L.lmoe_gemm.restype = i
    L.lmoe_gemm.argtypes = [vp, i, i, i, vp, i, vp, i, i, vp, sz, vp]
    L._model_bound = True
    return L


@dataclasses.dataclass
class ModelConfig:
    """lmoe::ModelConfig (model.hpp:18-40)."""
    hidden: int = 256
    ffn_dim: int = 128
    num_heads: int = 2
    num_experts: int = 4
    num_active: int = 2
    vocab_size: int = 64
    instance: int = LsmInstance.MAMBA2
    pattern: str = "LL"
    max_seq_len: int = 256
    norm_eps: float = 1e-6
    chunk_size: int = 16

    def validate(self):
        if not self.pattern:
            raise RuntimeError("ModelConfig: empty layer pattern")
        for c in self.pattern:
            if c not in "LN":
                raise RuntimeError("ModelConfig: invalid pattern char '%s' (want L or N)" % c)
        if self.hidden % self.num_heads:
            raise RuntimeError("ModelConfig: hidden must be divisible by num_heads")

    def head_dim(self):
        return self.hidden // self.num_heads


@dataclasses.dataclass
class Block:
    kind: str
    norm_mixer: torch.Tensor
    norm_moe: torch.Tensor
    w_qkv: torch.Tensor                 # [hidden, 3 hidden | 4 hidden]
    wo: torch.Tensor
    router: torch.Tensor
    w_gate: torch.Tensor
    w_up: torch.Tensor
    w_down: torch.Tensor
    w_gate_b: Optional[torch.Tensor] = None  # [hidden, 64] (Mamba2)
    a_raw: Optional[torch.Tensor] = None     # [heads] (Mamba2)


class Model:
    def __init__(self, cfg: ModelConfig, embedding, pos_embedding, blocks: List[Block], final_norm, lm_head):
        cfg.validate()
        self.cfg = cfg
        self.embedding, self.pos_embedding = embedding, pos_embedding
        self.blocks, self.final_norm, self.lm_head = blocks, final_norm, lm_head
        self.spec = LsmSpec.make(cfg.instance, cfg.head_dim())
        self.spec.use_normalizer = False  # the block executor runs the normaliser-free kinds

    # ------------------------------------------------------------------ construction
    @staticmethod
    def _block(cfg, kind, wq, wk, wv, wo, router, wg, wu, wd, w_gate_a=None, w_gate_b=None, a_raw=None,
               device="cuda"):
        dev = torch.device(device)
        cols = [wq, wk, wv] + ([w_gate_a] if (kind == "L" and w_gate_a is not None) else [])
        b = Block(kind=kind, norm_mixer=torch.ones(cfg.hidden, device=dev), norm_moe=torch.ones(cfg.hidden, device=dev),
                  w_qkv=torch.cat([torch.as_tensor(c, dtype=torch.float32) for c in cols], 1).to(dev, BF16).contiguous(),
                  wo=torch.as_tensor(wo, dtype=torch.float32).to(dev, BF16).contiguous(),
                  router=torch.as_tensor(router, dtype=torch.float32).to(dev, BF16).contiguous(),
                  w_gate=torch.as_tensor(wg, dtype=torch.float32).to(dev, BF16).contiguous(),
                  w_up=torch.as_tensor(wu, dtype=torch.float32).to(dev, BF16).contiguous(),
                  w_down=torch.as_tensor(wd, dtype=torch.float32).to(dev, BF16).contiguous())
        if kind == "L" and w_gate_b is not None:
            wgb = torch.as_tensor(w_gate_b, dtype=torch.float32)
            g = torch.zeros(cfg.hidden, 64, device=wgb.device)
            g[:, :cfg.num_heads] = wgb
            b.w_gate_b = g.to(dev, BF16).contiguous()
            b.a_raw = torch.as_tensor(a_raw, dtype=torch.float32).to(dev).contiguous()
        return b

    @staticmethod
    def init(cfg: ModelConfig, seed=0, device="cuda", draw_on_device=False):
        """build_model (model.hpp:336-362) shapes and scales: N(0, 0.02) embeddings, N(0, 1/hidden)
        mixer and router weights, N(0, 1/hidden) / N(0, 1/ffn) experts (moe.hpp:37-41).
        draw_on_device: draw the weights with a device generator (large configs; a different
        random stream than the host draw, same distributions)."""
        cfg.validate()
        gdev = torch.device(device) if draw_on_device else torch.device("cpu")
        g = torch.Generator(device=gdev).manual_seed(seed)
        h, H, E, F = cfg.hidden, cfg.num_heads, cfg.num_experts, cfg.ffn_dim
        rn = lambda *shape, s: torch.randn(*shape, generator=g, device=gdev) * s
        sh = 1.0 / math.sqrt(h)
        blocks = []
        for kind in cfg.pattern:
            vec = cfg.instance in (LsmInstance.GLA, LsmInstance.HGRN2, LsmInstance.RWKV6)
            blocks.append(Model._block(
                cfg, kind, rn(h, h, s=sh), rn(h, h, s=sh), rn(h, h, s=sh), rn(h, h, s=sh), rn(h, E, s=sh),
                rn(E, h, F, s=sh), rn(E, h, F, s=sh), rn(E, F, h, s=1.0 / math.sqrt(F)),
                w_gate_a=rn(h, h, s=sh) if (kind == "L" and vec) else None,
                w_gate_b=rn(h, H, s=sh) if (kind == "L" and cfg.instance == LsmInstance.MAMBA2) else None,
                a_raw=rn(H, s=0.5) if cfg.instance == LsmInstance.MAMBA2 else None, device=device))
        dev = torch.device(device)
        return Model(cfg, rn(cfg.vocab_size, h, s=0.02).to(dev, BF16), rn(cfg.max_seq_len, h, s=0.02).to(dev, BF16),
                     blocks, torch.ones(h, device=dev), rn(h, cfg.vocab_size, s=sh).to(dev, BF16))

    @staticmethod
    def from_arrays(cfg: ModelConfig, a, device="cuda"):
        """Parameters by reference name: embedding, pos_embedding, b{i}/{norm_mixer, wq, ...},
        final_norm, lm_head (the layout tests/golden/model.npz stores)."""
        dev = torch.device(device)
        blocks = []
        for i, kind in enumerate(cfg.pattern):
            p = "b%d/" % i
            blk = Model._block(cfg, kind, a[p + "wq"], a[p + "wk"], a[p + "wv"], a[p + "wo"], a[p + "router"],
                               a[p + "w_gate"], a[p + "w_up"], a[p + "w_down"], a.get(p + "w_gate_a"),
                               a.get(p + "w_gate_b"), a.get(p + "a_raw"), device=device)
            blk.norm_mixer = torch.as_tensor(a[p + "norm_mixer"], dtype=torch.float32).to(dev)
            blk.norm_moe = torch.as_tensor(a[p + "norm_moe"], dtype=torch.float32).to(dev)
            blocks.append(blk)
        T = lambda x: torch.as_tensor(x, dtype=torch.float32).to(dev)
        return Model(cfg, T(a["embedding"]).to(BF16), T(a["pos_embedding"]).to(BF16), blocks, T(a["final_norm"]),
                     T(a["lm_head"]).to(BF16).contiguous())

    # ------------------------------------------------------------------ forward
    def _desc(self, kind):
        c = self.cfg
        d = _BlockDesc(kind=ord(kind), hidden=c.hidden, heads=c.num_heads, num_experts=c.num_experts,
                       top_k=c.num_active, ffn_dim=c.ffn_dim, norm_eps=c.norm_eps)
        d.lsm = make_desc(self.spec, c.chunk_size, check=False)
        return d

    @staticmethod
    def _weights(b: Block):
        P = lambda t: None if t is None else t.data_ptr()
        return _BlockWeights(P(b.norm_mixer), P(b.norm_moe), P(b.w_qkv), P(b.w_gate_b), P(b.a_raw), P(b.wo),
                             P(b.router), P(b.w_gate), P(b.w_up), P(b.w_down))

    def run_block(self, i, x, B, N, comm=None, n_total=None, aux=None, stream=None, moe=True):
        """Block i on the fp32 residual stream x [B*N, hidden] in place (lmoe_block_fwd).
        moe=False: the mixer layer alone (x += mixer(rms_norm(x)) W_o; descriptor num_experts = 0)."""
        L = _bind()
        b = self.blocks[i]
        dev = x.device
        world = comm.world if comm is not None else 1
        rank = comm.rank if comm is not None else 0
        n_total = n_total or N
        st = stream if stream is not None else torch.cuda.current_stream(dev).cuda_stream
        if aux is None:
            aux = torch.zeros(1, dtype=torch.float32, device=dev)
        d = self._desc(b.kind)
        if not moe:
            d.num_experts = 0
        ws = _workspace(L.lmoe_block_workspace_size(ctypes.byref(d), B, N, n_total, world), dev)
        w = self._weights(b)
        _lib.check(L.lmoe_block_fwd(ctypes.byref(d), ctypes.byref(w), B, N, n_total, x.data_ptr(), aux.data_ptr(),
                                    comm.handle if comm is not None else None, rank, world, ws.data_ptr(),
                                    ws.numel(), st))
        return aux

    def _check_tokens(self, tok):
        """model.hpp:377-378: every id must index the embedding table (lmoe_embed reads
        embedding[tok] unchecked on the device)."""
        if tok.numel() and (int(tok.min()) < 0 or int(tok.max()) >= self.cfg.vocab_size):
            raise RuntimeError("model_forward: token id out of vocabulary range")

    def forward_packed(self, tokens, boundaries, stream=None):
        """model_forward (model.hpp:374-405) over one flat token stream with ascending document
        boundaries (PackedBatch, model.hpp:86-121): per-document positions, the mixer per
        document (lmoe_block_fwd_varlen), the MoE over all tokens.
        Returns (logits fp32 [T, vocab], aux = mean block load-balance loss)."""
        import numpy as np
        L = _bind()
        c = self.cfg
        dev = self.embedding.device
        cu = np.ascontiguousarray(np.asarray(list(boundaries), dtype=np.int32))
        n_docs = len(cu) - 1
        T = int(cu[-1])
        tok = tokens.reshape(-1).to(dev, torch.int32).contiguous()
        if len(cu) < 2 or cu[0] != 0 or tok.numel() != T:
            raise RuntimeError("PackedBatch: boundaries must run from 0 to total length")
        if (np.diff(cu) <= 0).any():
            raise RuntimeError("PackedBatch: boundaries must be strictly ascending")
        if int(np.diff(cu).max()) > c.max_seq_len:
            raise RuntimeError("model_forward: document longer than max_seq_len")
        self._check_tokens(tok)
        st = stream if stream is not None else torch.cuda.current_stream(dev).cuda_stream
        x = torch.empty(T, c.hidden, dtype=torch.float32, device=dev)
        for i in range(n_docs):  # positions restart per document (model.hpp:379-384)
            r0, n = int(cu[i]), int(cu[i + 1] - cu[i])
            _lib.check(L.lmoe_embed(tok[r0:].data_ptr(), n, n, 0, c.hidden, self.embedding.data_ptr(),
                                    self.pos_embedding.data_ptr(), x[r0:].data_ptr(), st))
        aux = torch.zeros(len(self.blocks), dtype=torch.float32, device=dev)
        cu_p = cu.ctypes.data_as(ctypes.c_void_p)
        for i, b in enumerate(self.blocks):
            d = self._desc(b.kind)
            ws = _workspace(L.lmoe_block_varlen_workspace_size(ctypes.byref(d), T, cu_p, n_docs), dev)
            w = self._weights(b)
            _lib.check(L.lmoe_block_fwd_varlen(ctypes.byref(d), ctypes.byref(w), T, cu_p, n_docs, x.data_ptr(),
                                               aux[i:].data_ptr(), ws.data_ptr(), ws.numel(), st))
        h = torch.empty(T, c.hidden, dtype=BF16, device=dev)
        _lib.check(L.lmoe_rmsnorm(x.data_ptr(), T, c.hidden, self.final_norm.data_ptr(), c.norm_eps, h.data_ptr(), st))
        logits = torch.empty(T, c.vocab_size, dtype=torch.float32, device=dev)
        ws = _workspace(L.lmoe_gemm_workspace_size(T), dev)
        _lib.check(L.lmoe_gemm(h.data_ptr(), T, c.hidden, c.hidden, self.lm_head.data_ptr(), c.vocab_size,
                               logits.data_ptr(), c.vocab_size, 1, ws.data_ptr(), ws.numel(), st))
        return logits, aux.mean()

    def forward(self, tokens, comm=None, n_total=None, stream=None):
        """tokens: int [B, N] (B equal-length documents), or this rank's [1, N_local] slice of
        one n_total-token document when `comm` (sp.NcclComm) spans > 1 rank.
        Returns (logits fp32 [B*N, vocab], aux = mean block load-balance loss)."""
        L = _bind()
        c = self.cfg
        B, N = tokens.shape
        dev = self.embedding.device
        world = comm.world if comm is not None else 1
        rank = comm.rank if comm is not None else 0
        n_total = n_total or N * (world if B == 1 else 1)
        pos0 = 0
        if world > 1:
            if B != 1:
                raise RuntimeError("hybrid_sp_forward: single-document batches only")
            from .sp import chunk_range
            pos0 = chunk_range(n_total, world, rank)[0]
        if pos0 + N > c.max_seq_len:  # model.hpp:382-383 (positions are document-relative)
            raise RuntimeError("model_forward: document longer than max_seq_len")
        st = stream if stream is not None else torch.cuda.current_stream(dev).cuda_stream
        T = B * N
        tok = tokens.to(dev, torch.int32).contiguous()
        self._check_tokens(tok)
        x = torch.empty(T, c.hidden, dtype=torch.float32, device=dev)
        _lib.check(L.lmoe_embed(tok.data_ptr(), T, N, pos0, c.hidden, self.embedding.data_ptr(),
                                self.pos_embedding.data_ptr(), x.data_ptr(), st))
        aux = torch.zeros(len(self.blocks), dtype=torch.float32, device=dev)
        for i in range(len(self.blocks)):
            self.run_block(i, x, B, N, comm, n_total, aux[i:], st)
        h = torch.empty(T, c.hidden, dtype=BF16, device=dev)
        _lib.check(L.lmoe_rmsnorm(x.data_ptr(), T, c.hidden, self.final_norm.data_ptr(), c.norm_eps, h.data_ptr(), st))
        logits = torch.empty(T, c.vocab_size, dtype=torch.float32, device=dev)
        ws = _workspace(L.lmoe_gemm_workspace_size(T), dev)
        _lib.check(L.lmoe_gemm(h.data_ptr(), T, c.hidden, c.hidden, self.lm_head.data_ptr(), c.vocab_size,
                               logits.data_ptr(), c.vocab_size, 1, ws.data_ptr(), ws.numel(), st))
        return logits, aux.mean()
