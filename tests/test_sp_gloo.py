"""CPU multi-process check of the SP decomposition (world 2 and 4, gloo): each process
computes its slice's payload [M | z | D] with the oracle, the payloads are exchanged with
ONE torch.distributed all_gather (the role ncclAllGather plays on the GPUs), each rank
folds the decayed exclusive prefix and evaluates its slice with the carried-in state.
The concatenated outputs must equal the sequential oracle (parallel.hpp:303-418)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, inst, q, k, v, b_pre, result):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    import oracle
    from paper_2503_05447_b200.sp import chunk_range
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    spec = oracle.spec_default(inst)
    spec["mamba2_a_raw"] = 0.25
    n = q.shape[0]
    r0, r1 = chunk_range(n, world, rank)
    sl = slice(r0, r1)
    b = None if b_pre is None else b_pre[sl]
    payload = oracle.sp_local_payload(spec, q[sl], k[sl], v[sl], b_pre=b, chunk=16)
    bufs = [torch.zeros(payload.shape, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(bufs, torch.from_numpy(payload))
    gathered = np.stack([x.numpy() for x in bufs])
    M_in, z_in = oracle.sp_combine(spec, gathered, rank, v.shape[1])
    o, _, _ = oracle.lsm_chunked(spec, q[sl], k[sl], v[sl], b_pre=b, chunk=16, M0=M_in,
                                 z0=z_in if spec["use_normalizer"] else None)
    result[rank] = o
    dist.destroy_process_group()


@pytest.mark.parametrize("inst,world", [("bla", 2), ("lightning", 2), ("mamba2", 4), ("retnet", 4)])
def test_sp_gloo_matches_sequential(inst, world):
    import oracle
    rng = np.random.default_rng(11)
    n, d = 64, 8
    q, k, v = (rng.normal(0, 0.5, (n, d)) for _ in range(3))
    b_pre = rng.normal(-1, 1, n) if inst == "mamba2" else None
    mgr = mp.Manager()
    result = mgr.dict()
    port = _free_port()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_worker, args=(r, world, port, inst, q, k, v, b_pre, result))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    o = np.concatenate([result[r] for r in range(world)])
    spec = oracle.spec_default(inst)
    spec["mamba2_a_raw"] = 0.25
    want, _, _ = oracle.lsm_sequential(spec, q, k, v, b_pre=b_pre)
    assert np.abs(o - want).max() < 1e-10


def _spawn(worker, world, *args):
    mgr = mp.Manager()
    result = mgr.dict()
    port = _free_port()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=worker, args=(r, world, port) + args + (result,)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    return result


def _nomask_worker(rank, world, port, fm, q, k, v, result):
    """sp_lsm_nomask_rank (parallel.hpp:282-297): M_r = phi(K_r)^T V_r, ONE all-gather,
    O_r = phi(Q_r) . sum_r M_r (Alg. 1: no mask, no decay, no normaliser)."""
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    from paper_2503_05447_b200.sp import chunk_range
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    phi = (lambda x: x) if fm == 0 else (lambda x: x * x)  # identity / squared (lsm.hpp:291-298)
    r0, r1 = chunk_range(q.shape[0], world, rank)
    M = phi(k[r0:r1]).T @ v[r0:r1]
    bufs = [torch.zeros(M.shape, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(bufs, torch.from_numpy(np.ascontiguousarray(M)))
    result[rank] = (phi(q[r0:r1]) @ sum(b.numpy() for b in bufs), world * M.size)
    dist.destroy_process_group()


@pytest.mark.parametrize("case", ["bla_plain", "rebased_plain"])
@pytest.mark.parametrize("world", [2, 4])
def test_sp_nomask_gloo_matches_reference(case, world):
    """The unmasked SP decomposition over real processes reproduces the reference's own
    sp_forward_nomask outputs (tests/golden/spn.npz, generated from the reference headers) and
    its comm count T * d * d (test_parallel.cpp:124-148)."""
    from conftest import load_golden
    g = load_golden("spn")
    q, k, v = (g[case + "/" + x] for x in "qkv")
    fm = int(g[case + "/feature_map"][0])
    res = _spawn(_nomask_worker, world, fm, q, k, v)
    o = np.concatenate([res[r][0] for r in range(world)])
    assert np.abs(o - g[case + "/o_t%d" % world]).max() < 1e-10
    assert res[0][1] == int(g[case + "/comm_elems_t%d" % world][0])


def _attn_worker(rank, world, port, q, k, v, result):
    """sp_attention_rank (parallel.hpp:380-387): all-gather K and V (two collectives), then causal
    attention of the local queries with row_offset = r0 (attention.hpp:18-38)."""
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    import oracle
    from paper_2503_05447_b200.sp import chunk_range
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = q.shape[0]
    r0, r1 = chunk_range(n, world, rank)
    out = []
    for x in (k, v):  # equal slices here (n divisible by world): all_gather needs equal shapes
        bufs = [torch.zeros((r1 - r0, x.shape[1]), dtype=torch.float64) for _ in range(world)]
        dist.all_gather(bufs, torch.from_numpy(np.ascontiguousarray(x[r0:r1])))
        out.append(np.concatenate([b.numpy() for b in bufs]))
    K, V = out
    result[rank] = (oracle.attention(q[r0:r1], K, V, True, r0), 2 * K.size)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_sp_attention_gloo_matches_reference(world):
    """K/V all-gather SP over real processes equals the reference's sp_attention_allgather output
    and full causal attention (tests/golden/attn.npz), moving 2 N d elements (test_parallel.cpp:195-210)."""
    from conftest import load_golden
    g = load_golden("attn")
    q, k, v = g["q"], g["k"], g["v"]
    res = _spawn(_attn_worker, world, q, k, v)
    o = np.concatenate([res[r][0] for r in range(world)])
    assert np.abs(o - g["o_sp_t%d" % world]).max() < 1e-10
    assert np.abs(o - g["o_full"]).max() < 1e-10
    assert res[0][1] == int(g["comm_elems_t%d" % world][0])
