"""Randomised forward / SP parity sweep against the float64 oracle (developer aid): random
instance, feature map, normaliser, length (including 1 and ragged), heads, world size."""
import sys
import zlib

import numpy as np
import torch

sys.path.insert(0, "tests")
import oracle  # noqa: E402
from conftest import norm_rel_err  # noqa: E402

import paper_2503_05447_b200 as pk  # noqa: E402
from paper_2503_05447_b200 import sp  # noqa: E402

KINDS = ["bla", "rebased", "lightning", "retnet", "mamba2", "gla", "hgrn2", "rwkv6"]
NORM_OK = {"bla", "rebased", "lightning", "retnet", "gla", "rwkv6"}
rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
n_cases = int(sys.argv[2]) if len(sys.argv) > 2 else 60
fails = 0
for case in range(n_cases):
    inst = KINDS[rng.integers(len(KINDS))]
    N = int(rng.choice([1, 2, 63, 64, 65, 127, 128, 129, 300, 1000, 2500]))
    H = int(rng.integers(1, 4))
    D = 128
    fm = int(rng.integers(0, 3)) if inst in ("bla", "rebased") else 0
    norm = bool(rng.integers(0, 2)) and inst in NORM_OK and fm != 0
    world = int(rng.choice([1, 2, 3, 8]))
    world = min(world, N)
    q, k, v = (rng.normal(0, 0.5, (1, N, H, D)) for _ in range(3))
    to = lambda x: torch.tensor(x, dtype=torch.float32, device="cuda").to(torch.bfloat16)
    Q, K, V = to(q), to(k), to(v)
    q, k, v = (t.float().cpu().numpy().astype(np.float64) for t in (Q, K, V))
    spec_d = oracle.spec_default(inst)
    spec_d["feature_map"], spec_d["use_normalizer"] = fm, int(norm)
    spec = pk.LsmSpec.make(inst, D)
    spec.feature_map, spec.use_normalizer = fm, norm
    gates, a_pre, b_pre = None, None, None
    a_raw = rng.normal(0, 1.0, H)
    if inst == "mamba2":
        spec.mamba2_a_raw = torch.tensor(a_raw, dtype=torch.float32, device="cuda")
        a_raw = spec.mamba2_a_raw.cpu().numpy().astype(np.float64)
        bt = torch.tensor(rng.normal(rng.normal(0, 2), 1.0, (1, N, H)), dtype=torch.float32, device="cuda")
        gates = pk.LsmGates(b_pre=bt)
        b_pre = bt.cpu().numpy().astype(np.float64)
    if inst in ("gla", "hgrn2", "rwkv6"):
        at = to(rng.normal(rng.normal(2, 1), 1.0, (1, N, H, D)))
        gates = pk.LsmGates(a_pre=at)
        a_pre = at.float().cpu().numpy().astype(np.float64)
    try:
        o = pk.lsm_forward_batched(Q, K, V, gates, spec, 64, check=False).float().cpu().numpy()
        osp = sp.sp_forward_masked_loopback(Q, K, V, gates, spec, world, check=False).float().cpu().numpy() \
            if not (inst in ("gla", "hgrn2", "rwkv6") and False) else o
    except Exception as e:  # noqa: BLE001
        print("case %d %s N=%d H=%d fm=%d norm=%d world=%d: EXCEPTION %s" % (case, inst, N, H, fm, norm, world, e))
        fails += 1
        continue
    worst = 0.0
    for h in range(H):
        sh = dict(spec_d, mamba2_a_raw=float(a_raw[h]))
        want, _, _ = oracle.lsm_sequential(sh, q[0, :, h], k[0, :, h], v[0, :, h],
                                           a_pre=None if a_pre is None else a_pre[0, :, h],
                                           b_pre=None if b_pre is None else b_pre[0, :, h])
        if not np.isfinite(want).all():
            continue
        worst = max(worst, norm_rel_err(o[0, :, h], want), norm_rel_err(osp[0, :, h], want))
    flag = "FAIL" if worst > 2e-2 else "ok"
    if flag == "FAIL":
        fails += 1
    print("case %d %-9s N=%4d H=%d fm=%d norm=%d world=%d: %.2e %s" % (case, inst, N, H, fm, norm, world, worst, flag))
print("failures:", fails)
