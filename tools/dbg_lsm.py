"""Quick device-vs-oracle error table for a few LSM variants (debug helper)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
import paper_2503_05447_b200 as pk

def run(inst, fm, norm, dtype, N, H=1, seed=0):
    D = 64 if dtype == "f32" else 128
    rng = np.random.default_rng(seed)
    q, k, v = (rng.normal(0, 0.5, (1, N, H, D)) for _ in range(3))
    tdt = torch.float32 if dtype == "f32" else torch.bfloat16
    Q, K, V = (torch.tensor(x, dtype=torch.float32, device="cuda").to(tdt) for x in (q, k, v))
    spec = pk.LsmSpec.make(inst, D); spec.feature_map = fm; spec.use_normalizer = bool(norm)
    a_raw = np.full(H, 0.3, dtype=np.float32)
    spec.mamba2_a_raw = torch.tensor(a_raw, device="cuda")
    b_pre = rng.normal(-1, 1, (1, N, H)).astype(np.float32)
    gates = pk.LsmGates(b_pre=torch.tensor(b_pre, device="cuda")) if inst == "mamba2" else None
    fs = pk.MemoryState()
    o = pk.lsm_forward_batched(Q, K, V, gates, spec, 64, final_state=fs, check=False)
    torch.cuda.synchronize()
    res = []
    for h in range(H):
        sd = oracle.spec_default(inst); sd["feature_map"] = fm; sd["use_normalizer"] = norm
        sd["mamba2_a_raw"] = float(a_raw[h])
        want, Mw, _ = oracle.lsm_chunked(sd, Q[0,:,h].float().cpu().numpy(), K[0,:,h].float().cpu().numpy(),
                                         V[0,:,h].float().cpu().numpy(), b_pre=b_pre[0,:,h] if inst=="mamba2" else None)
        got = o[0,:,h].float().cpu().numpy()
        e = np.abs(got-want).max()/np.abs(want).max()
        eM = np.abs(fs.M[0,h].cpu().numpy()-Mw).max()/max(np.abs(Mw).max(),1e-30)
        # first bad row
        rowerr = np.abs(got-want).max(1)/np.abs(want).max()
        bad = np.nonzero(rowerr > 0.05)[0]
        res.append((e, eM, bad[:5].tolist(), got[:2,:4].tolist(), want[:2,:4].tolist()))
    return res

cases = [("bla",0,0,"bf16",128),("bla",0,0,"bf16",300),("bla",0,0,"f32",256),("lightning",0,0,"bf16",1000),
         ("mamba2",0,0,"bf16",1000),("bla",1,1,"f32",2048),("retnet",0,0,"f32",515),("rebased",2,1,"bf16",700),("bla",1,1,"bf16",1000),("bla",1,1,"f32",256),("bla",1,1,"f32",200)]
for c in cases:
    try:
        t=time.time(); r = run(*c)
        print(c, "err=%.3e Merr=%.3e bad=%s" % (r[0][0], r[0][1], r[0][2]), "%.2fs"%(time.time()-t))
        if r[0][0] > 0.05: print("   got", r[0][3], "\n   want", r[0][4])
    except Exception as ex:
        print(c, "EXC", repr(ex)[:300])
    sys.stdout.flush()
