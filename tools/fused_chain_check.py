"""Developer aid: dumps what every (head, segment) of lsm_fused_fwd used -- its own state
S_seg, its total log decay, the entering state M_in read from the hand-off ring -- and checks
(1) S_seg and logD against float64 host values, (2) M_in(s) == D(s-1) M_in(s-1) + S_seg(s-1)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2503_05447_b200 as pk

D = 128
N = int(sys.argv[1]) if len(sys.argv) > 1 else 40000
H = int(sys.argv[2]) if len(sys.argv) > 2 else 16
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
g = torch.Generator(device="cuda").manual_seed(3)
q, k, v = (torch.randn(1, N, H, D, device="cuda", generator=g).mul_(0.5).bfloat16() for _ in range(3))
b = torch.randn(1, N, H, device="cuda", generator=g).mul_(0.5).sub_(3.0)
spec = pk.LsmSpec.make("mamba2", D)
a_raw = torch.linspace(-0.6, 0.4, H, device="cuda")
spec.mamba2_a_raw = a_raw
gates = pk.LsmGates(b_pre=b)
plan = pk.lsm.forward_plan(spec, 1, N, H, D)
nseg, L = plan["segments"], plan["seg_len"]
print("plan", plan)
dbg = torch.zeros(H * nseg * 2 * D * D + H * nseg + 4, device="cuda")
os.environ["LMOE_FUSED_DEBUG_PTR"] = str(dbg.data_ptr())

sp = lambda x: np.log1p(np.exp(-np.abs(x))) + np.maximum(x, 0)
kk, vv, bb = k[0].double().cpu().numpy(), v[0].double().cpu().numpy(), b[0].double().cpu().numpy()
ar = a_raw.double().cpu().numpy()
Sref, Lref = np.zeros((H, nseg, D, D)), np.zeros((H, nseg))
parts = {}  # (h, s) -> list of (chunk c, token quarter q, k-column group hh, partial S rows of hh)
for h in range(H):
    spb = sp(bb[:, h])
    la = -spb * sp(ar[h])
    for s in range(nseg):
        t0, t1 = s * L, min(N, (s + 1) * L)
        lseg = la[t0:t1]
        suffix = np.concatenate([np.cumsum(lseg[::-1])[::-1][1:], [0.0]])  # sum over t' > t
        w = np.exp(suffix) * spb[t0:t1]
        Sref[h, s] = (kk[t0:t1, h] * w[:, None]).T @ vv[t0:t1, h]
        parts[(h, s)] = (t0, t1, w)
        Lref[h, s] = lseg.sum()
prevM = None
for r in range(reps):
    dbg.zero_()
    pk.lsm_forward_batched(q, k, v, gates, spec, 64, check=False)
    torch.cuda.synchronize()
    x = dbg.cpu().numpy().astype(np.float64)
    SM = x[:H * nseg * 2 * D * D].reshape(H, nseg, 2, D, D)
    S, M = SM[:, :, 0], SM[:, :, 1]
    lg = x[H * nseg * 2 * D * D:H * nseg * 2 * D * D + H * nseg].reshape(H, nseg)
    cnt = dbg[H * nseg * 2 * D * D + H * nseg:].view(torch.int32).cpu().numpy()
    print("   stale A-step ring reads %d, non-positive A weights %d, stale C-step ring reads %d" % tuple(cnt[:3]))
    bad = []
    for h in range(H):
        for s in range(nseg):
            eS = np.abs(S[h, s] - Sref[h, s]).max() / max(np.abs(Sref[h, s]).max(), 1e-30)
            eL = abs(lg[h, s] - Lref[h, s])
            if s > 0:
                want = np.exp(lg[h, s - 1]) * M[h, s - 1] + S[h, s - 1]
                eM = np.abs(M[h, s] - want).max() / max(np.abs(want).max(), 1e-30)
            else:
                eM = np.abs(M[h, s]).max()
            if eS > 1e-2 or eL > 1e-3 or eM > 1e-4:
                bad.append((h, s, round(eS, 4), round(eL, 5), round(eM, 5), round(float(np.abs(M[h, s]).max()), 4)))
                if eS > 1e-2:  # which (chunk, token quarter, column group) carries the wrong factor
                    t0, t1, w = parts[(h, s)]
                    for hh in range(4):
                        cols, ys = [], S[h, s][hh * 32:(hh + 1) * 32].ravel()
                        keys = []
                        for c0 in range(t0, t1, 128):
                            for qq in range(4):
                                a0, a1 = c0 + qq * 32, min(t1, c0 + qq * 32 + 32)
                                if a0 >= a1:
                                    continue
                                part = (kk[a0:a1, h, hh * 32:(hh + 1) * 32] * w[a0 - t0:a1 - t0, None]).T @ vv[a0:a1, h]
                                cols.append(part.ravel())
                                keys.append(((c0 - t0) // 128, qq))
                        A = np.stack(cols, 1)
                        alpha = np.linalg.lstsq(A, ys, rcond=None)[0]
                        off = [(kq, round(float(al), 3)) for kq, al in zip(keys, alpha) if abs(al - 1) > 0.05]
                        print("   head %d seg %d col group %d: factors != 1 at (chunk, token quarter): %s" % (h, s, hh, off))
    for (h, s_, *_r) in bad:
        X = (S[h, s_] - Sref[h, s_]).ravel()
        best = []
        for nm, src in (("M_in this rep", M), ("M_in prev rep", prevM)):
            if src is None:
                continue
            Y = src.reshape(H * nseg, -1)
            c = Y @ X / (np.linalg.norm(Y, axis=1) * np.linalg.norm(X) + 1e-30)
            i = int(np.argmax(np.abs(c)))
            best.append((nm, divmod(i, nseg), round(float(c[i]), 4), round(float(np.linalg.norm(X) / (np.linalg.norm(Y[i]) + 1e-30)), 3)))
        t0, t1, w = parts[(h, s_)]
        Xm = (S[h, s_] - Sref[h, s_])
        cands = []
        for c0 in range(t0, t1, 128):
            for qq in range(4):
                a0, a1 = c0 + qq * 32, min(t1, c0 + qq * 32 + 32)
                if a0 >= a1:
                    continue
                for hh in range(4):
                    Y = np.zeros((D, D))
                    Y[hh * 32:(hh + 1) * 32] = (kk[a0:a1, h, hh * 32:(hh + 1) * 32] * (1 - w[a0 - t0:a1 - t0, None])).T @ vv[a0:a1, h]
                    c = float((Y * Xm).sum() / (np.linalg.norm(Y) * np.linalg.norm(Xm) + 1e-30))
                    cands.append((round(c, 3), (c0 - t0) // 128, qq, hh, round(float(np.linalg.norm(Xm) / np.linalg.norm(Y)), 3)))
        cands.sort(reverse=True)
        print("      best 'one warp block left unweighted' (corr, chunk, token quarter, col group, |X|/|Y|): %s" % cands[:3])
        blk = [(hh, qq, round(float(np.abs(Xm[hh * 32:(hh + 1) * 32]).max()), 3)) for hh in range(4) for qq in range(1)]
        print("      max|X| per S row block (col group): %s" % blk)
        print("   X = S_gpu - S_ref of (head %d, seg %d): best-correlated dumped state (name, (head, seg), corr, |X|/|Y|): %s" % (h, s_, best))
    prevM = M.copy()
    print("rep %d: %d bad (head, seg, S err, logD err, M_in hand-off err, max|M_in|): %s" % (r, len(bad), bad[:12]))
