"""bench.py -- LSM-layer tokens/s on B200 with LSM sequence parallelism (BASELINE.json
config 3: per-token-decay LSM, seq 256K, H=16, d=128, bf16; SP over 1/2/4/8 GPUs).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...   (one process per GPU, NCCL)

A step = one LSM forward over the whole 256K-token sequence, all 16 heads, split across
ranks by chunk_range (parallel.hpp:192-197) through lmoe_sp_lsm_fwd.  For Mamba2 that is the
local-state forward: the output pass from zero segment states, the segment combine (and at
N > 1 ONE ncclAllGather of the per-rank state payload plus the decayed rank prefix), then the
correction of each segment's first chunks.  Inputs (3 x 1 GiB)
are resident in HBM and larger than L2, so no flush is needed between steps.  Timing:
CUDA events on the launching stream, barrier + synchronize on both sides, max over ranks.
Prints ONE JSON line on rank 0.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SEQ, HEADS, HEAD_DIM = 262144, 16, 128
METRIC = "LSM-layer tokens/sec at 1/2/4/8 B200 (SP); % tensor-pipe peak vs CPU ref"
# algorithmic bytes per (token, head): 3*d*s_in + d*s_out + g
#   Mamba2: g = 4 (fp32 b_pre); flops per (token, head) = 4 d^2 + 2 C d, C = 64
ALG_BYTES_TH = {"mamba2": 3 * 128 * 2 + 128 * 2 + 4, "lightning": 4 * 128 * 2,
                "retnet": 4 * 128 * 2, "bla": 4 * 128 * 2}
ALG_FLOPS_TH = 4 * 128 * 128 + 2 * 64 * 128


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], p["bf16_tflops"], "measured"
    except Exception:  # noqa: BLE001
        return 6650.0, 1590.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + self.FIELDS,
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:  # noqa: BLE001
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:  # noqa: BLE001
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus > 1 and world == 1:
        print("note: --gpus %d without torchrun; running 1 rank" % args.gpus, file=sys.stderr)
    return world, rank, local


def cpu_reference(instance, tokens, threads, budget_s, gate_mean=0.0):
    """Times the reference CPU path (oracle/_ref/ref_driver: the unmodified reference
    headers' lsm_forward_chunked, f32 mode, C=64, one (b,h) per thread).  Falls back to
    the oracle C restatement when the reference build is absent."""
    drv = os.path.join(ROOT, "oracle", "_ref", "ref_driver")
    if os.path.exists(drv):
        # chunk 16 = the reference model default (model.hpp:36); at chunk 64 its f32-mode
        # K/p closed form overflows ("non-finite output in div") for Mamba2 gates
        out = subprocess.run([drv, "bench-lsm", instance, "1", str(tokens), str(HEADS),
                              str(HEAD_DIM), "16", str(threads), str(budget_s), str(gate_mean)],
                             capture_output=True, text=True, timeout=budget_s * 4 + 120)
        if out.returncode == 0 and out.stdout.strip():
            r = json.loads(out.stdout.strip().splitlines()[-1])
            if r["heads_done"] > 0:
                return {"value": r["tokens_per_sec"], "unit": "tokens/s", "cores": r["threads"],
                        "kind": "reference",
                        "sample": "%d of %d (b,h) sequences of %d tokens within a %.0fs budget, "
                                  "reference lsm_forward_chunked, f32 mode, chunk 16, "
                                  "extrapolated to all %d heads" % (r["heads_done"], r["heads_total"],
                                                                    tokens, budget_s, HEADS)}
    # port fallback: float64 C restatement, single thread, one head sample
    import numpy as np
    import oracle
    n = 8192
    rng = np.random.default_rng(0)
    q, k, v = (rng.normal(0, 0.5, (n, HEAD_DIM)) for _ in range(3))
    spec = oracle.spec_default(instance)
    spec["mamba2_a_raw"] = 0.3
    t0 = time.time()
    oracle.lsm_chunked(spec, q, k, v, b_pre=rng.normal(0, 1, n), chunk=64)
    dt = time.time() - t0
    return {"value": n / dt / HEADS, "unit": "tokens/s", "cores": 1, "kind": "port",
            "sample": "1 head x %d tokens, f64 oracle, extrapolated to %d heads" % (n, HEADS)}


def run_reference(args, world, rank):
    """--impl reference: the reference's CPU implementation on the box's host cores."""
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    budget = max(5.0, min(40.0, 60.0 / max(1, args.steps + args.warmup)))
    vals = []
    cb = None
    for i in range(args.warmup + args.steps):
        cb = cpu_reference(args.instance, SEQ, threads, budget)
        if i >= args.warmup:
            vals.append(cb["value"])
    v = statistics.median(vals) if vals else cb["value"]
    cb["value"] = v
    line = {"metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": SEQ / v * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32 (reference f32 mode)",
            "data": "synthetic N(0,0.5^2) q,k,v; N(0,1) gates", "impl": "reference",
            "config": headline_config(args.instance, world),
            "cpu_baseline": cb,
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def headline_config(instance, world, rank=0):
    """The config dict both arms print (ours and --impl reference), so the driver can match them."""
    base, rem = divmod(SEQ, world)
    n_loc = base + (1 if rank < rem else 0)
    return {"workload": "cfg3 per-token-decay LSM (%s) with LSM sequence parallelism" % instance,
            "seq_len": SEQ, "heads": HEADS, "head_dim": HEAD_DIM, "batch": 1,
            "tokens_per_rank": n_loc, "parallelism": "sp%d" % world}


def make_inputs(dev, n_loc, rank, instance="mamba2"):
    """Synthetic inputs of the config-3 shape, this rank's slice [1, n_loc, H, d] (also used by
    tests/test_fullshape_gpu.py, so parity is checked on exactly the benchmarked data):
    q, k, v ~ N(0, 0.5^2) bf16; Mamba2 b_pre ~ N(0, 1) fp32 and a_raw ~ N(0, 0.5^2) per head
    (the reference's LsmSpec::make / LsmGates defaults, lsm.hpp:177, 222-253)."""
    import torch
    import paper_2503_05447_b200 as pk
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    q, k, v = (torch.randn(1, n_loc, HEADS, HEAD_DIM, device=dev, generator=g).mul_(0.5)
               .to(torch.bfloat16) for _ in range(3))
    b_pre = torch.randn(1, n_loc, HEADS, device=dev, generator=g)
    spec = pk.LsmSpec.make(instance, HEAD_DIM)
    # a_raw is a per-head parameter of the whole sequence: the same on every rank
    spec.mamba2_a_raw = torch.randn(HEADS, device=dev, generator=torch.Generator(device=dev).manual_seed(99)).mul_(0.5)
    gates = pk.LsmGates(b_pre=b_pre) if instance == "mamba2" else None
    return q, k, v, b_pre, spec, gates


def make_gla_inputs(dev, n=SEQ):
    """cfg3 GLA side inputs (gla_bench): q, k, v ~ N(0, 0.5^2), dO, a_pre ~ N(0, 1), bf16."""
    import torch
    g = torch.Generator(device=dev).manual_seed(21)
    return tuple(torch.randn(1, n, HEADS, HEAD_DIM, device=dev, generator=g).mul_(s).to(torch.bfloat16)
                 for s in (0.5, 0.5, 0.5, 1.0, 1.0))


def layer_bench(dev, steps=5, warmup=3, cpu=True):
    """SURVEY 8(d) second number: LSM-layer tokens/s on cfg4 (A0.3B-2B Linear-MoE block:
    hidden 1024, 8 heads x 128, GLA, FFN 896, 64 experts top-8; 8 documents x 8192 tokens)
    through lmoe_block_fwd: RMSNorm, fused QKV+gate GEMM, LSM, W_o, RMSNorm, MoE, residuals."""
    import torch
    from paper_2503_05447_b200.lsm import LsmInstance
    from paper_2503_05447_b200.model import Model, ModelConfig
    cfg = ModelConfig(hidden=1024, ffn_dim=896, num_heads=8, num_experts=64, num_active=8, vocab_size=256,
                      instance=LsmInstance.GLA, pattern="L", max_seq_len=8192)
    m = Model.init(cfg, seed=0, device=str(dev))
    B, N = 8, 8192
    g = torch.Generator(device=dev).manual_seed(7)
    x0 = torch.randn(B * N, cfg.hidden, device=dev, generator=g)
    x = x0.clone()
    for _ in range(warmup):
        x.copy_(x0)
        m.run_block(0, x, B, N)
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        m.run_block(0, x, B, N)
    e1.record()
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1) / steps
    T, h, H, d, F, E, K = B * N, cfg.hidden, cfg.num_heads, 128, cfg.ffn_dim, cfg.num_experts, cfg.num_active
    flops = T * (2 * h * 4 * h + 2 * h * h + 2 * h * E + 6 * K * h * F + H * (4 * d * d + 2 * 64 * d))
    tflops_peak = 1373.0
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            tflops_peak = json.load(f)["bf16_tflops_sustained"]
    except Exception:  # noqa: BLE001
        pass
    tf = flops / (ms / 1e3) / 1e12
    res = {"workload": "cfg4 A0.3B-2B Linear-MoE block (GLA LSM + 64-expert top-8 MoE), 8 x 8192 tokens",
           "tokens_per_s": T / (ms / 1e3), "ms_per_step": ms, "steps": steps,
           "roofline": {"bound": "tensor", "achieved": tf, "peak": tflops_peak, "unit": "TFLOP/s",
                        "frac": tf / tflops_peak, "flops_per_step": flops,
                        "note": "GEMM + LSM flops per block; peak = MEASURED_PEAKS bf16_tflops_sustained"}}
    # end to end: the fp32 residual stream in from pinned host memory, the block, and back out
    hx = x0.cpu().pin_memory()
    hy = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
    ems, bi, bo = e2e_ms(dev, (hx,), (x,), lambda: m.run_block(0, x, B, N), hy, x, steps)
    res["e2e"] = {"value": T / (ems / 1e3), "unit": "tokens/s", "h2d_bytes_per_step": bi, "d2h_bytes_per_step": bo,
                  "path": "pinned host x -> H2D -> lmoe_block_fwd (C-ABI) -> D2H"}
    if cpu:
        r = ref_driver(["bench-block", "gla", "L", 256, cfg.hidden, cfg.num_heads, cfg.ffn_dim, cfg.num_experts,
                        cfg.num_active, os.cpu_count() or 1, 15], 300)
        if r and r.get("tokens_done", 0) > 0:
            res["cpu_baseline"] = {
                "value": r["tokens_per_sec"], "unit": "tokens/s", "cores": r["threads"], "kind": "reference",
                "sample": "reference Block body of model_forward (rms_norm, LsmMixer GLA, residual, rms_norm, "
                          "MoeLayer, residual), f32 mode, 256-token documents for 15 s on all host threads "
                          "(per-token cost is length-independent for the LSM mixer)"}
    return res


def backward_bench(dev, steps=3, warmup=2):
    """LSM backward (lmoe_lsm_bwd) at the cfg3 shape on one GPU: Mamba2, N = 262144, 16 x 128."""
    import torch
    import paper_2503_05447_b200 as pk
    g = torch.Generator(device=dev).manual_seed(11)
    q, k, v, dO = (torch.randn(1, SEQ, HEADS, HEAD_DIM, device=dev, generator=g).mul_(0.5).to(torch.bfloat16)
                   for _ in range(4))
    gates = pk.LsmGates(b_pre=torch.randn(1, SEQ, HEADS, device=dev, generator=g))
    spec = pk.LsmSpec.make("mamba2", HEAD_DIM)
    spec.mamba2_a_raw = torch.randn(HEADS, device=dev, generator=g).mul_(0.5)
    for _ in range(warmup):
        pk.lsm_backward_batched(q, k, v, gates, spec, dO, check=False)
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        pk.lsm_backward_batched(q, k, v, gates, spec, dO, check=False)
    e1.record()
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1) / steps
    hbm, _, _ = peaks()
    # backward bytes per (token, head) = 4 d s_in + 3 d s_out + 2 g
    alg = (4 * HEAD_DIM * 2 + 3 * HEAD_DIM * 2 + 2 * 4) * SEQ * HEADS
    gbs = alg / (ms / 1e3) / 1e9
    return {"workload": "cfg3 Mamba2 LSM backward (dq, dk, dv, db_pre, da_raw, dM0), N=262144, 16 x 128",
            "tokens_per_s": SEQ / (ms / 1e3), "ms_per_step": ms, "steps": steps,
            "roofline": {"bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm,
                         "note": "algorithmic bytes of the op / step time (three chunk passes + gate kernel)"}}


OUTPASS_NCU = "profiles/r2_lsm_output_pass.ncu.txt"
FUSED_NCU = "profiles/r2_lsm_fused_fwd.ncu.txt"
LOCAL_NCU = "profiles/r2_local_output_pass.ncu.txt"  # the output pass in local-state mode (default)


def ncu_traffic(rel=OUTPASS_NCU):
    """dram read + write bytes per launch of the dominant kernel from the committed ncu --set full
    capture (profiles/), or None when absent."""
    path = os.path.join(ROOT, rel)
    try:
        vals = {}
        for line in open(path):
            parts = line.split()
            if len(parts) >= 3 and parts[0] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}[parts[2]]
                vals[parts[0]] = float(parts[1]) * scale
        return vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"]
    except (OSError, KeyError, ValueError):
        return None


def gla_bench(dev, steps=3, warmup=2):
    """TokenVector side numbers at the cfg3 shape (GLA, N = 262144, 16 x 128, a_pre ~ N(0, 1) as
    the reference's gate default): forward (lmoe_lsm_fwd) and backward (lmoe_lsm_bwd: dq, dk, dv,
    da_pre, dM0), each against the HBM roofline of its algorithmic bytes (SURVEY 8(d):
    fwd 3 d s_in + d s_out + d s_gate = 1280 B, bwd 4 d s_in + 3 d s_out + 2 d s_gate = 2304 B
    per (token, head))."""
    import torch
    import paper_2503_05447_b200 as pk
    q, k, v, dO, a = make_gla_inputs(dev)
    gates = pk.LsmGates(a_pre=a)
    spec = pk.LsmSpec.make("gla", HEAD_DIM)
    hbm, _, _ = peaks()
    out = {}
    for name, fn, per in (("forward", lambda: pk.lsm_forward_batched(q, k, v, gates, spec, 64, check=False), 1280),
                          ("backward", lambda: pk.lsm_backward_batched(q, k, v, gates, spec, dO, check=False), 2304)):
        for _ in range(warmup):
            fn()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            fn()
        e1.record()
        torch.cuda.synchronize(dev)
        ms = e0.elapsed_time(e1) / steps
        gbs = per * SEQ * HEADS / (ms / 1e3) / 1e9
        out[name] = {"tokens_per_s": SEQ / (ms / 1e3), "ms_per_step": ms, "steps": steps,
                     "roofline": {"bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm,
                                  "alg_bytes_per_token_head": per}}
    out["workload"] = "cfg3 GLA (TokenVector decay) LSM, N=262144, 16 x 128, bf16, a_pre ~ N(0,1)"
    return out


def ref_driver(cmd, timeout):
    """Runs oracle/_ref/ref_driver (the unmodified reference headers, compiled by
    oracle/Makefile) and returns its JSON line, or None when the build is absent."""
    drv = os.path.join(ROOT, "oracle", "_ref", "ref_driver")
    if not os.path.exists(drv):
        return None
    out = subprocess.run([drv] + [str(a) for a in cmd], capture_output=True, text=True, timeout=timeout)
    if out.returncode != 0 or not out.stdout.strip():
        return None
    return json.loads(out.stdout.strip().splitlines()[-1])


def graph_ms(dev, fn, steps, warmup):
    """Device ms per call of fn (launches on the current stream): captured once as a CUDA
    graph on a side stream and replayed `steps` times between CUDA events on that stream."""
    import torch
    st = torch.cuda.Stream(dev)
    with torch.cuda.stream(st):
        for _ in range(warmup):
            fn()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            fn()
        g.replay()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(steps):
            g.replay()
        e1.record(st)
        torch.cuda.synchronize(dev)
    return e0.elapsed_time(e1) / steps


def e2e_ms(dev, host_in, dev_in, fn, host_out, dev_out, steps):
    """End-to-end ms per step through the public API: every step copies its inputs from pinned
    host memory (H2D), runs fn, and copies the result back (D2H), all inside the timed region.
    Returns (ms, h2d_bytes, d2h_bytes)."""
    import torch
    st = torch.cuda.Stream(dev)
    with torch.cuda.stream(st):
        def one():
            for h, d in zip(host_in, dev_in):
                d.copy_(h, non_blocking=True)
            fn()
            host_out.copy_(dev_out, non_blocking=True)
        one()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(steps):
            one()
        e1.record(st)
        torch.cuda.synchronize(dev)
    h2d = sum(x.numel() * x.element_size() for x in host_in)
    return e0.elapsed_time(e1) / steps, h2d, host_out.numel() * host_out.element_size()


def cfg1_bench(dev, steps=50, warmup=5, cpu=True):
    """Config 1, the reference's own test shape: BLA without decay, B = 1,
    N = 2048, H = 8, d = 64, fp32 in / out (tf32 tensor cores, fp32 accumulation), chunk 64.
    Two variants: plain (identity phi, no normaliser; test_lsm.cpp:35, verify.hpp:77-78) and
    the reference default (elu+1 + normaliser, lsm.hpp:157-160).  16.8 MB per step: the HBM
    roofline is 2.6 us, so this shape is launch-latency bound; the number says by how much."""
    import torch
    import paper_2503_05447_b200 as pk
    n, h, d = 2048, 8, 64
    g = torch.Generator(device=dev).manual_seed(1)
    q, k, v = (torch.randn(1, n, h, d, device=dev, generator=g).mul_(0.5) for _ in range(3))
    o = torch.empty_like(q)
    hbm, _, _ = peaks()
    alg = 4 * d * 4 * n * h  # 3 d s_in + d s_out bytes per (token, head), fp32
    res = {"workload": "cfg1 BLA (no decay), B=1, N=2048, H=8, d=64, fp32, chunk 64, CUDA-graph replay"}
    for name, spec in (("plain", pk.LsmSpec(instance=0, feature_map=0)), ("default", pk.LsmSpec.make("bla", d))):
        fn = lambda: pk.lsm_forward_batched(q, k, v, None, spec, 64, out=o, check=False)
        ms = graph_ms(dev, fn, steps, warmup)
        gbs = alg / (ms / 1e3) / 1e9
        res[name] = {"tokens_per_s": n / (ms / 1e3), "us_per_step": ms * 1e3,
                     "roofline": {"bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s",
                                  "frac": gbs / hbm, "alg_bytes_per_step": alg}}
        hq, hk, hv = (x.cpu().pin_memory() for x in (q, k, v))
        ho = torch.empty(o.shape, dtype=o.dtype, pin_memory=True)
        ems, bi, bo = e2e_ms(dev, (hq, hk, hv), (q, k, v), fn, ho, o, steps)
        res[name]["e2e"] = {"value": n / (ems / 1e3), "unit": "tokens/s", "h2d_bytes_per_step": bi,
                            "d2h_bytes_per_step": bo}
    if cpu:
        r = ref_driver(["bench-lsm", "bla", 1, n, h, d, 64, os.cpu_count() or 1, 10], 200)
        if r and r.get("heads_done", 0) > 0:
            res["cpu_baseline"] = {"value": r["tokens_per_sec"], "unit": "tokens/s", "cores": r["threads"],
                                   "kind": "reference",
                                   "sample": "reference lsm_forward_chunked (bla default), f32 mode, chunk 64, "
                                             "%d of %d heads within 10 s, all host threads"
                                             % (r["heads_done"], r["heads_total"])}
    return res


def lsm_layer_bench(dev, steps=3, warmup=2):
    """SURVEY 8(d)'s second number at the headline shape: LSM-layer tokens/s for config 3
    (Mamba2, one 262144-token document, hidden 2048 = 16 heads x 128): rms_norm, the fused
    [Wq | Wk | Wv] GEMM, the W_gate_b GEMM (b_pre), the LSM, W_o and the residual add --
    lmoe_block_fwd with num_experts = 0 (the mixer layer without the MoE)."""
    import torch
    from paper_2503_05447_b200.lsm import LsmInstance
    from paper_2503_05447_b200.model import Model, ModelConfig
    cfg = ModelConfig(hidden=2048, ffn_dim=128, num_heads=HEADS, num_experts=8, num_active=2, vocab_size=256,
                      instance=LsmInstance.MAMBA2, pattern="L", max_seq_len=SEQ)
    m = Model.init(cfg, seed=0, device=str(dev), draw_on_device=True)
    g = torch.Generator(device=dev).manual_seed(12)
    x0 = torch.randn(SEQ, cfg.hidden, device=dev, generator=g)
    x = x0.clone()
    for _ in range(warmup):
        m.run_block(0, x, 1, SEQ, moe=False)
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        m.run_block(0, x, 1, SEQ, moe=False)
    e1.record()
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1) / steps
    h, d = cfg.hidden, HEAD_DIM
    flops = SEQ * (2 * h * 3 * h + 2 * h * 64 + 2 * h * h + HEADS * (4 * d * d + 2 * 64 * d))
    tflops_peak = 1373.0
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            tflops_peak = json.load(f)["bf16_tflops_sustained"]
    except Exception:  # noqa: BLE001
        pass
    tf = flops / (ms / 1e3) / 1e12
    del m
    torch.cuda.empty_cache()
    return {"workload": "cfg3 LSM layer (Mamba2, N=262144, hidden 2048 = 16 x 128): rms_norm + QKV/gate GEMMs + "
                        "LSM + W_o + residual, lmoe_block_fwd without MoE",
            "tokens_per_s": SEQ / (ms / 1e3), "ms_per_step": ms, "steps": steps,
            "roofline": {"bound": "tensor", "achieved": tf, "peak": tflops_peak, "unit": "TFLOP/s",
                         "frac": tf / tflops_peak, "flops_per_step": flops,
                         "note": "projection GEMM + LSM flops; peak = MEASURED_PEAKS bf16_tflops_sustained"}}


def hybrid_bench(dev, steps=2, warmup=1, cpu=True):
    """Config 5: the hybrid A1B-7B Linear-MoE stack -- hidden 2048, 16 heads x 128,
    FFN 1024, 64 experts top-8, 16 layers LLLNLLLNLLLNLLLN -- over ONE 131072-token
    document on one GPU (SP degree 1; the driver's multi-GPU run would split it by chunk_range).
    GLA LSM layers; N layers are causal softmax attention over the whole document.  Weights drawn
    on the device with the reference's init scales; x ~ N(0, 1) fp32 residual stream."""
    import torch
    from paper_2503_05447_b200.lsm import LsmInstance
    from paper_2503_05447_b200.model import Model, ModelConfig
    N = 131072
    cfg = ModelConfig(hidden=2048, ffn_dim=1024, num_heads=16, num_experts=64, num_active=8, vocab_size=256,
                      instance=LsmInstance.GLA, pattern="LLLN" * 4, max_seq_len=N)
    m = Model.init(cfg, seed=0, device=str(dev), draw_on_device=True)
    g = torch.Generator(device=dev).manual_seed(8)
    x0 = torch.randn(N, cfg.hidden, device=dev, generator=g)
    x = x0.clone()
    nb = len(cfg.pattern)

    def stack():
        for i in range(nb):
            m.run_block(i, x, 1, N)
    for _ in range(warmup):
        x.copy_(x0)
        stack()
    torch.cuda.synchronize(dev)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(nb + 1)]
    tot, per = 0.0, [0.0] * nb
    for _ in range(steps):
        x.copy_(x0)
        ev[0].record()
        for i in range(nb):
            m.run_block(i, x, 1, N)
            ev[i + 1].record()
        torch.cuda.synchronize(dev)
        tot += ev[0].elapsed_time(ev[nb])
        for i in range(nb):
            per[i] += ev[i].elapsed_time(ev[i + 1])
    ms = tot / steps
    h, H, d, F, E, K = cfg.hidden, cfg.num_heads, 128, cfg.ffn_dim, cfg.num_experts, cfg.num_active
    moe = 2 * h * E + 6 * K * h * F
    fl_L = N * (2 * h * 4 * h + 2 * h * h + moe + H * (4 * d * d + 2 * 64 * d))
    fl_N = N * (2 * h * 3 * h + 2 * h * h + moe) + H * 2 * N * N * d  # causal QK^T + PV
    flops = 12 * fl_L + 4 * fl_N
    tflops_peak = 1373.0
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            tflops_peak = json.load(f)["bf16_tflops_sustained"]
    except Exception:  # noqa: BLE001
        pass
    tf = flops / (ms / 1e3) / 1e12
    msL = sum(per[i] for i in range(nb) if cfg.pattern[i] == "L") / steps / 12
    msN = sum(per[i] for i in range(nb) if cfg.pattern[i] == "N") / steps / 4
    res = {"workload": "cfg5 hybrid A1B-7B stack (16 layers LLLN x 4, GLA + causal attention, 64-expert top-8 MoE), "
                       "one 131072-token document, 1 GPU",
           "tokens_per_s": N / (ms / 1e3), "ms_per_step": ms, "steps": steps,
           "ms_per_L_block": msL, "ms_per_N_block": msN,
           "roofline": {"bound": "tensor", "achieved": tf, "peak": tflops_peak, "unit": "TFLOP/s",
                        "frac": tf / tflops_peak, "flops_per_step": flops,
                        "note": "GEMM + LSM + causal attention flops of the 16 blocks; peak = bf16_tflops_sustained"},
           "sp8_kv_gather": {"bytes_received_per_rank_per_N_layer": 2 * 7 * (N // 8) * H * d * 2,
                             "note": "K and V bf16 of the 7 other ranks (SURVEY 8(d) cfg5); not exercised on 1 GPU"}}
    if cpu:
        rates = {}
        for kind in ("L", "N"):
            r = ref_driver(["bench-block", "gla", kind, 256, h, H, F, E, K, os.cpu_count() or 1, 12], 300)
            if r and r.get("tokens_done", 0) > 0:
                rates[kind] = r
        if len(rates) == 2:
            v = 1.0 / (12.0 / rates["L"]["tokens_per_sec"] + 4.0 / rates["N"]["tokens_per_sec"])
            res["cpu_baseline"] = {
                "value": v, "unit": "tokens/s", "cores": rates["L"]["threads"], "kind": "reference",
                "sample": "reference Block body of model_forward, f32 mode, L (GLA) and N (dense causal attention) "
                          "blocks each timed 12 s on 256-token documents on all host threads, composed as "
                          "12 L + 4 N per token; the reference's dense attention is quadratic, so at the 128K "
                          "document the CPU is slower than this"}
    del m
    torch.cuda.empty_cache()
    return res


def cfg2_bench(dev, steps=20, warmup=3, cpu=True):
    """Config-2 side numbers: Lightning (a = 0.95) and RetNet (a = 1 - 1/32)
    scalar-decay LSM forward, B = 1, N = 32768, H = 16, d = 128, bf16 in / out, through the
    same call as the headline (world 1: the local pass), CUDA-graph replay; HBM roofline of
    3 d s_in + d s_out = 1024 B per (token, head) (537 MB per step > L2, no flush needed)."""
    import torch
    import paper_2503_05447_b200 as pk
    from paper_2503_05447_b200 import sp
    n = 32768
    comm = sp.NcclComm(0, 1)
    g = torch.Generator(device=dev).manual_seed(2)
    q, k, v = (torch.randn(1, n, HEADS, HEAD_DIM, device=dev, generator=g).mul_(0.5).to(torch.bfloat16)
               for _ in range(3))
    out_t = torch.empty_like(q)
    hbm, _, _ = peaks()
    res = {}
    st = torch.cuda.Stream(dev)
    for inst in ("lightning", "retnet"):
        spec = pk.LsmSpec.make(inst, HEAD_DIM)
        gates = pk.LsmGates()
        with torch.cuda.stream(st):
            for _ in range(warmup):
                sp.sp_lsm_masked_rank(comm, q, k, v, gates, spec, 64, out=out_t, check=False, stream=st.cuda_stream)
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=st):
                sp.sp_lsm_masked_rank(comm, q, k, v, gates, spec, 64, out=out_t, check=False, stream=st.cuda_stream)
            graph.replay()
            torch.cuda.synchronize(dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(steps):
                graph.replay()
            e1.record(st)
            torch.cuda.synchronize(dev)
        ms = e0.elapsed_time(e1) / steps
        gbs = 1024 * n * HEADS / (ms / 1e3) / 1e9
        res[inst] = {"tokens_per_s": n / (ms / 1e3), "ms_per_step": ms, "steps": steps,
                     "roofline": {"bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm,
                                  "alg_bytes_per_token_head": 1024, "note": "whole step (3 kernels)"}}
        hq, hk, hv = (x.cpu().pin_memory() for x in (q, k, v))
        ho = torch.empty(out_t.shape, dtype=out_t.dtype, pin_memory=True)
        fn = lambda: sp.sp_lsm_masked_rank(comm, q, k, v, gates, spec, 64, out=out_t, check=False)
        ems, bi, bo = e2e_ms(dev, (hq, hk, hv), (q, k, v), fn, ho, out_t, 5)
        res[inst]["e2e"] = {"value": n / (ems / 1e3), "unit": "tokens/s", "h2d_bytes_per_step": bi,
                            "d2h_bytes_per_step": bo}
        if cpu:
            r = ref_driver(["bench-lsm", inst, 1, n, HEADS, HEAD_DIM, 64, os.cpu_count() or 1, 10], 200)
            if r and r.get("heads_done", 0) > 0:
                res[inst]["cpu_baseline"] = {
                    "value": r["tokens_per_sec"], "unit": "tokens/s", "cores": r["threads"], "kind": "reference",
                    "sample": "reference lsm_forward_chunked, f32 mode, chunk 64, %d of %d heads of %d tokens "
                              "within 10 s, extrapolated to all heads" % (r["heads_done"], r["heads_total"], n)}
    res["workload"] = "cfg2 scalar-decay LSM forward, N=32768, 16 x 128, bf16, CUDA-graph replay"
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--instance", default="mamba2", choices=["mamba2", "lightning", "retnet", "bla"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the layer / backward side numbers")
    ap.add_argument("--no-graph", action="store_true", help="time direct calls instead of a CUDA-graph replay")
    args = ap.parse_args()
    world, rank, local = dist_setup(args)
    if args.impl == "reference":
        if world > 1:
            import torch.distributed as dist
            dist.init_process_group("gloo")
        run_reference(args, world, rank)
        return

    import torch
    import torch.distributed as dist

    import paper_2503_05447_b200 as pk
    from paper_2503_05447_b200 import sp as spm
    from paper_2503_05447_b200 import _lib

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    comm = spm.NcclComm(rank, world, dev)
    r0, r1 = spm.chunk_range(SEQ, world, rank)
    n_loc = r1 - r0

    q, k, v, b_pre, spec, gates = make_inputs(dev, n_loc, rank, args.instance)
    out = torch.empty_like(q)
    stream = torch.cuda.Stream(dev)  # a side stream (CUDA-graph capture needs a non-default stream)

    def step(timing=False):
        spm.sp_lsm_masked_rank(comm, q, k, v, gates, spec, 64, out=out, check=False,
                               timing=timing, stream=stream.cuda_stream)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step()
    barrier()
    _lib.timing_read(8)  # drop warm-up timings

    # The step (kernels + the NCCL all-gather) is captured once as a CUDA graph and replayed:
    # the timed region is then free of host submission gaps.  --no-graph times direct calls.
    graph, per_step = None, None
    if not args.no_graph:
        try:
            n0 = pk.launch_count()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                step()
            per_step = pk.launch_count() - n0
            graph = g
            graph.replay()
            barrier()
        except Exception as exc:  # noqa: BLE001 -- capture unsupported here: time direct calls
            print("bench: CUDA graph capture failed (%s); timing direct calls" % exc, file=sys.stderr)
            graph = None
            barrier()

    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    launches0 = pk.launch_count()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    with torch.cuda.stream(stream):
        for _ in range(args.steps):
            if graph is not None:
                graph.replay()
            else:
                step()
    e1.record(stream)
    barrier()
    launches = per_step * args.steps if graph is not None else pk.launch_count() - launches0
    ms_total = e0.elapsed_time(e1)
    clk = clocks.stop()
    # per-phase device times (roofline of the dominant kernel): the same step with CUDA events
    # between its kernels, outside the timed region
    with torch.cuda.stream(stream):
        for _ in range(args.steps):
            step(timing=True)
    barrier()
    calls, phase_ms = _lib.timing_read(8)
    # phases of lmoe_sp_lsm_fwd: 0 state pass, 1 local combine, 2 all-gather,
    # 3 rank combine, 4 segment combine, 5 output pass
    t = torch.tensor([ms_total], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = t.item() / args.steps
    value = SEQ / (ms_step / 1e3)

    # ---- end to end through the public API, host buffers, copies inside the timed region
    hq, hk, hv = (x.cpu().pin_memory() for x in (q, k, v))
    hb = b_pre.cpu().pin_memory()
    hout = torch.empty(out.shape, dtype=out.dtype, pin_memory=True)
    h2d = sum(x.numel() * x.element_size() for x in (hq, hk, hv)) + (
        hb.numel() * 4 if args.instance == "mamba2" else 0)
    d2h = hout.numel() * hout.element_size()
    dq, dk, dv, db = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v), torch.empty_like(b_pre)
    dgates = pk.LsmGates(b_pre=db) if args.instance == "mamba2" else None

    # Pipelined like a serving loop: step i+1's H2D (copy stream) overlaps step i's D2H (second
    # copy stream; PCIe is full duplex), inputs / outputs double-buffered in HBM.
    bufs = [(dq, dk, dv, db, dgates, out)]
    q2, k2, v2, b2 = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v), torch.empty_like(b_pre)
    bufs.append((q2, k2, v2, b2, pk.LsmGates(b_pre=b2) if args.instance == "mamba2" else None, torch.empty_like(out)))
    s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    done = [torch.cuda.Event(), torch.cuda.Event()]  # output of slot j copied out
    done[0].record(s_out)
    done[1].record(s_out)

    def e2e_step(i):
        xq, xk, xv, xb, xg, xo = bufs[i & 1]
        s_in.wait_event(done[i & 1])  # slot free: its previous output has left the device
        with torch.cuda.stream(s_in):
            xq.copy_(hq, non_blocking=True)
            xk.copy_(hk, non_blocking=True)
            xv.copy_(hv, non_blocking=True)
            if xg is not None:
                xb.copy_(hb, non_blocking=True)
        stream.wait_stream(s_in)
        spm.sp_lsm_masked_rank(comm, xq, xk, xv, xg, spec, 64, out=xo, check=False,
                               stream=stream.cuda_stream)
        s_out.wait_stream(stream)
        with torch.cuda.stream(s_out):
            hout.copy_(xo, non_blocking=True)
        done[i & 1].record(s_out)

    e2e_step(0)
    barrier()
    e0.record(stream)
    s_in.wait_stream(stream)  # the timed region starts before the first H2D
    for i in range(args.e2e_steps):
        e2e_step(i + 1)
    e1.record(s_out)
    barrier()
    te = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = SEQ / (te.item() / args.e2e_steps / 1e3)

    # ---- roofline of the dominant kernel: the single-read kernel (world 1, one launch) or the
    # output pass (SP): either moves the full algorithmic bytes of the op (reads q,k,v,gate,
    # writes o) for this rank's tokens x heads
    hbm, tflops, src = peaks()
    plan = pk.lsm.forward_plan(spec, 1, n_loc, HEADS, HEAD_DIM)
    fused = plan["fused"] and world == 1
    local = plan["local"]  # local-state forward: output pass first (phase 0)
    out_pass_ms = (phase_ms[0] if (fused or local) else phase_ms[5]) / max(calls, 1)
    units = n_loc * HEADS
    alg_bytes = ALG_BYTES_TH[args.instance] * units
    achieved = alg_bytes / (out_pass_ms / 1e3) / 1e9
    step_alg = ALG_BYTES_TH[args.instance] * units / (ms_step / 1e3) / 1e9
    phase_names = ["state_pass", "local_combine", "all_gather", "rank_combine(fused into next)",
                   "rank_seg_combine", "output_pass"]
    if fused:
        phase_names = ["lsm_fused_fwd"]
    if local:
        phase_names = (["output_pass(local state)", "-", "seg_combine", "local_fix", "-", "-"] if world == 1 else
                       ["output_pass(local state)", "-", "local_combine", "all_gather", "rank_seg_combine",
                        "local_fix"])

    if rank == 0:
        cb = None
        extra = {}
        if world == 1 and not args.no_extra:
            extra["layer"] = layer_bench(dev, cpu=not args.no_cpu_baseline)
            extra["lsm_layer"] = lsm_layer_bench(dev)
            extra["backward"] = backward_bench(dev)
            extra["gla"] = gla_bench(dev)
            extra["cfg2"] = cfg2_bench(dev, cpu=not args.no_cpu_baseline)
            extra["cfg1"] = cfg1_bench(dev, cpu=not args.no_cpu_baseline)
            extra["hybrid"] = hybrid_bench(dev, cpu=not args.no_cpu_baseline)
        if world == 1 and not args.no_cpu_baseline:
            cb = cpu_reference(args.instance, SEQ, os.cpu_count() or 1, 20.0)
        prof_file = FUSED_NCU if fused else (LOCAL_NCU if plan.get("local") else OUTPASS_NCU)
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic: q,k,v ~ N(0,0.5^2) bf16, Mamba2 b_pre ~ N(0,1) fp32, a_raw ~ N(0,0.5^2)",
            "config": headline_config(args.instance, world, rank),
            "timing": {"timed": "CUDA-graph replay of the step" if graph is not None else "direct calls",
                       "l2": "inputs 3 GiB > L2; no flush needed"},
            "gpu_launches": launches,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": achieved / hbm, "traffic": ncu_traffic(prof_file),
                         "peak_source": src,
                         "traffic_source": prof_file + " (ncu --set full, one launch)",
                         "kernel": "lsm_fused_fwd" if fused else "lsm_output_pass",
                         "plan": plan,
                         "alg_bytes_per_launch": alg_bytes,
                         "alg_bytes_per_token_head": ALG_BYTES_TH[args.instance]},
            "step_roofline": {"achieved": step_alg, "frac": step_alg / hbm, "unit": "GB/s",
                              "note": "whole-step algorithmic bytes / step time"},
            "phase_ms_per_step": {n: phase_ms[i] / max(calls, 1) for i, n in enumerate(phase_names)},
            "clocks": clk,
            "e2e": {"value": e2e_value, "unit": "tokens/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h,
                    "path": "pinned host -> H2D -> lmoe_sp_lsm_fwd (C-ABI) -> D2H, H2D(i+1) overlapping D2H(i)"},
            "cpu_baseline": cb,
        }
        line.update(extra)
        print(json.dumps(line))
    comm.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
