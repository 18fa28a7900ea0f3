"""ctypes binding of the float64 CPU oracle (oracle/lmoe_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline leg of bench.py -- never by the product package
paper_2503_05447_b200, which fails loudly without its CUDA library.
"""
import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liblmoe_oracle.so")
REF_DRIVER = os.path.join(HERE, "_ref", "ref_driver")

# lmoe::LsmInstance numbering (lsm.hpp:30-48)
INSTANCES = ["bla", "lightning", "retnet", "gla", "deltanet", "gated_deltanet", "rebased",
             "gfw", "gateloop", "ttt", "titans", "s4", "mamba", "mamba2", "hgrn2", "rwkv6",
             "rwkv7"]
FM_IDENTITY, FM_ELU1, FM_SQUARED = 0, 1, 2


class OracleError(RuntimeError):
    pass


class _Spec(ctypes.Structure):
    _fields_ = [("instance", ctypes.c_int), ("feature_map", ctypes.c_int),
                ("use_normalizer", ctypes.c_int), ("scalar_decay", ctypes.c_double),
                ("mamba2_a_raw", ctypes.c_double)]


def build():
    subprocess.check_call(["make", "-s", "-C", HERE], stdout=subprocess.DEVNULL)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        _lib = ctypes.CDLL(LIB_PATH)
    return _lib


def _p(a):
    if a is None:
        return None
    return a.ctypes.data_as(ctypes.c_void_p)


def _f64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


def spec_default(instance):
    if isinstance(instance, str):
        instance = INSTANCES.index(instance)
    s = _Spec()
    lib().lmo_spec_default(ctypes.byref(s), ctypes.c_int(instance))
    return {"instance": s.instance, "feature_map": s.feature_map,
            "use_normalizer": s.use_normalizer, "scalar_decay": s.scalar_decay,
            "mamba2_a_raw": s.mamba2_a_raw}


def _spec(d):
    s = _Spec()
    s.instance = int(d["instance"])
    s.feature_map = int(d.get("feature_map", 0))
    s.use_normalizer = int(d.get("use_normalizer", 0))
    s.scalar_decay = float(d.get("scalar_decay", 1.0))
    s.mamba2_a_raw = float(d.get("mamba2_a_raw", 0.0))
    return s


def decay_kind(instance):
    return lib().lmo_decay_kind(ctypes.c_int(instance))


def _run(fn, *args):
    err = ctypes.create_string_buffer(256)
    rc = fn(*args, err, ctypes.c_int(256))
    if rc != 0:
        raise OracleError(err.value.decode())


def lsm_chunked(spec, q, k, v, a_pre=None, b_pre=None, chunk=64, M0=None, z0=None):
    """lsm_forward_chunked (lsm.hpp:668) for one head: q,k (n,d_k), v (n,d_v)."""
    q, k, v, a_pre, b_pre, M0, z0 = map(_f64, (q, k, v, a_pre, b_pre, M0, z0))
    n, dk = q.shape
    dv = v.shape[1]
    o = np.zeros((n, dv))
    M = np.zeros((dk, dv))
    z = np.zeros(dk)
    sp = _spec(spec)
    _run(lib().lmo_lsm_chunked, ctypes.byref(sp), n, dk, dv, chunk, _p(q), _p(k), _p(v),
         _p(a_pre), _p(b_pre), _p(M0), _p(z0), _p(o), _p(M), _p(z))
    return o, M, z


def lsm_sequential(spec, q, k, v, a_pre=None, b_pre=None, M0=None, z0=None):
    q, k, v, a_pre, b_pre, M0, z0 = map(_f64, (q, k, v, a_pre, b_pre, M0, z0))
    n, dk = q.shape
    dv = v.shape[1]
    o = np.zeros((n, dv))
    M = np.zeros((dk, dv))
    z = np.zeros(dk)
    sp = _spec(spec)
    _run(lib().lmo_lsm_sequential, ctypes.byref(sp), n, dk, dv, _p(q), _p(k), _p(v),
         _p(a_pre), _p(b_pre), _p(M0), _p(z0), _p(o), _p(M), _p(z))
    return o, M, z


def lsm_recurrent(spec, q, k, v, a_pre=None, b_pre=None, alpha_pre=None, beta_pre=None, s4_delta_raw=None,
                  s4_b=None, s4_A_raw=None, mamba_A_raw=None, M0=None):
    """recurrent_step (lsm.hpp:335-441) for the kinds without a chunk-parallel form."""
    arrs = list(map(_f64, (q, k, v, a_pre, b_pre, alpha_pre, beta_pre, s4_delta_raw, s4_b, s4_A_raw,
                           mamba_A_raw, M0)))
    n, dk = arrs[0].shape
    dv = arrs[2].shape[1]
    o = np.zeros((n, dv))
    M = np.zeros((dk, dv))
    sp = _spec(spec)
    _run(lib().lmo_lsm_recurrent, ctypes.byref(sp), n, dk, dv, *[_p(x) for x in arrs], _p(o), _p(M))
    return o, M


def lsm_backward(spec, q, k, v, dO, a_pre=None, b_pre=None, M0=None, dM_final=None):
    q, k, v, a_pre, b_pre, M0, dO, dM_final = map(_f64, (q, k, v, a_pre, b_pre, M0, dO, dM_final))
    n, dk = q.shape
    dv = v.shape[1]
    dq, dkk, dvv = np.zeros((n, dk)), np.zeros((n, dk)), np.zeros((n, dv))
    da = np.zeros((n, dk))
    db = np.zeros(n)
    draw = ctypes.c_double(0.0)
    dM0 = np.zeros((dk, dv))
    sp = _spec(spec)
    _run(lib().lmo_lsm_backward, ctypes.byref(sp), n, dk, dv, _p(q), _p(k), _p(v), _p(a_pre),
         _p(b_pre), _p(M0), _p(dO), _p(dq), _p(dkk), _p(dvv), _p(da), _p(db), ctypes.byref(draw),
         _p(dM0), _p(dM_final))
    return {"dq": dq, "dk": dkk, "dv": dvv, "da_pre": da, "db_pre": db, "da_raw": draw.value,
            "dM0": dM0}


def route(logits, top_k):
    logits = _f64(logits)
    t, e = logits.shape
    ids = np.zeros((t, top_k), dtype=np.int32)
    gates = np.zeros((t, e))
    probs = np.zeros((t, e))
    _run(lib().lmo_route, _p(logits), t, e, top_k, _p(ids), _p(gates), _p(probs))
    return ids, gates, probs


def load_balance_loss(ids, probs):
    ids = np.ascontiguousarray(ids, dtype=np.int32)
    probs = _f64(probs)
    f = lib().lmo_load_balance_loss
    f.restype = ctypes.c_double
    return f(_p(ids), _p(probs), probs.shape[0], probs.shape[1], ids.shape[1])


def moe_forward(x, router, w_gate, w_up, w_down, top_k):
    x, router, w_gate, w_up, w_down = map(_f64, (x, router, w_gate, w_up, w_down))
    t, hidden = x.shape
    e = router.shape[1]
    ffn = w_gate.shape[2]
    y = np.zeros((t, hidden))
    logits = np.zeros((t, e))
    aux = ctypes.c_double(0.0)
    _run(lib().lmo_moe_forward, _p(x), t, hidden, ffn, e, top_k, _p(router), _p(w_gate),
         _p(w_up), _p(w_down), _p(y), ctypes.byref(aux), _p(logits))
    return y, aux.value, logits


def chunk_range(n, t, rank):
    r0, r1 = ctypes.c_int(0), ctypes.c_int(0)
    lib().lmo_chunk_range(n, t, rank, ctypes.byref(r0), ctypes.byref(r1))
    return r0.value, r1.value


def sp_forward_masked(spec, q, k, v, world, a_pre=None, b_pre=None, rank_chunk=0):
    q, k, v, a_pre, b_pre = map(_f64, (q, k, v, a_pre, b_pre))
    n, dk = q.shape
    dv = v.shape[1]
    o = np.zeros((n, dv))
    sp = _spec(spec)
    _run(lib().lmo_sp_forward_masked, ctypes.byref(sp), n, dk, dv, world, rank_chunk, _p(q),
         _p(k), _p(v), _p(a_pre), _p(b_pre), _p(o))
    return o


def sp_forward_nomask(spec, q, k, v, world):
    """sp_forward_nomask (parallel.hpp:391-403): non-causal O = phi(Q) sum_r phi(K_r)^T V_r."""
    q, k, v = map(_f64, (q, k, v))
    n, dk = q.shape
    dv = v.shape[1]
    o = np.zeros((n, dv))
    _run(lib().lmo_sp_forward_nomask, ctypes.byref(_spec(spec)), n, dk, dv, world, _p(q), _p(k), _p(v), _p(o))
    return o


def sp_payload_width(spec, dv):
    sp = _spec(spec)
    return lib().lmo_sp_payload_width(ctypes.byref(sp), dv)


def sp_local_payload(spec, q, k, v, a_pre=None, b_pre=None, chunk=0):
    q, k, v, a_pre, b_pre = map(_f64, (q, k, v, a_pre, b_pre))
    n, dk = q.shape
    dv = v.shape[1]
    pw = sp_payload_width(spec, dv)
    out = np.zeros((dk, pw))
    sp = _spec(spec)
    _run(lib().lmo_sp_local_payload, ctypes.byref(sp), n, dk, dv, chunk, _p(q), _p(k), _p(v),
         _p(a_pre), _p(b_pre), _p(out))
    return out


def sp_combine(spec, gathered, rank, dv):
    gathered = _f64(gathered)
    dk = gathered.shape[1]
    M = np.zeros((dk, dv))
    z = np.zeros(dk)
    sp = _spec(spec)
    lib().lmo_sp_combine(ctypes.byref(sp), dk, dv, rank, _p(gathered), _p(M), _p(z))
    return M, z


def attention(q, k, v, causal=True, row_offset=0):
    q, k, v = map(_f64, (q, k, v))
    o = np.zeros((q.shape[0], v.shape[1]))
    lib().lmo_attention(_p(q), _p(k), _p(v), q.shape[0], k.shape[0], q.shape[1], v.shape[1],
                        int(causal), int(row_offset), _p(o))
    return o


def spec_from_golden(d, prefix):
    return {"instance": int(d[prefix + "/instance"][0]),
            "feature_map": int(d[prefix + "/feature_map"][0]),
            "use_normalizer": int(d[prefix + "/use_normalizer"][0]),
            "scalar_decay": float(d[prefix + "/scalar_decay"][0]),
            "mamba2_a_raw": float(d[prefix + "/mamba2_a_raw"][0])}
