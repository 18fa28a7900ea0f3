"""ctypes loader for liblmoe_cuda.so (the C-ABI in include/lmoe_cuda.h).

There is no CPU fallback: if the library cannot be loaded (or built, on a box with nvcc)
every entry point raises.  The library is built in-tree so it travels with the repo.
"""
import ctypes
import os

from . import _build

_lib = None


class LmoeError(RuntimeError):
    """Raised with the library's message (the reference's error text where one exists)."""

    def __init__(self, status, msg):
        super().__init__(msg)
        self.status = status


STATUS = {0: "OK", 1: "ARG", 2: "SHAPE", 3: "DEGENERATE", 4: "NONFINITE", 5: "CUDA", 6: "NCCL",
          7: "UNSUPPORTED"}


class LsmDesc(ctypes.Structure):
    _fields_ = [("instance", ctypes.c_int), ("feature_map", ctypes.c_int),
                ("use_normalizer", ctypes.c_int), ("scalar_decay", ctypes.c_float),
                ("chunk_size", ctypes.c_int), ("flags", ctypes.c_int)]


def lib():
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("LMOE_LIB") or _build.LIB  # LMOE_LIB: developer A/B of a prebuilt library
    if not os.environ.get("LMOE_LIB") and not _build.up_to_date():
        try:
            _build.build()
        except Exception as e:  # noqa: BLE001
            if not os.path.exists(path):
                raise RuntimeError("liblmoe_cuda.so is missing and could not be built: %s" % e)
    L = ctypes.CDLL(path, mode=ctypes.RTLD_GLOBAL)
    vp, sz, i, f = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_float
    L.lmoe_last_error.restype = ctypes.c_char_p
    L.lmoe_version.restype = ctypes.c_char_p
    L.lmoe_launch_count.restype = ctypes.c_longlong
    L.lmoe_lsm_fwd_workspace_size.restype = sz
    L.lmoe_lsm_fwd_workspace_size.argtypes = [ctypes.POINTER(LsmDesc), i, i, i, i, i]
    L.lmoe_lsm_fwd.restype = i
    L.lmoe_lsm_fwd.argtypes = [ctypes.POINTER(LsmDesc), i, i, i, i, i, vp, vp, vp, vp, vp, vp,
                               vp, vp, vp, vp, vp, vp, sz, vp]
    L.lmoe_lsm_bwd_workspace_size.restype = sz
    L.lmoe_lsm_bwd_workspace_size.argtypes = [ctypes.POINTER(LsmDesc), i, i, i, i, i]
    L.lmoe_lsm_bwd.restype = i
    L.lmoe_lsm_bwd.argtypes = [ctypes.POINTER(LsmDesc), i, i, i, i, i] + [vp] * 17 + [sz, vp]
    L.lmoe_lsm_varlen_workspace_size.restype = sz
    L.lmoe_lsm_varlen_workspace_size.argtypes = [ctypes.POINTER(LsmDesc), i, vp, i, i, i, i, i]
    L.lmoe_lsm_fwd_varlen.restype = i
    L.lmoe_lsm_fwd_varlen.argtypes = [ctypes.POINTER(LsmDesc), i, vp, i, i, i, i] + [vp] * 9 + [sz, vp]
    L.lmoe_lsm_bwd_varlen.restype = i
    L.lmoe_lsm_bwd_varlen.argtypes = [ctypes.POINTER(LsmDesc), i, vp, i, i, i, i] + [vp] * 14 + [sz, vp]
    L.lmoe_lsm_fwd_plan.restype = i
    L.lmoe_lsm_fwd_plan.argtypes = [ctypes.POINTER(LsmDesc), i, i, i, i, i, vp]
    L.lmoe_timing_read.restype = i
    L.lmoe_timing_read.argtypes = [ctypes.POINTER(ctypes.c_float), i]
    _lib = L
    return L


def check(rc):
    if rc != 0:
        raise LmoeError(rc, lib().lmoe_last_error().decode())


def ptr(t):
    """Device pointer of a torch tensor (or None)."""
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def launch_count():
    return int(lib().lmoe_launch_count())


def timing_read(nphase=3):
    arr = (ctypes.c_float * nphase)()
    calls = lib().lmoe_timing_read(arr, nphase)
    if calls < 0:
        raise LmoeError(-calls, lib().lmoe_last_error().decode())
    return calls, [float(x) for x in arr]
