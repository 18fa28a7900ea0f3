import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run under gpurun)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def load_golden(group):
    return dict(np.load(os.path.join(GOLDEN, group + ".npz")))


def golden_cases(d):
    """Case prefixes of a golden group (keys look like '<case>/<array>')."""
    return sorted({k.rsplit("/", 1)[0] for k in d})


def norm_rel_err(got, want):
    """max|got-want| / max|want| -- the north-star error definition."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    scale = max(np.abs(want).max(), 1e-30)
    return float(np.abs(got - want).max() / scale)


@pytest.fixture(scope="session")
def cuda_ok():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return True


def record_parity(name, err, tol, **extra):
    """Logs an achieved parity error next to its bound (how much of the budget a test uses):
    printed, and appended as JSON to $LMOE_PARITY_LOG or gpurun_out/parity_errors.jsonl when
    that directory exists (the GPU box copies it back; profiles/ keeps the summaries)."""
    import json
    rec = {"test": name, "err": float(err), "tol": float(tol), "used": float(err) / float(tol)}
    rec.update(extra)
    print("PARITY", json.dumps(rec))
    path = os.environ.get("LMOE_PARITY_LOG")
    if not path and os.path.isdir(os.path.join(ROOT, "gpurun_out")):
        path = os.path.join(ROOT, "gpurun_out", "parity_errors.jsonl")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(rec) + "\n")
