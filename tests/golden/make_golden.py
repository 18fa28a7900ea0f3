"""Regenerates tests/golden/*.npz from the UNMODIFIED reference.

Runs oracle/_ref/ref_driver (oracle/ref_driver.cpp compiled against
/root/reference/proj/include by oracle/Makefile) and packs its record stream
into one .npz per group.  Only runnable where /root/reference exists (the
build container); the committed .npz files are what travels to the GPU box.

    python tests/golden/make_golden.py
"""
import os
import struct
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
DRIVER = os.path.join(ROOT, "oracle", "_ref", "ref_driver")

# groups whose large arrays are stored as float32 (inputs are bf16-exact there); in "model"
# only the parameters (rounded to bf16 by the driver), never the logits
F32_GROUPS = {"lsm_dev", "model"}


def read_records(path):
    out = {}
    with open(path, "rb") as f:
        data = f.read()
    off = 0
    while off < len(data):
        (nl,) = struct.unpack_from("<I", data, off)
        off += 4
        name = data[off:off + nl].decode()
        off += nl
        (nd,) = struct.unpack_from("<I", data, off)
        off += 4
        shape = struct.unpack_from("<%dI" % nd, data, off)
        off += 4 * nd
        cnt = int(np.prod(shape)) if nd else 1
        arr = np.frombuffer(data, dtype="<f8", count=cnt, offset=off).reshape(shape)
        off += 8 * cnt
        out[name] = arr.copy()
    return out


def main():
    subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "oracle")])
    if not os.path.exists(DRIVER):
        sys.exit("oracle/_ref/ref_driver missing: /root/reference is needed to regenerate")
    with tempfile.TemporaryDirectory() as td:
        raw = os.path.join(td, "golden.bin")
        subprocess.check_call([DRIVER, "golden", raw])
        recs = read_records(raw)
    groups = {}
    for name, arr in recs.items():
        g, rest = name.split("/", 1)
        if g in F32_GROUPS and arr.size > 1 and "logits" not in rest:
            arr = arr.astype(np.float32)
        groups.setdefault(g, {})[rest] = arr
    for g, d in groups.items():
        np.savez_compressed(os.path.join(HERE, g + ".npz"), **d)
        print("wrote %s.npz (%d arrays)" % (g, len(d)))


if __name__ == "__main__":
    main()
