# SPDX-License-Identifier: Apache-2.0
"""Golden QueryEncoder outputs (pipeline.cpp:29-57, the encode at the start
of Engine::step, :222) from the REFERENCE's own code (oracle/_ref, verbatim
extract of pipeline.cpp:29-57).  Needs /root/reference.

    python tests/golden/make_encoder_golden.py
"""
import ctypes
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle_bind import ref_lib  # noqa: E402

CASES = [(16, 1 ^ 0x71c9de52ae0aef), (64, 7 ^ 0x71c9de52ae0aef), (96, 12345)]


def ref_encode(width, seed, x):
    lib = ref_lib()
    P = ctypes.POINTER(ctypes.c_double)
    lib.ref_encode.argtypes = [ctypes.c_int, ctypes.c_uint64, P, P, P, P]
    q, k, v = (np.zeros(width) for _ in range(3))
    rc = lib.ref_encode(width, seed, x.ctypes.data_as(P), q.ctypes.data_as(P), k.ctypes.data_as(P),
                        v.ctypes.data_as(P))
    assert rc == 0
    return q, k, v


def main():
    if ref_lib() is None:
        raise SystemExit("reference objects unavailable (needs /root/reference)")
    rng = np.random.default_rng(222)
    out = {}
    for width, seed in CASES:
        x = rng.standard_normal(width)
        q, k, v = ref_encode(width, seed, x)
        out["w%d_seed" % width] = np.uint64(seed)
        out["w%d_x" % width], out["w%d_q" % width] = x, q
        out["w%d_k" % width], out["w%d_v" % width] = k, v
    np.savez_compressed(os.path.join(HERE, "encoder", "query_encoder.npz"), **out)
    print("wrote", len(CASES), "cases")


if __name__ == "__main__":
    main()
