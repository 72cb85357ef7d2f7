# SPDX-License-Identifier: Apache-2.0
"""Golden traces from the REFERENCE's own generate_trace and
save_trace (trace.cpp, compiled unchanged into oracle/_ref).  Needs
/root/reference.

    python tests/golden/make_trace_golden.py
"""
import ctypes
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle_bind import ref_lib  # noqa: E402

CASES = [  # steps, width, vocab, skew, seed, layers
    (64, 16, 64, 1.0, 1, 4),
    (200, 32, 17, 0.0, 99, 3),
    (50, 8, 5, 2.5, 12345678901234, 1),
]


def ref_trace(steps, width, vocab, skew, seed, layers, path=None):
    lib = ref_lib()
    lib.ref_generate_trace.argtypes = [ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                       ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p,
                                       ctypes.c_void_p, ctypes.c_void_p, ctypes.c_char_p]
    voc = np.zeros((vocab, width))
    ids = np.zeros(steps, dtype=np.uint32)
    sal = np.zeros((steps, layers), dtype=np.float32)
    rc = lib.ref_generate_trace(steps, width, vocab, skew, seed, layers, voc.ctypes.data,
                                ids.ctypes.data, sal.ctypes.data,
                                None if path is None else path.encode())
    assert rc == 0, rc
    return voc, ids, sal


def main():
    if ref_lib() is None:
        raise SystemExit("reference objects unavailable (needs /root/reference)")
    for i, c in enumerate(CASES):
        path = os.path.join(HERE, "trace", "trace_%d.pikt" % i)
        voc, ids, sal = ref_trace(*c, path=path)
        np.savez_compressed(os.path.join(HERE, "trace", "trace_%d.npz" % i), spec=np.array(c, dtype=np.float64),
                            seed=np.uint64(c[4]), vocabulary=voc, embed_ids=ids, saliency=sal)
    print(len(CASES), "traces")


if __name__ == "__main__":
    main()
