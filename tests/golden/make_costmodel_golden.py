# SPDX-License-Identifier: Apache-2.0
"""Golden vectors for the analytic cost model from the
REFERENCE's own costmodel.cpp (compiled unchanged into oracle/_ref, wrapped
by ref_cost_report in oracle/ref_driver.cpp).  Needs /root/reference.

    python tests/golden/make_costmodel_golden.py
"""
import ctypes
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle_bind import ref_lib  # noqa: E402
from paper_2508_06526_b200.config import EngineConfig, ModelConfig  # noqa: E402

N_OUT = 27


def ref_report(m: ModelConfig, hw, batch, active, thr):
    lib = ref_lib()
    lib.ref_cost_report.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_double), ctypes.c_double,
                                    ctypes.c_int, ctypes.c_double, ctypes.POINTER(ctypes.c_double)]
    cfg = EngineConfig()
    cfg.model = m
    cfg.router.k = m.k  # pikv_config.k is the router's k (EngineConfig.to_c)
    c = cfg.to_c()
    h = (ctypes.c_double * 5)(*hw)
    out = (ctypes.c_double * N_OUT)()
    rc = lib.ref_cost_report(ctypes.byref(c), h, batch, active, thr, out)
    return rc, list(out)


def cases():
    rng = np.random.default_rng(2508)
    out = []
    # the reference KAT configs (test_costmodel.cpp cost_config) + B200 workloads
    out.append(dict(d=64, head_width=1, rho=2.0, L=1024, G=4, S=8, K=2, E=8, k=2, elem_bytes=2))
    out.append(dict(d=512, head_width=64, rho=1.0, L=4096, G=1, S=1, K=1, E=64, k=4, elem_bytes=2))
    out.append(dict(d=4096, head_width=128, rho=1.0, L=32768, G=1, S=6144, K=4, E=16, k=2,
                    elem_bytes=2))
    out.append(dict(d=4096, head_width=128, rho=4.0, L=65536, G=8, S=8192, K=4, E=16, k=2,
                    elem_bytes=2))
    for _ in range(60):
        d = int(rng.integers(8, 8192))
        E = int(rng.integers(1, 128))
        out.append(dict(d=d, head_width=int(rng.integers(1, d + 1)), rho=float(1 + rng.random() * 7),
                        L=int(rng.integers(1, 1 << 20)), G=int(rng.integers(1, 17)),
                        S=int(rng.integers(1, 1 << 15)), K=int(rng.integers(1, 64)), E=E,
                        k=int(rng.integers(1, E + 1)), elem_bytes=int(rng.integers(1, 5))))
    res = []
    for i, m in enumerate(out):
        hw = [float(10 ** rng.uniform(9, 13)), float(10 ** rng.uniform(9, 13)),
              float(rng.uniform(0.1, 2.0)), float(10 ** rng.uniform(11, 16)),
              float(10 ** rng.uniform(10, 13))]
        if i == 2:
            hw = [6456.8e9, 6456.8e9, 1.0, 1672.3e12, 6456.8e9]
        res.append(dict(model=m, hw=hw, batch=float(rng.integers(1, 257)),
                        active=int(rng.integers(0, m["E"] + 1)), thr=float(rng.random() * 0.5)))
    return res


def main():
    if ref_lib() is None:
        raise SystemExit("reference objects unavailable (needs /root/reference)")
    rows = []
    for c in cases():
        rc, out = ref_report(ModelConfig(**c["model"]), c["hw"], c["batch"], c["active"], c["thr"])
        c["rc"] = rc
        c["out"] = [x.hex() for x in out] if rc == 0 else []
        c["hw"] = [x.hex() for x in c["hw"]]
        c["model"]["rho"] = float(c["model"]["rho"]).hex()
        c["batch"] = c["batch"].hex()
        c["thr"] = c["thr"].hex()
        rows.append(c)
    with open(os.path.join(HERE, "costmodel.json"), "w") as f:
        json.dump(rows, f, indent=0)
    print(len(rows), "cases")


if __name__ == "__main__":
    main()
