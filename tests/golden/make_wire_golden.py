# SPDX-License-Identifier: Apache-2.0
"""Golden fixtures for the store-dump / eviction-report wire formats (SURVEY
§8 f2), from the REFERENCE's own objects and JSON library:

* the records: oracle/_ref/libpikv_ref.so (reference kvstore/router/... driven
  in Engine::step order) -- every eviction record of a run and the final
  KVStore::snapshot(now);
* the lines: oracle/wire_golden.cpp, which builds the objects as runner.cpp
  does and serialises them with nlohmann::json (the reference's JSON library;
  found in this image under cudnn_frontend/thirdparty).

Needs /root/reference and g++ (build container only); the fixtures travel.

    python tests/golden/make_wire_golden.py
"""
import glob
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from cases import engine_config  # noqa: E402
from oracle_bind import RefEngine, make_stream, ref_lib  # noqa: E402
from paper_2508_06526_b200.wire import REASONS  # noqa: E402

CASES = [
    # name, engine_config kwargs, steps, stream seed
    ("h2o_h2", dict(router="LoadBalanced", sched="H2O", H=2), 80, 23),
    ("lruplus_overwrite", dict(router="TopK", sched="LRUPlus", S=8, budget=16), 80, 31),
    ("adakv_theta", dict(router="CacheAware", sched="AdaKV"), 80, 29),
]
# doubles whose nlohmann layout or grisu2 digits are worth pinning
EDGE_SCORES = [0.0, -0.0, 1.0, -5.0, 0.1, 1 / 3, 1e-7, 1e-5, 1e-4, 123456.789, 1e15, 1e16,
               1e21, 5e-324, 1.7976931348623157e308, -1234567890123.25, 2.0 ** 53, 1e23, 0.3]


def wire_tool():
    inc = glob.glob(os.path.join(sys.prefix, "lib", "python3*", "site-packages", "include",
                                 "cudnn_frontend", "thirdparty"))
    if not inc:
        raise SystemExit("nlohmann/json.hpp not found")
    exe = os.path.join(ROOT, "oracle", "_ref", "wire_golden")
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", inc[0],
                    os.path.join(ROOT, "oracle", "wire_golden.cpp"), "-o", exe], check=True)
    return exe


def main():
    if ref_lib() is None:
        raise SystemExit("reference objects unavailable (needs /root/reference)")
    exe = wire_tool()
    for name, kw, T, seed in CASES:
        cfg = engine_config(**kw)
        eng = RefEngine(cfg)
        st = make_stream(T, cfg.model.d, seed, cfg.kv_dtype, cfg.n_layers)
        evs = []
        for t in range(T):
            r = eng.step(st[0][t], st[1][t], st[2][t], None if cfg.n_layers == 0 else st[3][t])
            evs += [(e[1], e[2], e[3], e[4], e[5], e[6]) for e in r["evictions"]]
        snap = eng.snapshot(T)
        if name == "h2o_h2":  # crafted scores ride along with real records
            evs += [(1000 + i, i, i % 4, i % 2, sc, i % 3) for i, sc in enumerate(EDGE_SCORES)]
        inp = "".join("S %d %d %d %d %d %d\n" % (r["device"], r["shard"], r["token"], r["expert"],
                                                  r["age"], r["freq"]) for r in snap)
        inp += "".join("E %d %d %d %d %s %s\n" % (i, tk, ex, dv, float(sc).hex(), REASONS[rs])
                       for i, tk, ex, dv, sc, rs in evs)
        out = subprocess.run([exe], input=inp, capture_output=True, text=True, check=True).stdout
        lines = out.splitlines()
        ev = np.array(evs, dtype=[("id", "<u8"), ("token", "<i8"), ("expert", "<i4"),
                                  ("device", "<i4"), ("score", "<f8"), ("reason", "<i4")])
        np.savez_compressed(os.path.join(HERE, "wire", "wire_%s.npz" % name), snapshot=snap, evictions=ev,
                            steps=T, seed=seed, now=T)
        with open(os.path.join(HERE, "wire", "wire_%s.jsonl" % name), "w") as f:
            f.write("\n".join(lines) + "\n")
        print(name, len(snap), "store lines,", len(evs), "eviction lines")


if __name__ == "__main__":
    main()
