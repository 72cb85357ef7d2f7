# SPDX-License-Identifier: Apache-2.0
"""Generate golden step traces from the REFERENCE's own objects.

Runs oracle/_ref/libpikv_ref.so (reference kvstore/router/mathops compiled
unchanged + verbatim scheduler/pipeline extracts, driven by
oracle/ref_driver.cpp in Engine::step order) on fixed configs and seeds and
stores every step's outputs plus the final slot state in tests/golden/*.npz.
Needs /root/reference (build container only); the fixtures travel.

    python tests/golden/make_golden.py
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from cases import engine_config  # noqa: E402
from oracle_bind import RefEngine, make_stream, ref_lib  # noqa: E402

CASES = [
    # name, engine_config kwargs, steps, stream seed
    ("lossless_topk_h1", dict(router="TopK", unbounded=True, S=256), 80, 13),
    ("lossless_hier_h2", dict(router="Hierarchical", unbounded=True, S=256, H=2), 80, 13),
    ("lossless_adaptive", dict(router="Adaptive", unbounded=True, S=256), 80, 17),
    ("lru_budget", dict(router="TopK", sched="LRU"), 80, 19),
    ("h2o_budget_h2", dict(router="LoadBalanced", sched="H2O", H=2), 80, 23),
    ("adakv_theta", dict(router="CacheAware", sched="AdaKV"), 80, 29),
    ("adakv_budget_h2", dict(router="TopK", sched="AdaKV", theta0=-1e18, H=2, budget=6), 80, 47),
    ("sl_overwrite", dict(router="EntropyLB", sched="SL", S=8, budget=16), 80, 31),
    ("duo_layers", dict(router="Base", sched="Duo"), 60, 37),
    ("flex_ragged_ring", dict(router="TopK", sched="Flex", S=10, ps=4, budget=3), 80, 41),
    ("lruplus_g1_ntok1", dict(router="TopK", sched="LRUPlus", G=1, n_tok=1, n_exp=8), 80, 43),
]


def main():
    if ref_lib() is None:
        sys.exit("reference objects unavailable (needs /root/reference)")
    for name, kw, T, seed in CASES:
        cfg = engine_config(**kw)
        eng = RefEngine(cfg)
        q, k, v, sal = make_stream(T, cfg.model.d, seed, cfg.kv_dtype, cfg.n_layers)
        rec = {"experts": [], "gates": [], "y": [], "hits": [], "n_attended": [], "fetch": [],
               "ev": [], "ev_step": [], "att": [], "att_step": [], "pages": []}
        for t in range(T):
            r = eng.step(q[t], k[t], v[t], None if sal is None else sal[t])
            rec["experts"].append(r["experts"])
            rec["gates"].append(r["gates"])
            rec["y"].append(r["y"])
            rec["hits"].append(r["hits"])
            rec["n_attended"].append(r["n_attended"])
            rec["fetch"].append(r["fetch_elements"])
            rec["pages"].append((r["pages_before"], r["pages_after"]))
            for e in r["evictions"]:
                rec["ev"].append(e)
                rec["ev_step"].append(t)
            for a in zip(r["att_token"], r["att_expert"], r["att_weight"]):
                rec["att"].append(a)
                rec["att_step"].append(t)
        n_slots = cfg.model.G * eng.lib.ref_shards_per_device(eng.h) * cfg.model.S
        slots = eng.slots(n_slots)
        rs = eng.router_state()
        ss = eng.sched_state()
        np.savez_compressed(
            os.path.join(HERE, name + ".npz"),
            config=json.dumps({"kw": kw, "steps": T, "seed": seed}),
            experts=np.array(rec["experts"], dtype=np.int32),
            gates=np.array(rec["gates"]), y=np.array(rec["y"]),
            hits=np.array(rec["hits"]), n_attended=np.array(rec["n_attended"]),
            fetch=np.array(rec["fetch"]), pages=np.array(rec["pages"]),
            ev=np.array([e[:5] + (e[6],) for e in rec["ev"]], dtype=np.int64).reshape(-1, 6),
            ev_score=np.array([e[5] for e in rec["ev"]]), ev_step=np.array(rec["ev_step"]),
            att_te=np.array([(a[0], a[1]) for a in rec["att"]], dtype=np.int64).reshape(-1, 2),
            att_w=np.array([a[2] for a in rec["att"]]), att_step=np.array(rec["att_step"]),
            **{"slot_" + k: v for k, v in slots.items()},
            router_load=rs["load"], router_miss=rs["miss"], router_bias=rs["bias"],
            sched=np.array([ss["theta"], ss["running_hit"], ss["step"]]))
        print(name, "evictions", len(rec["ev"]), "attended", len(rec["att"]))
    # pikv::Rng golden vector (rng.hpp)
    out = np.zeros(64)
    import ctypes
    lib = ref_lib()
    lib.ref_normal_vector.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_double,
                                      ctypes.POINTER(ctypes.c_double)]
    lib.ref_normal_vector(42, 64, 0.5, out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    np.save(os.path.join(HERE, "rng_seed42_n64_scale0.5.npy"), out)


if __name__ == "__main__":
    main()
