# SPDX-License-Identifier: Apache-2.0
"""Wire formats of the reference's run output.

* store dump: one JSON object per live entry, runner.cpp:215-222, from
  KVStore::snapshot (kvstore.cpp:206-221) -> ``Engine.snapshot()``;
* eviction report: runner.cpp:58-65 (``eviction_json``), one object per
  EvictionRecord (scheduler.hpp:90-98);
* step event line: runner.cpp:183-196.

The reference serialises with nlohmann::json ``dump()``: object keys in
sorted order (std::map), no spaces, integers as integers, doubles as the
grisu2 digit string with nlohmann's layout rules (fixed notation for decimal
exponents -4 < n <= 15, else d.ddde+XX), NaN/inf as null.  ``json_double``
reproduces the layout rules on Python's shortest round-trip digits; grisu2
emits a longer digit string for a small fraction of doubles (e.g. 1e23 ->
9.999999999999999e+22), which parses to the identical double
(tests/test_wire.py checks both against golden lines nlohmann produced).
"""
from __future__ import annotations

import json
import math
from decimal import Decimal

import numpy as np

# pikv_snapshot_record (include/pikv_b200.h)
SNAPSHOT_DTYPE = np.dtype([("device", "<i4"), ("shard", "<i4"), ("token", "<i8"),
                           ("expert", "<i4"), ("reserved", "<i4"), ("age", "<u8"),
                           ("freq", "<u8")])

REASONS = {0: "budget", 1: "threshold", 2: "overwrite"}  # scheduler.cpp:40-46


def json_double(x: float) -> str:
    """A double as nlohmann::json dump() writes it (dtoa_impl::format_buffer
    layout with min_exp = -4, max_exp = 15)."""
    x = float(x)
    if math.isnan(x) or math.isinf(x):
        return "null"
    if x == 0.0:
        return "-0.0" if math.copysign(1.0, x) < 0 else "0.0"
    sign = "-" if x < 0 else ""
    t = Decimal(repr(abs(x))).normalize().as_tuple()
    ds = "".join(str(c) for c in t.digits)
    k = len(ds)
    n = k + t.exponent  # value = 0.d1..dk * 10^n
    if k <= n <= 15:
        return sign + ds + "0" * (n - k) + ".0"
    if 0 < n <= 15:
        return sign + ds[:n] + "." + ds[n:]
    if -4 < n <= 0:
        return sign + "0." + "0" * (-n) + ds
    e = n - 1
    es = ("+" if e >= 0 else "-") + "%02d" % abs(e)
    return sign + ds[0] + ("." + ds[1:] if k > 1 else "") + "e" + es


def _value(v) -> str:
    if isinstance(v, (bool, np.bool_)):
        return "true" if v else "false"
    if isinstance(v, (int, np.integer)):
        return str(int(v))
    if isinstance(v, (float, np.floating)):
        return json_double(v)
    if isinstance(v, str):
        return json.dumps(v)
    if isinstance(v, dict):
        return dumps(v)
    if isinstance(v, (list, tuple, np.ndarray)):
        return "[" + ",".join(_value(x) for x in v) + "]"
    raise TypeError("unsupported JSON value %r" % (v,))


def dumps(obj: dict) -> str:
    """nlohmann::json(obj).dump(): sorted keys, compact."""
    return "{" + ",".join(json.dumps(k) + ":" + _value(obj[k]) for k in sorted(obj)) + "}"


def store_dump_lines(records) -> list[str]:
    """runner.cpp:215-222 for snapshot records (SNAPSHOT_DTYPE array)."""
    return [dumps({"device": int(r["device"]), "shard": int(r["shard"]), "token": int(r["token"]),
                   "expert": int(r["expert"]), "age": int(r["age"]), "freq": int(r["freq"])})
            for r in records]


def eviction_line(entry_id, token, expert, device, score, reason) -> str:
    """runner.cpp:58-65 (eviction_json)."""
    if not isinstance(reason, str):
        reason = REASONS[int(reason)]
    return dumps({"id": int(entry_id), "token": int(token), "expert": int(expert),
                  "device": int(device), "score": float(score), "reason": reason})


def step_event_line(t, experts, gates, inserts, fetch_bytes, hits, lookups, latency_s,
                    fidelity, evictions) -> str:
    """runner.cpp:183-196: one line of the event log; ``evictions`` holds
    eviction_line() objects' fields as dicts or (id, token, expert, device,
    score, reason) tuples."""
    evs = []
    for ev in evictions:
        if not isinstance(ev, dict):
            ev = dict(zip(("id", "token", "expert", "device", "score", "reason"), ev))
        reason = ev["reason"] if isinstance(ev["reason"], str) else REASONS[int(ev["reason"])]
        evs.append({"id": int(ev["id"]), "token": int(ev["token"]), "expert": int(ev["expert"]),
                    "device": int(ev["device"]), "score": float(ev["score"]), "reason": reason})
    return dumps({"t": int(t), "experts": [int(e) for e in experts],
                  "gates": [float(g) for g in gates], "inserts": int(inserts),
                  "fetch_bytes": int(fetch_bytes), "hits": int(hits), "lookups": int(lookups),
                  "latency_s": float(latency_s), "fidelity": float(fidelity), "evictions": evs})
