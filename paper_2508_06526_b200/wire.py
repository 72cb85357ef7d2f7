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
runs the same Grisu2 digit generation (Loitsch 2010 with the 64-bit cached
powers of ten; nlohmann's dtoa_impl), so even the doubles where grisu2 is not
shortest (1e23 -> 9.999999999999999e+22, 2.9849183999999998e-05) print
byte-identically (tests/test_wire.py, tests/test_replay.py against lines the
reference's nlohmann produced).
"""
from __future__ import annotations

import json
import math
import struct

import numpy as np

# pikv_snapshot_record (include/pikv_b200.h)
SNAPSHOT_DTYPE = np.dtype([("device", "<i4"), ("shard", "<i4"), ("token", "<i8"),
                           ("expert", "<i4"), ("reserved", "<i4"), ("age", "<u8"),
                           ("freq", "<u8")])

REASONS = {0: "budget", 1: "threshold", 2: "overwrite"}  # scheduler.cpp:40-46


# ---- Grisu2 (nlohmann dtoa_impl): digits d1..dk and exponent with value =
# d1..dk * 10^exp -------------------------------------------------------------
_M64 = (1 << 64) - 1


def _cached_powers():
    """(f, e, k): 10^k ~= f 2^e, 2^63 <= f < 2^64 rounded to nearest, for
    k = -300, -292, ..., 332 (kCachedPowers)."""
    out = []
    for i in range(79):
        k = -300 + 8 * i
        num, den = (10 ** k, 1) if k >= 0 else (1, 10 ** (-k))
        e = (num.bit_length() - den.bit_length()) - 64
        while True:
            q, r = divmod(num, den << e) if e >= 0 else divmod(num << -e, den)
            d = (den << e) if e >= 0 else den
            if q >= 1 << 64:
                e += 1
            elif q < 1 << 63:
                e -= 1
            else:
                break
        if 2 * r >= d:
            q += 1
        out.append((q, e, k))
    return out


_POW = _cached_powers()


def _normalize(f, e):
    s = 64 - f.bit_length()
    return (f << s) & _M64, e - s


def _mul(a, b):  # diyfp::mul: the high 64 bits of the product, rounded half up
    return ((a[0] * b[0] + (1 << 63)) >> 64) & _M64, a[1] + b[1] + 64


def _grisu2(v: float):
    bits = struct.unpack("<Q", struct.pack("<d", v))[0]
    E, F = bits >> 52, bits & ((1 << 52) - 1)
    f, e = (F, 1 - 1075) if E == 0 else (F + (1 << 52), E - 1075)
    closer = F == 0 and E > 1
    mp = _normalize(2 * f + 1, e - 1)
    mm_f, mm_e = (4 * f - 1, e - 2) if closer else (2 * f - 1, e - 1)
    mm = ((mm_f << (mm_e - mp[1])) & _M64, mp[1])
    w = _normalize(f, e)
    # cached power with alpha <= e_c + e + 64 <= gamma (alpha -60, gamma -32)
    fx = -60 - mp[1] - 1
    k = int(fx * 78913 / (1 << 18)) + (fx > 0)
    c = _POW[(300 + k + 7) // 8]
    cw, cmm, cmp = _mul(w, c[:2]), _mul(mm, c[:2]), _mul(mp, c[:2])
    Mm, Mp = (cmm[0] + 1, cmm[1]), (cmp[0] - 1, cmp[1])
    dec = -c[2]
    # digit generation (grisu2_digit_gen)
    delta, dist = Mp[0] - Mm[0], Mp[0] - cw[0]
    shift = -Mp[1]
    one = 1 << shift
    p1, p2 = Mp[0] >> shift, Mp[0] & (one - 1)
    digits = []
    n = len(str(p1))
    pow10 = 10 ** (n - 1)

    def rnd(rest, ten_k):  # grisu2_round
        nonlocal delta, dist
        while (rest < dist and delta - rest >= ten_k
               and (rest + ten_k < dist or dist - rest > rest + ten_k - dist)):
            digits[-1] -= 1
            rest += ten_k

    while n > 0:
        d, p1 = divmod(p1, pow10)
        digits.append(d)
        n -= 1
        rest = (p1 << shift) + p2
        if rest <= delta:
            rnd(rest, pow10 << shift)
            return "".join(map(str, digits)), dec + n
        pow10 //= 10
    m = 0
    while True:
        p2 *= 10
        delta *= 10
        dist *= 10
        digits.append(p2 >> shift)
        p2 &= one - 1
        m += 1
        if p2 <= delta:
            break
    rnd(p2, one)
    return "".join(map(str, digits)), dec - m


def json_double(x: float) -> str:
    """A double as nlohmann::json dump() writes it: grisu2 digits in
    dtoa_impl::format_buffer's layout (min_exp = -4, max_exp = 15)."""
    x = float(x)
    if math.isnan(x) or math.isinf(x):
        return "null"
    if x == 0.0:
        return "-0.0" if math.copysign(1.0, x) < 0 else "0.0"
    sign = "-" if x < 0 else ""
    ds, ex = _grisu2(abs(x))
    k = len(ds)
    n = k + ex  # value = 0.d1..dk * 10^n
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
