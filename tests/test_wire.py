# SPDX-License-Identifier: Apache-2.0
"""Store-dump / eviction-report wire formats on CPU.

Golden fixtures (tests/golden/make_wire_golden.py): records from the
reference's own objects, lines from nlohmann::json as runner.cpp builds them.
* our writer (paper_2508_06526_b200.wire) reproduces every golden line byte
  for byte, except doubles where grisu2 emits a non-shortest digit string:
  those lines must parse to the identical values (bit-identical doubles);
* the oracle's KVStore::snapshot restatement and eviction records equal the
  golden records, and (with /root/reference) live reference runs.
The GPU snapshot is compared with the oracle in test_engine_gpu.py."""
import json
import os
import struct
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))

from cases import engine_config  # noqa: E402
from make_wire_golden import CASES  # noqa: E402
from oracle_bind import OracleEngine, RefEngine, make_stream, ref_lib  # noqa: E402
from paper_2508_06526_b200.wire import (dumps, eviction_line, json_double,  # noqa: E402
                                        store_dump_lines)


def load_case(name):
    z = np.load(os.path.join(HERE, "golden", "wire", "wire_%s.npz" % name))
    with open(os.path.join(HERE, "golden", "wire", "wire_%s.jsonl" % name)) as f:
        lines = f.read().splitlines()
    return z["snapshot"], z["evictions"], int(z["now"]), lines


def bits(x):
    return struct.pack("<d", x)


def same_json(a, b):
    """Equal values, doubles bit for bit."""
    if isinstance(a, float) or isinstance(b, float):
        return isinstance(a, float) and isinstance(b, float) and bits(a) == bits(b)
    if isinstance(a, dict):
        return isinstance(b, dict) and a.keys() == b.keys() and all(same_json(a[k], b[k]) for k in a)
    if isinstance(a, list):
        return isinstance(b, list) and len(a) == len(b) and all(map(same_json, a, b))
    return type(a) is type(b) and a == b


@pytest.mark.parametrize("name", [c[0] for c in CASES])
def test_wire_lines_match_nlohmann(name):
    snap, evs, now, golden = load_case(name)
    ours = store_dump_lines(snap) + [eviction_line(*e) for e in evs]
    assert len(ours) == len(golden)
    non_byte = 0
    for a, b in zip(ours, golden):
        if a == b:
            continue
        non_byte += 1
        assert same_json(json.loads(a), json.loads(b)), (a, b)
        # only the score's digit string may differ (grisu2 non-shortest)
        ja, jb = json.loads(a), json.loads(b)
        assert repr(ja["score"]) != b.split('"score":')[1].split(",")[0], (a, b)
    assert non_byte <= 2, non_byte


def test_json_double_layout():
    """nlohmann's fixed/exponent switch points (dtoa_impl::format_buffer)."""
    assert [json_double(x) for x in (1e15, 1e14, 0.0001, 1e-5, 100.0, -0.0, 2.0 ** 53)] == [
        "1e+15", "100000000000000.0", "0.0001", "1e-05", "100.0", "-0.0", "9.007199254740992e+15"]
    assert json_double(float("nan")) == "null"
    assert dumps({"b": 1, "a": [1.5, 2]}) == '{"a":[1.5,2],"b":1}'


@pytest.mark.parametrize("name", [c[0] for c in CASES])
def test_oracle_snapshot_and_evictions_match_golden(name):
    kw, T, seed = next((c[1], c[2], c[3]) for c in CASES if c[0] == name)
    snap, evs, now, _ = load_case(name)
    cfg = engine_config(**kw)
    eng = OracleEngine(cfg)
    st = make_stream(T, cfg.model.d, seed, cfg.kv_dtype, cfg.n_layers)
    got = []
    for t in range(T):
        r = eng.step(st[0][t], st[1][t], st[2][t], None if cfg.n_layers == 0 else st[3][t])
        got += [(e[1], e[2], e[3], e[4], e[5], e[6]) for e in r["evictions"]]
    real = [tuple(e) for e in evs][:len(got)]
    assert [tuple(map(float, g)) for g in got] == [tuple(map(float, g)) for g in real]
    assert np.array_equal(eng.snapshot(now), snap)


@pytest.mark.skipif(ref_lib() is None, reason="reference objects need /root/reference")
@pytest.mark.parametrize("kw", [dict(router="TopK", sched="LRU", S=10, ps=4, budget=3),
                                dict(router="Hierarchical", unbounded=True, S=64, E=16, k=4,
                                     G=4, n_tok=4, n_exp=8),
                                dict(router="Adaptive", sched="SL", S=8, budget=16)])
def test_oracle_snapshot_matches_reference_live(kw):
    cfg = engine_config(**kw)
    a, b = OracleEngine(cfg), RefEngine(cfg)
    st = make_stream(70, cfg.model.d, 5, cfg.kv_dtype, cfg.n_layers)
    for t in range(70):
        a.step(st[0][t], st[1][t], st[2][t])
        b.step(st[0][t], st[1][t], st[2][t])
        if t % 10 == 9:
            for now in (t + 1, t + 1000, 0):
                assert np.array_equal(a.snapshot(now), b.snapshot(now))


@pytest.fixture(scope="module")
def cpp_writer(tmp_path_factory):
    import shutil
    import subprocess
    if shutil.which("g++") is None:
        pytest.skip("g++ not available")
    exe = str(tmp_path_factory.mktemp("wire") / "test_wire")
    root = os.path.dirname(HERE)
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(root, "include"),
                    os.path.join(HERE, "cpp", "test_wire.cpp"), "-o", exe], check=True)
    return exe


@pytest.mark.parametrize("name", [c[0] for c in CASES])
def test_cpp_facade_wire_lines_match_nlohmann(cpp_writer, name):
    """include/pikv_b200.hpp pikv::b200::wire writers, same bar as above."""
    import subprocess
    snap, evs, now, golden = load_case(name)
    inp = "".join("S %d %d %d %d %d %d\n" % (r["device"], r["shard"], r["token"], r["expert"],
                                              r["age"], r["freq"]) for r in snap)
    inp += "".join("E %d %d %d %d %s %d\n" % (e["id"], e["token"], e["expert"], e["device"],
                                              float(e["score"]).hex(), e["reason"]) for e in evs)
    ours = subprocess.run([cpp_writer], input=inp, capture_output=True, text=True,
                          check=True).stdout.splitlines()
    assert len(ours) == len(golden)
    non_byte = 0
    for a, b in zip(ours, golden):
        if a != b:
            non_byte += 1
            assert same_json(json.loads(a), json.loads(b)), (a, b)
    assert non_byte <= 2, non_byte


def test_json_double_is_nlohmanns_grisu2():
    """json_double == nlohmann::json::dump() for 6000 doubles across the whole
    range (golden strings from tests/golden/make_grisu_golden.py), including
    those where grisu2 is not the shortest representation."""
    import os
    import struct
    from paper_2508_06526_b200.wire import json_double
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "wire",
                        "doubles_nlohmann.txt")
    n = 0
    for line in open(path):
        bits, text = line.split()
        x = struct.unpack("<d", struct.pack("<Q", int(bits, 16)))[0]
        assert json_double(x) == text, (bits, x, text)
        n += 1
    assert n >= 5000


def test_cpp_facade_json_double_is_nlohmanns_grisu2(tmp_path):
    """The C++ facade's wire::json_double against the same nlohmann golden."""
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = str(tmp_path / "test_grisu")
    r = subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(root, "include"),
                        os.path.join(root, "tests", "cpp", "test_grisu.cpp"), "-o", exe],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([exe, os.path.join(root, "tests", "golden", "wire", "doubles_nlohmann.txt")],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stdout
