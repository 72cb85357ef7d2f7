# SPDX-License-Identifier: Apache-2.0
"""CPU checks of the product boundary: the C-ABI library loads and exports
every symbol include/pikv_b200.h declares, and the Python mirror agrees with
the C layouts.  No compute calls (no GPU here)."""
import ctypes
import os
import re

from paper_2508_06526_b200 import _capi
from paper_2508_06526_b200.build import build
from paper_2508_06526_b200.config import EngineConfig, PikvConfigC

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pikv_b200.h")


def header_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\*\s]+?\b(pikv_\w+)\s*\(", text, re.M)))


def test_library_builds_and_loads():
    path = build()
    assert os.path.exists(path)
    L = _capi.lib()
    assert L.pikv_version().decode().startswith("pikv-b200")


def test_every_header_symbol_is_exported():
    L = _capi.lib()
    syms = header_symbols()
    assert len(syms) >= 38
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_capi.SIGNATURES), set(syms) ^ set(_capi.SIGNATURES)


def test_config_layout_matches():
    assert _capi.lib().pikv_config_size() == ctypes.sizeof(PikvConfigC)
    assert ctypes.sizeof(_capi.PikvEvictRecord) == 48
    c = PikvConfigC()
    _capi.lib().pikv_config_default(ctypes.byref(c))
    # reference defaults (config.hpp, router.hpp:24-37, scheduler.hpp:30-47)
    assert (c.d, c.E, c.k, c.S, c.G) == (64, 8, 2, 16, 2)
    assert c.page_size == 16 and c.budget_pages == 4 and c.theta0 == -1e18
    assert c.load_decay == 0.99 and c.hit_decay == 0.9
    d = EngineConfig().to_c()
    for f, _ in PikvConfigC._fields_:
        if f in ("n_heads", "kv_dtype", "seed", "batch", "world_size", "rank_id",
                 "pool_entries", "n_layers", "flex_plan", "adakv_weights", "k", "rank",
                 "unbounded_budget"):
            continue
        assert getattr(c, f) == getattr(d, f), f


def test_no_gpu_path_fails_loudly_without_library(tmp_path, monkeypatch):
    monkeypatch.setattr(_capi, "LIB_PATH", str(tmp_path / "missing.so"))
    monkeypatch.setattr(_capi, "_LIB", None)
    try:
        _capi.lib()
        raise AssertionError("expected ImportError")
    except ImportError as e:
        assert "no CPU fallback" in str(e)
