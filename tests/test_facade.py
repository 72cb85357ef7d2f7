# SPDX-License-Identifier: Apache-2.0
"""The C++ facade (include/pikv_b200.hpp): compiles here against the C-ABI
library; on a GPU the reference's known-answer tests run through it."""
import os
import subprocess

import pytest

from paper_2508_06526_b200.build import LIB, build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_facade.cpp")
EXE = os.path.join(ROOT, "tests", "cpp", "test_facade")


def compile_facade_test():
    build()
    libdir = os.path.dirname(LIB)
    cmd = ["g++", "-std=c++20", "-O1", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"),
           SRC, "-L", libdir, "-lpikv_b200", "-Wl,-rpath," + libdir, "-o", EXE]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return EXE


def test_facade_compiles():
    assert os.path.exists(compile_facade_test())


@pytest.mark.gpu
def test_facade_reference_kats_on_gpu():
    exe = compile_facade_test()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ok: 0 failure(s)" in r.stdout
