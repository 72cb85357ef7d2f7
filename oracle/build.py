# SPDX-License-Identifier: Apache-2.0
"""TEST INFRASTRUCTURE — build recipe for the CPU checkers.

* ``build_oracle()`` compiles the C restatement ``oracle/pikv_oracle.c`` into
  ``oracle/libpikv_oracle.so`` (gcc; travels to the GPU box with the repo).
* ``build_ref()`` compiles the REFERENCE's own code from /root/reference
  (present only in the build container) into ``oracle/_ref/libpikv_ref.so``:
    - mathops.cpp, kvstore.cpp, router.cpp: compiled unchanged, in place;
    - scheduler.cpp lines 49-80 and 162-350 and pipeline.cpp lines 29-57
      (QueryEncoder) and 59-85 (attention):
      line-extracted (sha256-verified) into oracle/_ref/ because the rest of
      those files needs Eigen (absent) and scheduler.cpp:352-377 does not
      compile.  The extracted lines are byte-identical;
    - oracle/ref_driver.cpp: our step driver over those objects.
  Nothing from /root/reference is written into the tracked tree; oracle/_ref/
  is git-ignored.
"""
from __future__ import annotations

import hashlib
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.environ.get("PIKV_REFERENCE", "/root/reference/proj")
REF_OUT = os.path.join(HERE, "_ref")

EXTRACTS = [
    # (source, first line, last line, sha256 of those lines)
    ("src/scheduler.cpp", 49, 80,
     "ffe9e3842f8af007dec2f1e5e0af5ead963d84c537284e88fda66b405db2030e"),
    ("src/scheduler.cpp", 162, 350,
     "30cdc95c732fad259c0eb492ffc0422286c3f75f7833e1c7581609580d9900f7"),
    ("src/pipeline.cpp", 59, 85,
     "0b7a58bb7cf2a88e9dc9a5104abcacda680d760ba71f6d5b5c4e2ddb930bc5f2"),
    ("src/pipeline.cpp", 29, 57,  # QueryEncoder (the step's encode, pipeline.cpp:222)
     "94bea718658aadb9356db62905d46ab4460b919e090f97e3d4d0d2f1a581388a"),
    # runner build only: strategy / scheme names (the parts of those files
    # before their Eigen code)
    ("src/scheduler.cpp", 14, 48,
     "2d6cf5cf8afb020c51acd9485f85b5839f9669a547525bb53cae1c95c08640de"),
    ("src/compressor.cpp", 117, 163,
     "13f37d069754dcbe1e2a4f94c8d908497ef58acfe59848d75f962dcdca0b309d"),
]


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("command failed: %s\n%s%s" % (" ".join(cmd), r.stdout, r.stderr))


def oracle_lib_path() -> str:
    return os.path.join(HERE, "libpikv_oracle.so")


def ref_lib_path() -> str:
    return os.path.join(REF_OUT, "libpikv_ref.so")


def build_oracle(force: bool = False) -> str:
    out = oracle_lib_path()
    src = os.path.join(HERE, "pikv_oracle.c")
    hdr = os.path.join(HERE, "pikv_oracle.h")
    if (not force and os.path.exists(out)
            and os.path.getmtime(out) >= max(os.path.getmtime(src), os.path.getmtime(hdr))):
        return out
    _run(["gcc", "-O2", "-std=gnu11", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
          "-shared", "-Wall", "-o", out, src, "-lm"])
    return out


def _extract(rel, a, b, digest):
    with open(os.path.join(REF, rel), "rb") as f:
        lines = f.read().split(b"\n")
    chunk = b"\n".join(lines[a - 1:b]) + b"\n"
    got = hashlib.sha256(chunk).hexdigest()
    if got != digest:
        raise RuntimeError("reference %s:%d-%d changed (sha256 %s)" % (rel, a, b, got))
    return chunk.decode()


def build_ref(force: bool = False) -> str | None:
    """Build oracle/_ref/libpikv_ref.so from /root/reference; None if absent."""
    out = ref_lib_path()
    if not os.path.isdir(REF):
        return out if os.path.exists(out) else None
    drv = os.path.join(HERE, "ref_driver.cpp")
    if not force and os.path.exists(out) and os.path.getmtime(out) >= os.path.getmtime(drv):
        return out
    os.makedirs(REF_OUT, exist_ok=True)
    inc = os.path.join(REF, "include")
    sched = ('#include "pikv/scheduler.hpp"\n#include <algorithm>\n#include <cmath>\n'
             '#include "pikv/errors.hpp"\n#include "pikv/mathops.hpp"\n#include "pikv/rng.hpp"\n'
             "namespace pikv {\n"
             + _extract(*EXTRACTS[0]) + _extract(*EXTRACTS[1]) + "}  // namespace pikv\n")
    pipe = ('#include "pikv/pipeline.hpp"\n#include <cmath>\n#include "pikv/errors.hpp"\n'
            '#include "pikv/mathops.hpp"\n#include "pikv/rng.hpp"\nnamespace pikv {\n'
            + _extract(*EXTRACTS[3]) + _extract(*EXTRACTS[2]) + "}  // namespace pikv\n")
    gen = {"scheduler_extract.cpp": sched, "pipeline_extract.cpp": pipe}
    for name, text in gen.items():
        with open(os.path.join(REF_OUT, name), "w") as f:
            f.write(text)
    srcs = [os.path.join(REF, "src", s)
            for s in ("mathops.cpp", "kvstore.cpp", "router.cpp", "costmodel.cpp", "trace.cpp")]
    srcs += [os.path.join(REF_OUT, n) for n in gen] + [drv]
    flags = ["g++", "-std=c++20", "-O2", "-fPIC", "-include", "unordered_map", "-I", inc,
             "-I", HERE, "-I", os.path.join(HERE, "..", "include")]
    objs = []
    for s in srcs:
        o = os.path.join(REF_OUT, os.path.basename(s) + ".o")
        _run(flags + ["-c", s, "-o", o])
        objs.append(o)
    _run(["g++", "-shared", "-o", out] + objs + ["-lpthread"])
    return out


def runner_lib_path() -> str:
    return os.path.join(REF_OUT, "libpikv_runner.so")


def build_runner(force: bool = False) -> str | None:
    """oracle/_ref/libpikv_runner.so: the reference's run_experiment
    (runner.cpp) with pipeline.cpp, runconfig.cpp, costmodel.cpp, trace.cpp,
    kvstore.cpp, router.cpp, mathops.cpp compiled unchanged, the Eigen-free
    scheduler.cpp / compressor.cpp extracts, nlohmann json.hpp from the
    image's cudnn_frontend wheel, and oracle/ref_runner.cpp (Identity codec
    + driver).  None when /root/reference or json.hpp is absent."""
    out = runner_lib_path()
    drv = os.path.join(HERE, "ref_runner.cpp")
    if not os.path.isdir(REF):
        return out if os.path.exists(out) else None
    if not force and os.path.exists(out) and os.path.getmtime(out) >= os.path.getmtime(drv):
        return out
    import glob
    js = glob.glob(os.path.join(sys.prefix, "lib", "python3*", "site-packages", "include",
                                "cudnn_frontend", "thirdparty", "nlohmann", "json.hpp"))
    if not js:
        return None
    os.makedirs(REF_OUT, exist_ok=True)
    inc = os.path.join(REF, "include")
    hdr = ('#include "pikv/scheduler.hpp"\n#include <algorithm>\n#include <cmath>\n'
           '#include "pikv/errors.hpp"\n#include "pikv/mathops.hpp"\n#include "pikv/rng.hpp"\n')
    sched = (hdr + "namespace pikv {\n" + _extract(*EXTRACTS[4]) + _extract(*EXTRACTS[0]) +
             _extract(*EXTRACTS[1]) + "}  // namespace pikv\n")
    comp = ('#include "pikv/compressor.hpp"\n#include "pikv/errors.hpp"\nnamespace pikv {\n' +
            _extract(*EXTRACTS[5]) + "}  // namespace pikv\n")
    gen = {"runner_sched_extract.cpp": sched, "runner_comp_extract.cpp": comp}
    for name, text in gen.items():
        with open(os.path.join(REF_OUT, name), "w") as f:
            f.write(text)
    srcs = [os.path.join(REF, "src", s) for s in
            ("mathops.cpp", "kvstore.cpp", "router.cpp", "costmodel.cpp", "trace.cpp",
             "pipeline.cpp", "runconfig.cpp", "runner.cpp")]
    srcs += [os.path.join(REF_OUT, n) for n in gen] + [drv]
    flags = ["g++", "-std=c++20", "-O2", "-fPIC", "-include", "unordered_map", "-I", inc,
             "-I", os.path.dirname(js[0])]
    objs = []
    for s in srcs:
        o = os.path.join(REF_OUT, "runner_" + os.path.basename(s) + ".o")
        _run(flags + ["-c", s, "-o", o])
        objs.append(o)
    _run(["g++", "-shared", "-o", out] + objs + ["-lpthread"])
    return out


if __name__ == "__main__":
    print(build_oracle(force="-f" in sys.argv))
    print(build_ref(force="-f" in sys.argv))
