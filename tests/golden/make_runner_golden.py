# SPDX-License-Identifier: Apache-2.0
"""Regenerate tests/golden/runner/*.json: the reference's own run_experiment
(runner.cpp:69-261, compiled from /root/reference by oracle/build.py's
build_runner) on the cases of runner_cases.py.  Each file holds the config
text, the report line, the event lines and the store dump lines exactly as
the reference printed them.  Needs /root/reference (build container only)."""
import ctypes
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, HERE)

from oracle import build  # noqa: E402
from runner_cases import CASES, config_text  # noqa: E402


def main():
    lib = ctypes.CDLL(build.build_runner())
    lib.ref_run_experiment.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]
    lib.ref_free.argtypes = [ctypes.c_void_p]
    os.makedirs(os.path.join(HERE, "runner"), exist_ok=True)
    for name, c in CASES.items():
        text = config_text(c)
        out = ctypes.c_void_p()
        rc = lib.ref_run_experiment(text.encode(), ctypes.byref(out))
        s = ctypes.string_at(out).decode()
        lib.ref_free(out)
        if rc:
            raise RuntimeError("%s: %s" % (name, s))
        lines = s.rstrip("\n").split("\n")
        T = c["T"]
        doc = {"case": name, "config": text, "report": lines[0], "events": lines[1:1 + T],
               "store": lines[1 + T:]}
        with open(os.path.join(HERE, "runner", name + ".json"), "w") as f:
            json.dump(doc, f, indent=0)
        print(name, len(doc["events"]), "events,", len(doc["store"]), "store lines")


if __name__ == "__main__":
    main()
