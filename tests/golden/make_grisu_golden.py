# SPDX-License-Identifier: Apache-2.0
"""Regenerate tests/golden/wire/doubles_nlohmann.txt: 6000 doubles (random
bit patterns over the whole exponent range plus decimal-looking values) and
the strings nlohmann::json::dump() writes for them -- the JSON library of the
reference's runner (runner.cpp:7) -- compiled from the json.hpp the image
carries (cudnn_frontend's vendored copy).  Lines: <hex bits> <dump text>."""
import glob
import os
import struct
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = r'''
#include <cstdio>
#include <cstring>
#include <cstdint>
#include <json.hpp>
int main() {
    unsigned long long b;
    while (std::scanf("%llx", &b) == 1) {
        double x;
        std::memcpy(&x, &b, 8);
        std::printf("%016llx %s\n", b, nlohmann::json(x).dump().c_str());
    }
}
'''


def main():
    js = glob.glob(os.path.join(sys.prefix, "lib", "python3*", "site-packages", "include",
                                "cudnn_frontend", "thirdparty", "nlohmann", "json.hpp"))
    rng = np.random.default_rng(2025)
    vals = list(rng.integers(0, 1 << 63, 3000, dtype=np.uint64))             # any positive double
    vals += [struct.unpack("<Q", struct.pack("<d", float(x)))[0]
             for x in np.round(rng.random(2000) * 10.0 ** rng.integers(-8, 9, 2000), 12)]
    vals += [struct.unpack("<Q", struct.pack("<d", float(x)))[0]
             for x in rng.standard_normal(1000) * 1e-5]
    vals = [v for v in vals if (int(v) >> 52) & 0x7FF != 0x7FF]               # finite only
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "dump")
        with open(exe + ".cpp", "w") as f:
            f.write(SRC)
        subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.dirname(js[0]), exe + ".cpp", "-o", exe],
                       check=True)
        out = subprocess.run([exe], input="\n".join("%x" % int(v) for v in vals), capture_output=True,
                             text=True, check=True).stdout
    with open(os.path.join(HERE, "wire", "doubles_nlohmann.txt"), "w") as f:
        f.write(out)
    print(len(out.splitlines()), "doubles")


if __name__ == "__main__":
    main()
