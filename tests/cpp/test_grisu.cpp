// SPDX-License-Identifier: Apache-2.0
// pikv::b200::wire::json_double (include/pikv_b200.hpp) against the strings
// nlohmann::json::dump() wrote for the same doubles (the reference runner's
// JSON library, runner.cpp:7; golden: tests/golden/make_grisu_golden.py).
// Host-only: no GPU.  Exit code = number of mismatches.
#include <cstdio>
#include <cstring>
#include <fstream>
#include <string>

#include "pikv_b200.hpp"

int main(int argc, char** argv) {
    if (argc < 2) return 1;
    std::ifstream f(argv[1]);
    std::string hex, txt;
    int bad = 0, n = 0;
    while (f >> hex >> txt) {
        const unsigned long long b = std::stoull(hex, nullptr, 16);
        double x;
        std::memcpy(&x, &b, 8);
        const std::string got = pikv::b200::wire::json_double(x);
        if (got != txt) {
            if (bad < 5) std::printf("FAIL %s: want %s got %s\n", hex.c_str(), txt.c_str(), got.c_str());
            ++bad;
        }
        ++n;
    }
    std::printf("%d doubles, %d mismatch(es)\n", n, bad);
    return n < 5000 ? 1 : bad;
}
