// SPDX-License-Identifier: Apache-2.0
// CPU check of the facade's wire writers (pikv::b200::wire) against the golden
// nlohmann lines: stdin = records as written by tests/test_wire.py
//   S device shard token expert age freq
//   E id token expert device <score hex> reason_code
// stdout = one line per record.
#include <cstdlib>
#include <iostream>
#include <sstream>
#include <string>

#include "pikv_b200.hpp"

int main() {
    using namespace pikv::b200;
    std::string line;
    while (std::getline(std::cin, line)) {
        std::istringstream in(line);
        std::string kind;
        in >> kind;
        if (kind == "S") {
            SnapshotRecord r;
            in >> r.device >> r.shard >> r.token_id >> r.expert_id >> r.age >> r.freq;
            std::cout << wire::store_dump_line(r) << "\n";
        } else if (kind == "E") {
            EvictionRecord r;
            std::string hex;
            int reason = 0;
            in >> r.entry_id >> r.token_id >> r.expert_id >> r.device >> hex >> reason;
            r.score = std::strtod(hex.c_str(), nullptr);
            r.reason = static_cast<EvictReason>(reason);
            std::cout << wire::eviction_line(r) << "\n";
        }
    }
    return 0;
}
