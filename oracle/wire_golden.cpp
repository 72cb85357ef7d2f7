// SPDX-License-Identifier: Apache-2.0
// TEST INFRASTRUCTURE: golden JSON lines for the store-dump and eviction-report
// wire formats, produced by nlohmann::json (the library the reference's runner
// uses, runner.cpp:7) with the objects built exactly as runner.cpp builds them:
//   eviction_json      runner.cpp:58-65   {id, token, expert, device, score, reason}
//   store dump line    runner.cpp:215-222 {device, shard, token, expert, age, freq}
// Input (stdin), one record per line:
//   S <device> <shard> <token> <expert> <age> <freq>
//   E <id> <token> <expert> <device> <score as C99 hex float> <reason string>
// Output (stdout): json::dump() of each record, one per line.
// Built by tests/golden/make_wire_golden.py with -I <dir holding nlohmann/json.hpp>.
#include <cstdint>
#include <cstdlib>
#include <iostream>
#include <nlohmann/json.hpp>
#include <sstream>
#include <string>

using nlohmann::json;

int main() {
    std::string line;
    while (std::getline(std::cin, line)) {
        std::istringstream in(line);
        std::string kind;
        in >> kind;
        if (kind == "S") {
            int device, shard, expert;
            std::int64_t token;
            std::uint64_t age, freq;
            in >> device >> shard >> token >> expert >> age >> freq;
            json r{{"device", device}, {"shard", shard}, {"token", token},
                   {"expert", expert}, {"age", age},     {"freq", freq}};
            std::cout << r.dump() << "\n";
        } else if (kind == "E") {
            std::uint64_t id;
            std::int64_t token;
            int expert, device;
            std::string score_hex, reason;
            in >> id >> token >> expert >> device >> score_hex >> reason;
            const double score = std::strtod(score_hex.c_str(), nullptr);
            json r{{"id", id},         {"token", token}, {"expert", expert},
                   {"device", device}, {"score", score}, {"reason", reason}};
            std::cout << r.dump() << "\n";
        }
    }
    return 0;
}
