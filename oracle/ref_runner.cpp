// SPDX-License-Identifier: Apache-2.0
//
// TEST INFRASTRUCTURE -- drives the reference's own run_experiment
// (/root/reference/proj/src/runner.cpp:69-261, compiled unchanged together
// with pipeline.cpp, runconfig.cpp, costmodel.cpp, trace.cpp, kvstore.cpp,
// router.cpp, mathops.cpp and the Eigen-free scheduler.cpp extracts) to
// produce golden MetricsReport / event-log / store-dump lines for the trace
// replay.  Built by oracle/build.py into oracle/_ref/ (never
// shipped, never on the product path).
//
// compressor.cpp needs Eigen (absent here), so the Identity codec the
// golden runs use is supplied below: Codec::fit / encode / decode for
// Scheme::Identity only (compressor.cpp:186-230, 364-371, 413-419: the
// identity scheme copies the vectors; every other scheme throws).  The
// utility tracker's bookkeeping (scheduler.cpp:352-359, whose lookup at
// :363-375 does not compile) is a no-op: run_experiment never reads it.
#include <cstring>
#include <string>
#include <vector>

#include "pikv/compressor.hpp"
#include "pikv/errors.hpp"
#include "pikv/runconfig.hpp"
#include "pikv/runner.hpp"
#include "pikv/scheduler.hpp"

namespace pikv {

Codec Codec::fit(Scheme scheme, const std::vector<std::vector<double>>& calibration,
                 const CompressorConfig& cfg) {
    if (scheme != Scheme::Identity) throw NotFitted("oracle runner: Identity codec only");
    if (calibration.empty()) throw InsufficientCalibration("oracle runner: no calibration rows");
    Codec c;
    c.scheme_ = scheme;
    c.d_ = static_cast<int>(calibration[0].size());
    c.stored_width_ = c.d_;
    c.cfg_ = cfg;
    return c;
}

std::vector<double> Codec::encode_vector(std::span<const double> x) const {
    if (static_cast<int>(x.size()) != d_) throw InvalidEntry("encode: width mismatch");
    return {x.begin(), x.end()};
}

std::vector<double> Codec::decode_vector(std::span<const double> payload, int) const {
    if (static_cast<int>(payload.size()) != stored_width_) throw CodecMismatch("decode: payload width mismatch");
    return {payload.begin(), payload.end()};
}

CompressedKV Codec::encode(std::span<const double> key, std::span<const double> value) const {
    CompressedKV c;
    c.scheme = scheme_;
    c.original_width = d_;
    c.stored_width = stored_width_;
    c.key = encode_vector(key);
    c.value = encode_vector(value);
    return c;
}

std::vector<CompressedKV> Codec::encode_chunk(
    const std::vector<std::pair<std::vector<double>, std::vector<double>>>& entries) const {
    std::vector<CompressedKV> out;
    for (const auto& [k, v] : entries) out.push_back(encode(k, v));
    return out;
}

// Composition and QUEST are outside the golden runs (Identity codec, Table
// schedulers): refuse loudly if a config asks for them.
CompositeCodec CompositeCodec::fit(const std::vector<Scheme>&, const std::vector<std::vector<double>>&,
                                   const CompressorConfig&) {
    throw NotFitted("oracle runner: codec composition needs compressor.cpp (Eigen)");
}
CompressedKV CompositeCodec::encode(std::span<const double>, std::span<const double>) const {
    throw NotFitted("oracle runner: no composition");
}
std::pair<std::vector<double>, std::vector<double>> CompositeCodec::decode(const CompressedKV&) const {
    throw NotFitted("oracle runner: no composition");
}
std::vector<double> CompositeCodec::encode_vector(std::span<const double>) const {
    throw NotFitted("oracle runner: no composition");
}
int CompositeCodec::stored_width() const { throw NotFitted("oracle runner: no composition"); }
void QuestScorer::fit(const std::vector<std::vector<double>>&, const std::vector<double>&, int, double,
                      std::uint64_t) {
    throw NotFitted("oracle runner: QUEST needs scheduler.cpp's fit (Eigen)");
}

void ExpertUtilityTracker::note_query(int) {}
void ExpertUtilityTracker::note_attention(int, std::int64_t, double) {}

}  // namespace pikv

extern "C" {

// run_experiment(parse_config_text(text)): report line, then the event
// lines, then the store dump lines ("run.dump_store" set), '\n'-separated,
// into a malloc'ed string.  0 ok, 1 on an exception (message in *out).
int ref_run_experiment(const char* config_text, char** out) {
    std::string s;
    int rc = 0;
    try {
        const pikv::RunConfig cfg = pikv::parse_config_text(config_text);
        const pikv::RunOutput r = pikv::run_experiment(cfg);
        s = r.report_line + "\n";
        for (const auto& l : r.event_log) s += l + "\n";
        for (const auto& l : r.store_dump) s += l + "\n";
    } catch (const std::exception& e) {
        s = e.what();
        rc = 1;
    }
    *out = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(*out, s.c_str(), s.size() + 1);
    return rc;
}

void ref_free(char* p) { std::free(p); }

}  // extern "C"
