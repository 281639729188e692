// Host-only check of the streaming driver's chunk planner (csrc/stream_plan.hpp) against the
// one-shot scheduler (host_circuit.cpp schedule_windows, itself checked against the reference's
// schedule.hpp in tests/test_host.py): for generated and hand-made circuits and random chunk
// splits, the non-empty buckets in key order are the schedule's windows, gate for gate, and the
// reference's scheduling errors are raised by both. Prints "ok <cases>" or the first mismatch.
#include <cstdio>
#include <random>
#include <string>

#include "stream_plan.hpp"

using namespace qsr;

static std::string plan_error(const Circuit &c, std::mt19937_64 &rng, std::vector<std::vector<uint64_t>> *out) {
    const uint64_t G = c.gates.size();
    BucketDir buckets(2 * G + 4);
    auto fresh = [](std::vector<uint64_t> &b) { b.reserve(16); };
    ChunkPlanner<decltype(fresh)> planner(c.num_qubits, buckets, fresh);
    try {
        for (uint64_t i0 = 0; i0 < G;) {
            const uint64_t i1 = std::min<uint64_t>(G, i0 + 1 + rng() % 97);
            planner.plan(c.gates.data(), i0, i1);
            i0 = i1;
        }
    } catch (const Error &e) {
        return e.what();
    }
    for (uint64_t key = 0; key <= planner.max_key() + 1; ++key) {
        std::vector<uint64_t> *b = buckets.find(key);
        if (b && !b->empty()) out->push_back(*b);
    }
    return "";
}

int main() {
    std::mt19937_64 rng(7);
    int cases = 0;
    for (int t = 0; t < 400; ++t) {
        Circuit c;
        if (t % 4 == 3) { // hand-made: single-qubit runs, chained measurements, idle wires
            c.num_qubits = 2 + uint32_t(rng() % 9);
            const int len = int(rng() % 60);
            for (int i = 0; i < len; ++i) {
                const uint8_t kind = uint8_t(rng() % 12);
                const uint32_t q0 = uint32_t(rng() % c.num_qubits);
                uint32_t q1 = uint32_t(rng() % c.num_qubits);
                if (kind >= QSR_CX && kind <= QSR_ISWAP && q1 == q0) q1 = (q0 + 1) % c.num_qubits;
                c.gates.push_back({kind, q0, kind >= QSR_CX && kind <= QSR_ISWAP ? q1 : 0});
            }
        } else {
            c = generate_random(1 + uint32_t(rng() % 300), 1 + uint32_t(rng() % 40), rng(),
                                (t % 4) == 0 ? 0.0 : (t % 4) == 1 ? 0.3 : 1.0);
        }
        std::vector<std::vector<uint64_t>> got;
        const std::string perr = plan_error(c, rng, &got);
        std::string serr;
        Schedule s;
        try {
            c.check_valid();
            s = schedule_windows(c, QSR_SINGLE_SHOT);
            // A measurement chained behind another on its wire lands in the same window: the
            // streaming planner rejects it while planning (measure_window would, measure.hpp:394).
            std::vector<uint32_t> stamp;
            for (uint64_t w = 0; w < s.num_windows(); ++w)
                validate_window(c.num_qubits, s.gates.data() + s.offsets[w], s.offsets[w + 1] - s.offsets[w],
                                s.is_meas[w] != 0, stamp, uint32_t(w + 1));
        } catch (const Error &e) {
            serr = e.what();
        }
        if (perr.empty() != serr.empty()) {
            std::printf("case %d: planner error '%s' vs scheduler error '%s'\n", t, perr.c_str(), serr.c_str());
            return 1;
        }
        ++cases;
        if (!perr.empty()) continue;
        if (got.size() != s.num_windows()) {
            std::printf("case %d: %zu buckets vs %llu windows\n", t, got.size(), (unsigned long long)s.num_windows());
            return 1;
        }
        for (uint64_t w = 0; w < s.num_windows(); ++w) {
            const uint64_t b = s.offsets[w], e = s.offsets[w + 1];
            bool same = got[w].size() == e - b;
            for (uint64_t i = 0; same && i < e - b; ++i) same = got[w][i] == pack_gate(s.gates[b + i]);
            if (!same) {
                std::printf("case %d: window %llu differs\n", t, (unsigned long long)w);
                return 1;
            }
        }
    }
    std::printf("ok %d\n", cases);
    return 0;
}
