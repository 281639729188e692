// Circuit input pipeline and window scheduler (host side of the hot path).
//
// generate_random restates circuit.hpp:132-173 draw for draw (the benchmark circuits must
// be the reference's own). schedule_windows replaces the reference's O(G*W) greedy
// front advancement (schedule.hpp:51-137) by a one-pass closed form with identical output:
//   round(U) = 1 + max_{wires} round(previous gate on the wire)   (0 if none)
//   round(M) = max(1, round(previous gate on its wire))
// and for r = 1..R the schedule emits the unitary gates of round r (index order) as one
// window, then the measurements of round r (index order) as one measurement window.
// A unitary gate is frontier in the reference's round r exactly when every wire's previous
// gate was consumed in an earlier round (busy never blocks a frontier gate, because a busy
// wire means an earlier-indexed gate on that wire was taken in this very scan). Measurements
// are flushed after the unitary scan of the round in which their wire's predecessor was
// taken, chaining through consecutive measurements on one wire (the reference's quirk that
// later makes measure_window reject the window is therefore preserved).
#include <cstdio>
#include <algorithm>
#include <atomic>
#include <cstring>
#include <thread>

#include "host.hpp"

namespace qsr {

bool trace_on() {
    static const bool on = [] {
        const char *e = getenv("QSR_TRACE");
        return e && e[0] == '1';
    }();
    return on;
}

namespace {
std::atomic<unsigned> g_threads{0};
}
void set_host_threads(unsigned t) { g_threads = t; }
unsigned host_threads() {
    const unsigned t = g_threads.load();
    return t ? t : std::max(1u, std::thread::hardware_concurrency());
}

void trace(const char *phase, double ms) { fprintf(stderr, "[qsr] %-28s %10.2f ms\n", phase, ms); }


void philox_block(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int r = 0; r < 10; ++r) {
        uint64_t p0 = uint64_t(0xD2511F53u) * c0;
        uint64_t p1 = uint64_t(0xCD9E8D57u) * c2;
        uint32_t n0 = uint32_t(p1 >> 32) ^ c1 ^ k0;
        uint32_t n1 = uint32_t(p1);
        uint32_t n2 = uint32_t(p0 >> 32) ^ c3 ^ k1;
        uint32_t n3 = uint32_t(p0);
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

uint64_t philox_word(uint64_t seed, uint32_t stream, uint32_t ctx, uint64_t index) {
    uint32_t ctr[4] = {stream, ctx, uint32_t(index), uint32_t(index >> 32)};
    uint32_t key[2] = {uint32_t(seed), uint32_t(seed >> 32)};
    uint32_t out[4];
    philox_block(ctr, key, out);
    return (uint64_t(out[1]) << 32) | out[0];
}

uint64_t Circuit::measure_count() const {
    uint64_t m = 0;
    for (const auto &g : gates)
        m += g.kind == QSR_MEASURE;
    return m;
}

void Circuit::check_valid() const {
    for (const auto &g : gates) {
        if (g.kind > QSR_MEASURE)
            fail(QSR_INVALID_ARGUMENT, "unknown gate kind");
        int ar = gate_arity(g.kind);
        if (g.q0 >= num_qubits || (ar == 2 && g.q1 >= num_qubits))
            fail(QSR_OUT_OF_RANGE, "gate operand out of range");
        if (ar == 2 && g.q0 == g.q1)
            fail(QSR_INVALID_ARGUMENT, "two-qubit gate with equal operands");
    }
}

namespace {
// Sequential view of one (seed, stream) Philox lane (rng.hpp:61-95).
struct Stream {
    uint64_t seed;
    uint32_t stream;
    uint64_t index = 0;
    uint64_t next() { return philox_word(seed, stream, 0, index++); }
    uint64_t below(uint64_t bound) {
        if (bound <= 1)
            return 0;
        uint64_t limit = bound * (~uint64_t{0} / bound);
        for (;;) {
            uint64_t w = next();
            if (w < limit)
                return w % bound;
        }
    }
    bool bernoulli(double p) {
        double u = double(next() >> 11) * 0x1.0p-53;
        return u < p;
    }
};
} // namespace

Circuit generate_random(uint32_t n, uint32_t depth, uint64_t seed, double measure_prob) {
    if (n < 1 || depth < 1)
        fail(QSR_INVALID_ARGUMENT, "generate_random: n and depth must be >= 1");
    if (!(measure_prob >= 0.0 && measure_prob <= 1.0))
        fail(QSR_INVALID_ARGUMENT, "generate_random: measure_prob must be in [0,1]");
    if (n > kMaxQubits)
        fail(QSR_INVALID_ARGUMENT, "generate_random: n exceeds the packed-gate limit");
    static const uint8_t kUnitary[11] = {QSR_X,  QSR_Y,  QSR_Z,  QSR_H,    QSR_S,    QSR_SDG,
                                         QSR_CX, QSR_CY, QSR_CZ, QSR_SWAP, QSR_ISWAP};
    static const uint8_t kSingle[6] = {QSR_X, QSR_Y, QSR_Z, QSR_H, QSR_S, QSR_SDG};
    Stream rng{seed, 2 /* kStreamGenerator */};
    Circuit c;
    c.num_qubits = n;
    c.num_clbits = n; // circuit.hpp:171
    // ~0.6875 gates per qubit per layer for the uniform 11-kind draw.
    c.gates.reserve(size_t(double(n) * depth * 0.69) + n / 8 + 16);
    std::vector<uint32_t> order(n);
    for (uint32_t layer = 0; layer < depth; ++layer) {
        for (uint32_t i = 0; i < n; ++i)
            order[i] = i;
        for (uint32_t i = n; i > 1; --i) {
            uint32_t j = uint32_t(rng.below(i));
            std::swap(order[i - 1], order[j]);
        }
        uint32_t i = 0;
        while (i < n) {
            uint8_t kind = kUnitary[rng.below(11)];
            if (gate_arity(kind) == 2) {
                if (i + 1 >= n) {
                    kind = kSingle[rng.below(6)];
                    c.gates.push_back({kind, order[i], 0});
                    i += 1;
                } else {
                    c.gates.push_back({kind, order[i], order[i + 1]});
                    i += 2;
                }
            } else {
                c.gates.push_back({kind, order[i], 0});
                i += 1;
            }
        }
    }
    for (uint32_t q = 0; q < n; ++q)
        if (rng.bernoulli(measure_prob))
            c.gates.push_back({QSR_MEASURE, q, 0});
    return c;
}

WindowPlan plan_windows(const Circuit &c) {
    const uint64_t G = c.gates.size();
    const uint32_t n = c.num_qubits;
    WindowPlan p;
    p.key.resize(G);
    // wire state = round << 1 | (last gate on the wire was a MEASURE)
    std::vector<uint32_t> wire(n, 0);
    uint32_t max_round = 0, dup = 0;
    const qsr_gate *gates = c.gates.data();
    uint32_t *key = p.key.data();
    for (uint64_t i = 0; i < G; ++i) {
        const qsr_gate g = gates[i];
        const uint32_t kind = g.kind;
        // check_valid (circuit.hpp:108-115), fused into the same pass
        if (kind > QSR_MEASURE) fail(QSR_INVALID_ARGUMENT, "unknown gate kind");
        const bool two = kind >= QSR_CX && kind <= QSR_ISWAP;
        const uint32_t q0 = g.q0, q1 = two ? g.q1 : g.q0;
        if (q0 >= n || q1 >= n) fail(QSR_OUT_OF_RANGE, "gate operand out of range");
        if (two && q0 == q1) fail(QSR_INVALID_ARGUMENT, "two-qubit gate with equal operands");
        const uint32_t w0 = wire[q0], w1 = wire[q1];
        const uint32_t r0 = w0 >> 1, r1 = w1 >> 1;
        const uint32_t meas = kind == QSR_MEASURE;
        const uint32_t r = meas ? (r0 > 1 ? r0 : 1) : 1 + (r0 > r1 ? r0 : r1);
        // A measurement chained behind another on the same wire lands in the same window;
        // the reference's measure_window then rejects it (measure.hpp:394-395).
        dup |= meas & w0 & 1u;
        wire[q0] = (r << 1) | meas;
        wire[q1] = (r << 1) | meas;
        key[i] = 2 * r + meas;
        max_round = r > max_round ? r : max_round;
    }
    p.duplicate_measure = dup != 0;
    p.nkeys = 2 * uint64_t(max_round) + 2;
    // Per-thread key histograms over contiguous gate chunks -> stable scatter offsets
    // (key-major, chunk-minor), so the parallel scatter keeps circuit index order per window.
    const unsigned T = p.threads = std::max(1u, std::min<unsigned>(host_threads(),
                                                                     unsigned(G / (1 << 16)) + 1));
    p.chunk_offsets.assign(uint64_t(T) * p.nkeys, 0);
    {
        std::vector<std::thread> th;
        for (unsigned t = 0; t < T; ++t)
            th.emplace_back([&, t] {
                uint64_t *h = p.chunk_offsets.data() + uint64_t(t) * p.nkeys;
                for (uint64_t i = G * t / T; i < G * (t + 1) / T; ++i) ++h[p.key[i]];
            });
        for (auto &x : th) x.join();
    }
    uint64_t pos = 0;
    p.offsets.push_back(0);
    for (uint64_t key = 0; key < p.nkeys; ++key) {
        uint64_t total = 0;
        for (unsigned t = 0; t < T; ++t) {
            uint64_t &h = p.chunk_offsets[uint64_t(t) * p.nkeys + key];
            uint64_t cnt = h;
            h = pos + total;
            total += cnt;
        }
        if (total) {
            pos += total;
            p.offsets.push_back(pos);
            p.is_meas.push_back(uint8_t(key & 1));
        }
    }
    return p;
}

Schedule schedule_windows(const Circuit &c, int mode) {
    WindowPlan p = [&] {
        TraceScope tr("plan_windows");
        return plan_windows(c);
    }();
    Schedule s;
    s.mode = mode;
    s.gates.resize(c.gates.size());
    scatter_windows(c, p, s.gates.data(), [](const qsr_gate &g) { return g; });
    s.offsets = std::move(p.offsets);
    s.is_meas = std::move(p.is_meas);
    return s;
}

void validate_window(uint64_t n, const qsr_gate *gates, uint64_t ngates, bool is_measurement,
                     std::vector<uint32_t> &stamp, uint32_t stamp_id) {
    if (stamp.size() < n)
        stamp.assign(n, 0);
    if (is_measurement) {
        for (uint64_t i = 0; i < ngates; ++i) {
            const qsr_gate &g = gates[i];
            if (g.kind != QSR_MEASURE)
                fail(QSR_INVALID_ARGUMENT, "measure_window: unitary gate in window");
            if (g.q0 >= n)
                fail(QSR_OUT_OF_RANGE, "measure_window: qubit out of range");
            if (stamp[g.q0] == stamp_id)
                fail(QSR_INVALID_ARGUMENT, "measure_window: qubit measured twice");
            stamp[g.q0] = stamp_id;
        }
        return;
    }
    for (uint64_t i = 0; i < ngates; ++i) {
        const qsr_gate &g = gates[i];
        if (g.kind == QSR_MEASURE)
            fail(QSR_INVALID_ARGUMENT, "apply_window: window contains measurements");
        if (g.kind > QSR_MEASURE)
            fail(QSR_INVALID_ARGUMENT, "apply_window: unknown gate kind");
        int ar = gate_arity(g.kind);
        for (int op = 0; op < ar; ++op) {
            uint32_t q = op == 0 ? g.q0 : g.q1;
            if (q >= n)
                fail(QSR_OUT_OF_RANGE, "apply_window: gate operand out of range");
            if (stamp[q] == stamp_id)
                fail(QSR_INVALID_ARGUMENT, "apply_window: operands not disjoint");
            stamp[q] = stamp_id;
        }
    }
}

} // namespace qsr
