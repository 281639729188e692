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
#include <immintrin.h>
#include <condition_variable>
#include <functional>
#include <memory>
#include <mutex>
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
    // Cached: a c5 circuit is 1.5 GB of gates, and the count is asked for by every run.
    if (cached_measures_for_ == gates.size() && cached_data_ == gates.data()) return cached_measures_;
    const uint64_t G = gates.size();
    const unsigned T = std::max(1u, std::min<unsigned>(host_threads(), unsigned(G >> 20) + 1));
    std::vector<uint64_t> part(T, 0);
    parallel_chunks(G, T, [&](unsigned t, uint64_t b, uint64_t e) {
        uint64_t m = 0;
        for (uint64_t i = b; i < e; ++i) m += gates[i].kind == QSR_MEASURE;
        part[t] = m;
    });
    uint64_t m = 0;
    for (uint64_t v : part) m += v;
    cached_measures_ = m;
    cached_measures_for_ = G;
    cached_data_ = gates.data();
    return m;
}

void Circuit::check_valid() const {
    // The reference reports the first offending gate (circuit.hpp:108-115): chunks are checked in
    // parallel, and the earliest failing index wins.
    const uint64_t G = gates.size();
    const unsigned T = std::max(1u, std::min<unsigned>(host_threads(), unsigned(G >> 20) + 1));
    std::vector<uint64_t> first(T, ~uint64_t(0));
    std::vector<int> why(T, 0);
    parallel_chunks(G, T, [&](unsigned t, uint64_t b, uint64_t e) {
        for (uint64_t i = b; i < e; ++i) {
            const qsr_gate &g = gates[i];
            int w = 0;
            if (g.kind > QSR_MEASURE) {
                w = 1;
            } else {
                const int ar = gate_arity(g.kind);
                if (g.q0 >= num_qubits || (ar == 2 && g.q1 >= num_qubits)) w = 2;
                else if (ar == 2 && g.q0 == g.q1) w = 3;
            }
            if (w) {
                first[t] = i;
                why[t] = w;
                return;
            }
        }
    });
    for (unsigned t = 0; t < T; ++t) {
        if (why[t] == 1) fail(QSR_INVALID_ARGUMENT, "unknown gate kind");
        if (why[t] == 2) fail(QSR_OUT_OF_RANGE, "gate operand out of range");
        if (why[t] == 3) fail(QSR_INVALID_ARGUMENT, "two-qubit gate with equal operands");
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

namespace {
const uint8_t kUnitary[11] = {QSR_X, QSR_Y, QSR_Z, QSR_H, QSR_S, QSR_SDG, QSR_CX, QSR_CY, QSR_CZ, QSR_SWAP, QSR_ISWAP};
const uint8_t kSingle[6] = {QSR_X, QSR_Y, QSR_Z, QSR_H, QSR_S, QSR_SDG};

// One layer of the reference generator from stream position rng.index (circuit.hpp:142-164).
void sequential_layer(Stream &rng, uint32_t n, std::vector<uint32_t> &order, GateVec &out) {
    {
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
                    out.push_back({kind, order[i], 0});
                    i += 1;
                } else {
                    out.push_back({kind, order[i], order[i + 1]});
                    i += 2;
                }
            } else {
                out.push_back({kind, order[i], 0});
                i += 1;
            }
        }
    }
}

// Persistent workers for the Philox fills of the parallel generator: launch(f) runs f(t, T) on
// every worker; wait() blocks until all have returned.
class FillPool {
  public:
    explicit FillPool(unsigned T) : T_(T) {
        for (unsigned t = 0; t < T; ++t) th_.emplace_back([this, t] { loop(t); });
    }
    ~FillPool() {
        {
            std::lock_guard<std::mutex> g(m_);
            stop_ = true;
            ++gen_;
        }
        cv_.notify_all();
        for (auto &x : th_) x.join();
    }
    void launch(std::function<void(unsigned, unsigned)> f) {
        {
            std::lock_guard<std::mutex> g(m_);
            job_ = std::move(f);
            pending_ = T_;
            ++gen_;
        }
        cv_.notify_all();
    }
    void wait() {
        std::unique_lock<std::mutex> g(m_);
        done_.wait(g, [this] { return pending_ == 0; });
    }

  private:
    void loop(unsigned t) {
        uint64_t seen = 0;
        for (;;) {
            std::function<void(unsigned, unsigned)> f;
            {
                std::unique_lock<std::mutex> g(m_);
                cv_.wait(g, [&] { return gen_ != seen; });
                seen = gen_;
                if (stop_) return;
                f = job_;
            }
            f(t, T_);
            {
                std::lock_guard<std::mutex> g(m_);
                if (--pending_ == 0) done_.notify_all();
            }
        }
    }
    unsigned T_;
    std::vector<std::thread> th_;
    std::mutex m_;
    std::condition_variable cv_, done_;
    std::function<void(unsigned, unsigned)> job_;
    uint64_t gen_ = 0;
    unsigned pending_ = 0;
    bool stop_ = false;
};

// Words of one layer, drawn ahead on the workers assuming no rejection (probability < 2^-40
// per draw for bounds <= 2^24): j[t] = w % (n - t) for the n-1 Fisher-Yates draws at S + t, and
// kinds[u] = the kind of draw w % 11 at S + n - 1 + u. `reject` is set if any of those words
// would be rejected by next_below; the layer is then redone sequentially.
struct LayerWords {
    std::vector<uint32_t> j;
    std::vector<uint8_t> kinds; // per kind word: kind, bit 7 = two-qubit (gates = first m)
    uint32_t m = 0;             // gates of the layer
    uint64_t ku[33] = {};       // kind-word range [ku[t], ku[t+1]) drawn by worker t
    uint64_t steps[32] = {};    // sum over that range of the qubits each draw would take (1 or 2)
    std::atomic<bool> reject{false};
};

// Eight consecutive stream words philox(seed, 2, 0, idx .. idx+7) (rng.hpp:50-55) in AVX2 lanes:
// the 32x32->64 multiplies of a round are two vpmuludq per constant (even / odd lanes).
__attribute__((target("avx2"))) void philox8_avx2(uint64_t seed, uint64_t idx, uint64_t *out) {
    const __m256i M0 = _mm256_set1_epi64x(0xD2511F53u), M1 = _mm256_set1_epi64x(0xCD9E8D57u);
    __m256i c0 = _mm256_set1_epi32(2), c1 = _mm256_setzero_si256();
    const __m256i lane = _mm256_setr_epi32(0, 1, 2, 3, 4, 5, 6, 7);
    // (callers keep the 8 indices within one 2^32 block: the high counter word is common)
    __m256i c2 = _mm256_add_epi32(_mm256_set1_epi32(int(uint32_t(idx))), lane);
    __m256i c3 = _mm256_set1_epi32(int(uint32_t(idx >> 32)));
    uint32_t k0 = uint32_t(seed), k1 = uint32_t(seed >> 32);
    for (int r = 0; r < 10; ++r) {
        const __m256i pe0 = _mm256_mul_epu32(c0, M0), po0 = _mm256_mul_epu32(_mm256_srli_epi64(c0, 32), M0);
        const __m256i pe1 = _mm256_mul_epu32(c2, M1), po1 = _mm256_mul_epu32(_mm256_srli_epi64(c2, 32), M1);
        const __m256i hi0 = _mm256_blend_epi32(_mm256_srli_epi64(pe0, 32), po0, 0xAA);
        const __m256i lo0 = _mm256_blend_epi32(pe0, _mm256_slli_epi64(po0, 32), 0xAA);
        const __m256i hi1 = _mm256_blend_epi32(_mm256_srli_epi64(pe1, 32), po1, 0xAA);
        const __m256i lo1 = _mm256_blend_epi32(pe1, _mm256_slli_epi64(po1, 32), 0xAA);
        const __m256i n0 = _mm256_xor_si256(_mm256_xor_si256(hi1, c1), _mm256_set1_epi32(int(k0)));
        const __m256i n2 = _mm256_xor_si256(_mm256_xor_si256(hi0, c3), _mm256_set1_epi32(int(k1)));
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    // word = c1:c0 per lane
    const __m256i a = _mm256_unpacklo_epi32(c0, c1), b = _mm256_unpackhi_epi32(c0, c1); // lanes 0,1,4,5 / 2,3,6,7
    _mm256_storeu_si256(reinterpret_cast<__m256i *>(out), _mm256_permute2x128_si256(a, b, 0x20));
    _mm256_storeu_si256(reinterpret_cast<__m256i *>(out + 4), _mm256_permute2x128_si256(a, b, 0x31));
}

bool have_avx2() {
    static const bool v = __builtin_cpu_supports("avx2");
    return v;
}

void fill_layer(LayerWords &L, uint64_t seed, uint32_t n, uint64_t S, unsigned t, unsigned T) {
    const uint64_t total = uint64_t(n - 1) + uint64_t(n) + 1;
    const uint64_t lim11 = 11 * (~uint64_t(0) / 11);
    bool rej = false;
    const uint64_t x0 = total * t / T, x1 = total * (t + 1) / T;
    uint64_t steps = 0;
    const bool vec = have_avx2();
    uint64_t wb[8];
    for (uint64_t x = x0; x < x1; ++x) {
        uint64_t w;
        if (vec) {
            if (((x - x0) & 7) == 0) {
                const uint64_t i0 = S + x;
                if (uint32_t(i0) <= 0xFFFFFFF8u) philox8_avx2(seed, i0, wb);
                else for (int l = 0; l < 8; ++l) wb[l] = philox_word(seed, 2, 0, i0 + l); // low word wraps
            }
            w = wb[(x - x0) & 7];
        } else {
            w = philox_word(seed, 2, 0, S + x);
        }
        if (x < n - 1) {
            const uint64_t bound = n - x;
            if ((w >> 24) == 0xFFFFFFFFFFull && w >= bound * (~uint64_t(0) / bound)) rej = true;
            L.j[x] = uint32_t(w % bound);
        } else {
            if (w >= lim11) rej = true;
            const uint32_t kk = uint32_t(w % 11), two = kk >= 6;
            L.kinds[x - (n - 1)] = uint8_t(kUnitary[kk] | (two << 7));
            steps += 1 + two;
        }
    }
    L.ku[t] = std::max<uint64_t>(x0, n - 1) - (n - 1);
    if (t + 1 == T) L.ku[T] = total - (n - 1);
    L.steps[t] = steps;
    if (rej) L.reject = true;
}
} // namespace

// generate_random (circuit.hpp:132-173), word for word the reference's stream. Large circuits
// draw each layer's Philox words on all host threads (the stream is counter-based: word i is
// philox(seed, 2, 0, i)); only the layer-to-layer stream offset is sequential, and it is known
// as soon as the layer's kind draws are scanned, so the next layer's words are drawn while this
// layer is shuffled and emitted.
Circuit generate_random(uint32_t n, uint32_t depth, uint64_t seed, double measure_prob) {
    if (n < 1 || depth < 1)
        fail(QSR_INVALID_ARGUMENT, "generate_random: n and depth must be >= 1");
    if (!(measure_prob >= 0.0 && measure_prob <= 1.0))
        fail(QSR_INVALID_ARGUMENT, "generate_random: measure_prob must be in [0,1]");
    if (n > kMaxQubits)
        fail(QSR_INVALID_ARGUMENT, "generate_random: n exceeds the packed-gate limit");
    Stream rng{seed, 2 /* kStreamGenerator */};
    Circuit c;
    c.num_qubits = n;
    c.num_clbits = n; // circuit.hpp:171
    // ~0.6875 gates per qubit per layer for the uniform 11-kind draw.
    c.gates.reserve(size_t(double(n) * depth * 0.69) + n / 8 + 16);
    std::vector<uint32_t> order(n);
    const unsigned T = std::min(host_threads(), 32u); // LayerWords holds 32 chunk sums
    if (T < 2 || n < 4096 || uint64_t(n) * depth < (uint64_t(1) << 20)) {
        for (uint32_t layer = 0; layer < depth; ++layer) sequential_layer(rng, n, order, c.gates);
    } else {
        // Three stages over a ring of R layer buffers: workers draw layer L+1's words while the
        // main thread scans layer L's kinds (which fixes the layer's gate count, hence its output
        // offset) and E emitter threads shuffle and write earlier layers in place.
        const unsigned E = std::max(1u, std::min(4u, T / 2)), R = 2 + E;
        FillPool pool(T);
        std::unique_ptr<LayerWords[]> buf(new LayerWords[R]);
        for (unsigned r = 0; r < R; ++r) {
            buf[r].j.resize(n);
            buf[r].kinds.resize(size_t(n) + 1);
        }
        std::mutex em;
        std::condition_variable ecv;
        struct Job { uint32_t layer; uint64_t off; };
        std::vector<Job> jobs;  // FIFO (head index below)
        size_t head = 0;
        std::vector<uint8_t> done(depth, 0);
        uint32_t prefix = 0;    // layers [0, prefix) are written
        uint32_t in_flight = 0;
        bool quit = false;
        auto finish = [&](uint32_t L) { // under em
            done[L] = 1;
            while (prefix < depth && done[prefix]) ++prefix;
        };
        std::vector<std::thread> emitters;
        for (unsigned e = 0; e < E; ++e)
            emitters.emplace_back([&] {
                std::vector<uint32_t> ord(n);
                for (;;) {
                    Job j;
                    qsr_gate *out;
                    {
                        std::unique_lock<std::mutex> g(em);
                        ecv.wait(g, [&] { return quit || head < jobs.size(); });
                        if (head == jobs.size()) return;
                        j = jobs[head++];
                        out = c.gates.data() + j.off; // no reallocation while jobs are in flight
                    }
                    LayerWords &b = buf[j.layer % R];
                    for (uint32_t i = 0; i < n; ++i) ord[i] = i;
                    for (uint32_t t = 0; t + 1 < n; ++t) std::swap(ord[n - 1 - t], ord[b.j[t]]);
                    uint32_t pos = 0;
                    for (uint32_t g = 0; g < b.m; ++g) {
                        const uint8_t kk = b.kinds[g];
                        const uint32_t two = kk >> 7;
                        out[g] = qsr_gate{uint8_t(kk & 0x7F), ord[pos], two ? ord[pos + 1] : 0u};
                        pos += 1 + two;
                    }
                    {
                        std::lock_guard<std::mutex> g(em);
                        finish(j.layer);
                        --in_flight;
                    }
                    ecv.notify_all();
                }
            });
        auto wait_prefix = [&](uint32_t upto) {
            std::unique_lock<std::mutex> g(em);
            ecv.wait(g, [&] { return prefix >= upto; });
        };
        auto launch = [&](uint32_t L, uint64_t S) {
            if (L >= R) wait_prefix(L - R + 1); // the buffer's previous layer is written
            LayerWords &b = buf[L % R];
            b.reject = false;
            pool.launch([&b, seed, n, S](unsigned t, unsigned TT) { fill_layer(b, seed, n, S, t, TT); });
        };
        launch(0, 0);
        for (uint32_t layer = 0; layer < depth; ++layer) {
            LayerWords &b = buf[layer % R];
            pool.wait();
            const uint64_t S = rng.index;
            if (b.reject) { // exact fallback: the reference loop from the same stream position
                wait_prefix(layer);
                sequential_layer(rng, n, order, c.gates);
                if (layer + 1 < depth) launch(layer + 1, rng.index);
                std::lock_guard<std::mutex> g(em);
                finish(layer);
                continue;
            }
            // Kind scan (circuit.hpp:150-163): fixes the stream offset of the next layer.
            // The workers summed each chunk's steps; skip whole chunks, scan the crossing one.
            uint64_t pos = 0, u = 0;
            unsigned t = 0;
            while (t < T && pos + b.steps[t] < n) pos += b.steps[t++];
            u = b.ku[t];
            uint8_t *kinds = b.kinds.data();
            for (;;) {
                const uint32_t two = kinds[u] >> 7;
                if (two && pos + 1 >= n) { // a two-qubit draw on the last qubit: redraw single
                    rng.index = S + (n - 1) + u + 1;
                    kinds[u] = kSingle[rng.below(6)];
                    b.m = uint32_t(u + 1);
                    u = rng.index - S - (n - 1);
                    break;
                }
                pos += 1 + two;
                ++u;
                if (pos >= n) {
                    b.m = uint32_t(u);
                    break;
                }
            }
            rng.index = S + (n - 1) + u;
            if (layer + 1 < depth) launch(layer + 1, rng.index);
            // Output slot of the layer; growing past the reserved capacity waits for the
            // emitters (a reallocation moves the gates they write into).
            const uint64_t off = c.gates.size();
            if (off + b.m > c.gates.capacity()) {
                std::unique_lock<std::mutex> g(em);
                ecv.wait(g, [&] { return in_flight == 0; });
                c.gates.reserve(std::max<uint64_t>(2 * c.gates.capacity(), off + b.m));
            }
            c.gates.resize(off + b.m);
            {
                std::lock_guard<std::mutex> g(em);
                jobs.push_back({layer, off});
                ++in_flight;
            }
            ecv.notify_all();
        }
        pool.wait();
        {
            std::lock_guard<std::mutex> g(em);
            quit = true;
        }
        ecv.notify_all();
        for (auto &x : emitters) x.join();
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
    p.key.resize(G); // no zero fill (NoInitAlloc); first touch in parallel, off the serial scan
    parallel_chunks(G, std::max(1u, std::min<unsigned>(host_threads(), unsigned(G >> 22) + 1)),
                    [&](unsigned, uint64_t b, uint64_t e) {
                        if (e > b) std::memset(p.key.data() + b, 0, (e - b) * sizeof(uint32_t));
                    });
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
