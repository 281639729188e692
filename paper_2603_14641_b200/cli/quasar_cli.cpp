// `quasar` command-line driver on the B200 engine: the reference CLI (tools/quasar.cpp) with the
// same subcommands, options, outputs and exit codes, computing through libqsr.so.
//
//   quasar run <in.qasm> [--out F] [--json F] [--seed S] [--word-size W] [--threads T] [--device D]
//   quasar sample <in.qasm> [--shots N] [--format text|binary] [--out F] [--json F] [--seed S] ...
//   quasar gen [--qubits N] [--depth D] [--measure-prob P] [--out F] [--seed S]
//   quasar schedule <in.qasm>
//   quasar verify [--n-min --n-max --depth-min --depth-max --trials --seed --threads --device]
//   quasar bench [in.qasm] [--qubits --depth --measure-prob --reps --seed --word-size --device]
//
// Exit codes: 0 ok, 1 verification failure, 2 input error (QasmError / bad input / library
// error), 3 resource error (host or device memory) — tools/quasar.cpp:40-43, 386-395. Usage
// errors use CLI11's codes (104 conversion, 105 validation, 106 required, 109 extras).
//
// `verify` does not link the reference's scalar CHP / state-vector oracles (they are test
// infrastructure here). Its differential leg checks the fused, streamed whole-circuit run
// against (a) window-by-window calls on a device tableau and (b) an independent scalar cell
// tableau of its own (the role of oracle::run_scalar, tools/quasar.cpp:165-236), record and
// final tableau bit for bit, and checks the final tableau is a stabilizer group (device
// kernel); the statistical leg keeps the reference's chi-square test with a small state-vector
// checker of its own.
#include <algorithm>
#include <cerrno>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <functional>
#include <iostream>
#include <map>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "qsr.h"

namespace {

constexpr int kExitOk = 0, kExitVerifyFailure = 1, kExitInputError = 2, kExitResourceError = 3;

// ---- errors -------------------------------------------------------------------------------

struct UsageError : std::runtime_error {
    int code;
    UsageError(int c, const std::string &m) : std::runtime_error(m), code(c) {}
};
struct LibError : std::runtime_error {
    qsr_status status;
    LibError(qsr_status s, const std::string &m) : std::runtime_error(m), status(s) {}
};

void check(qsr_status st) {
    if (st != QSR_OK) throw LibError(st, qsr_last_error());
}

// RAII handles
struct CircuitH {
    qsr_circuit *p = nullptr;
    ~CircuitH() { if (p) qsr_circuit_destroy(p); }
};
struct ScheduleH {
    qsr_schedule *p = nullptr;
    ~ScheduleH() { if (p) qsr_schedule_destroy(p); }
};
struct TableauH {
    qsr_tableau *p = nullptr;
    ~TableauH() { if (p) qsr_tableau_destroy(p); }
};
struct FramesH {
    qsr_frames *p = nullptr;
    ~FramesH() { if (p) qsr_frames_destroy(p); }
};

// ---- a small CLI11-compatible option parser -------------------------------------------------

struct Opt {
    std::string name;       // "--seed"
    std::function<void(const std::string &)> set;
    bool flag = false;
};

struct Command {
    std::string name, help;
    std::vector<Opt> opts;
    std::string *positional = nullptr;
    bool positional_required = false;
    std::string positional_name;
    bool parsed = false;

    template <typename T>
    void num(const std::string &n, T &dst, std::function<void(T)> check_fn = nullptr) {
        opts.push_back({n, [n, &dst, check_fn](const std::string &v) {
            errno = 0;
            char *end = nullptr;
            T out{};
            if constexpr (std::is_floating_point_v<T>) {
                out = T(std::strtod(v.c_str(), &end));
            } else {
                if (!v.empty() && v[0] == '-') throw UsageError(104, n + ": negative value " + v);
                out = T(std::strtoull(v.c_str(), &end, 10));
            }
            if (v.empty() || !end || *end || errno) throw UsageError(104, n + ": could not convert '" + v + "'");
            if (check_fn) check_fn(out);
            dst = out;
        }});
    }
    void str(const std::string &n, std::string &dst, std::vector<std::string> members = {}) {
        opts.push_back({n, [n, &dst, members](const std::string &v) {
            if (!members.empty() && std::find(members.begin(), members.end(), v) == members.end())
                throw UsageError(105, n + ": " + v + " not in {" + [&] {
                    std::string s;
                    for (auto &m : members) s += (s.empty() ? "" : ",") + m;
                    return s;
                }() + "}");
            dst = v;
        }});
    }
};

template <typename T>
std::function<void(T)> positive(const std::string &n) {
    return [n](T v) { if (!(v > 0)) throw UsageError(105, n + ": value must be positive"); };
}
std::function<void(double)> unit_range(const std::string &n) {
    return [n](double v) { if (!(v >= 0.0 && v <= 1.0)) throw UsageError(105, n + ": value not in range [0, 1]"); };
}
std::function<void(unsigned)> word_member(const std::string &n) {
    return [n](unsigned v) {
        if (v != 8 && v != 16 && v != 32 && v != 64) throw UsageError(105, n + ": " + std::to_string(v) + " not in {8,16,32,64}");
    };
}

void parse_command(Command &cmd, int argc, char **argv, int first) {
    bool have_pos = false;
    for (int i = first; i < argc; ++i) {
        std::string a = argv[i];
        if (a.rfind("--", 0) == 0) {
            std::string key = a, val;
            const size_t eq = a.find('=');
            bool inline_val = eq != std::string::npos;
            if (inline_val) {
                key = a.substr(0, eq);
                val = a.substr(eq + 1);
            }
            auto it = std::find_if(cmd.opts.begin(), cmd.opts.end(), [&](const Opt &o) { return o.name == key; });
            if (it == cmd.opts.end()) throw UsageError(109, "The following argument was not expected: " + a);
            if (!inline_val) {
                if (i + 1 >= argc) throw UsageError(114, key + ": 1 required argument missing");
                val = argv[++i];
            }
            it->set(val);
        } else if (cmd.positional && !have_pos) {
            *cmd.positional = a;
            have_pos = true;
        } else {
            throw UsageError(109, "The following argument was not expected: " + a);
        }
    }
    if (cmd.positional_required && !have_pos) throw UsageError(106, cmd.positional_name + " is required");
    cmd.parsed = true;
}

// ---- IO -----------------------------------------------------------------------------------

std::string read_file(const std::string &path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error("cannot open input file: " + path);
    in.seekg(0, std::ios::end);
    const std::streamoff sz = in.tellg();
    in.seekg(0);
    std::string s(size_t(std::max<std::streamoff>(sz, 0)), '\0');
    if (sz > 0) in.read(&s[0], sz);
    return s;
}

void write_file(const std::string &path, const char *data, size_t len) {
    FILE *f = std::fopen(path.c_str(), "wb");
    if (!f) throw std::runtime_error("cannot open output file: " + path);
    const size_t w = len ? std::fwrite(data, 1, len, f) : 0;
    std::fclose(f);
    if (w != len) throw std::runtime_error("cannot write output file: " + path);
}

struct QasmFail : std::runtime_error {
    using std::runtime_error::runtime_error;
};

void load_circuit(const std::string &path, CircuitH &c) {
    const std::string text = read_file(path);
    qsr_qasm_error err{};
    const qsr_status st = qsr_parse_qasm(text.data(), text.size(), &c.p, &err);
    if (st == QSR_PARSE_ERROR) throw QasmFail(qsr_last_error());
    check(st);
}

std::string text_of(const std::function<qsr_status(char *, uint64_t, uint64_t *)> &fn) {
    uint64_t len = 0;
    check(fn(nullptr, 0, &len));
    std::string s(len, '\0');
    check(fn(len ? &s[0] : nullptr, len, &len));
    return s;
}

// nlohmann::json's number format (shortest round-trip digits; integral values keep ".0").
std::string json_double(double v) {
    if (!std::isfinite(v)) return "null";
    if (v == 0) return std::signbit(v) ? "-0.0" : "0.0";
    char buf[64];
    int prec = 1;
    for (; prec <= 17; ++prec) {
        std::snprintf(buf, sizeof buf, "%.*e", prec - 1, v);
        if (std::strtod(buf, nullptr) == v) break;
    }
    // buf = [-]d.ddde[+-]XX  -> digits and decimal exponent
    std::string s(buf);
    const bool neg = s[0] == '-';
    if (neg) s = s.substr(1);
    const size_t epos = s.find('e');
    const int e10 = std::atoi(s.c_str() + epos + 1);
    std::string digits;
    for (size_t i = 0; i < epos; ++i)
        if (s[i] != '.') digits += s[i];
    while (digits.size() > 1 && digits.back() == '0') digits.pop_back();
    const int k = int(digits.size()), n = e10 + 1; // value = 0.digits * 10^n
    std::string out;
    if (k <= n && n <= 15) {
        out = digits + std::string(size_t(n - k), '0') + ".0";
    } else if (0 < n && n <= 15) {
        out = digits.substr(0, size_t(n)) + "." + digits.substr(size_t(n));
    } else if (-4 < n && n <= 0) {
        out = "0." + std::string(size_t(-n), '0') + digits;
    } else {
        out = digits.substr(0, 1);
        if (k > 1) out += "." + digits.substr(1);
        const int ex = n - 1;
        char eb[16];
        std::snprintf(eb, sizeof eb, "e%c%02d", ex < 0 ? '-' : '+', std::abs(ex));
        out += eb;
    }
    return neg ? "-" + out : out;
}

// ---- report (tools/quasar.cpp:76-102) -----------------------------------------------------

void print_report(uint32_t qubits, const qsr_run_report &r, const std::string &json_path) {
    auto ms = [](double s) { return s * 1e3; };
    std::cout << "qubits=" << qubits << "\n"
              << "gates=" << r.gate_count << "\n"
              << "measures=" << r.measure_count << "\n"
              << "windows=" << r.window_count << "\n"
              << "probabilistic=" << r.probabilistic_count << "\n"
              << "to_ms=" << ms(r.timers.to_seconds) << "\n"
              << "t_ms=" << ms(r.timers.t_seconds) << "\n"
              << "cmp_ms=" << ms(r.timers.cmp_seconds) << "\n"
              << "ge_ms=" << ms(r.timers.ge_seconds) << "\n"
              << "total_ms=" << ms(r.total_seconds) << "\n";
    if (json_path.empty()) return;
    // nlohmann::json objects are std::map-ordered: keys sorted.
    std::map<std::string, std::string> j = {
        {"qubits", std::to_string(qubits)},
        {"gates", std::to_string(r.gate_count)},
        {"measures", std::to_string(r.measure_count)},
        {"windows", std::to_string(r.window_count)},
        {"probabilistic", std::to_string(r.probabilistic_count)},
        {"to_ms", json_double(ms(r.timers.to_seconds))},
        {"t_ms", json_double(ms(r.timers.t_seconds))},
        {"cmp_ms", json_double(ms(r.timers.cmp_seconds))},
        {"ge_ms", json_double(ms(r.timers.ge_seconds))},
        {"total_ms", json_double(ms(r.total_seconds))}};
    std::string out = "{\n";
    size_t i = 0;
    for (auto &[k, v] : j) out += "  \"" + k + "\": " + v + (++i < j.size() ? ",\n" : "\n");
    out += "}\n";
    write_file(json_path, out.data(), out.size());
}

uint32_t num_qubits(const qsr_circuit *c) {
    uint32_t n = 0;
    check(qsr_circuit_info(c, &n, nullptr, nullptr));
    return n;
}
uint64_t num_measures(const qsr_circuit *c) {
    uint64_t m = 0;
    check(qsr_circuit_info(c, nullptr, nullptr, &m));
    return m;
}

// MeasurementRecord::per_qubit (measure.hpp:50-64): last outcome per qubit, first-measured order.
std::vector<std::pair<uint32_t, bool>> per_qubit(const std::vector<qsr_record_entry> &rec) {
    std::vector<std::pair<uint32_t, bool>> out;
    std::map<uint32_t, size_t> pos;
    for (const auto &e : rec) {
        auto it = pos.find(e.qubit);
        if (it == pos.end()) {
            pos[e.qubit] = out.size();
            out.emplace_back(e.qubit, e.outcome != 0);
        } else {
            out[it->second].second = e.outcome != 0;
        }
    }
    return out;
}

struct Shot {
    std::vector<qsr_record_entry> record;
    qsr_run_report report{};
};

Shot run_shot(const qsr_circuit *c, const qsr_schedule *s, uint64_t seed, int device, TableauH *keep = nullptr) {
    Shot r;
    r.record.resize(num_measures(c));
    TableauH t;
    check(qsr_run_single_shot(c, s, seed, device, &t.p, r.record.data(), &r.report));
    if (keep) std::swap(keep->p, t.p);
    return r;
}

// ---- run ------------------------------------------------------------------------------------

int cmd_run(const std::string &in, uint64_t seed, int device, const std::string &out_path,
            const std::string &json_path) {
    CircuitH c;
    load_circuit(in, c);
    // Records are identical for every word type (the reference tests all W against one scalar
    // run, test_measure.cpp:315-335), so W only selects the reference's storage width.
    Shot r = run_shot(c.p, nullptr, seed, device);
    std::string outcomes;
    for (const auto &[q, bit] : per_qubit(r.record)) outcomes += bit ? '1' : '0';
    outcomes += '\n';
    if (!out_path.empty()) {
        if (r.record.empty()) write_file(out_path, "", 0);
        else write_file(out_path, outcomes.data(), outcomes.size());
    } else if (!r.record.empty()) {
        std::cout << "outcomes=" << outcomes;
    }
    print_report(num_qubits(c.p), r.report, json_path);
    return kExitOk;
}

// ---- sample ---------------------------------------------------------------------------------

struct Samples {
    uint64_t shots = 0, kf = 0;
    std::vector<uint32_t> measured;
    std::vector<uint64_t> words; // rows x kf (64-bit words)
    qsr_run_report report{};
};

Samples sample_all(const qsr_circuit *c, uint64_t shots, uint64_t seed, unsigned wbits, int device) {
    Samples s;
    FramesH f;
    check(qsr_sample_word(c, shots, seed, wbits, device, &f.p, &s.report));
    uint64_t n = 0, sh = 0, kf = 0, rows = 0;
    check(qsr_frames_info(f.p, &n, &sh, &kf));
    check(qsr_frames_record(f.p, &rows, nullptr, nullptr));
    s.shots = sh;
    s.kf = kf;
    s.measured.resize(rows);
    s.words.resize(rows * kf);
    check(qsr_frames_record(f.p, &rows, s.measured.data(), s.words.data()));
    return s;
}

// One line per shot, one character per record row (tools/quasar.cpp:131-137); rows are
// transposed 64 shots at a time on all host threads.
std::string shots_text(const Samples &s) {
    const uint64_t R = s.measured.size(), line = R + 1;
    std::string out(s.shots * line, '\0');
    const unsigned T = std::max(1u, std::min<unsigned>(qsr_get_num_threads(), unsigned(s.kf)));
    std::vector<std::thread> th;
    for (unsigned t = 0; t < T; ++t)
        th.emplace_back([&, t] {
            for (uint64_t j = s.kf * t / T; j < s.kf * (t + 1) / T; ++j) {
                const uint64_t s0 = j * 64, s1 = std::min<uint64_t>(s.shots, s0 + 64);
                for (uint64_t sh = s0; sh < s1; ++sh) out[sh * line + R] = '\n';
                for (uint64_t r = 0; r < R; ++r) {
                    const uint64_t w = s.words[r * s.kf + j];
                    for (uint64_t sh = s0; sh < s1; ++sh) out[sh * line + r] = char('0' + ((w >> (sh - s0)) & 1));
                }
            }
        });
    for (auto &x : th) x.join();
    return out;
}

// Per measured qubit: ceil(shots/W) little-endian W-bit words (tools/quasar.cpp:138-144). The
// first bytes of a row of 64-bit words are exactly those W-words.
std::string shots_binary(const Samples &s, unsigned wbits) {
    const uint64_t R = s.measured.size();
    const uint64_t rb = (s.shots + wbits - 1) / wbits * (wbits / 8);
    std::string out(R * rb, '\0');
    for (uint64_t r = 0; r < R; ++r) {
        const uint64_t *row = s.words.data() + r * s.kf;
        for (uint64_t b = 0; b < rb; ++b) out[r * rb + b] = char((row[b / 8] >> (8 * (b % 8))) & 0xFF);
    }
    return out;
}

int cmd_sample(const std::string &in, uint64_t shots, uint64_t seed, unsigned wbits, int device,
               const std::string &out_path, const std::string &format, const std::string &json_path) {
    CircuitH c;
    load_circuit(in, c);
    Samples s = sample_all(c.p, shots, seed, wbits, device);
    std::string payload;
    if (format == "text") payload = shots_text(s);
    else if (format == "binary") payload = shots_binary(s, wbits);
    else throw std::runtime_error("unknown format: " + format);
    if (!out_path.empty()) write_file(out_path, payload.data(), payload.size());
    else std::cout.write(payload.data(), std::streamsize(payload.size()));
    print_report(num_qubits(c.p), s.report, json_path);
    return kExitOk;
}

// ---- verify ---------------------------------------------------------------------------------

// Minimal dense state vector (n <= 12): exact distribution of the last outcome of every
// measured qubit, walking both branches at each measurement in circuit order.
using cplx = std::complex<double>;

void sv_gate(std::vector<cplx> &a, const qsr_gate &g) {
    const double r = 1.0 / std::sqrt(2.0);
    const cplx I(0, 1);
    const size_t b0 = size_t(1) << g.q0;
    if (g.kind <= QSR_SDG) {
        cplx m[4];
        switch (g.kind) {
        case QSR_X: m[0] = 0; m[1] = 1; m[2] = 1; m[3] = 0; break;
        case QSR_Y: m[0] = 0; m[1] = -I; m[2] = I; m[3] = 0; break;
        case QSR_Z: m[0] = 1; m[1] = 0; m[2] = 0; m[3] = -1; break;
        case QSR_H: m[0] = r; m[1] = r; m[2] = r; m[3] = -r; break;
        case QSR_S: m[0] = 1; m[1] = 0; m[2] = 0; m[3] = I; break;
        default: m[0] = 1; m[1] = 0; m[2] = 0; m[3] = -I; break;
        }
        for (size_t i = 0; i < a.size(); ++i)
            if (!(i & b0)) {
                const cplx x = a[i], y = a[i | b0];
                a[i] = m[0] * x + m[1] * y;
                a[i | b0] = m[2] * x + m[3] * y;
            }
        return;
    }
    const size_t c = b0, t = size_t(1) << g.q1;
    for (size_t i = 0; i < a.size(); ++i) {
        if (i & (c | t)) continue;
        cplx &a00 = a[i], &a01 = a[i | t], &a10 = a[i | c], &a11 = a[i | c | t];
        switch (g.kind) {
        case QSR_CX: std::swap(a10, a11); break;
        case QSR_CY: { const cplx x = a10; a10 = -I * a11; a11 = I * x; break; }
        case QSR_CZ: a11 = -a11; break;
        case QSR_SWAP: std::swap(a01, a10); break;
        default: { const cplx x = a01; a01 = I * a10; a10 = I * x; break; } // ISWAP
        }
        (void)a00;
    }
}

void sv_walk(std::vector<cplx> a, const std::vector<qsr_gate> &gates, size_t i, std::vector<int8_t> &last,
             double w, const std::vector<uint32_t> &rows, std::map<std::vector<bool>, double> &dist) {
    for (; i < gates.size(); ++i) {
        const qsr_gate &g = gates[i];
        if (g.kind != QSR_MEASURE) {
            sv_gate(a, g);
            continue;
        }
        const size_t b = size_t(1) << g.q0;
        double p1 = 0;
        for (size_t k = 0; k < a.size(); ++k)
            if (k & b) p1 += std::norm(a[k]);
        for (int o = 0; o < 2; ++o) {
            const double p = o ? p1 : 1 - p1;
            if (p < 1e-9) continue;
            std::vector<cplx> br = a;
            const double s = 1.0 / std::sqrt(p);
            for (size_t k = 0; k < br.size(); ++k) br[k] = (bool(k & b) == bool(o)) ? br[k] * s : 0.0;
            const int8_t saved = last[g.q0];
            last[g.q0] = int8_t(o);
            sv_walk(std::move(br), gates, i + 1, last, w * p, rows, dist);
            last[g.q0] = saved;
        }
        return;
    }
    std::vector<bool> key;
    for (uint32_t q : rows) key.push_back(last[q] == 1);
    dist[key] += w;
}

// Regularized upper incomplete gamma Q(a, x) (series / continued fraction).
double gamma_q(double a, double x) {
    if (x <= 0) return 1.0;
    const double lg = std::lgamma(a);
    if (x < a + 1) {
        double sum = 1.0 / a, del = sum, ap = a;
        for (int n = 0; n < 1000 && std::fabs(del) > std::fabs(sum) * 1e-15; ++n) {
            ap += 1;
            del *= x / ap;
            sum += del;
        }
        return 1.0 - sum * std::exp(-x + a * std::log(x) - lg);
    }
    double b = x + 1 - a, c = 1e300, d = 1 / b, h = d;
    for (int i = 1; i < 1000; ++i) {
        const double an = -i * (i - a);
        b += 2;
        d = an * d + b;
        if (std::fabs(d) < 1e-300) d = 1e-300;
        c = b + an / c;
        if (std::fabs(c) < 1e-300) c = 1e-300;
        d = 1 / d;
        const double del = d * c;
        h *= del;
        if (std::fabs(del - 1) < 1e-15) break;
    }
    return std::exp(-x + a * std::log(x) - lg) * h;
}

// Chi-square p-value with cells of expectation < 5 pooled; an observation the exact
// distribution forbids fails outright.
double chi_square_p(const std::map<std::vector<bool>, size_t> &obs, const std::map<std::vector<bool>, double> &exp,
                    size_t total) {
    for (const auto &[k, n] : obs)
        if (n && !exp.count(k)) return 0.0;
    double chi2 = 0, pe = 0, po = 0;
    size_t cells = 0;
    for (const auto &[k, p] : exp) {
        const double e = p * double(total);
        auto it = obs.find(k);
        const double o = it == obs.end() ? 0.0 : double(it->second);
        if (e < 5) {
            pe += e;
            po += o;
            continue;
        }
        chi2 += (o - e) * (o - e) / e;
        ++cells;
    }
    if (pe > 0) {
        chi2 += (po - pe) * (po - pe) / pe;
        ++cells;
    }
    if (cells <= 1) return 1.0;
    return gamma_q(double(cells - 1) / 2, chi2 / 2);
}

// Philox word stream for trial parameters (the library's counter-based generator).
struct Pick {
    uint64_t seed, i = 0;
    uint64_t word() { return qsr_philox_word(seed, 12, 0, i++); }
    uint64_t below(uint64_t bound) {
        if (bound <= 1) return 0;
        const uint64_t limit = bound * (~uint64_t(0) / bound);
        for (;;) {
            const uint64_t w = word();
            if (w < limit) return w % bound;
        }
    }
};

struct VerifyOpts {
    uint32_t n_min = 2, n_max = 32, depth_min = 4, depth_max = 32, trials = 50;
    uint64_t seed = 1;
};

// Independent scalar check for the differential leg (the role oracle::run_scalar plays in
// tools/quasar.cpp:165-236): one byte per tableau cell, every gate a loop over the 2n rows and
// every collapse the strictly ordered row products of the CHP algorithm, no bit packing, no
// device code. Semantics it must agree with: gate rules gates.hpp:35-115, products and their
// mod-4 phase tableau.hpp:337-350, the collapse measure.hpp:381-442 (pivot = lowest stabilizer
// with X at q; later pivots absorb it; other anticommuting destabilizers absorb it; D_c <- S_c,
// S_c <- Z_q with the coin as sign), deterministic outcomes as the ordered product of the
// stabilizers whose destabilizer has X at q, and the window order of simulator.hpp:46-76
// (probabilistic at window start -> collapse in order; the rest resolved after the collapses).
class CellTableau {
  public:
    explicit CellTableau(uint32_t n) : n_(n), x_(size_t(2) * n * n, 0), z_(size_t(2) * n * n, 0), s_(2 * n, 0) {
        for (uint32_t i = 0; i < n; ++i) {
            x(i, i) = 1;     // destabilizer i = X_i
            z(n + i, i) = 1; // stabilizer i = Z_i
        }
    }
    uint8_t &x(size_t g, size_t q) { return x_[g * n_ + q]; }
    uint8_t &z(size_t g, size_t q) { return z_[g * n_ + q]; }
    uint8_t x(size_t g, size_t q) const { return x_[g * n_ + q]; }
    uint8_t z(size_t g, size_t q) const { return z_[g * n_ + q]; }
    uint8_t sign(size_t g) const { return s_[g]; }

    void gate(const qsr_gate &g) {
        for (size_t r = 0; r < 2 * size_t(n_); ++r) {
            uint8_t &a = x(r, g.q0), &b = z(r, g.q0);
            uint8_t dummy_x = 0, dummy_z = 0;
            const bool two = g.kind >= QSR_CX;
            uint8_t &c = two ? x(r, g.q1) : dummy_x, &d = two ? z(r, g.q1) : dummy_z;
            s_[r] ^= conjugate(g.kind, a, b, c, d);
        }
    }

    // Single-cell Clifford conjugation; returns the sign flip.
    static uint8_t conjugate(uint8_t kind, uint8_t &x0, uint8_t &z0, uint8_t &x1, uint8_t &z1) {
        uint8_t f = 0;
        switch (kind) {
        case QSR_X: f = z0; break;
        case QSR_Y: f = x0 ^ z0; break;
        case QSR_Z: f = x0; break;
        case QSR_H: f = x0 & z0; std::swap(x0, z0); break;
        case QSR_S: f = x0 & z0; z0 ^= x0; break;
        case QSR_SDG: f = x0 & (z0 ^ 1); z0 ^= x0; break;
        case QSR_CX: f = x0 & z1 & ((x1 ^ z0) ^ 1); x1 ^= x0; z0 ^= z1; break;
        case QSR_CZ: f = x0 & x1 & (z0 ^ z1); z1 ^= x0; z0 ^= x1; break;
        case QSR_CY: // SDG(t), CX, S(t)
            f = conjugate(QSR_SDG, x1, z1, x1, z1);
            f ^= conjugate(QSR_CX, x0, z0, x1, z1);
            f ^= conjugate(QSR_S, x1, z1, x1, z1);
            break;
        case QSR_SWAP: std::swap(x0, x1); std::swap(z0, z1); break;
        case QSR_ISWAP: // SWAP, CZ, S(c), S(t)
            std::swap(x0, x1);
            std::swap(z0, z1);
            f = conjugate(QSR_CZ, x0, z0, x1, z1);
            f ^= conjugate(QSR_S, x0, z0, x0, z0);
            f ^= conjugate(QSR_S, x1, z1, x1, z1);
            break;
        default: throw std::runtime_error("verify: unknown gate kind");
        }
        return f & 1;
    }

    // i-exponent (mod 4) of P(xc,zc) * P(xt,zt) for one qubit: +1 / -1 / 0.
    static int phase(uint8_t xc, uint8_t zc, uint8_t xt, uint8_t zt) {
        if (xc && zc) return (zt && !xt) ? 1 : (xt && !zt) ? -1 : 0;          // Y * (Z | X)
        if (xc) return (xt && zt) ? 1 : (zt && !xt) ? -1 : 0;                 // X * (Y | Z)
        if (zc) return (xt && !zt) ? 1 : (xt && zt) ? -1 : 0;                 // Z * (X | Y)
        return 0;
    }

    // row t <- row c * row t (bits XOR, sign with the product's phase).
    void mult(size_t t, size_t c) {
        int e = 0;
        for (size_t q = 0; q < n_; ++q) e += phase(x(c, q), z(c, q), x(t, q), z(t, q));
        if (e & 1) throw std::runtime_error("verify: product of anticommuting rows");
        for (size_t q = 0; q < n_; ++q) {
            x(t, q) ^= x(c, q);
            z(t, q) ^= z(c, q);
        }
        s_[t] ^= s_[c] ^ uint8_t((e & 3) == 2);
    }

    int lowest_pivot(uint32_t q) const {
        for (uint32_t t = 0; t < n_; ++t)
            if (x(n_ + t, q)) return int(t);
        return -1;
    }

    bool deterministic(uint32_t q) const {
        std::vector<uint8_t> ax(n_, 0), az(n_, 0);
        int e = 0;
        for (uint32_t g = 0; g < n_; ++g) {
            if (!x(g, q)) continue;
            e += 2 * s_[n_ + g];
            for (uint32_t p = 0; p < n_; ++p) {
                e += phase(ax[p], az[p], x(n_ + g, p), z(n_ + g, p));
                ax[p] ^= x(n_ + g, p);
                az[p] ^= z(n_ + g, p);
            }
        }
        if (e & 1) throw std::runtime_error("verify: imaginary deterministic phase");
        return ((e >> 1) & 1) != 0;
    }

    // Collapse of a probabilistic Z_q; the coin is the next word of the measurement stream.
    bool collapse(uint32_t q, uint64_t coin) {
        const int c = lowest_pivot(q);
        for (uint32_t t = uint32_t(c) + 1; t < n_; ++t)
            if (x(n_ + t, q)) mult(n_ + t, n_ + c); // (D_c absorbing D_t is overwritten below)
        for (uint32_t g = 0; g < n_; ++g)
            if (g != uint32_t(c) && x(g, q)) mult(g, n_ + c);
        for (uint32_t p = 0; p < n_; ++p) {
            x(c, p) = x(n_ + c, p);
            z(c, p) = z(n_ + c, p);
            x(n_ + c, p) = 0;
            z(n_ + c, p) = p == q;
        }
        s_[c] = s_[n_ + c];
        s_[n_ + c] = uint8_t(coin & 1);
        return s_[n_ + c] != 0;
    }

  private:
    uint32_t n_;
    std::vector<uint8_t> x_, z_, s_;
};

// Scalar run in the schedule's window order; coins from Philox stream 0 (rng.hpp:98).
std::vector<qsr_record_entry> scalar_run(uint32_t n, const qsr_schedule *s, uint64_t seed, CellTableau &t) {
    uint64_t nw = 0, ng = 0;
    int mode = 0;
    check(qsr_schedule_info(s, &nw, &ng, &mode));
    const qsr_gate *g = qsr_schedule_gates(s);
    const uint64_t *off = qsr_schedule_offsets(s);
    const uint8_t *ism = qsr_schedule_is_measurement(s);
    std::vector<qsr_record_entry> rec;
    uint64_t coin = 0;
    (void)n;
    for (uint64_t w = 0; w < nw; ++w) {
        const uint64_t b = off[w], e = off[w + 1];
        if (!ism[w]) {
            for (uint64_t i = b; i < e; ++i) t.gate(g[i]);
            continue;
        }
        std::vector<qsr_record_entry> out(e - b);
        std::vector<char> prob(e - b);
        for (uint64_t m = b; m < e; ++m) prob[m - b] = t.lowest_pivot(g[m].q0) >= 0;
        for (uint64_t m = b; m < e; ++m) {
            const uint32_t q = g[m].q0;
            out[m - b] = {q, 0, 0};
            if (!prob[m - b]) continue;
            if (t.lowest_pivot(q) < 0) { // decided by an earlier collapse of this window
                out[m - b] = {q, uint8_t(t.deterministic(q)), 1};
                continue;
            }
            out[m - b] = {q, uint8_t(t.collapse(q, qsr_philox_word(seed, 0, 0, coin++))), 0};
        }
        for (uint64_t m = b; m < e; ++m)
            if (!prob[m - b]) out[m - b] = {g[m].q0, uint8_t(t.deterministic(g[m].q0)), 1};
        rec.insert(rec.end(), out.begin(), out.end());
    }
    return rec;
}

// Device tableau (reference layout, downloaded) against the scalar cells, bit for bit.
bool same_as_cells(const qsr_tableau *d, const CellTableau &c, uint32_t n) {
    uint64_t nn = 0, k = 0, npad = 0;
    int layout = 0;
    check(qsr_tableau_info(d, &nn, &k, &npad, &layout));
    std::vector<uint64_t> x(npad * 2 * k), z(npad * 2 * k), s(2 * k);
    check(qsr_tableau_download(d, x.data(), z.data(), s.data()));
    for (uint64_t g = 0; g < 2 * uint64_t(n); ++g) {
        const uint64_t col = g < n ? g : npad + (g - n); // tableau.hpp:90 rm_col
        const uint64_t sidx = g < n ? g : k * 64 + (g - n);
        if (((s[sidx / 64] >> (sidx % 64)) & 1) != c.sign(g)) return false;
        for (uint64_t q = 0; q < n; ++q) {
            // ColumnMajor: word (q, col / 64); RowMajor: word (q / 64, col) with pitch 2 n_pad.
            const uint64_t wi = layout == QSR_COLUMN_MAJOR ? q * 2 * k + col / 64 : (q / 64) * 2 * npad + col;
            const unsigned bit = unsigned(layout == QSR_COLUMN_MAJOR ? col % 64 : q % 64);
            if (((x[wi] >> bit) & 1) != c.x(g, q) || ((z[wi] >> bit) & 1) != c.z(g, q)) return false;
        }
    }
    return true;
}

// Window-by-window run on a device tableau (apply_window / measure_window per window: no
// fusion, no streaming, no batching across windows).
std::vector<qsr_record_entry> stepwise(const qsr_circuit *c, const qsr_schedule *s, uint64_t seed, int device,
                                       TableauH &t) {
    uint64_t nw = 0, ng = 0;
    int mode = 0;
    check(qsr_schedule_info(s, &nw, &ng, &mode));
    const qsr_gate *g = qsr_schedule_gates(s);
    const uint64_t *off = qsr_schedule_offsets(s);
    const uint8_t *ism = qsr_schedule_is_measurement(s);
    check(qsr_tableau_create(num_qubits(c), device, &t.p));
    check(qsr_tableau_basis_state(t.p, nullptr)); // |0...0> (tableau.hpp:130)
    std::vector<qsr_record_entry> rec(num_measures(c));
    uint64_t coin = 0, pos = 0;
    for (uint64_t w = 0; w < nw; ++w) {
        const uint64_t b = off[w], e = off[w + 1];
        if (!ism[w]) {
            check(qsr_apply_window(t.p, g + b, e - b));
        } else {
            check(qsr_measure_window(t.p, g + b, e - b, seed, &coin, rec.data() + pos, nullptr));
            pos += e - b;
        }
    }
    return rec;
}

bool same_tableau(const qsr_tableau *a, const qsr_tableau *b) {
    uint64_t n = 0, k = 0, npad = 0;
    int layout = 0;
    check(qsr_tableau_info(a, &n, &k, &npad, &layout));
    const uint64_t pw = npad * 2 * k;
    std::vector<uint64_t> xa(pw), za(pw), sa(2 * k), xb(pw), zb(pw), sb(2 * k);
    check(qsr_tableau_download(a, xa.data(), za.data(), sa.data()));
    check(qsr_tableau_download(b, xb.data(), zb.data(), sb.data()));
    return xa == xb && za == zb && sa == sb;
}

int cmd_verify(const VerifyOpts &opt, int device) {
    if (opt.trials == 0) {
        std::cout << "warning: trials=0, nothing verified\n";
        std::cout << "verify=pass (vacuous)\n";
        return kExitOk;
    }
    if (opt.n_min < 1 || opt.n_max < opt.n_min || opt.depth_max < opt.depth_min)
        throw std::runtime_error("bad verify ranges");
    size_t failures = 0, differential = 0, statistical = 0;
    Pick pick{opt.seed};
    for (uint32_t trial = 0; trial < opt.trials; ++trial) {
        const uint32_t n = opt.n_min + uint32_t(pick.below(opt.n_max - opt.n_min + 1));
        const uint32_t depth = opt.depth_min + uint32_t(pick.below(opt.depth_max - opt.depth_min + 1));
        const uint64_t circuit_seed = pick.word();
        CircuitH c;
        check(qsr_generate_random(n, depth, circuit_seed, 0.5, &c.p));
        ScheduleH s;
        check(qsr_schedule_windows(c.p, QSR_SINGLE_SHOT, &s.p));
        const std::string valid = text_of([&](char *b, uint64_t cap, uint64_t *len) {
            return qsr_validate_schedule(c.p, s.p, b, cap, len);
        });
        auto fail_line = [&](const char *what, const std::string &extra = "") {
            std::cout << "FAIL " << what << " n=" << n << " depth=" << depth << " seed=" << circuit_seed << extra << "\n";
            ++failures;
        };
        if (valid != "valid") {
            fail_line("schedule");
            continue;
        }
        // Differential: fused, streamed whole-circuit run vs window-by-window device calls.
        const uint64_t run_seed = pick.word();
        TableauH whole, step;
        Shot a = run_shot(c.p, nullptr, run_seed, device, &whole);
        std::vector<qsr_record_entry> b = stepwise(c.p, s.p, run_seed, device, step);
        auto same_record = [](const std::vector<qsr_record_entry> &u, const std::vector<qsr_record_entry> &v) {
            bool eq = u.size() == v.size();
            for (size_t i = 0; eq && i < v.size(); ++i)
                eq = u[i].qubit == v[i].qubit && u[i].outcome == v[i].outcome &&
                     u[i].deterministic == v[i].deterministic;
            return eq;
        };
        if (!same_record(a.record, b) || !same_tableau(whole.p, step.p)) fail_line("differential");
        // Independent leg: the scalar cell tableau on the same schedule and coins.
        CellTableau cells(n);
        const std::vector<qsr_record_entry> sc = scalar_run(n, s.p, run_seed, cells);
        if (!same_record(a.record, sc) || !same_as_cells(whole.p, cells, n)) fail_line("differential-scalar");
        const std::string group = text_of([&](char *buf, uint64_t cap, uint64_t *len) {
            return qsr_tableau_check_validity(whole.p, buf, cap, len);
        });
        if (group != "valid") fail_line("group", " (" + group + ")");
        ++differential;
        // Statistical: sampler frequencies against the exact distribution.
        const uint64_t m = num_measures(c.p);
        if (n <= 6 && m >= 1 && m <= 10) {
            const size_t shots = 4096;
            Samples smp = sample_all(c.p, shots, run_seed, 64, device);
            std::vector<qsr_gate> gates(qsr_circuit_gates(c.p), qsr_circuit_gates(c.p) + [&] {
                uint64_t ng = 0;
                check(qsr_circuit_info(c.p, nullptr, &ng, nullptr));
                return ng;
            }());
            std::vector<cplx> amps(size_t(1) << n, 0.0);
            amps[0] = 1.0;
            std::vector<int8_t> last(n, 0);
            std::map<std::vector<bool>, double> expect;
            sv_walk(std::move(amps), gates, 0, last, 1.0, smp.measured, expect);
            std::map<std::vector<bool>, size_t> observed;
            for (size_t sh = 0; sh < shots; ++sh) {
                std::vector<bool> key;
                for (size_t r = 0; r < smp.measured.size(); ++r)
                    key.push_back((smp.words[r * smp.kf + sh / 64] >> (sh % 64)) & 1);
                observed[key]++;
            }
            const double p = chi_square_p(observed, expect, shots);
            if (p <= 0.001) {
                std::ostringstream e;
                e << " p=" << p;
                fail_line("statistical", e.str());
            }
            ++statistical;
        }
    }
    std::cout << "differential_trials=" << differential << "\n"
              << "statistical_trials=" << statistical << "\n"
              << "failures=" << failures << "\n"
              << "verify=" << (failures == 0 ? "pass" : "fail") << "\n";
    return failures == 0 ? kExitOk : kExitVerifyFailure;
}

// ---- bench (tools/quasar.cpp:240-266) --------------------------------------------------------

int cmd_bench(const qsr_circuit *c, uint64_t seed, unsigned reps, int device) {
    ScheduleH s;
    check(qsr_schedule_windows(c, QSR_SINGLE_SHOT, &s.p));
    std::vector<qsr_run_report> reps_out;
    std::cout << "rep\tto_ms\tt_ms\tcmp_ms\tge_ms\ttotal_ms\n";
    for (unsigned rep = 0; rep < reps; ++rep) {
        Shot r = run_shot(c, s.p, seed + rep, device);
        reps_out.push_back(r.report);
        const auto &tm = r.report.timers;
        std::cout << rep << '\t' << tm.to_seconds * 1e3 << '\t' << tm.t_seconds * 1e3 << '\t'
                  << tm.cmp_seconds * 1e3 << '\t' << tm.ge_seconds * 1e3 << '\t'
                  << r.report.total_seconds * 1e3 << "\n";
    }
    auto median = [&](auto get) {
        std::vector<double> v;
        for (const auto &r : reps_out) v.push_back(get(r));
        std::sort(v.begin(), v.end());
        return v[v.size() / 2] * 1e3;
    };
    std::cout << "median\t" << median([](const qsr_run_report &r) { return r.timers.to_seconds; }) << '\t'
              << median([](const qsr_run_report &r) { return r.timers.t_seconds; }) << '\t'
              << median([](const qsr_run_report &r) { return r.timers.cmp_seconds; }) << '\t'
              << median([](const qsr_run_report &r) { return r.timers.ge_seconds; }) << '\t'
              << median([](const qsr_run_report &r) { return r.total_seconds; }) << "\n";
    return kExitOk;
}

void usage(std::ostream &o) {
    o << "data-parallel stabilizer circuit simulator (B200 engine)\n"
         "Usage: quasar SUBCOMMAND [OPTIONS]\n\n"
         "Subcommands:\n"
         "  run       single-shot simulation of a QASM file\n"
         "  sample    many-shot Pauli-frame sampling\n"
         "  gen       generate a random Clifford benchmark circuit\n"
         "  schedule  dump the window schedule of a circuit\n"
         "  verify    differential and statistical self-checks\n"
         "  bench     phase-timing table (TO/T/CMP/GE)\n";
}

} // namespace

int main(int argc, char **argv) {
    uint64_t seed = 0;
    unsigned word_size = 64, threads = 0;
    int device = 0;
    std::string in_path, out_path, json_path, format = "text";
    uint64_t shots = 1024;
    uint32_t gen_qubits = 16, gen_depth = 16;
    double measure_prob = 0.1;
    unsigned reps = 3;
    VerifyOpts verify;

    Command run{"run", "single-shot simulation of a QASM file"}, smp{"sample", "many-shot Pauli-frame sampling"},
        gen{"gen", "generate a random Clifford benchmark circuit"}, sched{"schedule", "dump the window schedule"},
        ver{"verify", "differential and statistical self-checks"}, bench{"bench", "phase-timing table"};
    auto add_common = [&](Command &cmd, bool with_word) {
        cmd.num<uint64_t>("--seed", seed);
        if (with_word) cmd.num<unsigned>("--word-size", word_size, word_member("--word-size"));
        cmd.num<unsigned>("--threads", threads);
        cmd.num<int>("--device", device);
    };
    run.positional = &in_path; run.positional_required = true; run.positional_name = "input";
    run.str("--out", out_path);
    run.str("--json", json_path);
    add_common(run, true);
    smp.positional = &in_path; smp.positional_required = true; smp.positional_name = "input";
    smp.num<uint64_t>("--shots", shots, positive<uint64_t>("--shots"));
    smp.str("--format", format, {"text", "binary"});
    smp.str("--out", out_path);
    smp.str("--json", json_path);
    add_common(smp, true);
    gen.num<uint32_t>("--qubits", gen_qubits, positive<uint32_t>("--qubits"));
    gen.num<uint32_t>("--depth", gen_depth, positive<uint32_t>("--depth"));
    gen.num<double>("--measure-prob", measure_prob, unit_range("--measure-prob"));
    gen.str("--out", out_path);
    add_common(gen, false);
    sched.positional = &in_path; sched.positional_required = true; sched.positional_name = "input";
    ver.num<uint32_t>("--n-min", verify.n_min);
    ver.num<uint32_t>("--n-max", verify.n_max);
    ver.num<uint32_t>("--depth-min", verify.depth_min);
    ver.num<uint32_t>("--depth-max", verify.depth_max);
    ver.num<uint32_t>("--trials", verify.trials);
    ver.num<uint64_t>("--seed", verify.seed);
    ver.num<unsigned>("--threads", threads);
    ver.num<int>("--device", device);
    bench.positional = &in_path; bench.positional_name = "input";
    bench.num<uint32_t>("--qubits", gen_qubits);
    bench.num<uint32_t>("--depth", gen_depth);
    bench.num<double>("--measure-prob", measure_prob, unit_range("--measure-prob"));
    bench.num<unsigned>("--reps", reps, positive<unsigned>("--reps"));
    add_common(bench, true);

    Command *cmds[] = {&run, &smp, &gen, &sched, &ver, &bench};
    try {
        if (argc < 2) throw UsageError(106, "A subcommand is required");
        const std::string sub = argv[1];
        if (sub == "-h" || sub == "--help") {
            usage(std::cout);
            return kExitOk;
        }
        Command *cmd = nullptr;
        for (Command *c : cmds)
            if (c->name == sub) cmd = c;
        if (!cmd) throw UsageError(109, "The following argument was not expected: " + sub);
        for (int i = 2; i < argc; ++i)
            if (!std::strcmp(argv[i], "-h") || !std::strcmp(argv[i], "--help")) {
                usage(std::cout);
                return kExitOk;
            }
        parse_command(*cmd, argc, argv, 2);
    } catch (const UsageError &e) {
        std::cerr << e.what() << "\nRun with --help for more information.\n";
        return e.code;
    }

    try {
        if (threads == 0)
            if (const char *env = std::getenv("QUASAR_THREADS")) threads = unsigned(std::strtoul(env, nullptr, 10));
        if (threads != 0) qsr_set_num_threads(threads);
        if (run.parsed) return cmd_run(in_path, seed, device, out_path, json_path);
        if (smp.parsed) return cmd_sample(in_path, shots, seed, word_size, device, out_path, format, json_path);
        if (gen.parsed) {
            CircuitH c;
            check(qsr_generate_random(gen_qubits, gen_depth, seed, measure_prob, &c.p));
            const std::string text = text_of([&](char *b, uint64_t cap, uint64_t *len) {
                return qsr_emit_qasm(c.p, b, cap, len);
            });
            if (out_path.empty()) std::cout.write(text.data(), std::streamsize(text.size()));
            else write_file(out_path, text.data(), text.size());
            return kExitOk;
        }
        if (sched.parsed) {
            CircuitH c;
            load_circuit(in_path, c);
            ScheduleH s;
            check(qsr_schedule_windows(c.p, QSR_SINGLE_SHOT, &s.p));
            const std::string text = text_of([&](char *b, uint64_t cap, uint64_t *len) {
                return qsr_schedule_text(s.p, b, cap, len);
            });
            std::cout.write(text.data(), std::streamsize(text.size()));
            return kExitOk;
        }
        if (ver.parsed) return cmd_verify(verify, device);
        if (bench.parsed) {
            CircuitH c;
            if (in_path.empty()) check(qsr_generate_random(gen_qubits, gen_depth, seed, measure_prob, &c.p));
            else load_circuit(in_path, c);
            return cmd_bench(c.p, seed, reps, device);
        }
    } catch (const std::bad_alloc &) {
        std::cerr << "error: out of memory\n";
        return kExitResourceError;
    } catch (const LibError &e) {
        std::cerr << "error: " << e.what() << "\n";
        return e.status == QSR_OUT_OF_MEMORY ? kExitResourceError : kExitInputError;
    } catch (const std::exception &e) {
        std::cerr << "error: " << e.what() << "\n";
        return kExitInputError;
    }
    return kExitOk;
}
