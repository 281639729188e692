// OpenQASM 2.0 subset reader / writer (reference qasm.hpp:29-271) and the schedule text dump /
// validator (schedule.hpp:143-249): the formats either side of the hot path.
//
// The grammar, the accepted programs, the produced Circuit and every error (reason text, line,
// column) are the reference's. Column = characters consumed since the last newline eaten as
// whitespace + 1, exactly as the reference lexer counts (its quoted-string scan does not reset the
// column on a newline, and neither does this one).
//
// Scale: a c5 program is ~2.2 GB of text. After the header statements (OPENQASM / include / qreg /
// creg) are read in order, the body is split at line ends that follow a ';' and the pieces are
// parsed on all host threads with the register state of the header. A piece that sees anything
// but gate / measure statements (a late include / qreg / creg, a string literal, any error) aborts
// the parallel attempt and the body is parsed sequentially from the same point, so errors carry
// the exact reference position. Emission is two parallel passes (sizes, then bytes).
#include <algorithm>
#include <atomic>
#include <cstring>
#include <string_view>

#include "host.hpp"

namespace qsr {

namespace {

inline bool is_space(char c) {
    return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r';
}
inline bool is_digit(char c) { return c >= '0' && c <= '9'; }
inline bool is_ident(char c) {
    return is_digit(c) || (c >= 'a' && c <= 'z') || (c >= 'A' && c <= 'Z') || c == '_';
}

const char *const kNames[12] = {"x",  "y",  "z",  "h",    "s",     "sdg",
                                "cx", "cy", "cz", "swap", "iswap", "measure"};
inline std::string_view name_of(uint8_t k) { return k < 12 ? kNames[k] : "?"; }

// qasm.hpp:149-155 over kUnitaryKinds (circuit.hpp:81-83); -1 = not a unitary gate name.
inline int unitary_kind(std::string_view s) {
    switch (s.size()) {
    case 1:
        switch (s[0]) {
        case 'x': return QSR_X;
        case 'y': return QSR_Y;
        case 'z': return QSR_Z;
        case 'h': return QSR_H;
        case 's': return QSR_S;
        }
        return -1;
    case 2:
        if (s[0] != 'c') return -1;
        return s[1] == 'x' ? QSR_CX : s[1] == 'y' ? QSR_CY : s[1] == 'z' ? QSR_CZ : -1;
    case 3: return s == "sdg" ? QSR_SDG : -1;
    case 4: return s == "swap" ? QSR_SWAP : -1;
    case 5: return s == "iswap" ? QSR_ISWAP : -1;
    }
    return -1;
}

struct Abort {}; // a body piece could not be parsed on its own

// Register state after the header (qasm.hpp:162-164).
struct Regs {
    bool have_qreg = false;
    std::string_view qreg, creg; // creg empty = none declared
    uint32_t num_qubits = 0, num_clbits = 0;
};

// Piece = true: any failure or header statement throws Abort (the caller re-parses sequentially).
template <bool Piece>
struct Lexer {
    const char *p, *e;
    const char *ls; // first character of the current line
    int line = 1;

    [[noreturn]] void fail(const std::string &m) const {
        if constexpr (Piece) throw Abort{};
        else throw QasmFailure(m, line, int(p - ls) + 1);
    }
    void skip_space() {
        while (p < e) {
            const char c = *p;
            if (c == '\n') {
                ++line;
                ls = ++p;
            } else if (is_space(c)) {
                ++p;
            } else if (c == '/' && p + 1 < e && p[1] == '/') {
                while (p < e && *p != '\n') ++p;
            } else {
                break;
            }
        }
    }
    bool eof() {
        skip_space();
        return p >= e;
    }
    char peek() const { return p < e ? *p : '\0'; }
    void expect(char c) {
        skip_space();
        if (peek() != c) fail(std::string("expected '") + c + "'");
        ++p;
    }
    bool accept(char c) {
        skip_space();
        if (peek() == c) {
            ++p;
            return true;
        }
        return false;
    }
    std::string_view ident() {
        skip_space();
        const char *s = p;
        while (p < e && is_ident(*p)) ++p;
        if (p == s) fail("expected identifier");
        return std::string_view(s, size_t(p - s));
    }
    uint64_t number() {
        skip_space();
        if (!is_digit(peek())) fail("expected number");
        uint64_t v = 0;
        while (p < e && is_digit(*p)) v = v * 10 + uint64_t(*p++ - '0'); // wraps like the reference
        return v;
    }
    void version() {
        number();
        if (accept('.')) number();
    }
    void quoted() {
        skip_space();
        if (peek() != '"') fail("expected string literal");
        ++p;
        while (p < e && *p != '"') ++p;
        if (p >= e) fail("unterminated string literal");
        ++p;
    }
};

template <bool Piece>
uint32_t qubit_operand(Lexer<Piece> &L, const Regs &r) {
    std::string_view reg = L.ident();
    if (!r.have_qreg || reg != r.qreg) L.fail("unknown quantum register '" + std::string(reg) + "'");
    L.expect('[');
    const uint64_t idx = L.number();
    L.expect(']');
    if (idx >= r.num_qubits) L.fail("qubit index " + std::to_string(idx) + " out of range");
    return uint32_t(idx);
}

// One gate or measure statement whose keyword `kw` has been read (qasm.hpp:211-244). Returns
// false if `kw` is not one.
template <bool Piece>
bool gate_statement(Lexer<Piece> &L, const Regs &r, std::string_view kw, GateVec &out) {
    if (kw == "measure") {
        if (!r.have_qreg) L.fail("measure before qreg declaration");
        const uint32_t q = qubit_operand(L, r);
        L.skip_space();
        if (L.accept('-')) {
            L.expect('>');
            std::string_view reg = L.ident();
            if (r.creg.empty() || reg != r.creg)
                L.fail("unknown classical register '" + std::string(reg) + "'");
            L.expect('[');
            const uint64_t idx = L.number();
            L.expect(']');
            if (idx >= r.num_clbits) L.fail("classical index " + std::to_string(idx) + " out of range");
        }
        L.expect(';');
        out.push_back(qsr_gate{QSR_MEASURE, q, 0});
        return true;
    }
    const int k = unitary_kind(kw);
    if (k < 0) return false;
    if (!r.have_qreg) L.fail("gate before qreg declaration");
    qsr_gate g{uint8_t(k), 0, 0};
    g.q0 = qubit_operand(L, r);
    if (gate_arity(uint8_t(k)) == 2) {
        L.expect(',');
        g.q1 = qubit_operand(L, r);
        if (g.q0 == g.q1) L.fail("two-qubit gate with identical operands");
    }
    L.expect(';');
    out.push_back(g);
    return true;
}

// Fast path for the canonical statement shapes emit_qasm writes ("h q[3];", "cx q[0],q[1];",
// "measure q[5] -> c[5];", no comments or line breaks inside): recognised without the general
// lexer and with the same checks; anything else (or any error) returns false with nothing
// consumed, and the general path takes the statement (so error positions stay exact).
template <bool Piece>
bool fast_statement(Lexer<Piece> &L, const Regs &r, GateVec &out) {
    if (!r.have_qreg) return false;
    const char *p = L.p, *const e = L.e;
    const char *s = p;
    while (p < e && *p >= 'a' && *p <= 'z') ++p;
    if (p >= e || *p != ' ') return false;
    const std::string_view name(s, size_t(p - s));
    const int k = unitary_kind(name);
    const bool meas = k < 0 && name == "measure";
    if (k < 0 && !meas) return false;
    ++p;
    auto index = [&](std::string_view reg, uint64_t bound, uint32_t &out_idx) {
        if (size_t(e - p) < reg.size() + 3 || std::memcmp(p, reg.data(), reg.size()) != 0) return false;
        p += reg.size();
        if (*p != '[') return false;
        ++p;
        uint64_t v = 0;
        int nd = 0;
        while (p < e && is_digit(*p)) {
            v = v * 10 + uint64_t(*p++ - '0');
            if (++nd > 18) return false;
        }
        if (nd == 0 || p >= e || *p != ']' || v >= bound) return false;
        ++p;
        out_idx = uint32_t(v);
        return true;
    };
    qsr_gate g{uint8_t(meas ? QSR_MEASURE : k), 0, 0};
    if (!index(r.qreg, r.num_qubits, g.q0)) return false;
    if (meas) {
        if (size_t(e - p) >= 4 && p[0] == ' ' && p[1] == '-' && p[2] == '>' && p[3] == ' ') {
            p += 4;
            uint32_t cl = 0;
            if (r.creg.empty() || !index(r.creg, r.num_clbits, cl)) return false;
        }
    } else if (gate_arity(uint8_t(k)) == 2) {
        if (p >= e || *p != ',') return false;
        ++p;
        if (!index(r.qreg, r.num_qubits, g.q1) || g.q0 == g.q1) return false;
    }
    if (p >= e || *p != ';') return false;
    out.push_back(g);
    L.p = p + 1;
    return true;
}

// Header statements (qasm.hpp:190-210). Returns false if `kw` is not one.
bool header_statement(Lexer<false> &L, Regs &r, std::string_view kw) {
    if (kw == "include") {
        L.quoted();
        L.expect(';');
    } else if (kw == "qreg") {
        if (r.have_qreg) L.fail("multiple quantum registers are not supported");
        r.qreg = L.ident();
        L.expect('[');
        const uint64_t n = L.number();
        L.expect(']');
        L.expect(';');
        if (n == 0) L.fail("quantum register must have at least one qubit");
        r.num_qubits = uint32_t(n);
        r.have_qreg = true;
    } else if (kw == "creg") {
        r.creg = L.ident();
        L.expect('[');
        r.num_clbits = uint32_t(L.number());
        L.expect(']');
        L.expect(';');
    } else {
        return false;
    }
    return true;
}

// Piece boundaries: just after a '\n' whose line's last non-blank character before it is ';'.
const char *next_boundary(const char *p, const char *lo, const char *e) {
    while (p < e) {
        const char *nl = static_cast<const char *>(memchr(p, '\n', size_t(e - p)));
        if (!nl) return e;
        const char *b = nl;
        while (b > lo && (b[-1] == ' ' || b[-1] == '\t' || b[-1] == '\r')) --b;
        if (b > lo && b[-1] == ';') return nl + 1;
        p = nl + 1;
    }
    return e;
}

// Parallel body parse; false = some piece aborted (nothing of `out` is kept then).
bool parse_body_parallel(const char *b, const char *e, const Regs &r, GateVec &out) {
    const uint64_t len = uint64_t(e - b);
    const unsigned T = std::max(1u, std::min<unsigned>(host_threads(), unsigned(len >> 22)));
    if (T < 2) return false;
    std::vector<const char *> cut(T + 1);
    cut[0] = b;
    cut[T] = e;
    for (unsigned t = 1; t < T; ++t)
        cut[t] = std::max(cut[t - 1], next_boundary(b + len * t / T, b, e));
    std::vector<GateVec> part(T);
    std::atomic<bool> bad{false};
    parallel_chunks(T, T, [&](unsigned, uint64_t t0, uint64_t t1) {
        for (uint64_t t = t0; t < t1 && !bad.load(std::memory_order_relaxed); ++t) {
            try {
                Lexer<true> L{cut[t], cut[t + 1], cut[t]};
                auto &v = part[t];
                v.reserve(size_t(cut[t + 1] - cut[t]) / 14 + 16);
                while (!L.eof()) {
                    if (fast_statement(L, r, v)) continue;
                    std::string_view kw = L.ident();
                    if (!gate_statement(L, r, kw, v)) throw Abort{};
                }
            } catch (const Abort &) {
                bad = true;
            }
        }
    });
    if (bad) return false;
    std::vector<uint64_t> off(T + 1, 0);
    for (unsigned t = 0; t < T; ++t) off[t + 1] = off[t] + part[t].size();
    const uint64_t base = out.size();
    out.resize(base + off[T]);
    parallel_chunks(T, T, [&](unsigned, uint64_t t0, uint64_t t1) {
        for (uint64_t t = t0; t < t1; ++t) {
            if (!part[t].empty())
                std::memcpy(out.data() + base + off[t], part[t].data(), part[t].size() * sizeof(qsr_gate));
            GateVec().swap(part[t]);
        }
    });
    return true;
}

// ---- writers -------------------------------------------------------------------------

inline unsigned digits(uint32_t v) {
    unsigned d = 1;
    while (v >= 10) { v /= 10; ++d; }
    return d;
}
inline char *put_u32(char *o, uint32_t v) {
    const unsigned d = digits(v);
    for (unsigned i = d; i-- > 0; v /= 10) o[i] = char('0' + v % 10);
    return o + d;
}
inline char *put(char *o, std::string_view s) {
    std::memcpy(o, s.data(), s.size());
    return o + s.size();
}

// emit_qasm line of one gate (qasm.hpp:261-269).
inline uint64_t qasm_line_size(const qsr_gate &g) {
    if (g.kind == QSR_MEASURE) return 20 + 2 * uint64_t(digits(g.q0)); // "measure q[A] -> c[A];\n"
    if (gate_arity(g.kind) == 1) return name_of(g.kind).size() + 6 + digits(g.q0);
    return name_of(g.kind).size() + 10 + digits(g.q0) + digits(g.q1);
}
inline char *qasm_line(char *o, const qsr_gate &g) {
    if (g.kind == QSR_MEASURE) {
        o = put(o, "measure q[");
        o = put_u32(o, g.q0);
        o = put(o, "] -> c[");
        o = put_u32(o, g.q0);
        return put(o, "];\n");
    }
    o = put(o, name_of(g.kind));
    o = put(o, " q[");
    o = put_u32(o, g.q0);
    if (gate_arity(g.kind) == 2) {
        o = put(o, "],q[");
        o = put_u32(o, g.q1);
    }
    return put(o, "];\n");
}

// schedule_to_text item of one gate (schedule.hpp:240-245): " name(q0[,q1])".
inline uint64_t sched_item_size(const qsr_gate &g) {
    return name_of(g.kind).size() + 3 + digits(g.q0) + (gate_arity(g.kind) == 2 ? 1 + digits(g.q1) : 0);
}
inline char *sched_item(char *o, const qsr_gate &g) {
    *o++ = ' ';
    o = put(o, name_of(g.kind));
    *o++ = '(';
    o = put_u32(o, g.q0);
    if (gate_arity(g.kind) == 2) {
        *o++ = ',';
        o = put_u32(o, g.q1);
    }
    *o++ = ')';
    return o;
}
inline uint64_t digits64(uint64_t v) {
    uint64_t d = 1;
    while (v >= 10) { v /= 10; ++d; }
    return d;
}

unsigned text_threads(uint64_t items) {
    return std::max(1u, std::min<unsigned>(host_threads(), unsigned(items >> 18) + 1));
}

} // namespace

Circuit parse_qasm(const char *text, uint64_t len) {
    Lexer<false> L{text, text + len, text};
    Regs r;
    Circuit c;
    {
        std::string_view kw = L.ident();
        if (kw != "OPENQASM") L.fail("expected OPENQASM header");
        L.version();
        L.expect(';');
    }
    // Header statements in order; stop before the first body statement.
    while (!L.eof()) {
        const Lexer<false> save = L;
        std::string_view kw = L.ident();
        if (!header_statement(L, r, kw)) {
            L = save;
            break;
        }
    }
    c.num_qubits = r.num_qubits;
    c.num_clbits = r.num_clbits;
    if (!L.eof() && r.have_qreg && uint64_t(L.e - L.p) >= (uint64_t(8) << 20) &&
        parse_body_parallel(L.p, L.e, r, c.gates)) {
        return c;
    }
    // Sequential body (also the exact-error path when a piece aborted).
    c.gates.reserve(size_t(L.e - L.p) / 14 + 16);
    while (!L.eof()) {
        if (fast_statement(L, r, c.gates)) continue;
        std::string_view kw = L.ident();
        if (header_statement(L, r, kw)) {
            c.num_qubits = r.num_qubits;
            c.num_clbits = r.num_clbits;
            continue;
        }
        if (!gate_statement(L, r, kw, c.gates)) L.fail("unsupported gate or statement '" + std::string(kw) + "'");
    }
    if (!r.have_qreg) L.fail("missing quantum register declaration");
    return c;
}

uint64_t emit_qasm(const Circuit &c, char *out) {
    const uint64_t G = c.gates.size();
    const unsigned T = text_threads(G);
    std::vector<uint64_t> size(T + 1, 0), meas(T, 0);
    parallel_chunks(G, T, [&](unsigned t, uint64_t b, uint64_t e) {
        uint64_t s = 0, m = 0;
        for (uint64_t i = b; i < e; ++i) {
            s += qasm_line_size(c.gates[i]);
            m += c.gates[i].kind == QSR_MEASURE;
        }
        size[t + 1] = s;
        meas[t] = m;
    });
    uint64_t nmeas = 0;
    for (unsigned t = 0; t < T; ++t) nmeas += meas[t];
    // Header (qasm.hpp:256-260).
    std::string head = "OPENQASM 2.0;\ninclude \"qelib1.inc\";\nqreg q[" + std::to_string(c.num_qubits) + "];\n";
    if (nmeas > 0) head += "creg c[" + std::to_string(c.num_qubits) + "];\n";
    size[0] = head.size();
    for (unsigned t = 0; t < T; ++t) size[t + 1] += size[t];
    if (!out) return size[T];
    std::memcpy(out, head.data(), head.size());
    parallel_chunks(G, T, [&](unsigned t, uint64_t b, uint64_t e) {
        char *o = out + size[t];
        for (uint64_t i = b; i < e; ++i) o = qasm_line(o, c.gates[i]);
    });
    return size[T];
}

uint64_t schedule_text(const Schedule &s, char *out) {
    // "W<wi> M:" / "W<wi> U:", then one item per gate, then '\n' (schedule.hpp:235-249).
    // Threads take contiguous window ranges of about equal gate counts.
    const uint64_t W = s.num_windows(), G = s.gates.size();
    const unsigned T = W ? std::min<unsigned>(text_threads(G), unsigned(std::min<uint64_t>(W, 1u << 16))) : 1;
    std::vector<uint64_t> wcut(T + 1, W);
    wcut[0] = 0;
    for (unsigned t = 1; t < T; ++t) {
        const uint64_t target = G * t / T;
        wcut[t] = std::max(wcut[t - 1],
                           uint64_t(std::lower_bound(s.offsets.begin(), s.offsets.end() - 1, target) -
                                    s.offsets.begin()));
    }
    auto win_size = [&](uint64_t w) {
        uint64_t z = 1 + digits64(w) + 3 + 1;
        for (uint64_t i = s.offsets[w]; i < s.offsets[w + 1]; ++i) z += sched_item_size(s.gates[i]);
        return z;
    };
    std::vector<uint64_t> size(T + 1, 0);
    parallel_chunks(T, T, [&](unsigned, uint64_t t0, uint64_t t1) {
        for (uint64_t t = t0; t < t1; ++t) {
            uint64_t z = 0;
            for (uint64_t w = wcut[t]; w < wcut[t + 1]; ++w) z += win_size(w);
            size[t + 1] = z;
        }
    });
    for (unsigned t = 0; t < T; ++t) size[t + 1] += size[t];
    if (!out) return size[T];
    parallel_chunks(T, T, [&](unsigned, uint64_t t0, uint64_t t1) {
        for (uint64_t t = t0; t < t1; ++t) {
            char *o = out + size[t];
            for (uint64_t w = wcut[t]; w < wcut[t + 1]; ++w) {
                *o++ = 'W';
                const std::string ws = std::to_string(w);
                o = put(o, ws);
                o = put(o, s.is_meas[w] ? " M:" : " U:");
                for (uint64_t i = s.offsets[w]; i < s.offsets[w + 1]; ++i) o = sched_item(o, s.gates[i]);
                *o++ = '\n';
            }
        }
    });
    return size[T];
}

// validate_schedule (schedule.hpp:143-233): the same checks in the same order, so the first
// violation reported is the reference's. O(G + n + W): per-window stamps instead of cleared
// busy vectors, wire sequences in CSR form, and the maximality scan reduced to "is there a
// unitary window in [earliest, wi)" (no window in that range touches either wire of the gate,
// because earliest is one past the last window that did).
std::string validate_schedule(const Circuit &c, const Schedule &s) {
    const uint64_t n = c.num_qubits, W = s.num_windows();
    auto gate_of = [&](uint64_t i) -> const qsr_gate & { return s.gates[i]; };
    {   // (a) window-internal structure
        std::vector<uint64_t> stamp(n, 0);
        for (uint64_t wi = 0; wi < W; ++wi) {
            const uint64_t b = s.offsets[wi], e = s.offsets[wi + 1];
            if (b == e) return "window " + std::to_string(wi) + " is empty";
            for (uint64_t i = b; i < e; ++i) {
                const qsr_gate &g = gate_of(i);
                const bool two = gate_arity(g.kind) == 2;
                if (bool(s.is_meas[wi]) != (g.kind == QSR_MEASURE))
                    return "window " + std::to_string(wi) + " mixes measurements and unitaries";
                if (g.q0 >= n || (two && g.q1 >= n))
                    return "window " + std::to_string(wi) + " has an operand out of range";
                if (stamp[g.q0] == wi + 1 || (two && stamp[g.q1] == wi + 1))
                    return "window " + std::to_string(wi) + " has overlapping operands";
                stamp[g.q0] = wi + 1;
                if (two) stamp[g.q1] = wi + 1;
            }
        }
    }
    // (b, c) per-wire order and conservation
    if (s.gates.size() != c.gates.size()) return "gate count mismatch";
    std::vector<uint64_t> start(n + 1, 0);
    for (const qsr_gate &g : c.gates) {
        ++start[g.q0 + 1];
        if (gate_arity(g.kind) == 2) ++start[g.q1 + 1];
    }
    for (uint64_t q = 0; q < n; ++q) start[q + 1] += start[q];
    std::vector<uint64_t> seq(start[n]), cursor(start.begin(), start.end() - 1);
    for (uint64_t i = 0; i < c.gates.size(); ++i) {
        const qsr_gate &g = c.gates[i];
        seq[cursor[g.q0]++] = i;
        if (gate_arity(g.kind) == 2) seq[cursor[g.q1]++] = i;
    }
    std::copy(start.begin(), start.end() - 1, cursor.begin());
    auto same = [](const qsr_gate &a, const qsr_gate &b) {
        return a.kind == b.kind && a.q0 == b.q0 && (gate_arity(a.kind) == 1 || a.q1 == b.q1);
    };
    for (uint64_t wi = 0; wi < W; ++wi)
        for (uint64_t i = s.offsets[wi]; i < s.offsets[wi + 1]; ++i) {
            const qsr_gate &g = gate_of(i);
            for (int op = 0; op < gate_arity(g.kind); ++op) {
                const uint32_t q = op == 0 ? g.q0 : g.q1;
                if (cursor[q] >= start[q + 1] || !same(c.gates[seq[cursor[q]]], g))
                    return "wire order violated on qubit " + std::to_string(q) + " at window " +
                           std::to_string(wi);
                ++cursor[q];
            }
        }
    for (uint64_t q = 0; q < n; ++q)
        if (cursor[q] != start[q + 1]) return "wire " + std::to_string(q) + " not fully scheduled";
    // (d) maximality
    std::vector<uint64_t> next_unitary(W + 1, W);
    for (uint64_t w = W; w-- > 0;) next_unitary[w] = s.is_meas[w] ? next_unitary[w + 1] : w;
    const uint64_t kNone = ~uint64_t(0);
    std::vector<uint64_t> last(n, kNone);
    for (uint64_t wi = 0; wi < W; ++wi) {
        const uint64_t b = s.offsets[wi], e = s.offsets[wi + 1];
        for (uint64_t i = b; i < e; ++i) {
            const qsr_gate &g = gate_of(i);
            if (g.kind == QSR_MEASURE) continue;
            uint64_t earliest = last[g.q0] != kNone ? last[g.q0] + 1 : 0;
            if (gate_arity(g.kind) == 2 && last[g.q1] != kNone) earliest = std::max(earliest, last[g.q1] + 1);
            if (earliest < wi && next_unitary[earliest] < wi)
                return "gate in window " + std::to_string(wi) + " could have joined window " +
                       std::to_string(next_unitary[earliest]);
        }
        for (uint64_t i = b; i < e; ++i) {
            const qsr_gate &g = gate_of(i);
            last[g.q0] = wi;
            if (gate_arity(g.kind) == 2) last[g.q1] = wi;
        }
    }
    return "valid";
}

} // namespace qsr
