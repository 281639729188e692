"""OpenQASM reader / writer, schedule text and schedule validator (reference qasm.hpp:29-271,
schedule.hpp:143-249) — CPU tests, no GPU needed.

The first group restates the reference's own cases (test_circuit.cpp:22-78). The rest are
differential against the reference compiled unmodified (oracle/_ref): the same accepted programs
and the same Circuit, and for rejected programs the same QasmError text, line and column, over a
mutation fuzz corpus, large bodies (the parallel parse path) and corrupted schedules.
"""
import random
import re

import numpy as np
import pytest

from oracle.oracle import Oracle, QasmFailure, available

needs_ref = pytest.mark.skipif(not available("reference"), reason="oracle/_ref not built")


@pytest.fixture(scope="module")
def ref():
    return Oracle("reference")


def gates_of(q, a):
    return [q.Gate(int(g["kind"]), int(g["q0"]), int(g["q1"])) for g in a]


# ---- the reference's own cases (test_circuit.cpp) -------------------------------------------

def test_parse_simple_program(q):  # test_circuit.cpp:22-29
    c = q.parse_qasm('OPENQASM 2.0;\ninclude "qelib1.inc";\nqreg q[2];\nh q[0]; cx q[0],q[1];\n')
    assert c.num_qubits == 2 and len(c) == 2
    assert c.gates[0] == q.Gate(q.GateKind.H, 0)
    assert c.gates[1] == q.Gate(q.GateKind.CX, 0, 1)


def test_parse_measure_targets(q):  # test_circuit.cpp:31-37
    c = q.parse_qasm("OPENQASM 2.0;\nqreg q[3];\ncreg c[3];\nmeasure q[1] -> c[2];\nmeasure q[0];\n")
    assert c.gates == [q.Gate(q.GateKind.MEASURE, 1), q.Gate(q.GateKind.MEASURE, 0)]
    assert c.num_clbits == 3


def test_parse_errors_carry_position(q):  # test_circuit.cpp:39-54
    with pytest.raises(q.QasmError) as e:
        q.parse_qasm("OPENQASM 2.0;\nqreg q[1];\nt q[0];\n")
    assert e.value.line == 3 and "unsupported" in str(e.value)
    for bad in ["OPENQASM 2.0;\nqreg q[2];\nh q[5];\n", "OPENQASM 2.0;\nqreg q[2];\nqreg r[2];\n",
                "qreg q[2];\n", "OPENQASM 2.0;\nqreg q[2];\nh q[0]\n",
                "OPENQASM 2.0;\nqreg q[2];\ncx q[1],q[1];\n"]:
        with pytest.raises(q.QasmError):
            q.parse_qasm(bad)


def test_emit_minimal(q):  # test_circuit.cpp:56-66
    c = q.Circuit(1, [q.Gate(q.GateKind.H, 0)])
    assert "h q[0];" in q.emit_qasm(c)
    text = q.emit_qasm(q.Circuit(3, []))
    assert "qreg q[3];" in text and "creg" not in text


def test_round_trip(q):  # test_circuit.cpp:68-78
    for seed in (1, 2, 3, 99):
        c = q.generate_random(100, 100, seed, 0.5)
        assert q.parse_qasm(q.emit_qasm(c)) == c
    c = q.generate_random(100, 100, 7, 0.0)
    text = q.emit_qasm(c)
    assert q.emit_qasm(q.parse_qasm(text)) == text


# ---- differential against the reference ---------------------------------------------------

def ours(q, text):
    try:
        c = q.parse_qasm(text)
        return ("ok", c.num_qubits, c.num_clbits, [(int(g["kind"]), int(g["q0"]), int(g["q1"]))
                                                   for g in c.gate_array])
    except q.QasmError as e:
        return ("err", str(e), e.line, e.column)


def theirs(ref, text):
    try:
        n, ncl, g = ref.parse_qasm(text)
        return ("ok", n, ncl, [(int(x["kind"]), int(x["q0"]), int(x["q1"])) for x in g])
    except QasmFailure as e:
        return ("err", e.msg, e.line, e.column)


BASES = [
    'OPENQASM 2.0;\ninclude "qelib1.inc";\nqreg q[5];\ncreg c[5];\nh q[0];\ncx q[0],q[1];\n'
    "sdg q[2]; iswap q[3],q[4];\nmeasure q[1] -> c[1];\nmeasure q[2];\nswap q[0],q[4];\n",
    "OPENQASM 2.0;\n// a comment; with a semicolon\nqreg qq[3];\n  y qq[2] ;\r\nz   qq[0];cz qq[0] , qq[2];\n"
    "creg m[2];\nmeasure qq[0]->m[1];\n",
    'OPENQASM 3;\ninclude "a;\nb";\nqreg r[2];\ns r[1];\ncy r[1],r[0];\n// tail',
    "OPENQASM 2.0;\n\n\nqreg q[70];\ncreg c[1];\nx q[69];\nmeasure q[69] -> c[0];\nmeasure q[3] -> c[1];\n",
]
ALPHABET = list(";[]->,/\"\n qcregxyzh0123456789_ .\t") + ["measure", "cx", "//", "qreg", "creg", "include"]


def mutate(rng, s):
    for _ in range(rng.randint(1, 3)):
        op = rng.randrange(5)
        i = rng.randrange(len(s) + 1)
        if op == 0 and s:
            s = s[:i] + s[i + 1:]
        elif op == 1:
            s = s[:i] + rng.choice(ALPHABET) + s[i:]
        elif op == 2 and s:
            s = s[:i] + rng.choice(ALPHABET) + s[i + 1:]
        else:
            lines = s.split("\n")
            a, b = rng.randrange(len(lines)), rng.randrange(len(lines))
            if op == 3:
                lines[a], lines[b] = lines[b], lines[a]
            else:
                lines.insert(a, lines[b])
            s = "\n".join(lines)
    return s


@needs_ref
def test_fuzz_matches_reference(q, ref):
    rng = random.Random(2603)
    for base in BASES:
        assert ours(q, base) == theirs(ref, base)
    checked_err = 0
    for i in range(1500):
        t = mutate(rng, BASES[i % len(BASES)])
        a, b = ours(q, t), theirs(ref, t)
        assert a == b, (t, a, b)
        checked_err += a[0] == "err"
    assert checked_err > 300  # the corpus exercises many error paths


@needs_ref
@pytest.mark.parametrize("n,depth,seed,p", [(1, 1, 5, 0.0), (7, 9, 3, 1.0), (64, 20, 8, 0.3), (300, 40, 11, 0.05)])
def test_emit_matches_reference(q, ref, n, depth, seed, p):
    c = q.generate_random(n, depth, seed, p)
    text = q.emit_qasm(c)
    assert text == ref.emit_qasm(n, c.gate_array)
    assert ours(q, text) == theirs(ref, text)


def big_program(q):
    c = q.generate_random(3000, 300, 17, 0.02)
    return c, q.emit_qasm(c)  # ~ 9e5 gates, > 8 MB: parsed in parallel pieces


@needs_ref
def test_large_body_parallel_parse(q, ref):
    c, text = big_program(q)
    assert len(text) > (8 << 20)
    assert q.parse_qasm(text) == c
    # Statements split across lines, comments with ';' and CRLF line ends.
    lines = text.split("\n")
    for i in range(5000, len(lines) - 10, 9973):
        lines[i] = lines[i].replace(" ", "\n  ", 1) + " // x; y;\r"
    t2 = "\n".join(lines)
    assert ours(q, t2) == theirs(ref, t2)


@needs_ref
@pytest.mark.parametrize("kind", ["late_error", "late_creg", "late_include", "late_qreg", "unterminated"])
def test_large_body_fallbacks(q, ref, kind):
    _, text = big_program(q)
    lines = text.split("\n")
    at = len(lines) * 7 // 8
    if kind == "late_error":
        lines[at] = "t q[0];"
    elif kind == "late_creg":
        lines[at] = "creg d[9]; measure q[5] -> d[8];"
    elif kind == "late_include":
        lines[at] = 'include "x;\nh q[0];\n";'
    elif kind == "late_qreg":
        lines[at] = "qreg r[2];"
    else:
        lines[at] = 'include "never closed;'
    t = "\n".join(lines)
    a, b = ours(q, t), theirs(ref, t)
    assert a[0] == b[0] and a[1:] == b[1:]


@needs_ref
@pytest.mark.parametrize("n,depth,seed,p,mode", [(5, 10, 1, 1.0, 0), (40, 30, 2, 0.5, 0), (40, 30, 2, 0.5, 1),
                                                  (200, 50, 3, 0.1, 0), (1, 4, 9, 1.0, 1)])
def test_schedule_text_matches_reference(q, ref, n, depth, seed, p, mode):
    c = q.generate_random(n, depth, seed, p)
    s = q.schedule_windows(c, q.ScheduleMode(mode))
    assert q.schedule_to_text(s) == ref.schedule_text(n, c.gate_array, mode)
    assert q.validate_schedule(c, s) == "valid"


def corrupt(rng, windows):
    """Random structural damage to a schedule (list of (is_meas, [gates]))."""
    w = [(m, list(g)) for m, g in windows]
    op = rng.randrange(7)
    a = rng.randrange(len(w))
    b = rng.randrange(len(w))
    if op == 0 and w[a][1]:  # move one gate to another window
        g = w[a][1].pop(rng.randrange(len(w[a][1])))
        w[b][1].insert(rng.randrange(len(w[b][1]) + 1), g)
    elif op == 1:  # swap windows
        w[a], w[b] = w[b], w[a]
    elif op == 2 and w[a][1]:  # drop a gate
        w[a][1].pop(rng.randrange(len(w[a][1])))
    elif op == 3 and w[a][1]:  # duplicate a gate
        w[a][1].append(w[a][1][0])
    elif op == 4:  # empty window
        w.insert(a, (w[a][0], []))
    elif op == 5:  # flip the measurement flag
        w[a] = (not w[a][0], w[a][1])
    elif op == 6 and len(w) > 1:  # merge two windows
        lo, hi = min(a, b), max(a, b)
        if lo != hi:
            w[lo] = (w[lo][0], w[lo][1] + w[hi][1])
            del w[hi]
    return w


@needs_ref
def test_validate_schedule_matches_reference(q, ref):
    rng = random.Random(7)
    seen = set()
    for trial in range(300):
        n = rng.choice([3, 6, 12])
        c = q.generate_random(n, rng.randint(2, 8), trial, rng.choice([0.0, 0.5, 1.0]))
        s = q.schedule_windows(c)
        wins = [(w.is_measurement, list(w.gates)) for w in s.windows]
        bad = corrupt(rng, wins)
        bad = [q.Window(g, m) for m, g in bad]
        sb = q.Schedule(bad)
        sg, off, fl = sb.arrays()
        want = ref.validate_schedule(n, c.gate_array, sg, off, fl)
        got = q.validate_schedule(c, sb)
        assert got == want, (trial, got, want)
        seen.add(re.sub(r"\d+", "#", want))
    assert len(seen) >= 6, seen  # several distinct violation kinds were exercised


def test_num_threads_roundtrip(q):
    q.set_num_threads(3)
    try:
        assert q._lib.lib.qsr_get_num_threads() == 3
        c = q.generate_random(50, 20, 1, 0.5)
        assert q.parse_qasm(q.emit_qasm(c)) == c
    finally:
        q.set_num_threads(0)


def test_text_output_convention(q):
    """qsr.h text outputs: NULL buffer -> size query; a short buffer is rejected with the size set."""
    import ctypes as C
    from paper_2603_14641_b200 import _lib
    c = q.generate_random(20, 5, 2, 0.5)
    n = C.c_uint64()
    _lib.check(_lib.lib.qsr_emit_qasm(c._h, None, 0, C.byref(n)))
    need = n.value
    assert need == len(q.emit_qasm(c).encode())
    small = C.create_string_buffer(need - 1)
    st = _lib.lib.qsr_emit_qasm(c._h, small, need - 1, C.byref(n))
    assert st == _lib.INVALID_ARGUMENT and n.value == need
    assert b"too small" in _lib.lib.qsr_last_error()


def test_qasm_error_struct_and_status(q):
    import ctypes as C
    from paper_2603_14641_b200 import _lib
    h, err = C.c_void_p(), _lib.QasmError_t()
    text = b"OPENQASM 2.0;\nqreg q[2];\n  cx q[0],q[0];\n"
    st = _lib.lib.qsr_parse_qasm(text, len(text), C.byref(h), C.byref(err))
    assert st == _lib.PARSE_ERROR and (err.line, err.column) == (3, 15)
    assert _lib.lib.qsr_last_error().decode() == "qasm:3:15: two-qubit gate with identical operands"
