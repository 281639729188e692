"""CPU tests of the product's host side (no GPU needed): C-ABI symbols, Philox, the circuit
generator and the O(G) scheduler against the oracle and the reference's golden vectors."""
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def test_every_declared_symbol_is_exported():
    from paper_2603_14641_b200 import _lib
    decl = set(re.findall(r"\b(qsr_[a-z0-9_]+)\s*\(", (ROOT / "include" / "qsr.h").read_text()))
    assert decl, "no declarations parsed"
    for name in sorted(decl):
        assert hasattr(_lib.lib, name), f"{name} declared in include/qsr.h but not exported"
    assert decl == set(_lib.SIGNATURES), sorted(decl ^ set(_lib.SIGNATURES))
    assert _lib.lib.qsr_abi_version() == 1


def test_philox_known_answers(q):
    # test_rng.cpp:24-37 (Random123 published vectors)
    assert q.Philox.block([0, 0, 0, 0], [0, 0]) == (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)
    f = 0xFFFFFFFF
    assert q.Philox.block([f] * 4, [f, f]) == (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)
    assert q.Philox.block([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0]) == \
        (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)


def test_philox_words_match_oracle(q, oracles):
    for o in oracles:
        for args in [(0, 0, 0, 0), (7, 0, 0, 123), (2**64 - 1, 1, 5, 2**40 + 3), (42, 2, 0, 99)]:
            assert q.Philox.word_at(*args) == o.philox_word(*args)


@pytest.mark.parametrize("n,depth,seed,p", [(1, 1, 0, 0.0), (2, 5, 1, 1.0), (17, 9, 3, 0.4),
                                            (64, 3, 42, 0.5), (1000, 100, 42, 1.0), (333, 7, 9, 0.01)])
def test_generate_random_matches_oracle(q, oracles, n, depth, seed, p):
    c = q.generate_random(n, depth, seed, p)
    for o in oracles:
        np.testing.assert_array_equal(c.gate_array, o.generate_random(n, depth, seed, p))


@pytest.mark.parametrize("threads", [2, 3, 8])
@pytest.mark.parametrize("n,depth,seed,p", [(5001, 300, 3, 0.3), (4096, 257, 9, 1.0), (4097, 256, 11, 0.5)])
def test_parallel_generator_matches_oracle(q, oracles, threads, n, depth, seed, p):
    """Sizes that take the multi-threaded generator (Philox words drawn ahead on workers, kind
    scan by chunk sums, layers emitted in place by several threads)."""
    q.set_num_threads(threads)
    try:
        c = q.generate_random(n, depth, seed, p)
    finally:
        q.set_num_threads(0)
    np.testing.assert_array_equal(c.gate_array, oracles[0].generate_random(n, depth, seed, p))


def test_generator_errors(q):
    with pytest.raises(q.InvalidArgument):
        q.generate_random(0, 5, 1, 0.5)
    with pytest.raises(q.InvalidArgument):
        q.generate_random(5, 0, 1, 0.5)
    with pytest.raises(q.InvalidArgument):
        q.generate_random(5, 5, 1, 1.5)


def _sched_eq(q, c, o, mode):
    s = q.schedule_windows(c, mode)
    g, off, fl = s.arrays()
    rg, roff, rfl = o.schedule(c.num_qubits, c.gate_array, int(mode))
    np.testing.assert_array_equal(off, roff)
    np.testing.assert_array_equal(fl, rfl)
    np.testing.assert_array_equal(g, rg)


def test_schedule_five_wire_golden(q, oracles):
    # test_schedule.cpp:28-55: 5 windows of sizes 3, 2 (M), 3, 2, 2
    G = q.GateKind
    c = q.Circuit(5, [(G.H, 0), (G.MEASURE, 3), (G.MEASURE, 1), (G.S, 4), (G.S, 0), (G.S, 2), (G.S, 3),
                      (G.CX, 0, 2), (G.CX, 3, 4), (G.H, 1), (G.H, 2), (G.S, 3)])
    s = q.schedule_windows(c)
    ws = s.windows
    assert [len(w.gates) for w in ws] == [3, 2, 3, 2, 2]
    assert [w.is_measurement for w in ws] == [False, True, False, False, False]
    assert ws[0].gates == [q.Gate(G.H, 0), q.Gate(G.S, 4), q.Gate(G.S, 2)]
    assert ws[1].gates == [q.Gate(G.MEASURE, 3), q.Gate(G.MEASURE, 1)]
    for o in oracles:
        _sched_eq(q, c, o, 0)


def test_schedule_record_order_quirk(q):
    # [H0, H0, M0, M1] -> U{h0} M{m1} U{h0} M{m0}
    G = q.GateKind
    c = q.Circuit(2, [(G.H, 0), (G.H, 0), (G.MEASURE, 0), (G.MEASURE, 1)])
    ws = q.schedule_windows(c).windows
    assert [(w.is_measurement, [g.q0 for g in w.gates]) for w in ws] == \
        [(False, [0]), (True, [1]), (False, [0]), (True, [0])]


def test_schedule_matches_oracle_sweep(q, oracles):
    rng = np.random.default_rng(2024)
    for trial in range(300):
        n = int(rng.integers(1, 40))
        ng = int(rng.integers(0, 200))
        kinds = rng.integers(0, 14, ng)
        gates = []
        for kd in kinds:
            kd = 11 if kd >= 11 else int(kd)  # 3/14 measurements
            a = int(rng.integers(0, n))
            if kd in (6, 7, 8, 9, 10):
                if n < 2:
                    kd = 3
                else:
                    b = int(rng.integers(0, n - 1))
                    b = b + 1 if b >= a else b
                    gates.append((kd, a, b))
                    continue
            gates.append((kd, a))
        c = q.Circuit(n, gates)
        for o in oracles:
            for mode in (0, 1):
                _sched_eq(q, c, o, mode)


@pytest.mark.parametrize("seed", range(20))
def test_schedule_matches_oracle_generated(q, oracles, seed):
    n = 1 + (seed * 13) % 64
    c = q.generate_random(n, 1 + (seed * 7) % 20, seed, 0.4)
    for o in oracles:
        _sched_eq(q, c, o, 0)


def test_circuit_validation(q):
    with pytest.raises(q.OutOfRange):
        q.Circuit(2, [(3, 2)])
    with pytest.raises(q.InvalidArgument):
        q.Circuit(3, [(6, 1, 1)])


def test_chunk_planner_matches_scheduler(tmp_path):
    """The streaming driver's chunk planner (csrc/stream_plan.hpp), host only: over 400 generated
    and hand-made circuits with random chunk splits, its buckets in key order are the one-shot
    scheduler's windows gate for gate, and both reject the same circuits (tests/cpp/plan_check.cpp)."""
    import shutil
    import subprocess
    if shutil.which("g++") is None:
        pytest.skip("g++ not available")
    root = Path(__file__).resolve().parents[1]
    exe = tmp_path / "plan_check"
    subprocess.run(["g++", "-O2", "-std=c++17", "-I", str(root / "include"), "-I",
                    str(root / "paper_2603_14641_b200" / "csrc"), str(root / "tests" / "cpp" / "plan_check.cpp"),
                    str(root / "paper_2603_14641_b200" / "csrc" / "host_circuit.cpp"), "-pthread", "-o", str(exe)],
                   check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0 and out.stdout.startswith("ok "), out.stdout + out.stderr
