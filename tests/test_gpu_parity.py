"""GPU parity: libqsr (CUDA, through the C ABI) vs the CPU oracle on the same inputs.

Bit-exact equality of raw storage (x, z, s words incl. padding, layout) and of every
measurement record entry, as the reference's own suites require (test_measure.cpp:315-335,
test_gates.cpp:176-201, test_tableau.cpp:141-178, test_frames.cpp:96-122).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CM, RM = 0, 1


def gpu_planes(t):
    return t.planes()


def assert_same(t, x, z, s, layout=CM):
    gx, gz, gs = t.planes()
    assert int(t.layout()) == layout
    np.testing.assert_array_equal(gx, x)
    np.testing.assert_array_equal(gz, z)
    np.testing.assert_array_equal(gs, s)


def scrambled(q, oracle, n, seed, depth=12):
    """Both engines evolved by generate_random(n, depth, seed, 0) (test_measure.cpp:27-35)."""
    c = q.generate_random(n, depth, seed, 0.0)
    sched = q.schedule_windows(c)
    t = q.Tableau.zero_state(n)
    x, z, s = oracle.basis_state(n)
    for w in sched.windows:
        q.apply_window(t, w)
        oracle.apply_window(n, CM, x, z, s, w.array())
    return t, x, z, s


@pytest.mark.parametrize("n", [1, 2, 5, 63, 64, 65, 130, 1000])
def test_zero_and_basis_state(q, oracle, n):
    t = q.Tableau.zero_state(n)
    assert_same(t, *oracle.basis_state(n))
    rng = np.random.default_rng(n)
    bits = rng.integers(0, 2, n).astype(np.uint8)
    t = q.Tableau.basis_state(list(bits.astype(bool)))
    assert_same(t, *oracle.basis_state(n, bits))


@pytest.mark.parametrize("n", [2, 7, 64, 65, 129, 300, 1100])
def test_gate_windows_match(q, oracle, n):
    t, x, z, s = scrambled(q, oracle, n, seed=n * 3 + 1, depth=9)
    assert_same(t, x, z, s)


def test_window_every_kind(q, oracle):
    n = 96
    t, x, z, s = scrambled(q, oracle, n, seed=5, depth=6)
    for kind in range(11):
        ar = 2 if kind >= 6 else 1
        w = q.Window([q.Gate(q.GateKind(kind), i, i + 1 if ar == 2 else 0) for i in range(0, n - 1, 2)])
        q.apply_window(t, w)
        oracle.apply_window(n, CM, x, z, s, w.array())
        assert_same(t, x, z, s)


def test_large_window_many_chunks(q, oracle):
    """Windows big enough that the gate kernel splits them into many chunks (partials path)."""
    n = 6000
    t, x, z, s = scrambled(q, oracle, n, seed=11, depth=3)
    assert_same(t, x, z, s)


@pytest.mark.parametrize("n", [1, 5, 63, 64, 65, 130, 700, 1088, 9000])
def test_transpose_matches_reference_layout(q, oracle, n):
    """k_transpose (TMA blocks of 8 row-tiles x 16 words, both planes per launch): partial blocks
    in both directions, RM row padding of up to 15 words (n = 1088: k = 17, rm_pitch = 32)."""
    t, x, z, s = scrambled(q, oracle, n, seed=100 + n, depth=5)
    t.transpose_in_place()
    lay = oracle.transpose(n, CM, x, z)
    assert lay == RM
    assert_same(t, x, z, s, RM)
    t.transpose_in_place()
    oracle.transpose(n, RM, x, z)
    assert_same(t, x, z, s, CM)


@pytest.mark.parametrize("seed", range(12))
def test_run_single_shot_random(q, oracle, seed):
    n = 2 + (seed * 37) % 150
    depth = 4 + seed % 10
    p = [0.0, 0.3, 0.5, 1.0][seed % 4]
    c = q.generate_random(n, depth, seed * 31 + 1, p)
    r = q.run_single_shot(c, seed)
    x, z, s, rec, rep = oracle.run_single_shot(n, c.gate_array, seed)
    assert_same(r.tableau, x, z, s)
    np.testing.assert_array_equal(r.record_array, rec)
    assert r.report.probabilistic_count == rep.probabilistic_count


@pytest.mark.parametrize("n,depth,p", [(64, 30, 1.0), (65, 40, 0.7), (200, 60, 1.0), (513, 25, 0.5)])
def test_run_single_shot_measure_heavy(q, oracle, n, depth, p):
    # Concatenated segments: mid-circuit measurements on scrambled states.
    segs = [q.generate_random(n, depth, 1000 + r, p).gate_array for r in range(3)]
    gates = np.concatenate(segs)
    c = q.Circuit(n, gates)
    r = q.run_single_shot(c, 7)
    x, z, s, rec, _ = oracle.run_single_shot(n, gates, 7)
    assert_same(r.tableau, x, z, s)
    np.testing.assert_array_equal(r.record_array, rec)


def test_config1_full(q, oracle):
    """BASELINE config 1: generate_random(1000, 100, 42, 1.0), run seed 7."""
    c = q.generate_random(1000, 100, 42, 1.0)
    r = q.run_single_shot(c, 7)
    x, z, s, rec, rep = oracle.run_single_shot(1000, c.gate_array, 7)
    assert_same(r.tableau, x, z, s)
    np.testing.assert_array_equal(r.record_array, rec)
    assert r.report.probabilistic_count == rep.probabilistic_count == 998


def test_measure_window_api(q, oracle):
    n = 90
    t, x, z, s = scrambled(q, oracle, n, seed=3, depth=14)
    w = q.Window([q.Gate(q.GateKind.MEASURE, i) for i in range(0, n, 3)], True)
    rng = q.RandomStream(77, q.kStreamMeasure)
    rng.index = 5
    rec = q.MeasurementRecord()
    q.measure_window(t, w, rng, rec)
    out, ci = oracle.measure_window(n, CM, x, z, s, w.array(), 77, 5)
    assert_same(t, x, z, s)
    np.testing.assert_array_equal(rec.array(), out)
    assert rng.index == ci


def test_rm_pipeline_ops(q, oracle):
    """find_probabilistic / pivots / parallel_ge / swap / inject_x / deterministic_outcome."""
    for seed in range(8):
        n = 4 + seed * 9
        t, x, z, s = scrambled(q, oracle, n, seed=seed, depth=12)
        t.transpose_in_place()
        oracle.transpose(n, CM, x, z)
        w = q.Window([q.Gate(q.GateKind.MEASURE, i) for i in range(n)], True)
        assert q.find_probabilistic(t, w) == list(oracle.find_probabilistic(n, RM, x, z, w.array()))
        qq = (seed * 13) % n
        piv = q.find_and_compact_pivots(t, qq)
        e, cnt = oracle.find_and_compact_pivots(n, RM, x, z, qq)
        assert piv.count == cnt and piv.entries == list(e)
        if cnt == 0:
            assert q.deterministic_outcome(t, qq) == oracle.deterministic_outcome(n, RM, x, z, s, qq)
            continue
        for block in (2, 256):
            t2 = t.copy()
            q.parallel_ge(t2, piv, block_targets=block)
            x2, z2, s2 = x.copy(), z.copy(), s.copy()
            oracle.parallel_ge(n, RM, x2, z2, s2, e, cnt, block)
            assert_same(t2, x2, z2, s2, RM)
        q.parallel_ge(t, piv)
        oracle.parallel_ge(n, RM, x, z, s, e, cnt)
        p = piv.entries[0]
        q.swap_anti_commuting(t, p, qq)
        oracle.swap_anti_commuting(n, RM, x, z, s, p, qq)
        assert_same(t, x, z, s, RM)
        q.inject_x(t, p)
        oracle.inject_x(n, s, p)
        assert_same(t, x, z, s, RM)
        assert q.deterministic_outcome(t, qq) == oracle.deterministic_outcome(n, RM, x, z, s, qq)


def test_error_behaviour(q):
    t = q.Tableau.zero_state(3)
    with pytest.raises(q.InvalidArgument):
        q.apply_window(t, q.Window([q.Gate(q.GateKind.H, 0), q.Gate(q.GateKind.CX, 0, 1)]))
    with pytest.raises(q.InvalidArgument):
        q.apply_window(t, q.Window([q.Gate(q.GateKind.MEASURE, 0)], True))
    rng = q.RandomStream(1, q.kStreamMeasure)
    rec = q.MeasurementRecord()
    with pytest.raises(q.InvalidArgument):
        q.measure_window(t, q.Window([q.Gate(q.GateKind.MEASURE, 0), q.Gate(q.GateKind.H, 1)], True), rng, rec)
    with pytest.raises(q.InvalidArgument):
        q.measure_window(t, q.Window([q.Gate(q.GateKind.MEASURE, 2), q.Gate(q.GateKind.MEASURE, 2)], True), rng, rec)
    t.transpose_in_place()
    with pytest.raises(q.InvalidArgument):
        q.apply_window(t, q.Window([q.Gate(q.GateKind.H, 0)]))
    with pytest.raises(q.InvalidArgument):
        q.parallel_ge(t, q.PivotList([-1, -1, -1], 0))
    with pytest.raises(q.InvalidArgument):
        q.swap_anti_commuting(t, 0, 0)  # stabilizer Z_0 commutes with Z_0
    # duplicate-measurement quirk of the reference scheduler surfaces from run_single_shot
    c = q.Circuit(1, [(11, 0), (11, 0)])
    with pytest.raises(q.InvalidArgument):
        q.run_single_shot(c, 3)


@pytest.mark.parametrize("shots", [1, 64, 70, 1000])
def test_sample_matches(q, oracle, shots):
    for seed in range(3):
        n = 5 + seed * 7
        c = q.generate_random(n, 10 + seed, 91 + seed, 0.7)
        rec = q.sample(c, shots, 1234 + seed)
        meas, words, _ = oracle.sample(n, c.gate_array, shots, 1234 + seed)
        assert rec.measured == [int(v) for v in meas]
        np.testing.assert_array_equal(rec.words, words)


def test_frames_ops_match(q, oracle):
    n, shots = 9, 150
    f = q.init_frames(n, shots, 21)
    xf, zf = oracle.init_frames(n, shots, 21)
    gx, gz = f.planes()
    np.testing.assert_array_equal(gx, xf)
    np.testing.assert_array_equal(gz, zf)
    c = q.generate_random(n, 15, 22, 0.0)
    for w in q.schedule_windows(c, q.ScheduleMode.sampling).windows:
        q.apply_window_frames(f, w)
        oracle.apply_window_frames(n, shots, xf, zf, w.array())
    gx, gz = f.planes()
    np.testing.assert_array_equal(gx, xf)
    np.testing.assert_array_equal(gz, zf)
    w = q.Window([q.Gate(q.GateKind.MEASURE, 2), q.Gate(q.GateKind.MEASURE, 5)], True)
    q.measure_sample(f, w, None, 31, 1)
    kf = (shots + 63) // 64
    measured = np.zeros(n, dtype=np.uint32)
    words = np.zeros(n * kf, dtype=np.uint64)
    nr = oracle.measure_sample(n, shots, xf, zf, w.array(), 31, 1, measured, 0, words)
    rec = f.record()
    assert rec.measured == [int(v) for v in measured[:nr]]
    np.testing.assert_array_equal(rec.words, words[:nr * kf])
    gx, gz = f.planes()
    np.testing.assert_array_equal(gz, zf)


def test_engine_matches_run_single_shot(q, oracle):
    n = 300
    c = q.generate_random(n, 40, 5, 0.2)
    e = q.Engine(c)
    e.run(9)
    x, z, s, rec, _ = oracle.run_single_shot(n, c.gate_array, 9)
    np.testing.assert_array_equal(e.record(), rec)
    gx, gz, gs = e.tableau_planes(n)
    np.testing.assert_array_equal(gx, x)
    np.testing.assert_array_equal(gz, z)
    np.testing.assert_array_equal(gs, s)
    # later runs on the same resident inputs are identical (state reset per run); from the
    # second run on, unitary runs replay as CUDA graphs (both plane-pointer parities)
    for seed in (9, 9, 9, 4):
        e.run(seed)
        x, z, s, rec, _ = oracle.run_single_shot(n, c.gate_array, seed)
        np.testing.assert_array_equal(e.record(), rec)
        gx, gz, gs = e.tableau_planes(n)
        np.testing.assert_array_equal(gx, x)
        np.testing.assert_array_equal(gz, z)
        np.testing.assert_array_equal(gs, s)


@pytest.mark.parametrize("n,depth,p", [(2000, 60, 0.0), (700, 80, 0.05), (130, 200, 0.5)])
def test_engine_graph_replay_matches(q, oracle, n, depth, p):
    """Resident-engine runs 2.. replay captured CUDA graphs of the unitary runs; every run must
    stay bit-exact (mid-circuit measurements swap the plane roles between runs)."""
    c = q.generate_random(n, depth, 11, p)
    e = q.Engine(c)
    for seed in (1, 2, 1, 3):
        e.run(seed)
        x, z, s, rec, _ = oracle.run_single_shot(n, c.gate_array, seed)
        np.testing.assert_array_equal(e.record(), rec)
        gx, gz, gs = e.tableau_planes(n)
        np.testing.assert_array_equal(gx, x)
        np.testing.assert_array_equal(gz, z)
        np.testing.assert_array_equal(gs, s)


@pytest.mark.parametrize("n", [3, 64, 200])
def test_ghz_chain_deterministic_breaks(q, oracle, n):
    """All qubits flagged at window start, all but the first become deterministic mid-window
    (exercises the batched path's deterministic break, measure.hpp:417-421)."""
    G = q.GateKind
    gates = [(G.H, 0)] + [(G.CX, i, i + 1) for i in range(n - 1)] + [(G.MEASURE, i) for i in range(n)]
    c = q.Circuit(n, gates)
    for seed in range(3):
        r = q.run_single_shot(c, seed)
        x, z, s, rec, _ = oracle.run_single_shot(n, c.gate_array, seed)
        assert_same(r.tableau, x, z, s)
        np.testing.assert_array_equal(r.record_array, rec)
        assert rec["deterministic"].tolist() == [0] + [1] * (n - 1)


def test_mixed_bell_and_random(q, oracle):
    G = q.GateKind
    n = 150
    g = list(q.generate_random(n, 30, 77, 0.0).gate_array)
    g = [(int(a["kind"]), int(a["q0"]), int(a["q1"])) for a in q.generate_random(n, 30, 77, 0.0).gate_array]
    g += [(G.H, 0), (G.CX, 0, 1)] + [(G.MEASURE, i) for i in range(0, n, 2)]
    g += [(int(a["kind"]), int(a["q0"]), int(a["q1"])) for a in q.generate_random(n, 10, 78, 1.0).gate_array]
    c = q.Circuit(n, g)
    r = q.run_single_shot(c, 11)
    x, z, s, rec, _ = oracle.run_single_shot(n, c.gate_array, 11)
    assert_same(r.tableau, x, z, s)
    np.testing.assert_array_equal(r.record_array, rec)


@pytest.mark.parametrize("env", [{"QSR_MEASURE_BATCH": "0"}, {"QSR_FUSE": "0"}, {"QSR_STREAM": "0"},
                                 {"QSR_GRAPHS": "0"}, {"QSR_PDL": "0"}, {"QSR_HOSTPOLL": "0"},
                                 {"QSR_FUSE_COLS": "0", "QSR_CHAIN": "0"}, {"QSR_CHAIN": "0"}])
def test_alternate_collapse_paths_match(q, env):
    """Every alternate path must agree with the default and the oracle: QSR_MEASURE_BATCH=0 (one
    collapse per pass, the path of uploaded tableaux), QSR_FUSE=0 (no gate fusion), QSR_STREAM=0
    (schedule first, then run), QSR_GRAPHS=0 (no graph replay), QSR_PDL=0 (plain launches instead
    of programmatic dependent launches), QSR_HOSTPOLL=0 (batch control words read back by a copy
    + event per batch instead of the sign pass's pinned-memory write), QSR_CHAIN=0 (every batch's
    select in its own launch after its column bits, which the previous sign pass computes) and with
    QSR_FUSE_COLS=0 (a column-bit launch per batch)."""
    import subprocess
    import sys
    code = (
        "import numpy as np, sys\n"
        "sys.path.insert(0, '.')\n"
        "from paper_2603_14641_b200 import quasar as q\n"
        "from oracle.oracle import best_available\n"
        "o = best_available()\n"
        "for seed in range(4):\n"
        "    n = 40 + 37 * seed\n"
        "    c = q.generate_random(n, 30, seed, 1.0)\n"
        "    r = q.run_single_shot(c, seed)\n"
        "    x, z, s, rec, _ = o.run_single_shot(n, c.gate_array, seed)\n"
        "    gx, gz, gs = r.tableau.planes()\n"
        "    assert np.array_equal(gx, x) and np.array_equal(gz, z) and np.array_equal(gs, s)\n"
        "    assert np.array_equal(r.record_array, rec)\n"
        "    e = q.Engine(c)\n"
        "    for _ in range(2):\n"
        "        e.run(seed)\n"
        "        assert np.array_equal(e.record(), rec)\n"
        "        gx, gz, gs = e.tableau_planes(n)\n"
        "        assert np.array_equal(gx, x) and np.array_equal(gz, z) and np.array_equal(gs, s)\n"
        "    se = q.ShardedEngine(c, min(3, (n + 63) // 64))\n"
        "    se.run(seed)\n"
        "    assert np.array_equal(se.record(), rec)\n"
        "    meas, words, _ = o.sample(n, c.gate_array, 200, seed)\n"
        "    smp = q.sample(c, 200, seed)\n"
        "    assert smp.measured == [int(v) for v in meas] and np.array_equal(smp.words, words)\n"
        "print('ok')\n")
    import os
    env = dict(os.environ, **env)
    root = __import__("pathlib").Path(__file__).resolve().parents[1]
    out = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    assert "ok" in out.stdout
