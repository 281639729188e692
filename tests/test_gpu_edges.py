"""Edge cases of the reference's tests and semantics on the B200 engine, each against the oracle:
empty circuits, measurement-only circuits, repeated measurement of one qubit across windows,
single-qubit registers, word-boundary register sizes, and boundary shot counts."""
import numpy as np
import pytest

from helpers import geometry

pytestmark = pytest.mark.gpu


def run_both(q, oracle, n, gates, seed):
    arr = q.gates_array(gates)
    c = q.Circuit(n, arr)
    r = q.run_single_shot(c, seed)
    x, z, s, rec, rep = oracle.run_single_shot(n, c.gate_array, seed)
    gx, gz, gs = r.tableau.planes()
    np.testing.assert_array_equal(gx, x)
    np.testing.assert_array_equal(gz, z)
    np.testing.assert_array_equal(gs, s)
    np.testing.assert_array_equal(r.record_array, rec)
    assert r.report.probabilistic_count == rep.probabilistic_count
    return r


@pytest.mark.parametrize("n", [1, 5, 64, 130])
def test_empty_circuit(q, oracle, n):
    r = run_both(q, oracle, n, [], 3)
    assert len(r.record_array) == 0 and r.report.window_count == 0


def test_measurement_only_is_deterministic_zero(q, oracle):
    n = 70
    r = run_both(q, oracle, n, [(11, i) for i in range(n)], 5)
    rec = r.record_array
    assert rec["outcome"].sum() == 0 and rec["deterministic"].all()


def test_repeated_measurement_of_one_qubit(q, oracle):
    # Qubit 0 measured again and again across windows: probabilistic first, then deterministic
    # repeats, then probabilistic again after an H; a bystander entangled in between.
    gates = [(3, 0), (11, 0), (0, 0), (11, 0), (3, 0), (11, 0), (6, 0, 1), (11, 1), (2, 0), (11, 0)]
    for seed in range(8):
        run_both(q, oracle, 2, gates, seed)
    # Two measurements of one qubit back to back land in one window (the reference scheduler's
    # flush) and measure_window rejects it — on both sides.
    from oracle.oracle import OracleError
    bad = q.gates_array([(3, 0), (11, 0), (11, 0)])
    with pytest.raises(q.InvalidArgument):
        q.run_single_shot(q.Circuit(1, bad), 1)
    with pytest.raises(OracleError):
        oracle.run_single_shot(1, bad, 1)


def test_single_qubit_register_every_kind(q, oracle):
    for seed in range(4):
        gates = [(k, 0) for k in (3, 4, 5, 0, 1, 2, 3)] + [(11, 0)] + [(3, 0), (4, 0), (11, 0)]
        run_both(q, oracle, 1, gates, seed)


@pytest.mark.parametrize("n", [63, 64, 65, 127, 128, 129, 191, 192, 193])
def test_word_boundary_registers(q, oracle, n):
    c = q.generate_random(n, 12, n, 0.6)
    run_both(q, oracle, n, c.gate_array, 1)


@pytest.mark.parametrize("shots", [1, 63, 64, 65, 128, 129])
def test_sample_boundary_shots(q, oracle, shots):
    for n in (1, 3, 64):
        c = q.generate_random(n, 6, 17 + n, 1.0)
        rec = q.sample(c, shots, 99)
        meas, words, _ = oracle.sample(n, c.gate_array, shots, 99)
        assert rec.measured == [int(v) for v in meas]
        np.testing.assert_array_equal(rec.words, words)


def test_sample_empty_and_unmeasured(q, oracle):
    c = q.generate_random(20, 5, 3, 0.0)  # no measurements
    rec = q.sample(c, 100, 1)
    assert rec.measured == [] and rec.words.size == 0


def test_geometry_helper_consistent():
    assert geometry(64) == (1, 64) and geometry(65) == (2, 128)


def test_shot_word_keying_prefix(q):
    """test_frames.cpp:188-196: a 64-shot run is a prefix of the 128-shot run (the Z frames are
    keyed by (seed, qubit, shot-word), not by the shot count); also across word sizes."""
    c = q.generate_random(6, 10, 91, 1.0)
    small = q.sample(c, 64, 1234)
    big = q.sample(c, 128, 1234)
    assert small.measured == big.measured
    for r in range(len(small.measured)):
        for shot in range(64):
            assert small.bit(r, shot) == big.bit(r, shot)
    # deterministic in (circuit, shots, seed)
    again = q.sample(c, 128, 1234)
    assert np.array_equal(again.words, big.words)


@pytest.mark.parametrize("n", [600, 1000])
def test_measure_all_window_block_order(q, oracle, n):
    """Measure-all windows (c3's shape) at sizes where the absorb pass visits 64-row blocks in a
    strided order (n = 600: 18 blocks, stride 11; n = 1000: 31 blocks) and collapsed stabilizers
    pile up at the low stabilizer rows batch after batch."""
    for seed in range(2):
        c = q.generate_random(n, 15, 300 + seed, 1.0)
        r = run_both(q, oracle, n, c.gate_array, seed)
        assert r.report.probabilistic_count > n // 2
