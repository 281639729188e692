"""Parity at the benchmarked scale (SURVEY.md §8(c) parity plan, items (2) and (3)), run by
default in the `-m gpu` suite against the reference compiled unmodified (oracle/_ref).

* every gate-window kernel instance (QSR_GATE_VARIANT 0-4, incl. the headline <1,1,4>)
  against the reference apply_window (gates.hpp:147-197);
* c3 shape in full at n = 8,000 (three 100-layer measure-all segments):
  run_single_shot and the resident Engine with CUDA-graph replay (simulator.hpp:46-76);
* c3 width, snapshot parity: a 50,000-qubit tableau scrambled by 100 layers on the device,
  then the first measurements of its measure-all window, the batched collapse path with the
  strided absorb order at 1,564 row blocks, against the reference measure_window
  (measure.hpp:381-442) run on the downloaded snapshot;
* c5 width, snapshot parity: a 180,000-qubit tableau scrambled by 150 layers of the c5
  circuit; layer 151 (a >= 16k-gate window, so k_gate_window<1,1,4>) on both sides, the fused
  streamed run of the same 151 layers against that, then the first measurements of c5's final
  Bernoulli(0.01) window on both sides.
The CPU work is bounded (tens of seconds to a few minutes on the box's host cores).
"""
import os
import subprocess
import sys
import textwrap
import time
from pathlib import Path

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def ref():
    from oracle.oracle import Oracle, available
    if not available("reference"):
        pytest.skip("oracle/_ref (compiled reference) not available")
    o = Oracle("reference")
    o.set_threads(os.cpu_count() or 1)
    return o


def _windows(q, c):
    g, off, fl = q.schedule_windows(c).arrays()
    return [(g[off[w]:off[w + 1]], bool(fl[w])) for w in range(len(fl))]


def _same(a, b):
    return a.shape == b.shape and np.array_equal(a, b)


# ---- every k_gate_window instance --------------------------------------------------------
VARIANT_SCRIPT = textwrap.dedent("""
    import sys, numpy as np
    sys.path.insert(0, {root!r})
    from paper_2603_14641_b200 import quasar as q
    from oracle.oracle import best_available
    o = best_available()
    n = {n}
    c = q.generate_random(n, 12, 99, 0.0)
    g, off, fl = q.schedule_windows(c).arrays()
    t = q.Tableau.zero_state(n)
    x, z, s = o.basis_state(n)
    for w in range(len(fl)):
        win = g[off[w]:off[w + 1]]
        q.apply_window(t, win)
        o.apply_window(n, 0, x, z, s, win)
    gx, gz, gs = t.planes()
    ok = np.array_equal(gx, x) and np.array_equal(gz, z) and np.array_equal(gs, s)
    print("variant", {v}, "windows", len(fl), "gates", len(g), "ok", ok)
    sys.exit(0 if ok else 1)
""")


@pytest.mark.parametrize("variant", [0, 1, 2, 3, 4])
@pytest.mark.parametrize("n", [333, 3000])
def test_every_gate_kernel_variant(q, ref, variant, n):
    """QSR_GATE_VARIANT forces one instance for the whole process (k_gates.cu gate_variant);
    variant 1 (<1,1,4>) is the default for >= 16k-gate windows (the c5 headline)."""
    env = dict(os.environ, QSR_GATE_VARIANT=str(variant))
    r = subprocess.run([sys.executable, "-c", VARIANT_SCRIPT.format(root=str(ROOT), n=n, v=variant)],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr


# ---- c3 shape in full at n = 8,000 --------------------------------------------------------
def _c3_circuit(q, n, rounds, depth=100):
    return q.Circuit(n, np.concatenate([q.generate_random(n, depth, 1000 + r, 1.0).gate_array
                                        for r in range(rounds)]))


@pytest.fixture(scope="module")
def c3_small(q, ref):
    c = _c3_circuit(q, 8000, 3)
    t0 = time.time()
    x, z, s, rec, rep = ref.run_single_shot(8000, c.gate_array, 7)
    print(f"reference c3 n=8000 x3: {time.time() - t0:.1f} s, {len(rec)} measurements, "
          f"{rep.probabilistic_count} probabilistic")
    return c, (x, z, s, rec)


def test_c3_shape_n8000_three_rounds(q, c3_small):
    c, (x, z, s, rec) = c3_small
    r = q.run_single_shot(c, 7)
    gx, gz, gs = r.tableau.planes()
    np.testing.assert_array_equal(r.record_array, rec)
    assert _same(gx, x) and _same(gz, z) and _same(gs, s)


def test_c3_shape_n8000_engine_graph_replay(q, c3_small):
    c, (x, z, s, rec) = c3_small
    e = q.Engine(c)
    for _ in range(3):  # first run eager, then CUDA-graph replay of the unitary runs
        e.run(7)
        np.testing.assert_array_equal(e.record(), rec)
    gx, gz, gs = e.tableau_planes(8000)
    assert _same(gx, x) and _same(gz, z) and _same(gs, s)


# ---- c3 width: measure-all window on a scrambled 50,000-qubit snapshot -------------------------
C3_MEASURE = int(os.environ.get("QSR_C3_SNAPSHOT_MEASURE", "1024"))


def test_c3_width_snapshot_measure_window(q, ref):
    n = 50000
    c = q.generate_random(n, 100, 1000, 1.0)  # c3 segment 0
    wins = _windows(q, c)
    t = q.Tableau.zero_state(n)
    for g, is_m in wins:
        if not is_m:
            q.apply_window(t, g)
    mwin = [g for g, is_m in wins if is_m]
    assert len(mwin) == 1 and len(mwin[0]) == n
    meas = mwin[0][:C3_MEASURE]
    x, z, s = t.planes()  # snapshot (reference CM layout)
    rng = q.RandomStream(7, 0)
    rec = q.MeasurementRecord()
    q.measure_window(t, q.Window(meas, True), rng, rec)
    t0 = time.time()
    out, coins = ref.measure_window(n, 0, x, z, s, meas, 7, 0)
    print(f"reference measure_window n={n} m={len(meas)}: {time.time() - t0:.1f} s, coins {coins}")
    assert coins == rng.index
    np.testing.assert_array_equal(rec.array(), out)
    gx, gz, gs = t.planes()
    assert _same(gs, s) and _same(gx, x) and _same(gz, z)


# ---- c5 width: a headline gate window and the first collapses of c5's final window ----------
C5_LAYERS = int(os.environ.get("QSR_C5_SNAPSHOT_LAYERS", "150"))
C5_MEASURE = int(os.environ.get("QSR_C5_SNAPSHOT_MEASURE", "33"))


def test_c5_width_snapshot_window_and_collapses(q, ref):
    n = 180000
    c = q.generate_random(n, C5_LAYERS + 1, 42, 0.01)  # the c5 circuit's first layers + its final window
    wins = _windows(q, c)
    unitary = [g for g, is_m in wins if not is_m]
    mwin = [g for g, is_m in wins if is_m]
    assert len(unitary) == C5_LAYERS + 1 and len(mwin) == 1
    t = q.Tableau.zero_state(n)
    for g in unitary[:-1]:
        q.apply_window(t, g)
    x, z, s = t.planes()  # scrambled snapshot
    last = unitary[-1]
    assert len(last) >= 1 << 14  # the <1,1,4> instance (k_gates.cu gate_variant)
    q.apply_window(t, last)
    t0 = time.time()
    ref.apply_window(n, 0, x, z, s, last)
    print(f"reference apply_window n={n} gates={len(last)}: {time.time() - t0:.1f} s")
    gx, gz, gs = t.planes()
    assert _same(gs, s) and _same(gx, x) and _same(gz, z)
    del gx, gz, gs
    # The fused, streamed product path (SWAP relabelling, single-qubit runs folded into the next
    # two-qubit gate, rows un-permuted at the end) over the same C5_LAYERS + 1 layers.
    fused = q.run_single_shot(q.generate_random(n, C5_LAYERS + 1, 42, 0.0), 7)
    fx, fz, fs = fused.tableau.planes()
    assert _same(fs, s) and _same(fx, x) and _same(fz, z)
    del fused, fx, fz, fs
    meas = mwin[0][:C5_MEASURE]
    rng = q.RandomStream(7, 0)
    rec = q.MeasurementRecord()
    q.measure_window(t, q.Window(meas, True), rng, rec)
    t0 = time.time()
    out, coins = ref.measure_window(n, 0, x, z, s, meas, 7, 0)
    print(f"reference measure_window n={n} m={len(meas)}: {time.time() - t0:.1f} s, coins {coins}, "
          f"outcomes {''.join(str(int(v)) for v in out['outcome'])}")
    assert coins == rng.index and coins > 0
    np.testing.assert_array_equal(rec.array(), out)
    gx, gz, gs = t.planes()
    assert _same(gs, s) and _same(gx, x) and _same(gz, z)
