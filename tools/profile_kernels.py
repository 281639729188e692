#!/usr/bin/env python
"""Small driver for ncu captures of the hot kernels at full width without generating the whole
124 M-gate circuit: `layers` random layers of the c5 circuit (n = 180,000) through the
apply_window API, then one measurement window on the scrambled state.

    ncu --set full -k regex:k_gate_window -s 20 -c 1 -o prof python tools/profile_kernels.py
"""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2603_14641_b200 import quasar as q  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=180000)
    ap.add_argument("--layers", type=int, default=60)
    ap.add_argument("--measure", type=int, default=3, help="qubits in the final measurement window")
    a = ap.parse_args()
    c = q.generate_random(a.n, a.layers, 42, 0.0)
    s = q.schedule_windows(c)
    t = q.Tableau.zero_state(a.n)
    t0 = time.time()
    for w in s.windows:
        q.apply_window(t, w)
    print(f"{len(c)} gates in {len(s)} windows: {time.time() - t0:.2f}s (API path, incl. uploads)")
    if a.measure:
        w = q.Window([q.Gate(q.GateKind.MEASURE, i * 997 % a.n) for i in range(a.measure)], True)
        rec = q.MeasurementRecord()
        q.measure_window(t, w, q.RandomStream(7, q.kStreamMeasure), rec)
        print("outcomes", [(e.qubit, e.outcome, e.deterministic) for e in rec.entries])


if __name__ == "__main__":
    main()
