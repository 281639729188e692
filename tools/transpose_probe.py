"""Times the CM<->RM transpose pair on a tableau of n qubits (python tools/transpose_probe.py n reps);
QSR_TR_GW / QSR_TR_GR select the CTA block grouping (k_transpose.cu)."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_2603_14641_b200 import quasar as q  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 180000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
k = (n + 63) // 64
t = q.Tableau.zero_state(n)
t.transpose_in_place()
t.transpose_in_place()
t0 = time.perf_counter()
for _ in range(reps):
    t.transpose_in_place()
    t.transpose_in_place()
dt = (time.perf_counter() - t0) / (2 * reps)
bytes_ = 2 * 2 * 8.0 * 64 * k * 2 * k
print(f"n={n} gw={os.environ.get('QSR_TR_GW', '-')} gr={os.environ.get('QSR_TR_GR', '-')} "
      f"{dt * 1e3:.2f} ms per transpose, {bytes_ / dt / 1e9:.0f} GB/s")
