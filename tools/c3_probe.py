"""One segment of the c3 shape (generate_random(n, depth, seed, 1.0): depth layers then
measure every qubit) through the resident engine; prints per-phase device times.

    python tools/c3_probe.py [n] [depth] [runs]
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2603_14641_b200 import quasar as q  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 50000
depth = int(sys.argv[2]) if len(sys.argv) > 2 else 100
runs = int(sys.argv[3]) if len(sys.argv) > 3 else 2
c = q.generate_random(n, depth, 1000, 1.0)
e = q.Engine(c)
for i in range(runs):
    t0 = time.perf_counter()
    ms = e.run(7)
    wall = time.perf_counter() - t0
    rec = e.record()
    print(f"run {i}: device {ms:.1f} ms wall {wall*1e3:.1f} ms {e.stats()} "
          f"probabilistic={int((rec['deterministic'] == 0).sum())}/{len(rec)}", flush=True)
