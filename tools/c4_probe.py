"""c4: many-shot sampling, generate_random(10000, 500, 42, 1.0), sample(shots=100000, seed=7)
(SURVEY.md §8(d)); prints the sample() wall time and its reference-shot part.

    python tools/c4_probe.py [n] [depth] [shots] [runs]
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2603_14641_b200 import quasar as q  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
depth = int(sys.argv[2]) if len(sys.argv) > 2 else 500
shots = int(sys.argv[3]) if len(sys.argv) > 3 else 100000
runs = int(sys.argv[4]) if len(sys.argv) > 4 else 2
c = q.generate_random(n, depth, 42, 1.0)
for i in range(runs):
    rep = q.RunReport()
    t0 = time.perf_counter()
    rec = q.sample(c, shots, 7, rep)
    dt = time.perf_counter() - t0
    t1 = time.perf_counter()
    del rec
    import gc
    gc.collect()
    print(f"  (record freed in {(time.perf_counter() - t1) * 1e3:.1f} ms)", flush=True)
    print(f"run {i}: sample {dt * 1e3:.1f} ms (reference shot {rep.total_seconds * 1e3:.1f} ms), "
          f"{len(c)} gates x {shots} shots = {len(c) * shots / dt / 1e9:.2f} G gate-shots/s; "
          f"reference-shot device phases: to {rep.timers.to_seconds * 1e3:.1f} t {rep.timers.t_seconds * 1e3:.1f} "
          f"ge {rep.timers.ge_seconds * 1e3:.1f} cmp {rep.timers.cmp_seconds * 1e3:.1f} ms", flush=True)
