"""One unitary segment (generate_random(n, depth, 42, 0), no measurements) through the resident
engine: the temporally blocked gate kernel alone, for ncu.

    python tools/seg_probe.py [n] [depth] [runs]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2603_14641_b200 import quasar as q  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 180000
depth = int(sys.argv[2]) if len(sys.argv) > 2 else 30
runs = int(sys.argv[3]) if len(sys.argv) > 3 else 1
c = q.generate_random(n, depth, 42, 0.0)
e = q.Engine(c)
for _ in range(runs):
    ms = e.run(7)
    print(f"n={n} depth={depth}: {ms:.1f} ms {e.stats()}", flush=True)
