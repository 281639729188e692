"""Gate-window throughput when the whole tableau fits in L2 (how much an L2-resident,
temporally blocked gate pass could gain over the HBM-bound one).

    python tools/gate_l2_probe.py [n ...]
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2603_14641_b200 import quasar as q  # noqa: E402

RW = np.array([(1, 0), (2, 0), (1, 0), (2, 2), (2, 1), (2, 1), (4, 2), (4, 3), (4, 2), (4, 4), (4, 4), (0, 0)])
for n in [int(a) for a in sys.argv[1:]] or [4000, 9000, 14000, 20000, 40000]:
    depth = 300
    c = q.generate_random(n, depth, 3, 0.0)
    k = (n + 63) // 64
    kinds = np.bincount(c.gate_array["kind"], minlength=12)
    gb = 8.0 * 2 * k * float((kinds * RW.sum(axis=1)).sum()) + 16.0 * 2 * k * depth
    e = q.Engine(c)
    e.run(1)
    best = 1e30
    for _ in range(3):
        e.run(1)
        best = min(best, e.stats()["gate_ms"])
    mb = 64 * k * ((2 * k + 15) // 16 * 16) * 16 / 1e6
    print(f"n={n:6d} tableau={mb:8.1f} MB  gate windows {best:8.2f} ms  {gb / best / 1e6:8.1f} GB/s algorithmic",
          flush=True)
