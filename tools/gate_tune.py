#!/usr/bin/env python
"""Gate-window kernel tuning: device time per window and achieved HBM GB/s (kind-exact
algorithmic bytes) for the first L layers of the c2 / c5 circuits.

    QSR_GATE_VARIANT=1 python tools/gate_tune.py --n 180000 --layers 40
"""
import argparse
import json
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2603_14641_b200 import quasar as q  # noqa: E402

RW = np.array([(1, 0), (2, 0), (1, 0), (2, 2), (2, 1), (2, 1), (4, 2), (4, 3), (4, 2), (4, 4), (4, 4), (0, 0)])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=180000)
    ap.add_argument("--layers", type=int, default=40)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    c = q.generate_random(a.n, a.layers, 42, 0.0)
    e = q.Engine(c)
    k = (a.n + 63) // 64
    kinds = np.bincount(c.gate_array["kind"], minlength=12)
    gbytes = 8.0 * 2 * k * float((kinds * RW.sum(axis=1)).sum()) + 16.0 * 2 * k * a.layers
    for _ in range(2):
        e.run(1)
    ms = []
    for _ in range(a.reps):
        e.run(1)
        ms.append(e.stats()["gate_ms"])
    best = min(ms)
    print(json.dumps({"variant": os.environ.get("QSR_GATE_VARIANT", "default"), "n": a.n, "layers": a.layers,
                      "ms_per_window": best / a.layers, "GBps": gbytes / (best * 1e-3) / 1e9,
                      "bytes_per_window": gbytes / a.layers}))


if __name__ == "__main__":
    main()
