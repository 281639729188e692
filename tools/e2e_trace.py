"""Phase trace of the end-to-end C-ABI call at c5 (QSR_TRACE=1): run_single_shot with host
buffers + final tableau download into pinned memory.

    QSR_TRACE=1 python tools/e2e_trace.py [n] [depth] [p] [runs]
"""
import ctypes as C
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2603_14641_b200 import _lib  # noqa: E402
from paper_2603_14641_b200 import quasar as q  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 180000
depth = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
p = float(sys.argv[3]) if len(sys.argv) > 3 else 0.01
runs = int(sys.argv[4]) if len(sys.argv) > 4 else 2
c = q.generate_random(n, depth, 42, p)
k = (n + 63) // 64
plane = 64 * k * 2 * k
px, pz = C.c_void_p(), C.c_void_p()
_lib.check(_lib.lib.qsr_host_alloc(plane * 8, C.byref(px)))
_lib.check(_lib.lib.qsr_host_alloc(plane * 8, C.byref(pz)))
ps = np.empty(2 * k, dtype=np.uint64)
rec = np.zeros(max(c.measure_count(), 1), dtype=_lib.ENTRY_DTYPE)
for i in range(runs):
    t0 = time.perf_counter()
    h = C.c_void_p()
    rep = _lib.Report_t()
    _lib.check(_lib.lib.qsr_run_single_shot(c._h, None, 7, 0, C.byref(h), _lib.ptr(rec), C.byref(rep)))
    t1 = time.perf_counter()
    _lib.check(_lib.lib.qsr_tableau_download(h, C.cast(px, _lib.pu64), C.cast(pz, _lib.pu64), _lib.ptr(ps, C.c_uint64)))
    t2 = time.perf_counter()
    _lib.lib.qsr_tableau_destroy(h)
    t3 = time.perf_counter()
    print(f"e2e {i}: run_single_shot {t1 - t0:.3f} s, download {t2 - t1:.3f} s, destroy {t3 - t2:.3f} s, "
          f"total {t3 - t0:.3f} s", file=sys.stderr, flush=True)
