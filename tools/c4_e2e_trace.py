"""Phase trace of the end-to-end sample() call at c4 (QSR_TRACE=1 prints libqsr's scopes):
generate_random(10000, 500, 42, 1.0), sample(100000, 7), the ShotRecord download split out.

    QSR_TRACE=1 python tools/c4_e2e_trace.py [n] [depth] [shots] [runs]
"""
import ctypes as C
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2603_14641_b200 import _lib  # noqa: E402
from paper_2603_14641_b200 import quasar as q  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
depth = int(sys.argv[2]) if len(sys.argv) > 2 else 500
shots = int(sys.argv[3]) if len(sys.argv) > 3 else 100000
runs = int(sys.argv[4]) if len(sys.argv) > 4 else 3
c = q.generate_random(n, depth, 42, 1.0)
for i in range(runs):
    t0 = time.perf_counter()
    h = C.c_void_p()
    rep = _lib.Report_t()
    _lib.check(_lib.lib.qsr_sample_word(c._h, shots, 7, 64, 0, C.byref(h), C.byref(rep)))
    t1 = time.perf_counter()
    f = q.FrameTableau(h)
    r = f.record()
    t2 = time.perf_counter()
    del f
    t3 = time.perf_counter()
    print(f"run {i}: qsr_sample {1e3 * (t1 - t0):.1f} ms, record download {1e3 * (t2 - t1):.1f} ms "
          f"({r.words.nbytes / 1e6:.0f} MB), free {1e3 * (t3 - t2):.1f} ms", flush=True)
