"""Timing probe of the device check_group_validity (k_validity.cu) after a run."""
import sys
import time

sys.path.insert(0, '.')
from paper_2603_14641_b200 import quasar as q  # noqa: E402

sizes = [(int(a), int(b)) for a, b in (s.split("x") for s in sys.argv[1:])] or [(20000, 100), (50000, 20)]
for n, d in sizes:
    c = q.generate_random(n, d, 42, 0.0)
    r = q.run_single_shot(c, 7)
    r.tableau.check_group_validity()  # warm
    t0 = time.time()
    v = r.tableau.check_group_validity()
    t1 = time.time()
    print(f"validity n={n}: {v} {t1 - t0:.3f} s", flush=True)
