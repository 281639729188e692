"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck / synccheck): every
kernel family of the hot path at small sizes, checked against the CPU oracle.

    compute-sanitizer --tool memcheck python tools/sanitize_probe.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_2603_14641_b200 import quasar as q  # noqa: E402
from oracle.oracle import best_available  # noqa: E402

o = best_available()
ok = True


def check(name, cond):
    global ok
    print(f"{name}: {'ok' if cond else 'MISMATCH'}", flush=True)
    ok &= bool(cond)


for n, depth, p, seed in [(130, 30, 1.0, 1), (200, 40, 0.5, 2), (65, 20, 1.0, 3), (2500, 40, 1.0, 4)]:
    c = q.generate_random(n, depth, seed, p)
    x, z, s, rec, _ = o.run_single_shot(n, c.gate_array, 7)
    r = q.run_single_shot(c, 7)  # streamed, fused, batched collapses (PDL chain)
    gx, gz, gs = r.tableau.planes()
    check(f"run_single_shot n={n}", np.array_equal(gx, x) and np.array_equal(gz, z) and np.array_equal(gs, s)
          and np.array_equal(r.record_array, rec))
    e = q.Engine(c)
    for _ in range(2):  # eager, then CUDA-graph replay
        e.run(7)
    check(f"engine n={n}", np.array_equal(e.record(), rec))
    se = q.ShardedEngine(c, min(2, (n + 63) // 64))  # local exchange (3 shards at n = 2,500 exhaust racecheck's host memory)
    se.run(7)
    check(f"sharded n={n}", np.array_equal(se.record(), rec))
    st = q.ShardedEngine(c, 1, exchange="local", streamed_seed=7)  # streamed driver + sharded protocol
    check(f"sharded streamed n={n}", np.array_equal(st.record(), rec))
    del st
    meas, words, _ = o.sample(n, c.gate_array, 300, 7)
    smp = q.sample(c, 300, 7)  # record staged through the pinned buffers (pageable destination)
    check(f"sample n={n}", np.array_equal(smp.words, words))
    pb = q.PinnedBuffer(8 * len(meas) * 5 + 8)
    smp = q.sample(c, 300, 7, out=pb.array)  # straight into a pinned buffer
    check(f"sample pinned n={n}", np.array_equal(smp.words, words))
    rs, _ = e.sample(300, 7)
    check(f"engine sample n={n}", np.array_equal(rs.words, words))
    t = q.Tableau.zero_state(n)
    g, off, fl = q.schedule_windows(q.generate_random(n, 8, seed, 0.0)).arrays()
    for w in range(len(fl)):
        q.apply_window(t, g[off[w]:off[w + 1]])
    t.transpose_in_place()
    t.transpose_in_place()
    piv = q.find_and_compact_pivots
    t.transpose_in_place()
    pl = piv(t, 0)
    if pl.count:
        q.parallel_ge(t, pl, block_targets=2)
    t.transpose_in_place()
    check(f"api ops n={n}", True)
print("SANITIZE PROBE", "OK" if ok else "FAILED")
sys.exit(0 if ok else 1)
