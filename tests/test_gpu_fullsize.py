"""Full-size parity on the BASELINE configs that the CPU oracle finishes in minutes
(SURVEY.md §8(c) parity plan). Slow (the reference CPU path runs at full size on the host's
cores, ~1-2 min per config); part of the default `-m gpu` suite.

  c2: generate_random(20000, 1000, 42, 0.0), run seed 7      — final tableau bit-identical
  c4: generate_random(10000, 500, 42, 1.0), sample(100000, 7) — every shot word identical
  c5 prefix: the first 6 layers of the c5 circuit at 180,000 qubits + its Bernoulli(0.01)
      final measurements — tableau and every record entry identical
Full c3 / c5 are hours on the CPU: tests/test_gpu_scale.py covers them by
snapshot parity at their widths (50,000 and 180,000 qubits).
"""
import hashlib
import os

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        if a.dtype.names:
            for f in a.dtype.names:
                h.update(np.ascontiguousarray(a[f]).tobytes())
        else:
            h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


@pytest.fixture(scope="module")
def ref():
    from oracle.oracle import Oracle, available
    if not available("reference"):
        pytest.skip("oracle/_ref (compiled reference) not available")
    o = Oracle("reference")
    o.set_threads(os.cpu_count() or 1)
    return o


def test_c2_full(q, ref):
    c = q.generate_random(20000, 1000, 42, 0.0)
    r = q.run_single_shot(c, 7)
    gx, gz, gs = r.tableau.planes()
    x, z, s, rec, _ = ref.run_single_shot(20000, c.gate_array, 7)
    print("c2 tableau sha256", digest(gx, gz, gs))
    assert digest(gx, gz, gs) == digest(x, z, s)


def test_c4_full(q, ref):
    c = q.generate_random(10000, 500, 42, 1.0)
    rec = q.sample(c, 100000, 7)
    meas, words, _ = ref.sample(10000, c.gate_array, 100000, 7)
    print("c4 shot-record sha256", digest(np.asarray(rec.measured, dtype=np.uint32), rec.words))
    assert rec.measured == [int(v) for v in meas]
    assert digest(rec.words) == digest(words)


def test_c5_prefix(q, ref):
    c = q.generate_random(180000, 6, 42, 0.01)
    r = q.run_single_shot(c, 7)
    gx, gz, gs = r.tableau.planes()
    x, z, s, rec, _ = ref.run_single_shot(180000, c.gate_array, 7)
    print("c5-prefix tableau sha256", digest(gx, gz, gs), "measurements", len(rec))
    assert digest(gx, gz, gs) == digest(x, z, s)
    np.testing.assert_array_equal(r.record_array, rec)
