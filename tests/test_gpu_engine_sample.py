"""Resident-engine sampling (qsr_engine_sample, the c4 bench step) and the measurement-pass
profile (qsr_engine_profile): results identical to the streamed sample() and to the reference
sample<uint64_t> (frames.hpp:163-204)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,depth,p,shots", [(130, 40, 1.0, 1000), (700, 30, 0.3, 4100), (64, 10, 0.0, 100)])
def test_engine_sample_matches_reference(q, oracle, n, depth, p, shots):
    c = q.generate_random(n, depth, 5 + n, p)
    meas, words, _ = oracle.sample(n, c.gate_array, shots, 9)
    e = q.Engine(c)
    for _ in range(2):  # repeated calls on one engine
        rec, ms = e.sample(shots, 9)
        assert ms > 0
        assert rec.measured == [int(v) for v in meas]
        np.testing.assert_array_equal(rec.words, words)
    s = q.sample(c, shots, 9)
    np.testing.assert_array_equal(s.words, words)
    # the engine still runs single shots bit-exactly afterwards
    x, z, sg, r, _ = oracle.run_single_shot(n, c.gate_array, 9)
    e.run(9)
    np.testing.assert_array_equal(e.record(), r)


def test_engine_sample_by_shot_slices(q, oracle):
    n, shots = 200, 4100
    c = q.generate_random(n, 25, 3, 1.0)
    meas, words, _ = oracle.sample(n, c.gate_array, shots, 4)
    kf = (shots + 63) // 64
    full = words.reshape(len(meas), kf)
    e = q.Engine(c)
    parts = []
    for rank in range(3):
        rec, _ = e.sample(shots, 4, world=3, rank=rank)
        parts.append(rec.words.reshape(len(meas), -1))
    np.testing.assert_array_equal(np.concatenate(parts, axis=1), full)


def test_engine_profile_counts_absorb_launches(q, oracle):
    n = 1000
    c = q.generate_random(n, 100, 42, 1.0)
    e = q.Engine(c)
    e.run(7)
    prof = e.profile(7)
    assert prof["absorb_launches"] >= (n + 31) // 32 // 2
    assert prof["absorb_rows"] > 0 and prof["absorb_ms"] > 0 and prof["row_words"] == (n + 63) // 64
    x, z, s, rec, _ = oracle.run_single_shot(n, c.gate_array, 7)
    np.testing.assert_array_equal(e.record(), rec)  # the profiled run is a normal run


def test_sample_record_into_pinned_buffer(q, oracle):
    """sample(..., out=PinnedBuffer.array): the record words land in the caller's page-locked
    buffer (the c4 e2e leg), identical to the reference; a too-small buffer is refused."""
    n, shots = 300, 2000
    c = q.generate_random(n, 20, 8, 1.0)
    meas, words, _ = oracle.sample(n, c.gate_array, shots, 6)
    buf = q.PinnedBuffer(8 * len(meas) * ((shots + 63) // 64) + 64)
    buf.array[:] = 0xDEADBEEF
    rec = q.sample(c, shots, 6, out=buf.array)
    np.testing.assert_array_equal(rec.words, words)
    assert rec.words.ctypes.data == buf.array.ctypes.data
    _, part = q.sample_shard(c, shots, 6, 2, 1, out=buf.array)
    kf = (shots + 63) // 64
    np.testing.assert_array_equal(part.words.reshape(len(meas), -1),
                                  words.reshape(len(meas), kf)[:, kf // 2:])
    with pytest.raises(ValueError):
        q.sample(c, shots, 6, out=buf.array[:10])
