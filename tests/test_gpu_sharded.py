"""GPU parity of the generator-row-sharded engine.

All shards run in one process on one GPU (exchange="local"): the exact multi-GPU algorithm,
with the collectives as device copies, so the leader protocol, the pivot-block broadcast and
the shard-ordered deterministic fold are checked bit-for-bit against the CPU oracle
(run_single_shot<uint64_t>, simulator.hpp:46-76) at every world size. The NCCL transport
differs only in who moves the same bytes (exchange.cu).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def check_sharded(q, oracle, c, seed, worlds):
    n = c.num_qubits
    x, z, s, rec, _ = oracle.run_single_shot(n, c.gate_array, seed)
    k = (n + 63) // 64
    for w in worlds:
        if w > k:
            continue
        e = q.ShardedEngine(c, w)
        e.run(seed)
        np.testing.assert_array_equal(e.record(), rec, err_msg=f"record, world={w}")
        gx, gz, gs = e.tableau_planes()
        np.testing.assert_array_equal(gx, x, err_msg=f"x, world={w}")
        np.testing.assert_array_equal(gz, z, err_msg=f"z, world={w}")
        np.testing.assert_array_equal(gs, s, err_msg=f"s, world={w}")
    return rec


@pytest.mark.parametrize("seed", range(8))
def test_sharded_random(q, oracle, seed):
    n = 130 + (seed * 97) % 500
    depth = 5 + seed % 20
    p = [0.2, 0.5, 1.0, 0.7][seed % 4]
    c = q.generate_random(n, depth, seed * 13 + 3, p)
    check_sharded(q, oracle, c, seed, [1, 2, 3, 8])


@pytest.mark.parametrize("depth", [1, 2, 3])
def test_sharded_shallow_pivots_on_every_shard(q, oracle, depth):
    """Shallow circuits keep stabilizers local, so batch leaders are shards > 0 and the
    leader's batch is cut by lower shards' masks (shard.cpp leader protocol)."""
    n = 600
    c = q.generate_random(n, depth, 100 + depth, 1.0)
    check_sharded(q, oracle, c, 5, [2, 3, 4, 7])


def test_sharded_h_layer_reverse_measure(q, oracle):
    G = q.GateKind
    n = 520
    gates = [(G.H, i) for i in range(n)] + [(G.MEASURE, i) for i in reversed(range(n))]
    c = q.Circuit(n, gates)
    rec = check_sharded(q, oracle, c, 3, [2, 5, 9])
    assert rec["deterministic"].sum() == 0


@pytest.mark.parametrize("n", [200, 700])
def test_sharded_ghz_deterministic(q, oracle, n):
    """All but the first measurement become deterministic mid-window: the shard-ordered
    partial-product fold decides them."""
    G = q.GateKind
    gates = [(G.H, 0)] + [(G.CX, i, i + 1) for i in range(n - 1)] + [(G.MEASURE, i) for i in range(n)]
    c = q.Circuit(n, gates)
    rec = check_sharded(q, oracle, c, 1, [2, 3, 4])
    assert rec["deterministic"].tolist() == [0] + [1] * (n - 1)


def test_sharded_mid_circuit_segments(q, oracle):
    """c3 shape in small: segments of random layers, each ending in measure-all."""
    n = 400
    gates = np.concatenate([q.generate_random(n, 30, 1000 + r, 1.0).gate_array for r in range(3)])
    c = q.Circuit(n, gates)
    check_sharded(q, oracle, c, 7, [2, 4, 7])


def test_sharded_engine_rerun_and_world_equals_k(q, oracle):
    n = 320  # k = 5: world 5 puts one generator-word on each shard
    c = q.generate_random(n, 40, 9, 0.5)
    x, z, s, rec, _ = oracle.run_single_shot(n, c.gate_array, 4)
    e = q.ShardedEngine(c, 5)
    for _ in range(2):
        e.run(4)
        np.testing.assert_array_equal(e.record(), rec)
        gx, gz, gs = e.tableau_planes()
        np.testing.assert_array_equal(gx, x)
        np.testing.assert_array_equal(gs, s)


def test_sharded_errors(q):
    c = q.generate_random(100, 3, 1, 0.0)
    with pytest.raises(q.InvalidArgument):
        q.ShardedEngine(c, 3)  # k = 2 < world
    with pytest.raises(q.InvalidArgument):
        q.ShardedEngine(c, 0)


def test_sharded_nccl_transport_single_rank(q, oracle):
    """The NCCL transport itself (ncclCommInitRank / Broadcast / AllGather / AllReduce through
    libqsr's dynamically bound NCCL) on the one GPU available: world 1, rank 0."""
    n = 300
    c = q.generate_random(n, 30, 21, 1.0)
    x, z, s, rec, _ = oracle.run_single_shot(n, c.gate_array, 2)
    e = q.ShardedEngine(c, 1, exchange="nccl", rank=0, nccl_id=q.nccl_unique_id())
    e.run(2)
    np.testing.assert_array_equal(e.record(), rec)
    gx, gz, gs = e.tableau_planes()
    np.testing.assert_array_equal(gx, x)
    np.testing.assert_array_equal(gz, z)
    np.testing.assert_array_equal(gs, s)


def test_sharded_tableau_local_layout(q, oracle):
    """qsr_sharded_tableau_local: per local shard, n_pad rows x 2kg words (destabilizer words
    then stabilizer words) — the same words as the shard's columns of the full CM layout."""
    import ctypes as C
    from paper_2603_14641_b200 import _lib
    n, world = 300, 3
    c = q.generate_random(n, 20, 4, 0.5)
    x, z, s, _, _ = oracle.run_single_shot(n, c.gate_array, 6)
    e = q.ShardedEngine(c, world)
    e.run(6)
    k = (n + 63) // 64
    n_pad = 64 * k
    lx = np.zeros(n_pad * 2 * k, dtype=np.uint64)
    lz = np.zeros_like(lx)
    ls = np.zeros(2 * k, dtype=np.uint64)
    _lib.check(_lib.lib.qsr_sharded_tableau_local(e._h, _lib.ptr(lx, C.c_uint64), _lib.ptr(lz, C.c_uint64),
                                                  _lib.ptr(ls, C.c_uint64)))
    X, Z = x.reshape(n_pad, 2 * k), z.reshape(n_pad, 2 * k)
    xo = so = 0
    for r in range(world):
        j0, kg = q.shard_range(n, world, r)
        cols = list(range(j0, j0 + kg)) + list(range(k + j0, k + j0 + kg))
        blk = n_pad * 2 * kg
        np.testing.assert_array_equal(lx[xo:xo + blk].reshape(n_pad, 2 * kg), X[:, cols])
        np.testing.assert_array_equal(lz[xo:xo + blk].reshape(n_pad, 2 * kg), Z[:, cols])
        np.testing.assert_array_equal(ls[so:so + 2 * kg], s[cols])
        xo += blk
        so += 2 * kg


def test_sharded_nccl_engine_rebuilt_with_same_id(q):
    """bench.py rebuilds the NCCL-sharded engine with one ncclUniqueId (timed steps, then every
    e2e step): the communicator is reused, never re-initialised on the spent id (which would
    wait for the bootstrap root forever). Run in a subprocess under a timeout."""
    import subprocess
    import sys
    code = (
        "import sys, numpy as np\n"
        "sys.path.insert(0, '.')\n"
        "from paper_2603_14641_b200 import quasar as q\n"
        "c = q.generate_random(200, 20, 3, 0.5)\n"
        "uid = q.nccl_unique_id()\n"
        "recs = []\n"
        "for _ in range(3):\n"
        "    e = q.ShardedEngine(c, 1, exchange='nccl', rank=0, nccl_id=uid)\n"
        "    e.run(5)\n"
        "    recs.append(e.record())\n"
        "    del e\n"
        "assert all(np.array_equal(r, recs[0]) for r in recs)\n"
        "print('ok')\n")
    root = __import__("pathlib").Path(__file__).resolve().parents[1]
    out = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    assert "ok" in out.stdout


@pytest.mark.parametrize("shots", [64, 130, 1000, 4100])
def test_sample_sharded_by_shot(q, oracle, shots):
    """Sampling sharded by shot-word (one rank per GPU in production): the ranks' record
    slices concatenated word-wise equal the oracle's ShotRecord (frames.hpp:163-204)."""
    n = 70
    c = q.generate_random(n, 15, 5, 0.6)
    meas, words, _ = oracle.sample(n, c.gate_array, shots, 99)
    kf = (shots + 63) // 64
    rows = len(meas)
    full = np.asarray(words, dtype=np.uint64).reshape(rows, kf)
    for world in [1, 2, 3, 5]:
        if world > kf:
            continue
        got = np.zeros((rows, kf), dtype=np.uint64)
        for rank in range(world):
            w0, rec = q.sample_shard(c, shots, 99, world, rank)
            assert rec.measured == [int(v) for v in meas]
            nw = rec.kf
            got[:, w0:w0 + nw] = np.asarray(rec.words, dtype=np.uint64).reshape(rows, nw)
        np.testing.assert_array_equal(got, full, err_msg=f"world={world}")


@pytest.mark.parametrize("exchange", ["local", "nccl"])
@pytest.mark.parametrize("case", ["final", "segments"])
def test_sharded_streamed_run_circuit(q, oracle, exchange, case):
    """qsr_sharded_run_circuit: the streamed driver (planning + fusion + upload overlapped with the
    device) on this process's shard, measurement windows through the sharded protocol — the N > 1
    e2e path of bench.py, exercised here at world 1 (one GPU)."""
    n = 300
    if case == "final":
        c = q.generate_random(n, 40, 31, 0.5)
    else:  # mid-circuit measure-all windows between unitary segments
        c = q.Circuit(n, np.concatenate([q.generate_random(n, 20, 40 + r, 1.0).gate_array for r in range(3)]))
    x, z, s, rec, _ = oracle.run_single_shot(n, c.gate_array, 5)
    kw = dict(rank=0, nccl_id=q.nccl_unique_id()) if exchange == "nccl" else {}
    e = q.ShardedEngine(c, 1, exchange=exchange, streamed_seed=5, **kw)
    assert e.device_ms > 0
    np.testing.assert_array_equal(e.record(), rec)
    gx, gz, gs = e.tableau_planes()
    np.testing.assert_array_equal(gx, x)
    np.testing.assert_array_equal(gz, z)
    np.testing.assert_array_equal(gs, s)
    with pytest.raises(q.InvalidArgument):  # a resident-engine call on a streamed object
        e.run(5)


def test_sharded_streamed_needs_one_shard_per_process(q):
    c = q.generate_random(200, 5, 1, 0.5)
    with pytest.raises(q.InvalidArgument):
        q.ShardedEngine(c, 2, exchange="local", streamed_seed=1)
