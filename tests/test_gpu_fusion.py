"""Gate fusion (csrc/fuse.cpp) parity: SWAP / ISWAP relabelling, single-qubit runs folded into the
next two-qubit gate, flushes before measurement windows, and the row un-permutation — against the
CPU oracle, through both whole-circuit paths (streaming run_single_shot and the resident Engine).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

K = dict(X=0, Y=1, Z=2, H=3, S=4, SDG=5, CX=6, CY=7, CZ=8, SWAP=9, ISWAP=10, M=11)


def layered(n, depth, seed, p_two, p_swap, p_meas_layer, p_meas):
    """Random layered circuit with a tunable share of SWAP / ISWAP and single-qubit runs, and
    measurement layers in the middle (each measuring a random subset once)."""
    rng = np.random.default_rng(seed)
    gates = []
    for layer in range(depth):
        perm = rng.permutation(n)
        i = 0
        while i < n:
            if i + 1 < n and rng.random() < p_two:
                a, b = int(perm[i]), int(perm[i + 1])
                r = rng.random()
                kind = (K["SWAP"] if r < p_swap / 2 else K["ISWAP"] if r < p_swap
                        else int(rng.choice([K["CX"], K["CY"], K["CZ"]])))
                gates.append((kind, a, b))
                i += 2
            else:
                gates.append((int(rng.integers(0, 6)), int(perm[i])))
                i += 1
        if layer + 1 < depth and rng.random() < p_meas_layer:  # (a qubit measured twice in one
            # window is the reference's invalid_argument, measure.hpp:394-395: see below)
            for q in range(n):
                if rng.random() < p_meas:
                    gates.append((K["M"], q))
    for q in range(n):
        if rng.random() < 0.5:
            gates.append((K["M"], q))
    return gates


CASES = [
    dict(n=70, depth=40, seed=1, p_two=0.5, p_swap=0.8, p_meas_layer=0.0, p_meas=0.0),
    dict(n=130, depth=30, seed=2, p_two=0.3, p_swap=0.5, p_meas_layer=0.2, p_meas=0.3),
    dict(n=200, depth=60, seed=3, p_two=0.1, p_swap=0.9, p_meas_layer=0.1, p_meas=0.5),
    dict(n=65, depth=80, seed=4, p_two=0.7, p_swap=1.0, p_meas_layer=0.3, p_meas=0.2),
    dict(n=257, depth=25, seed=5, p_two=0.05, p_swap=0.5, p_meas_layer=0.5, p_meas=0.1),
]


@pytest.mark.parametrize("case", CASES, ids=[f"n{c['n']}s{c['seed']}" for c in CASES])
def test_fused_paths_match_oracle(q, oracle, case):
    n = case["n"]
    c = q.Circuit(n, layered(**case))
    x, z, s, rec, _ = oracle.run_single_shot(n, c.gate_array, 9)
    r = q.run_single_shot(c, 9)                       # streaming driver, fused
    gx, gz, gs = r.tableau.planes()
    np.testing.assert_array_equal(r.record_array, rec)
    np.testing.assert_array_equal(gx, x)
    np.testing.assert_array_equal(gz, z)
    np.testing.assert_array_equal(gs, s)
    e = q.Engine(c)                                   # resident engine, fused schedule
    e.run(9)
    np.testing.assert_array_equal(e.record(), rec)
    ex, ez, es = e.tableau_planes(n)
    np.testing.assert_array_equal(ex, x)
    np.testing.assert_array_equal(ez, z)
    np.testing.assert_array_equal(es, s)
    sh = q.ShardedEngine(c, 2 if n >= 128 else 1)     # sharded engine, fused schedule
    sh.run(9)
    np.testing.assert_array_equal(sh.record(), rec)
    hx, hz, hs = sh.tableau_planes()
    np.testing.assert_array_equal(hx, x)
    np.testing.assert_array_equal(hs, s)


def test_fusion_moves_fewer_bytes(q):
    """The fused schedule of a SWAP-heavy circuit moves far fewer bytes than its unfused form."""
    import os
    import subprocess
    import sys
    code = (
        "import sys; sys.path.insert(0, '.')\n"
        "from paper_2603_14641_b200 import quasar as q\n"
        "c = q.generate_random(2000, 30, 5, 0.0)\n"
        "e = q.Engine(c); e.run(1); print(e.stats()['gate_bytes'])\n")
    root = __import__("pathlib").Path(__file__).resolve().parents[1]
    out = {}
    for fuse in ("1", "0"):
        env = dict(os.environ, QSR_FUSE=fuse)
        r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True,
                           timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        out[fuse] = float(r.stdout.strip().splitlines()[-1])
    assert out["1"] < 0.7 * out["0"], out


def test_duplicate_measurement_raises_like_reference(q, oracle):
    """Two measurements of one qubit landing in one window: every path raises invalid_argument."""
    G = q.GateKind
    gates = [(G.H, 0), (G.CX, 0, 1), (G.MEASURE, 0), (G.MEASURE, 0)]
    c = q.Circuit(2, gates)
    from oracle.oracle import OracleError
    with pytest.raises(OracleError):
        oracle.run_single_shot(2, c.gate_array, 1)
    with pytest.raises(q.InvalidArgument):
        q.run_single_shot(c, 1)
    with pytest.raises(q.InvalidArgument):
        q.Engine(c)
