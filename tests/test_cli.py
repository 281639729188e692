"""`quasar` CLI (paper_2603_14641_b200/bin/quasar) — the reference's tools/quasar.cpp on the B200
engine — plus the word-size-generic sampler and the device group-validity check.

CPU tests cover the commands that need no GPU (gen, schedule, usage errors, exit codes). GPU tests
compare run / sample outputs with the reference (oracle/_ref) on the same circuit and seeds, and
run verify / bench end to end.
"""
import json
import subprocess
from pathlib import Path

import numpy as np
import pytest

from oracle.oracle import Oracle, available

ROOT = Path(__file__).resolve().parents[1]
CLI = ROOT / "paper_2603_14641_b200" / "bin" / "quasar"
needs_ref = pytest.mark.skipif(not available("reference"), reason="oracle/_ref not built")
needs_cli = pytest.mark.skipif(not CLI.exists(), reason="CLI not built (python paper_2603_14641_b200/build.py)")


def cli(*args, check=True):
    p = subprocess.run([str(CLI), *map(str, args)], capture_output=True, timeout=600)
    if check and p.returncode != 0:
        raise AssertionError(f"quasar {' '.join(map(str, args))} -> {p.returncode}\n{p.stderr.decode()}")
    return p


@pytest.fixture(scope="module")
def ref():
    return Oracle("reference")


def write_qasm(q, tmp_path, n, depth, seed, p, name="c.qasm"):
    c = q.generate_random(n, depth, seed, p)
    path = tmp_path / name
    path.write_text(q.emit_qasm(c))
    return c, path


# ---- CPU ------------------------------------------------------------------------------------

@needs_cli
@needs_ref
@pytest.mark.parametrize("n,depth,seed,p", [(16, 16, 0, 0.1), (5, 3, 4, 0.5), (70, 9, 123, 1.0)])
def test_gen_matches_reference(q, ref, n, depth, seed, p):
    out = cli("gen", "--qubits", n, "--depth", depth, "--seed", seed, "--measure-prob", p).stdout.decode()
    gates = ref.generate_random(n, depth, seed, p)
    assert out == ref.emit_qasm(n, gates)


@needs_cli
def test_gen_out_file_and_defaults(q, tmp_path):
    path = tmp_path / "d.qasm"
    cli("gen", "--out", path)
    # defaults of tools/quasar.cpp:286-289: 16 qubits, depth 16, seed 0, measure-prob 0.1
    assert path.read_text() == q.emit_qasm(q.generate_random(16, 16, 0, 0.1))


@needs_cli
@needs_ref
def test_schedule_matches_reference(q, ref, tmp_path):
    c, path = write_qasm(q, tmp_path, 40, 20, 9, 0.5)
    out = cli("schedule", path).stdout.decode()
    assert out == ref.schedule_text(40, c.gate_array, 0)


@needs_cli
@pytest.mark.parametrize("args,code", [
    ([], 106), (["bogus"], 109), (["run"], 106), (["gen", "--qubits", "0"], 105),
    (["gen", "--measure-prob", "1.5"], 105), (["gen", "--qubits", "x"], 104),
    (["sample", "f.qasm", "--format", "xml"], 105), (["sample", "f.qasm", "--shots", "0"], 105),
    (["run", "f.qasm", "--word-size", "12"], 105), (["gen", "--nope", "1"], 109),
    (["run", "/nonexistent/in.qasm"], 2),
])
def test_usage_and_input_errors(args, code):
    p = cli(*args, check=False)
    assert p.returncode == code, p.stderr.decode()


@needs_cli
def test_parse_error_exit_code(tmp_path):
    bad = tmp_path / "bad.qasm"
    bad.write_text("OPENQASM 2.0;\nqreg q[1];\nt q[0];\n")
    p = cli("schedule", bad, check=False)
    assert p.returncode == 2
    assert "qasm:3:2: unsupported gate or statement 't'" in p.stderr.decode()


@needs_cli
def test_help_and_verify_vacuous():
    assert cli("--help").returncode == 0
    p = cli("verify", "--trials", "0")
    assert p.stdout.decode().endswith("verify=pass (vacuous)\n")


# ---- GPU ------------------------------------------------------------------------------------

def report_lines(text):
    return dict(line.split("=", 1) for line in text.strip().split("\n") if "=" in line)


def per_qubit_bits(rec):
    last, order = {}, []
    for e in rec:
        qb = int(e["qubit"])
        if qb not in last:
            order.append(qb)
        last[qb] = int(e["outcome"])
    return "".join(str(last[qb]) for qb in order)


@pytest.mark.gpu
@needs_cli
@pytest.mark.parametrize("n,depth,seed,p,run_seed", [(30, 20, 3, 1.0, 7), (200, 40, 5, 0.3, 11), (8, 4, 1, 0.0, 2)])
def test_run_matches_reference(q, oracle, tmp_path, n, depth, seed, p, run_seed):
    c, path = write_qasm(q, tmp_path, n, depth, seed, p)
    jpath = tmp_path / "r.json"
    out = cli("run", path, "--seed", run_seed, "--json", jpath).stdout.decode()
    _, _, _, rec, rep = oracle.run_single_shot(n, c.gate_array, run_seed)
    kv = report_lines(out)
    if len(rec):
        assert kv["outcomes"] == per_qubit_bits(rec)
    else:
        assert "outcomes" not in kv
    assert int(kv["qubits"]) == n and int(kv["gates"]) == rep.gate_count
    assert int(kv["measures"]) == rep.measure_count and int(kv["windows"]) == rep.window_count
    assert int(kv["probabilistic"]) == rep.probabilistic_count
    j = json.loads(jpath.read_text())
    assert list(j) == sorted(j)  # nlohmann object order
    assert j["gates"] == rep.gate_count and j["qubits"] == n
    # --out and other word sizes: identical outcome file
    o64, o8 = tmp_path / "o64", tmp_path / "o8"
    cli("run", path, "--seed", run_seed, "--out", o64)
    cli("run", path, "--seed", run_seed, "--out", o8, "--word-size", 8)
    assert o64.read_text() == o8.read_text() == (per_qubit_bits(rec) + "\n" if len(rec) else "")


@pytest.mark.gpu
@needs_cli
@needs_ref
@pytest.mark.parametrize("wbits", [8, 16, 32, 64])
def test_sample_formats_match_reference(q, ref, tmp_path, wbits):
    n, shots, seed = 24, 1000, 5
    c, path = write_qasm(q, tmp_path, n, 15, 77, 0.6)
    measured, kf, rows = ref.sample_w(n, c.gate_array, shots, seed, wbits)
    b = tmp_path / "s.bin"
    cli("sample", path, "--shots", shots, "--seed", seed, "--word-size", wbits, "--format", "binary", "--out", b)
    assert b.read_bytes() == rows.tobytes()
    t = tmp_path / "s.txt"
    cli("sample", path, "--shots", shots, "--seed", seed, "--word-size", wbits, "--out", t)
    lines = t.read_text().split("\n")
    assert len(lines) == shots + 1 and lines[-1] == ""
    bits = np.unpackbits(rows, axis=1, bitorder="little")[:, :shots]  # [rows, shots]
    want = ["".join("1" if bits[r, s] else "0" for r in range(len(measured))) for s in range(shots)]
    assert lines[:-1] == want


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("wbits,shots", [(8, 1), (8, 777), (16, 4097), (32, 100), (64, 130)])
def test_sample_word_sizes_api(q, ref, wbits, shots):
    n = 12
    c = q.generate_random(n, 10, 31, 1.0)
    rec = q.sample(c, shots, 9, word_bits=wbits)
    measured, kf, rows = ref.sample_w(n, c.gate_array, shots, 9, wbits)
    assert rec.measured == list(measured)
    assert np.array_equal(rec.row_bytes(wbits), rows)


@pytest.mark.gpu
@needs_cli
def test_verify_passes():
    p = cli("verify", "--trials", 12, "--n-max", 40, "--depth-max", 20, "--seed", 3)
    out = p.stdout.decode()
    assert out.endswith("verify=pass\n") and "failures=0" in out
    kv = report_lines(out)
    assert int(kv["differential_trials"]) == 12 and int(kv["statistical_trials"]) >= 1


@pytest.mark.gpu
@needs_cli
def test_bench_table(tmp_path):
    out = cli("bench", "--qubits", 300, "--depth", 30, "--reps", 3, "--measure-prob", 0.2).stdout.decode()
    lines = out.strip().split("\n")
    assert lines[0] == "rep\tto_ms\tt_ms\tcmp_ms\tge_ms\ttotal_ms"
    assert [l.split("\t")[0] for l in lines[1:]] == ["0", "1", "2", "median"]
    assert all(len(l.split("\t")) == 6 for l in lines[1:])


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("n,depth,p", [(1, 3, 1.0), (63, 20, 0.5), (130, 30, 0.3), (300, 25, 0.1)])
def test_group_validity_valid(q, ref, n, depth, p):
    c = q.generate_random(n, depth, n, p)
    r = q.run_single_shot(c, 4)
    t = r.tableau
    x, z, s = t.planes()
    assert q.check_group_validity(t) == "valid" == ref.check_validity(n, int(t.layout()), x, z)
    # the check leaves the tableau untouched
    x2, z2, s2 = t.planes()
    assert np.array_equal(x, x2) and np.array_equal(z, z2) and np.array_equal(s, s2)


@pytest.mark.gpu
@needs_ref
def test_group_validity_first_violation_matches_reference(q, ref):
    import random
    rng = random.Random(5)
    for trial in range(40):
        n = rng.choice([3, 17, 64, 90, 150])
        c = q.generate_random(n, 10, trial, 0.5)
        x, z, s = q.run_single_shot(c, trial).tableau.planes()
        x, z = x.copy(), z.copy()
        for _ in range(rng.randint(1, 3)):  # flip random tableau bits (real qubit rows only)
            plane = x if rng.random() < 0.5 else z
            k = (n + 63) // 64
            qb, j = rng.randrange(n), rng.randrange(2 * k)
            plane[qb * 2 * k + j] ^= np.uint64(1) << np.uint64(rng.randrange(64 if (j % k) < k - 1 else (n - 64 * (k - 1))))
        t = q.Tableau.from_planes(n, x, z, s)
        assert q.check_group_validity(t) == ref.check_validity(n, 0, x, z)
