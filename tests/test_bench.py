"""bench.py contract pieces that run without a GPU: the reference arm (`--impl reference`) runs
the reference CPU path only — the process must never map the product library (libqsr.so)."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]

PROBE = """
import contextlib, io, json, runpy, sys
sys.argv = ['bench.py', '--impl', 'reference', '--config', 'c1', '--steps', '2', '--warmup', '1']
buf = io.StringIO()
with contextlib.redirect_stdout(buf):
    runpy.run_path('bench.py', run_name='__main__')
maps = open('/proc/self/maps').read()
print(json.dumps({'line': buf.getvalue().strip().splitlines()[-1], 'libqsr': 'libqsr' in maps,
                  'ref': 'libquasar_ref' in maps}))
"""


def test_reference_arm_never_loads_the_product_library():
    from oracle.oracle import available
    if not available("reference") and not available("port"):
        pytest.skip("no oracle library built")
    r = subprocess.run([sys.executable, "-c", PROBE], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["libqsr"] is False
    line = json.loads(out["line"])
    assert line["impl"] == "reference" and line["unit"] == "gates/s" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["cores"] >= 1
    assert "CPU gate-window sample" in line["config"]["step"]


def test_reference_arm_other_ranks_exit_without_work():
    import os
    env = dict(os.environ, RANK="1", WORLD_SIZE="2")
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "c1"], cwd=ROOT,
                       env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.strip() == ""
