#!/bin/bash
# A/B: batch control words written by the sign pass into pinned memory (default) vs a copy +
# event per batch (QSR_HOSTPOLL=0): parity, c4 / c3 measure phases.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/hp
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_engine_sample.py \
    tests/test_gpu_fusion.py -m gpu -q -x > gpurun_out/hp/tests.log 2>&1; echo "rc=$?" >> gpurun_out/hp/tests.log
for v in 1 0 1 0; do
  QSR_HOSTPOLL=$v timeout 300 python tools/c4_probe.py 10000 500 100000 3 >> gpurun_out/hp/c4_$v.log 2>&1
  QSR_HOSTPOLL=$v timeout 300 python tools/c3_probe.py 50000 100 2 >> gpurun_out/hp/c3_$v.log 2>&1
done
for f in gpurun_out/hp/*.log; do echo "== $f"; grep -o "ge [0-9.]*\|measure_ms': [0-9.]*\|passed.*\|rc=.*" $f; done
