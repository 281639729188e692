#!/bin/bash
# Batch-chain change check: the measurement-path GPU tests (incl. scale parity), c4 / c3 benches.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/cc
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_sharded.py \
    tests/test_gpu_engine_sample.py tests/test_gpu_fusion.py tests/test_gpu_scale.py tests/test_gpu_fullsize.py \
    -m gpu -q -x > gpurun_out/cc/tests.log 2>&1; echo "rc=$?" >> gpurun_out/cc/tests.log
timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu > gpurun_out/cc/c4.json 2> gpurun_out/cc/c4.err
timeout 900 python bench.py --config c3 --steps 2 --warmup 2 --no-cpu > gpurun_out/cc/c3.json 2> gpurun_out/cc/c3.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"signs" -c 100 --csv \
    --log-file gpurun_out/cc/ncu_signs_c4.csv python tools/c4_probe.py 10000 500 1000 1 > /dev/null 2>&1
tail -3 gpurun_out/cc/tests.log
