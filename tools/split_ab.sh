#!/bin/bash
# sample(): frames on an SM partition (QSR_FRAMES_SMS) vs the shared GPU (0): parity + c4 bench.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/split
timeout 900 python -m pytest tests/test_gpu_engine_sample.py tests/test_gpu_fullsize.py -k "sample or c4" -m gpu -q -x \
    > gpurun_out/split/tests.log 2>&1; echo "rc=$?" >> gpurun_out/split/tests.log
for v in 96 0 64 112 80; do
  QSR_FRAMES_SMS=$v timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu --e2e-steps 0 \
      > gpurun_out/split/c4_$v.json 2> gpurun_out/split/c4_$v.err
done
for v in 96 0 64 112 80; do python -c "
import json
d=json.loads(open('gpurun_out/split/c4_$v.json').read().strip().splitlines()[-1])
print('$v', d['ms_per_step'], d['kernels']['frames_window']['ms_per_step'], d['kernels']['tableau_window']['ms_per_step'])
"; done
tail -3 gpurun_out/split/tests.log
