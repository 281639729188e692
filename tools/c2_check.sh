#!/bin/bash
# c2 end-to-end check: two bench runs and a QSR_TRACE run of the C-ABI call.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/c2
for i in 1 2; do
  timeout 600 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu > gpurun_out/c2/bench_$i.json 2> gpurun_out/c2/bench_$i.err
  grep "e2e" gpurun_out/c2/bench_$i.err
done
QSR_TRACE=1 timeout 300 python tools/e2e_trace.py 20000 1000 0.0 6 > gpurun_out/c2/trace.log 2>&1
tail -40 gpurun_out/c2/trace.log
