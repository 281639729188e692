mkdir -p gpurun_out/val
python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/val/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/val/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/val/smoke.log 2>&1
for c in c5 c3 c4 c2 c1; do python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/val/bench_$c.json 2> gpurun_out/val/bench_$c.err; done
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/val/bench_ref.json 2> gpurun_out/val/bench_ref.err
python bench.py > gpurun_out/val/bench_default.json 2> gpurun_out/val/bench_default.err
# launch lists (ncu, serialised, cold caches: per-kernel shares, not bench numbers)
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --metrics $M --clock-control none -c 3200 --csv --log-file gpurun_out/val/launches_c3seg.csv \
    python tools/c3_probe.py 50000 100 1 > /dev/null 2>&1
timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/val/launches_c4.csv \
    python tools/c4_probe.py 10000 500 100000 1 > /dev/null 2>&1
timeout 1800 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/val/launches_c5.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu --no-profile --e2e-steps 0 > /dev/null 2>&1
for f in c3seg c4 c5; do python tools/summarize_launches.py gpurun_out/val/launches_$f.csv gpurun_out/val/launches_${f}_summary.csv > /dev/null 2>&1; gzip -f gpurun_out/val/launches_$f.csv; done
