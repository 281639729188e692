# End-of-round evidence: the whole -m gpu suite, smoke(), and the bench line of every config
# plus the reference arm (the driver's own sequence), into gpurun_out/val3/.
mkdir -p gpurun_out/val3
python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/val3/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/val3/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/val3/smoke.log 2>&1
python bench.py --impl reference > gpurun_out/val3/bench_ref.json 2> gpurun_out/val3/bench_ref.err
python bench.py > gpurun_out/val3/bench_default.json 2> gpurun_out/val3/bench_default.err
for c in c3 c4 c2 c1; do python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/val3/bench_$c.json 2> gpurun_out/val3/bench_$c.err; done
