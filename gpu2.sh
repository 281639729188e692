mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
nproc; free -g | head -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -15
timeout 600 python bench.py --config c2 --steps 2 --warmup 1 --no-cpu 2>gpurun_out/bench_c2.err | tee gpurun_out/bench_c2.json
tail -5 gpurun_out/bench_c2.err
timeout 1200 python bench.py 2>gpurun_out/bench_c5.err | tee gpurun_out/bench_c5.json
tail -12 gpurun_out/bench_c5.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --config c2 --steps 1 --warmup 0 --e2e-steps 0 --no-cpu > /dev/null 2>&1; echo ncu1 $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gate_window -s 30 -c 1 -o gpurun_out/prof_gate_c5 python tools/profile_kernels.py --layers 60 --measure 0 > gpurun_out/ncu_gate.log 2>&1; echo ncu2 $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_rowmul -c 1 -o gpurun_out/prof_rowmul_c5 python tools/profile_kernels.py --layers 100 --measure 2 > gpurun_out/ncu_rowmul.log 2>&1; echo ncu3 $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_transpose -c 1 -o gpurun_out/prof_transpose_c5 python tools/profile_kernels.py --layers 4 --measure 1 > gpurun_out/ncu_tr.log 2>&1; echo ncu4 $?
ls -la gpurun_out
