#!/bin/bash
# ncu --set full captures of the batch chain's select and absorb kernels (c4 and c3 shapes).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/ncu
QSR_SELECT=0 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_pivot_select" -s 100 -c 1 \
    -o gpurun_out/ncu/select_c4_s0 python tools/c4_probe.py 10000 500 1000 1 > gpurun_out/ncu/select_c4_s0.log 2>&1
QSR_SELECT=16 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_pivot_select" -s 100 -c 1 \
    -o gpurun_out/ncu/select_c4_s16 python tools/c4_probe.py 10000 500 1000 1 > gpurun_out/ncu/select_c4_s16.log 2>&1
QSR_ABSORB=4 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_batch_absorb" -s 100 -c 1 \
    -o gpurun_out/ncu/absorb_c3_a4 python tools/c3_probe.py 50000 100 1 > gpurun_out/ncu/absorb_c3_a4.log 2>&1
QSR_ABSORB=7 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_batch_absorb" -s 100 -c 1 \
    -o gpurun_out/ncu/absorb_c3_a7 python tools/c3_probe.py 50000 100 1 > gpurun_out/ncu/absorb_c3_a7.log 2>&1
QSR_TRACE=1 timeout 300 python tools/c4_e2e_trace.py > gpurun_out/ncu/c4_e2e_trace.log 2>&1
timeout 300 python tools/c4_probe.py 10000 500 100000 3 > gpurun_out/ncu/c4_prio.log 2>&1
ls -la gpurun_out/ncu
