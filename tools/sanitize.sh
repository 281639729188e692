#!/bin/bash
# compute-sanitizer over tools/sanitize_probe.py: memcheck, racecheck, synccheck (and initcheck),
# with programmatic dependent launches on (default) and off (QSR_PDL=0).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for pdl in 1 0; do
  for tool in memcheck racecheck synccheck initcheck; do
    echo "=== tool=$tool QSR_PDL=$pdl" >> gpurun_out/sanitize.log
    QSR_PDL=$pdl timeout 1200 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 \
        python tools/sanitize_probe.py >> gpurun_out/sanitize.log 2>&1
    echo "=== exit=$? tool=$tool QSR_PDL=$pdl" >> gpurun_out/sanitize.log
  done
done
grep "===\|SANITIZE PROBE\|ERROR SUMMARY\|Error" gpurun_out/sanitize.log | head -60
