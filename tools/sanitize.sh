#!/bin/bash
# compute-sanitizer over the smoke path (tiny workload: every kernel class once). usage (under gpurun): bash tools/sanitize.sh <tag>
tag=${1:-r02}
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python __graft_entry__.py smoke > gpurun_out/sanitizer_${tool}_$tag.log 2>&1
  echo "== $tool: exit $?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|smoke:" gpurun_out/sanitizer_${tool}_$tag.log | tail -4
done
# the headline shape (7 channels, 3 speakers + noise, WPE, 40 s window): the tcgen05 kernels and the M = 7, K = 4 sweep
for tool in memcheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/parity_probe.py cfg2 > gpurun_out/sanitizer_${tool}_cfg2_$tag.log 2>&1
  echo "== $tool cfg2: exit $?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|SDR" gpurun_out/sanitizer_${tool}_cfg2_$tag.log | tail -4
done
# the row-owner sweep (8 channels, 4 speakers + noise): exchange-buffer hand-overs between its three phases
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/parity_probe.py custom:8,4,3,2.0,1.5 > gpurun_out/sanitizer_${tool}_m8_$tag.log 2>&1
  echo "== $tool m8: exit $?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|SDR" gpurun_out/sanitizer_${tool}_m8_$tag.log | tail -4
done
