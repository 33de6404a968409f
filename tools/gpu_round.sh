#!/bin/bash
# One GPU visit: parity tests, smoke, the bench line (both arms), the ncu launch list and full captures of every
# kernel class. usage (under gpurun): bash tools/gpu_round.sh <tag>
tag=${1:-r02}
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt; lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/nproc.txt
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt
timeout 900 python -m pytest tests -m gpu -q --timeout 300 2>&1 | tail -15 > gpurun_out/test_$tag.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_$tag.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_$tag.log 2>&1
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref_$tag.log 2>&1
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --headline-only --workload ${WL:-cfg3} --segments ${SEGS:-16}"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches_$tag.csv \
  $B > gpurun_out/ncu_launch_$tag.log 2>&1
N="ncu --set full --clock-control none --import-source on"
timeout 900 $N -k regex:"em_pass" -s 70 -c 2 -o gpurun_out/prof_em_$tag $B > gpurun_out/ncu_em_$tag.log 2>&1
timeout 900 $N -k regex:"^stft512|wpe_" -c 5 -o gpurun_out/prof_wpe_$tag $B > gpurun_out/ncu_wpe_$tag.log 2>&1
timeout 900 $N -k regex:"em_update" -s 3 -c 1 -o gpurun_out/prof_upd_$tag $B > gpurun_out/ncu_upd_$tag.log 2>&1
timeout 900 $N -k regex:"beamform_apply|istft|mvdr_|select_reference" -c 5 -o gpurun_out/prof_tail_$tag $B > gpurun_out/ncu_tail_$tag.log 2>&1
for w in tiny cfg1 cfg2 cfg3 cfg4; do (timeout 300 python tools/parity_probe.py $w) >> gpurun_out/probe_$tag.log 2>&1; done
tail -3 gpurun_out/test_$tag.log; tail -2 gpurun_out/smoke_$tag.log; tail -c 700 gpurun_out/bench_$tag.log; tail -c 400 gpurun_out/bench_ref_$tag.log
