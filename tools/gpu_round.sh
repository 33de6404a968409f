#!/bin/bash
# One GPU visit: parity tests, smoke, the bench line (both arms), the ncu launch list and full captures of every
# kernel class. usage (under gpurun): bash tools/gpu_round.sh <tag>
tag=${1:-r02}
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt; lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/nproc.txt
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 2>&1 | tail -15 > gpurun_out/test_$tag.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_$tag.log 2>&1
timeout 1500 python bench.py > gpurun_out/bench_$tag.log 2>&1
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref_$tag.log 2>&1
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --headline-only --workload ${WL:-cfg3} --segments ${SEGS:-16}"
# the launch list of the headline command itself (64 segments per step; the configs block is left out)
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches_$tag.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --headline-only > gpurun_out/ncu_launch_$tag.log 2>&1
N="ncu --set full --clock-control none --import-source on"
P=/tmp/gss_prof_$tag; rm -rf $P; mkdir -p $P   # reports stay on the box (gpurun brings back at most 64 MiB): summaries travel
timeout 900 $N -k regex:"em_pass" -s 70 -c 2 -o $P/prof_em_$tag $B > gpurun_out/ncu_em_$tag.log 2>&1
timeout 900 $N -k regex:"^stft512|wpe_" -c 5 -o $P/prof_wpe_$tag $B > gpurun_out/ncu_wpe_$tag.log 2>&1
timeout 900 $N -k regex:"em_update" -s 3 -c 1 -o $P/prof_upd_$tag $B > gpurun_out/ncu_upd_$tag.log 2>&1
timeout 900 $N -k regex:"beamform_apply|istft|mvdr_|select_reference" -c 5 -o $P/prof_tail_$tag $B > gpurun_out/ncu_tail_$tag.log 2>&1
# the two-phase sweep (M = 7) on the cfg2 shape
timeout 900 $N -k regex:"em_pass" -s 70 -c 1 -o $P/prof_em7_$tag python bench.py --steps 1 --warmup 3 --no-cpu-baseline --headline-only --workload cfg2 > gpurun_out/ncu_em7_$tag.log 2>&1
python tools/ncu_summary.py full $P/prof_em_$tag.ncu-rep $P/prof_wpe_$tag.ncu-rep $P/prof_upd_$tag.ncu-rep $P/prof_tail_$tag.ncu-rep \
  --segments ${SEGS:-16} --label "${WL:-cfg3}" --out gpurun_out/ncu_full_$tag.md --traffic gpurun_out/ncu_traffic_$tag.json > /dev/null 2>&1
(python tools/ncu_stalls.py $P/prof_em_$tag.ncu-rep; python tools/ncu_stalls.py $P/prof_em7_$tag.ncu-rep; python tools/ncu_stalls.py $P/prof_wpe_$tag.ncu-rep wpe_gram; python tools/ncu_stalls.py $P/prof_wpe_$tag.ncu-rep wpe_solve; python tools/ncu_stalls.py $P/prof_wpe_$tag.ncu-rep wpe_apply) > gpurun_out/ncu_stalls_$tag.txt 2>&1
cp $P/prof_em_$tag.ncu-rep $P/prof_em7_$tag.ncu-rep gpurun_out/ 2>/dev/null
timeout 900 python tools/parity_math.py cfg1 cfg2 2>&1 | grep "^\[" > gpurun_out/parity_math_$tag.log
timeout 1500 python -m pytest tests/test_gpu_enhance.py tests/test_synthbench.py -m gpu -q -s --timeout 900 2>&1 | grep -E "\[sweep|\[cfg|\[tiny|\[ragged|criterion|passed|failed" | cut -c1-400 > gpurun_out/parity_tests_$tag.log
for w in tiny cfg1 cfg2 cfg3 cfg4; do (timeout 300 python tools/parity_probe.py $w) >> gpurun_out/probe_$tag.log 2>&1; done
tail -3 gpurun_out/test_$tag.log; tail -2 gpurun_out/smoke_$tag.log; tail -c 700 gpurun_out/bench_$tag.log; tail -c 400 gpurun_out/bench_ref_$tag.log
