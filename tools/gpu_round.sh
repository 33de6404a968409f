#!/bin/bash
# One GPU visit: parity tests, smoke, the bench line, the ncu launch list and full captures of the hot kernels.
# usage (under gpurun): bash tools/gpu_round.sh <tag> [full]
tag=${1:-r01}
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt; lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/nproc.txt
timeout 900 python -m pytest tests -m gpu -q --timeout 300 2>&1 | tail -15 > gpurun_out/test_$tag.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_$tag.log 2>&1
if [ "$2" = "full" ]; then
  timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_$tag.log 2>&1
else
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$tag.log 2>&1
fi
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches_$tag.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_$tag.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"em_pass" -s 70 -c 2 -o gpurun_out/prof_em_$tag \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_em_$tag.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"wpe_|stft_kernel|istft_kernel|em_update|beamform_apply" -s 12 -c 14 -o gpurun_out/prof_misc_$tag \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_misc_$tag.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ffma2_probe tools/ffma2_probe.cu && timeout 120 /tmp/ffma2_probe > gpurun_out/ffma2_probe.log 2>&1
(timeout 300 python tools/parity_probe.py cfg1) > gpurun_out/probe_$tag.log 2>&1
tail -3 gpurun_out/test_$tag.log; tail -2 gpurun_out/smoke_$tag.log; tail -c 600 gpurun_out/bench_$tag.log
