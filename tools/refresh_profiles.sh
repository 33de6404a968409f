#!/bin/bash
# gpurun_out/ (scratch) of `tools/gpu_round.sh <tag>` -> the tracked summaries under profiles/
# (the ncu reports are summarised on the GPU box: gpurun brings back at most 64 MiB)
tag=${1:-r02}
python tools/ncu_summary.py launches gpurun_out/launches_$tag.csv profiles/ncu_launches_$tag.md | tail -1
sed 's/ %% / % /g' gpurun_out/ncu_full_$tag.md > profiles/ncu_full_$tag.md
cp gpurun_out/ncu_traffic_$tag.json profiles/ncu_traffic_$tag.json
cp gpurun_out/ncu_stalls_$tag.txt profiles/ncu_stalls_$tag.txt
python - "$tag" <<'PY'
import json, sys
tag = sys.argv[1]
for src, dst in (("bench", "bench"), ("bench_ref", "bench_reference")):
    d = json.loads([l for l in open(f"gpurun_out/{src}_{tag}.log") if l.startswith("{")][-1])
    json.dump(d, open(f"profiles/{dst}_{tag}.json", "w"), indent=1)
    print(dst, d["value"], d.get("ms_per_step"), d.get("e2e"))
    if src == "bench":
        print({k: v["ms_per_step"] for k, v in d["kernels"].items()}, d["roofline"]["frac"], d["cpu_baseline"]["value"])
        print({k: (v["value"], v["ms_per_step"], v["e2e"]["value"]) for k, v in d["configs"].items()})
PY
cp gpurun_out/probe_$tag.log profiles/parity_probe_$tag.log
cp gpurun_out/parity_tests_$tag.log profiles/parity_tests_$tag.log
(cat gpurun_out/gpu.txt gpurun_out/nproc.txt) > profiles/box_$tag.txt
tail -3 gpurun_out/test_$tag.log; tail -2 gpurun_out/smoke_$tag.log
