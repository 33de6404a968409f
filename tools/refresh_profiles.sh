#!/bin/bash
# gpurun_out/ (scratch) of `tools/gpu_round.sh <tag>` -> the tracked summaries under profiles/
tag=${1:-r01}
python tools/ncu_summary.py launches gpurun_out/launches_$tag.csv profiles/ncu_launches_$tag.md | tail -1
python tools/ncu_summary.py full gpurun_out/prof_em_$tag.ncu-rep gpurun_out/prof_wpe_$tag.ncu-rep gpurun_out/prof_upd_$tag.ncu-rep \
  gpurun_out/prof_tail_$tag.ncu-rep --segments 16 --out profiles/ncu_full_$tag.md --traffic profiles/ncu_traffic_$tag.json | tail -1
python - "$tag" <<'PY'
import json, sys
tag = sys.argv[1]
for src, dst in (("bench", "bench"), ("bench_ref", "bench_reference")):
    d = json.loads([l for l in open(f"gpurun_out/{src}_{tag}.log") if l.startswith("{")][-1])
    json.dump(d, open(f"profiles/{dst}_{tag}.json", "w"), indent=1)
    print(dst, d["value"], d.get("ms_per_step"), d.get("e2e"))
    if src == "bench":
        print({k: v["ms_per_step"] for k, v in d["kernels"].items()}, d["roofline"]["frac"], d["cpu_baseline"]["value"])
PY
cp gpurun_out/probe_$tag.log profiles/parity_probe_$tag.log
tail -3 gpurun_out/test_$tag.log; tail -2 gpurun_out/smoke_$tag.log
