#!/bin/bash
# usage (under gpurun): [WL=cfg3 SEGS=16] bash tools/exp_bench.sh tag1 tag2 ...   ("base" = the product library)
mkdir -p gpurun_out
WL=${WL:-cfg2}; SEGS=${SEGS:-16}
for tag in "$@"; do
  if [ "$tag" = base ]; then unset GSS_B200_LIB; else export GSS_B200_LIB=$PWD/paper_2212_05271_b200/lib/libgss_b200_$tag.so; fi
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --headline-only --workload $WL --segments $SEGS > gpurun_out/exp_$tag.log 2>&1
  python - "$tag" <<'PY'
import json, sys
tag = sys.argv[1]
try:
    d = json.loads([l for l in open(f"gpurun_out/exp_{tag}.log") if l.startswith("{")][-1])
    print(tag, "xRT", d["value"], "ms/step", d["ms_per_step"], "e2e", d["e2e"]["ms_per_step"], {k: v["ms_per_step"] for k, v in d["kernels"].items()}, d["failures"][:1])
except Exception as e:
    print(tag, "FAILED", e); print(open(f"gpurun_out/exp_{tag}.log").read()[-1500:])
PY
done
