#!/usr/bin/env python
"""Turns ncu output brought back in gpurun_out/ into the tracked summaries under profiles/.

    python tools/ncu_summary.py launches gpurun_out/launches_X.csv profiles/ncu_launches_rNN.md
    python tools/ncu_summary.py full gpurun_out/prof_A.ncu-rep [gpurun_out/prof_B.ncu-rep ...] \
        --segments 16 --out profiles/ncu_full_rNN.md --traffic profiles/ncu_traffic_r01.json

`launches`: per-kernel-class share of one bench step from the `--metrics gpu__time_duration.sum` pass
(cold-cache, serialised launches: the SHARE is what must agree with bench.py, not the absolute).
`full`: one row per captured launch from `--set full` reports: duration, DRAM bytes, pipe utilisation,
occupancy, registers; also writes the per-kernel-class DRAM traffic bench.py reports as roofline.traffic.
Test/measurement infrastructure, not product code.
"""
import argparse
import collections
import csv
import io
import json
import re
import subprocess
import sys

CLASSES = [("stft", r"^stft"), ("istft", r"^istft"), ("wpe_power", r"wpe_power"),
           ("wpe_gram", r"wpe_gram"), ("wpe_solve", r"wpe_solve"), ("wpe_apply", r"wpe_apply"),
           ("em_pass", r"em_pass"), ("em_update", r"em_update_kernel"),
           ("mvdr", r"mvdr_|select_reference"), ("apply", r"beamform_apply"), ("em_ll_sum", r"sum_ll"),
           ("bench_fp32_peak_probe (not part of a step)", r"fma_peak"), ("other", r".")]


def classify(name):
    base = name.split("(")[0].replace("void ", "").replace("gssb::", "")
    for c, pat in CLASSES:
        if re.search(pat, base):
            return c
    return "other"


def launches(path, out):
    rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    per = collections.OrderedDict()
    total = 0.0
    for r in rows[1:]:
        if r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        ns = float(r[ix["Metric Value"]].replace(",", ""))
        if r[ix["Metric Unit"]] in ("us", "usecond"):
            ns *= 1e3
        c = classify(r[ix["Kernel Name"]])
        d = per.setdefault(c, {"n": 0, "ns": 0.0, "grid": r[ix["Grid Size"]], "block": r[ix["Block Size"]],
                               "name": r[ix["Kernel Name"]][:70]})
        d["n"] += 1
        d["ns"] += ns
        total += ns
    with open(out, "w") as f:
        f.write("# ncu launch list (`--metrics gpu__time_duration.sum --clock-control none`)\n\n")
        f.write("Source: `%s` (%d launches, all launches of the profiled command incl. warm-up steps).\n"
                "Times are cold-cache and serialised; compare the SHARE column with bench.py's `kernels`.\n\n" % (path, sum(d["n"] for d in per.values())))
        f.write("| kernel class | launches | total ms | avg us | share | example grid x block | example name |\n|---|---|---|---|---|---|---|\n")
        for c, d in sorted(per.items(), key=lambda kv: -kv[1]["ns"]):
            f.write("| %s | %d | %.3f | %.1f | %.1f %% | %s x %s | `%s` |\n" % (
                c, d["n"], d["ns"] * 1e-6, d["ns"] / d["n"] * 1e-3, 100 * d["ns"] / total, d["grid"], d["block"], d["name"]))
        f.write("\ntotal %.3f ms\n" % (total * 1e-6))
    print(open(out).read())


KEYS = [("gpu__time_duration.sum", "time"), ("dram__bytes_read.sum", "dram_rd"), ("dram__bytes_write.sum", "dram_wr"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
        ("sm__inst_executed_pipe_fma.sum.pct_of_peak_sustained_active", "fma%"),
        ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64%"),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor%"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
        ("launch__registers_per_thread", "regs"), ("launch__grid_size", "grid"), ("launch__block_size", "block"),
        ("smsp__inst_executed.sum", "warp_inst")]

UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6,
        "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6}


def read_raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    rows = [r for r in rows if len(r) > 10]
    return rows[0], rows[1], rows[2:]


def full(reps, segments, out, traffic_path, label="cfg2"):
    lines = []
    traffic = {}
    for rep in reps:
        hdr, units, rows = read_raw(rep)
        ix = {h: i for i, h in enumerate(hdr)}
        for r in rows:
            name = r[ix["Kernel Name"]]
            rec = {"kernel": name.replace("void ", "").replace("gssb::", "")[:60], "class": classify(name), "src": rep.split("/")[-1]}
            for k, short in KEYS:
                if k not in ix:
                    rec[short] = None
                    continue
                v = r[ix[k]].replace(",", "")
                try:
                    v = float(v)
                except ValueError:
                    rec[short] = None
                    continue
                u = units[ix[k]]
                if short in ("time", "dram_rd", "dram_wr"):
                    v *= UNIT.get(u, 1.0)
                rec[short] = v
            lines.append(rec)
            t = traffic.setdefault(rec["class"], {"bytes": [], "us": []})
            t["bytes"].append((rec["dram_rd"] or 0) + (rec["dram_wr"] or 0))
            t["us"].append(rec["time"])
    with open(out, "w") as f:
        f.write("# ncu `--set full --clock-control none` captures (one row per captured launch)\n\n")
        f.write("Profiled command: `python bench.py --steps 1 --warmup 3 --no-cpu-baseline --headline-only --workload %s "
                "--segments %d`. Durations are under the profiler (replayed, cold cache) and are NOT bench values.\n\n"
                % (label, segments))
        f.write("| kernel | time us | DRAM rd MB | DRAM wr MB | DRAM % | SM % | issue % | fma pipe % | fp64 % | tensor % | occupancy % | regs | grid x block | report |\n")
        f.write("|---|---|---|---|---|---|---|---|---|---|---|---|---|---|\n")

        def fm(v, s="%.1f"):
            return "-" if v is None else s % v
        for r in lines:
            f.write("| `%s` | %s | %s | %s | %s | %s | %s | %s | %s | %s | %s | %s | %s x %s | %s |\n" % (
                r["kernel"], fm(r["time"]), fm(r["dram_rd"] and r["dram_rd"] / 1e6, "%.2f"), fm(r["dram_wr"] is not None and r["dram_wr"] / 1e6, "%.2f"),
                fm(r["dram%"]), fm(r["sm%"]), fm(r["issue%"]), fm(r["fma%"]), fm(r["fp64%"]), fm(r["tensor%"]), fm(r["occ%"]),
                fm(r["regs"], "%d"), fm(r["grid"], "%d"), fm(r["block"], "%d"), r["src"]))
    tj = {}
    for c, t in traffic.items():
        b = sum(t["bytes"]) / len(t["bytes"])
        tj[c] = {"dram_bytes_per_launch": b, "dram_bytes_per_segment_launch": b / segments, "launches_captured": len(t["bytes"]),
                 "segments": segments, "avg_us_under_ncu": sum(t["us"]) / len(t["us"])}
    if traffic_path:
        json.dump(tj, open(traffic_path, "w"), indent=1, sort_keys=True)
    print(open(out).read())
    print(json.dumps(tj, indent=1))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["launches", "full"])
    ap.add_argument("paths", nargs="+")
    ap.add_argument("--segments", type=int, default=16)
    ap.add_argument("--out", default=None)
    ap.add_argument("--traffic", default=None)
    ap.add_argument("--label", default="cfg2", help="workload name of the profiled command")
    a = ap.parse_args()
    if a.mode == "launches":
        launches(a.paths[0], a.paths[1])
    else:
        full(a.paths, a.segments, a.out, a.traffic, a.label)
