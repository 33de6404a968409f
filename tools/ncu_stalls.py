#!/usr/bin/env python
"""Stall / instruction-mix digest of one kernel from an `ncu --set full --import-source on` report.

    python tools/ncu_stalls.py gpurun_out/prof.ncu-rep [kernel-regex]

Prints duration, issue-active, pipe utilisation, bank conflicts, the warp-stall sample histogram, the SASS opcode
mix and the most-sampled instructions. Measurement helper (reads reports brought back from the GPU box)."""
import collections
import csv
import io
import subprocess
import sys


def page(rep, which, kern):
    cmd = ["ncu", "-i", rep, "--page", which, "--csv"] + (["--kernel-name", "regex:" + kern] if kern else [])
    return list(csv.reader(io.StringIO(subprocess.run(cmd, capture_output=True, text=True).stdout)))


def num(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return 0.0


def main():
    rep = sys.argv[1]
    kern = sys.argv[2] if len(sys.argv) > 2 else ""
    raw = page(rep, "raw", kern)
    hdr, row = raw[0], raw[2]
    g = {h: row[i] for i, h in enumerate(hdr)}
    print(g["Kernel Name"][:90])
    for k in ("gpu__time_duration.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
              "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
              "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers",
              "launch__occupancy_limit_shared_mem", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
              "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "smsp__inst_executed.sum",
              "dram__bytes_read.sum", "dram__bytes_write.sum"):
        print("  %-70s %s" % (k, g.get(k)))
    stalls = {h.replace("smsp__pcsamp_warps_issue_stalled_", ""): num(g[h]) for h in hdr
              if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued")}
    tot = sum(stalls.values()) or 1.0
    print("  stall samples: " + ", ".join("%s %.1f%%" % (k, 100 * v / tot) for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:9]))
    src = page(rep, "source", kern)
    h2 = src[1]
    ix = {h: i for i, h in enumerate(h2)}
    data = [r for r in src[2:] if len(r) == len(h2)]
    ins = sum(num(r[ix["Instructions Executed"]]) for r in data) or 1.0
    smp = sum(num(r[ix["# Samples"]]) for r in data) or 1.0
    mix, ms = collections.Counter(), collections.Counter()
    for r in data:
        t = r[ix["Source"]].split()
        op = (t[1] if t and t[0].startswith("@") and len(t) > 1 else (t[0] if t else "?")).split(".")[0]
        mix[op] += num(r[ix["Instructions Executed"]])
        ms[op] += num(r[ix["# Samples"]])
    print("  opcode mix: " + ", ".join("%s %.1f%% (%.1f%% of samples)" % (o, 100 * c / ins, 100 * ms[o] / smp) for o, c in mix.most_common(10)))
    print("  shared wavefronts: %d, excessive (bank conflicts): %d" % (
        sum(num(r[ix["L1 Wavefronts Shared"]]) for r in data), sum(num(r[ix["L1 Wavefronts Shared Excessive"]]) for r in data)))
    print("  most excessive shared wavefronts:")
    for r in sorted(data, key=lambda r: -num(r[ix["L1 Wavefronts Shared Excessive"]]))[:6]:
        if num(r[ix["L1 Wavefronts Shared Excessive"]]) > 0:
            print("    %10d of %10d  %s" % (num(r[ix["L1 Wavefronts Shared Excessive"]]), num(r[ix["L1 Wavefronts Shared"]]),
                                            r[ix["Source"]][:60]))
    print("  most sampled instructions:")
    for r in sorted(data, key=lambda r: -num(r[ix["# Samples"]]))[:12]:
        print("    %6d  %-60s short_sb %s mio %s long_sb %s" % (num(r[ix["# Samples"]]), r[ix["Source"]][:60], r[ix["stall_short_sb"]],
                                                                 r[ix["stall_mio"]], r[ix["stall_long_sb"]]))


if __name__ == "__main__":
    main()
