#!/usr/bin/env python
"""Opcode mix and stall summary of one kernel from `ncu -i X.ncu-rep --page source --csv --print-source sass`."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
# a report with several captured launches repeats the header: keep the section asked for (default the first)
starts = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
sec = int(sys.argv[2]) if len(sys.argv) > 2 else 0
end = starts[sec + 1] - 1 if sec + 1 < len(starts) else len(rows)
print(rows[starts[sec] - 1][1] if starts[sec] > 0 else "")
rows = rows[:2] + rows[starts[sec] + 1:end]
ix = {h: i for i, h in enumerate(hdr)}
ops = collections.Counter(); samples = collections.Counter(); total = 0
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
stalls = collections.Counter()
for r in rows[2:]:
    if len(r) < len(hdr): continue
    src = r[ix["Source"]].strip()
    toks = src.split()
    op = toks[1] if toks and toks[0].startswith("@") else (toks[0] if toks else "?")
    op = op.split(".")[0] if not op.startswith(("LDS", "STS", "LDG", "STG", "SHFL")) else ".".join(op.split(".")[:2])
    n = int(r[ix["Instructions Executed"]] or 0)
    ops[op] += n; total += n
    samples[op] += int(r[ix["# Samples"]] or 0)
    for c in stall_cols:
        stalls[c] += int(r[ix[c]] or 0)
print("total warp instr", total)
for op, n in ops.most_common(40):
    print(f"{op:14s} {n:12d} {100*n/total:6.2f}%  samples {samples[op]}")
ts = sum(stalls.values())
print("stalls:", ", ".join(f"{k[6:]} {100*v/ts:.1f}%" for k, v in stalls.most_common(10)))
