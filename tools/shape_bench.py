#!/usr/bin/env python
"""Resident-batch timing of one segment shape (run on the GPU box): which sweep wins for a channel / class count?

    python tools/shape_bench.py <channels> <speakers> [segments=16] [iterations=20] [target_s=10] [context_s=15]

Prints ms per step and the per-kernel clocks. GSS_B200_LIB selects a kernel-experiment build (tools/variant.py).
Measurement helper, not product code."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2212_05271_b200 import gss  # noqa: E402
import synthbench as synth  # noqa: E402


def main():
    a = sys.argv[1:]
    m, spk = int(a[0]), int(a[1])
    nseg = int(a[2]) if len(a) > 2 else 16
    iters = int(a[3]) if len(a) > 3 else 20
    dur = float(a[4]) if len(a) > 4 else 10.0
    ctxs = float(a[5]) if len(a) > 5 else 15.0
    cfg = synth.sweep_cfg(iters)
    segs = synth.make_sweep_segments([(9000 + i, m, spk, dur, iters) for i in range(nseg)]) if ctxs == 15.0 else \
        [synth.make_supersegment(9000 + i, m, spk, dur, ctxs, cfg) for i in range(nseg)]
    ctx = gss.default_context()
    rb = gss.scheduler.ResidentBatch(segs, cfg, ctx, pinned=True)
    rb.upload()
    for _ in range(3):
        rb.run()
    torch.cuda.synchronize()
    stream = torch.cuda.ExternalStream(ctx.stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    steps = 5
    e0.record(stream)
    for _ in range(steps):
        rb.run()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    ctx.profile(True)
    for _ in range(steps):
        rb.run()
    torch.cuda.synchronize()
    k = {n: round(v[0] / steps, 3) for n, v in ctx.kernel_ms().items() if v[1]}
    ctx.profile(False)
    bad = [str(r.error) for r in rb.fetch() if r.error is not None]
    print("M=%d K=%d segments=%d iters=%d: %.3f ms/step %s %s" % (m, spk + 1, nseg, iters, ms, k, bad[:1]))


if __name__ == "__main__":
    main()
