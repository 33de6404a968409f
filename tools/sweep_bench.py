#!/usr/bin/env python
"""BASELINE configs[4] in sample form (run on the GPU box): a seeded sample of the 4096-segment throughput sweep
-- target durations U[2,12] s with 15 s of context each side, 2-8 channels, 2-4 speakers + noise, 5/10/20/40
EM iterations, WPE on -- enhanced on one GPU through the public call (pinned host buffers, H2D/D2H inside the
timing), plus the static size-balanced shard the same sample would get on 1/2/4/8 GPUs (sharding.py's cost
model; the predicted scaling is the load balance, the data path has no collective). Prints one JSON line.
Measurement helper, not product code.

    python tools/sweep_bench.py [--segments 128] [--per-call 32]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2212_05271_b200 import gss, sharding  # noqa: E402
import synthbench as synth  # noqa: E402
from paper_2212_05271_b200.gss import scheduler, stft, wpe  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--segments", type=int, default=128)
    ap.add_argument("--per-call", type=int, default=32)
    a = ap.parse_args()
    rng = np.random.RandomState(5000)
    items = []
    for i in range(a.segments):
        iters = int(rng.choice([5, 10, 20, 40]))
        cfg = scheduler.PipelineConfig(stft.StftConfig(512, 128, 0, 16000), wpe.WpeConfig(10, 2, 3, 0, 1e-10), True, iters)
        ss = synth.make_supersegment(5000 + i, int(rng.randint(2, 9)), int(rng.randint(2, 5)),
                                     float(rng.uniform(2.0, 12.0)), 15.0, cfg)
        items.append((iters, cfg, ss))
    costs = [sharding.segment_cost(ss.activity.frames, ss.audio.num_channels(), ss.activity.num_classes(), it, 10, 3)
             for it, _, ss in items]
    ctx = gss.default_context()
    by_iter = {}
    for it, cfg, ss in items:
        by_iter.setdefault(it, (cfg, []))[1].append(ss)

    def run_all():
        failed = 0
        for it in sorted(by_iter):
            cfg, segs = by_iter[it]
            for p0 in range(0, len(segs), a.per_call):
                failed += sum(r.error is not None for r in scheduler.enhance_batches(segs[p0:p0 + a.per_call], cfg, ctx))
        return failed

    run_all()  # warm-up: module load, memory pool
    t0 = time.perf_counter()
    failed = run_all()
    wall = time.perf_counter() - t0
    out_s = sum((p.sample_end - p.sample_begin) / 16000.0 for _, _, ss in items for p in ss.parts)
    win_s = sum(ss.audio.num_samples() / 16000.0 for _, _, ss in items)
    balance = {}
    for n in (1, 2, 4, 8):
        loads = [sum(costs[i] for i in own) for own in sharding.shard(costs, n)]
        balance[str(n)] = round(sum(loads) / (n * max(loads)), 4)  # 1.0 = perfectly even shards
    print(json.dumps({"workload": "BASELINE configs[4] sample: %d segments, durations U[2,12] s + 2 x 15 s context, "
                                  "2-8 channels, 2-4 speakers + noise, EM iterations in {5,10,20,40}, WPE on" % a.segments,
                      "wall_s": round(wall, 3), "segments_per_s": round(a.segments / wall, 1),
                      "xrt_output": round(out_s / wall, 1), "xrt_processed": round(win_s / wall, 1),
                      "failed": failed, "per_call": a.per_call,
                      "shard_load_balance": balance}))


if __name__ == "__main__":
    main()
