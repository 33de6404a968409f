#!/usr/bin/env python
"""End-to-end pipeline throughput INCLUDING file I/O (run on the GPU box): a synthetic reverberant meeting is
written as a multi-channel WAV plus a JSONL segment manifest, then `scheduler.run_pipeline` reads, assembles,
enhances and writes every segment (the reference's acceptance C6 workload: a 10-minute 4-channel meeting,
acceptance.cpp:434-477). Prints one JSON line. Measurement helper, not product code.

    python tools/pipeline_bench.py [--minutes 10] [--channels 4] [--speakers 4] [--workers 4] [--gpu-batch 16]
"""
import argparse
import json
import os
import shutil
import sys
import tempfile
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2212_05271_b200 import gss  # noqa: E402
import synthbench as synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--minutes", type=float, default=10.0)
    ap.add_argument("--channels", type=int, default=4)
    ap.add_argument("--speakers", type=int, default=4)
    ap.add_argument("--workers", type=int, default=4)
    ap.add_argument("--gpu-batch", type=int, default=16)
    ap.add_argument("--one-per-batch", action="store_true")
    ap.add_argument("--repeat", type=int, default=3, help="runs of the same pipeline; the first one is cold "
                    "(CUDA module loading, memory pool growth, page cache) and is reported separately")
    a = ap.parse_args()
    sr, dur = 16000, a.minutes * 60.0
    rng = np.random.RandomState(11)
    layout = []
    for k in range(a.speakers):  # meeting-like turns: 2-8 s utterances, 1-10 s apart, speakers overlap freely
        pos, ivals = float(rng.uniform(0, 5)), []
        while pos < dur - 1.0:
            d = float(min(rng.uniform(2.0, 8.0), dur - pos))
            ivals.append((pos, d))
            pos += d + float(rng.uniform(1.0, 10.0))
        layout.append(ivals)
    root = tempfile.mkdtemp(prefix="gss_pipeline_")
    try:
        audio = synth.generate(dur, sr, a.channels, 77, layout)
        wav_path = os.path.join(root, "meeting.wav")
        gss.wav.write(wav_path, gss.stft.RealSignal(audio, sr))
        rec = gss.manifests.Recording("meeting", [gss.manifests.Source(wav_path, list(range(a.channels)))], sr, dur)
        segs = [gss.manifests.Segment("meeting", "spk%d" % k, s, d, "meeting-spk%d-%04d" % (k, i))
                for k, iv in enumerate(layout) for i, (s, d) in enumerate(iv)]
        cfg = gss.scheduler.PipelineConfig(gss.stft.StftConfig(512, 128, 0, sr), gss.wpe.WpeConfig(10, 2, 3, 0, 1e-10),
                                           True, 20, 15.0, True, out_dir=os.path.join(root, "out"), workers=a.workers,
                                           mode=gss.scheduler.ONE_PER_BATCH if a.one_per_batch else gss.scheduler.SUPER_SEGMENT)
        gss.default_context()  # context creation is not part of the run
        walls = []
        for _ in range(max(1, a.repeat)):
            shutil.rmtree(cfg.out_dir, ignore_errors=True)
            t0 = time.perf_counter()
            run = gss.scheduler.run_pipeline([rec], segs, cfg, gpu_batch=a.gpu_batch)
            walls.append(time.perf_counter() - t0)
        wall = min(walls[1:]) if len(walls) > 1 else walls[0]
        j = run.json
        speech = sum(s.duration for s in segs)
        print(json.dumps({"workload": "%.0f min, %d channels, %d speakers, %d segments (%.0f s of speech), WPE + 20 iterations, "
                                      "15 s context, %s" % (a.minutes, a.channels, a.speakers, len(segs), speech,
                                                            "one segment per batch" if a.one_per_batch else "super-segments <= 50 s"),
                          "wall_s": round(wall, 3), "walls_s": [round(w, 3) for w in walls], "recording_xrt": round(dur / wall, 1),
                          "enhanced_speech_xrt": round(speech / wall, 1),
                          "processed_xrt": round(j["processed_audio_seconds"] / wall, 1),
                          "batches": j["num_batches"], "segments_written": j["segments_written"],
                          "failed": run.failed_segments, "workers": a.workers, "gpu_batch": a.gpu_batch,
                          "stage_seconds": {k: round(v, 3) for k, v in j["stage_seconds"].items()}}))
    finally:
        shutil.rmtree(root, ignore_errors=True)


if __name__ == "__main__":
    main()
