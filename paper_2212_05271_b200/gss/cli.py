"""cli.hpp: the `gss` command line -- enhance, trim-to-segments, validate-manifests, bench.

    python -m paper_2212_05271_b200.gss.cli enhance recordings.jsonl segments.jsonl --out-dir out [...]

Same sub-commands, flags, defaults, messages and exit codes (0 ok, 1 failure, 2 usage) as the reference's
run_cli (cli.hpp:320-404). Two additions that only exist on this path: `--devices 0,1,...` (one compute slot per
GPU) and `--gpu-batch N` (super-segments per device call). `bench` needs the synthetic-mixture harness, which is
not part of the product package (repo root `synthbench/`); it is imported on demand.
"""
from __future__ import annotations

import argparse
import sys

from . import manifests, scheduler
from .common import ConfigError, ParseError

EXIT_OK, EXIT_FAILURE, EXIT_USAGE = 0, 1, 2


def _require_file(path: str) -> bool:  # cli.hpp:26-30
    import os
    if os.path.exists(path):
        return True
    print("gss: manifest not found: %s" % path, file=sys.stderr)
    return False


def pick_format(path: str, requested: str) -> str:  # cli.hpp:32-41
    if requested in (manifests.JSONL, manifests.RTTM):
        return requested
    p = path[:-3] if path.endswith(".gz") else path
    return manifests.RTTM if p.endswith(".rttm") else manifests.JSONL


def _int_list(text: str) -> list:
    return [int(x) for x in text.split(",") if x != ""]


def _float_list(text: str) -> list:
    return [float(x) for x in text.split(",") if x != ""]


def pipeline_config(a) -> scheduler.PipelineConfig:  # EnhanceOptions::pipeline, cli.hpp:61-78
    return scheduler.PipelineConfig(
        max_batch_duration=a.max_batch_duration, context_duration=a.context_duration,
        bss_iterations=a.bss_iterations, enable_wpe=not a.no_wpe, noise_class=not a.no_noise_class,
        channels=list(a.channels), mode=scheduler.ONE_PER_BATCH if a.one_per_batch else scheduler.SUPER_SEGMENT,
        workers=a.workers, queue_capacity=a.queue_capacity, seed=a.seed, out_dir=a.out_dir,
        extra_echo=[("recordings", a.recordings), ("segments", a.segments), ("segment-format", a.segment_format)])


def cmd_enhance(a) -> int:  # cli.hpp:81-106
    if not _require_file(a.recordings) or not _require_file(a.segments):
        return EXIT_USAGE
    try:
        recordings = manifests.load_recordings(a.recordings)
        skipped = [0]
        segments = manifests.load_segments(a.segments, pick_format(a.segments, a.segment_format), skipped)
        if skipped[0] > 0:
            print("warning: skipped %d zero-duration segment(s)" % skipped[0], file=sys.stderr)
        summary = scheduler.run_pipeline(recordings, segments, pipeline_config(a), devices=a.devices or None,
                                         gpu_batch=a.gpu_batch)
        print("wrote %d segment(s), %d failure(s), summary at %s/summary.json"
              % (summary.json["segments_written"], summary.failed_segments, a.out_dir))
        return EXIT_OK if summary.failed_segments == 0 else EXIT_FAILURE
    except Exception as e:  # noqa: BLE001 - every failure is reported and mapped to exit 1, as in the reference
        print("gss: enhance failed: %s" % e, file=sys.stderr)
        return EXIT_FAILURE


def cmd_trim_to_segments(a) -> int:  # cli.hpp:118-191
    """Recording-level cut lines (objects with a "supervisions" array) become one segment line per supervision;
    lines that already are segments pass through, so the command is a fixed point on its own output."""
    if not _require_file(a.cuts):
        return EXIT_USAGE
    if a.recordings and not _require_file(a.recordings):
        return EXIT_USAGE
    try:
        known = {r.id for r in manifests.load_recordings(a.recordings)} if a.recordings else set()
        out, counters = [], {}

        def one(j, line):
            t = manifests._typed
            rec_id = ""
            if "recording_id" in j:
                rec_id = t(j, "recording_id", str)
            elif "id" in j and "supervisions" in j:
                rec_id = t(j, "id", str)
            if not rec_id:
                raise ParseError("%s:%d: cut has no recording_id" % (a.cuts, line))
            if known and rec_id not in known:
                raise ConfigError("%s:%d: unknown recording_id '%s'" % (a.cuts, line, rec_id))
            if "supervisions" not in j:
                out.append(manifests.Segment(rec_id, t(j, "speaker", str), t(j, "start", float),
                                             t(j, "duration", float), t(j, "id", str)))
                return
            for sup in t(j, "supervisions", list):
                s = manifests.Segment(rec_id, t(sup, "speaker", str), t(sup, "start", float), t(sup, "duration", float))
                if "id" in sup:
                    s.id = t(sup, "id", str)
                else:
                    n = counters.get((rec_id, s.speaker), 0)
                    counters[(rec_id, s.speaker)] = n + 1
                    s.id = "%s-%s-%04d" % (rec_id, s.speaker, n)
                out.append(s)

        manifests._for_each_jsonl(a.cuts, one)
        manifests.save_segments(a.out, out)
        print("wrote %d segment(s) to %s" % (len(out), a.out))
        return EXIT_OK
    except Exception as e:  # noqa: BLE001
        print("gss: trim-to-segments failed: %s" % e, file=sys.stderr)
        return EXIT_FAILURE


def cmd_validate_manifests(a) -> int:  # cli.hpp:199-224
    if not _require_file(a.recordings) or not _require_file(a.segments):
        return EXIT_USAGE
    try:
        recordings = manifests.load_recordings(a.recordings)
        skipped = [0]
        segments = manifests.load_segments(a.segments, pick_format(a.segments, a.segment_format), skipped)
        problems = manifests.validate(recordings, segments)
        for p in problems:
            print("problem: %s" % p, file=sys.stderr)
        print("%d recording(s), %d segment(s), %d skipped, %d problem(s)"
              % (len(recordings), len(segments), skipped[0], len(problems)))
        return EXIT_OK if not problems else EXIT_FAILURE
    except Exception as e:  # noqa: BLE001
        print("gss: validate-manifests failed: %s" % e, file=sys.stderr)
        return EXIT_FAILURE


def cmd_bench(a) -> int:  # cli.hpp:230-318 (the grid itself lives with the harness: synthbench/harness.py)
    import os
    if not os.path.exists(a.spec):
        print("gss: spec not found: %s" % a.spec, file=sys.stderr)
        return EXIT_USAGE
    try:
        from synthbench import harness
    except ImportError as e:
        print("gss: bench needs the synthbench harness of the source tree on PYTHONPATH (%s)" % e, file=sys.stderr)
        return EXIT_FAILURE
    opt = harness.BenchOptions(a.spec, a.out_dir, list(a.contexts), list(a.iterations), list(a.channels), a.no_wpe,
                               a.max_batch_duration)
    return harness.cmd_bench(opt, devices=a.devices or None)


class _Parser(argparse.ArgumentParser):
    """argparse exits with 2 on bad usage already; --help exits 0. Messages go to stderr."""


def build_parser() -> argparse.ArgumentParser:  # cli.hpp:321-390
    app = _Parser(prog="gss", description="Guided source separation: WPE + guided CACGMM masks + MVDR",
                  epilog="GPU path: libgss_b200.so (sm_100a); there is no CPU fallback.")
    sub = app.add_subparsers(dest="command", required=True)

    en = sub.add_parser("enhance", help="Separate every manifest segment into a mono WAV")
    en.add_argument("recordings", help="Recordings JSONL")
    en.add_argument("segments", help="Segments JSONL or RTTM")
    en.add_argument("--out-dir", default="gss-out", help="Output directory")
    en.add_argument("--segment-format", default="auto", choices=["auto", "jsonl", "rttm"],
                    help="Segment manifest format")
    en.add_argument("--max-batch-duration", type=float, default=50.0, help="Per-batch speech budget in seconds")
    en.add_argument("--context-duration", type=float, default=15.0, help="Context seconds on each side of a batch")
    en.add_argument("--bss-iterations", type=int, default=20, help="EM iterations for mask estimation")
    en.add_argument("--no-wpe", action="store_true", help="Skip dereverberation")
    en.add_argument("--no-noise-class", action="store_true", help="Model only the listed speakers")
    en.add_argument("--channels", type=_int_list, default=[], help="Comma-separated stacked-channel subset, e.g. 0,1")
    en.add_argument("--one-per-batch", action="store_true", help="Process each segment in its own batch")
    en.add_argument("--workers", type=int, default=0, help="Data-loader threads")
    en.add_argument("--queue-capacity", type=int, default=2, help="Loader prefetch depth")
    en.add_argument("--seed", type=int, default=0, help="Echoed into the summary")
    en.add_argument("--devices", type=_int_list, default=[], help="GPUs to use, e.g. 0,1,2,3 (default: 0)")
    en.add_argument("--gpu-batch", type=int, default=16, help="Super-segments per device call")
    en.set_defaults(fn=cmd_enhance)

    tr = sub.add_parser("trim-to-segments", help="Expand recording-level cuts into segment lines")
    tr.add_argument("cuts", help="Cuts JSONL")
    tr.add_argument("--out", required=True, help="Segments JSONL to write")
    tr.add_argument("--recordings", default="", help="Optional recordings manifest to check ids against")
    tr.set_defaults(fn=cmd_trim_to_segments)

    va = sub.add_parser("validate-manifests", help="Cross-check recordings and segments")
    va.add_argument("recordings", help="Recordings JSONL")
    va.add_argument("segments", help="Segments JSONL or RTTM")
    va.add_argument("--segment-format", default="auto", choices=["auto", "jsonl", "rttm"],
                    help="Segment manifest format")
    va.set_defaults(fn=cmd_validate_manifests)

    be = sub.add_parser("bench", help="Sweep pipeline parameters over a synthetic mixture")
    be.add_argument("spec", help="Mixture spec JSON")
    be.add_argument("--out-dir", default="gss-bench", help="Output directory")
    be.add_argument("--contexts", type=_float_list, default=[5.0, 10.0, 15.0, 20.0], help="Context durations to sweep")
    be.add_argument("--iterations", type=_int_list, default=[1, 5, 10, 20], help="EM iteration counts")
    be.add_argument("--channels", type=_int_list, default=[], help="Channel counts to sweep")
    be.add_argument("--no-wpe", action="store_true", help="Skip dereverberation")
    be.add_argument("--max-batch-duration", type=float, default=50.0, help="Per-batch speech budget in seconds")
    be.add_argument("--devices", type=_int_list, default=[], help="GPUs to use (default: 0)")
    be.set_defaults(fn=cmd_bench)
    return app


def run_cli(argv=None) -> int:
    """cli.hpp:320-404. `argv` excludes the program name. Returns the exit code instead of exiting."""
    try:
        a = build_parser().parse_args(list(sys.argv[1:] if argv is None else argv))
    except SystemExit as e:  # argparse: 0 after --help, 2 on bad usage
        return EXIT_OK if e.code in (0, None) else EXIT_USAGE
    return a.fn(a)


if __name__ == "__main__":
    sys.exit(run_cli())
