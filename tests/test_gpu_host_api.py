"""The C++ host mirror (paper_2212_05271_b200/host/include/gss/*.hpp) compiled with g++ against the C ABI and
run on the device: the reference's own call sites compile unchanged against these headers."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def compile_check(out, source="host_api_check.cpp", extra=()):
    lib = os.path.join(ROOT, "paper_2212_05271_b200", "lib")
    cmd = ["g++", "-std=c++17", "-O1", "-Wall", "-I" + os.path.join(ROOT, "include"),
           "-I" + os.path.join(ROOT, "paper_2212_05271_b200", "host", "include"),
           os.path.join(ROOT, "tests", source), "-o", out, "-L" + lib, "-lgss_b200",
           "-Wl,-rpath," + lib, "-lpthread", *extra]
    subprocess.run(cmd, check=True)


def compile_pipeline_check(out):
    compile_check(out, "host_pipeline_check.cpp", ["-DGSS_WITH_ZLIB", "-lz"])


def test_host_mirror_compiles(tmp_path):
    from paper_2212_05271_b200 import build
    build.build(verbose=False)
    compile_check(str(tmp_path / "host_api_check"))


@pytest.mark.gpu
def test_host_mirror_runs_on_device(tmp_path):
    exe = str(tmp_path / "host_api_check")
    compile_check(exe)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.startswith("OK"), r.stdout + r.stderr


def test_host_mirror_pipeline_rows_on_cpu(tmp_path):
    """wav / manifests goldens / plan_batches / assemble / ordered queue of the C++ mirror (no device work)."""
    from paper_2212_05271_b200 import build
    build.build(verbose=False)
    exe = str(tmp_path / "host_pipeline_check")
    compile_pipeline_check(exe)
    work = tmp_path / "work"
    work.mkdir()
    r = subprocess.run([exe, "cpu", os.path.join(ROOT, "tests", "golden"), str(work)], capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.startswith("OK"), r.stdout + r.stderr


@pytest.mark.gpu
def test_host_mirror_run_pipeline_matches_the_python_mirror(tmp_path):
    """run_pipeline of the C++ mirror on device 0 (outputs, summary, executor invariance, failure isolation),
    then the Python mirror on the same manifests: both sit on the same C ABI, so the bytes must agree."""
    import json

    from paper_2212_05271_b200 import gss
    exe = str(tmp_path / "host_pipeline_check")
    compile_pipeline_check(exe)
    work = tmp_path / "work"
    work.mkdir()
    r = subprocess.run([exe, "gpu", str(work)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.startswith("OK"), r.stdout + r.stderr

    recs = gss.manifests.load_recordings(str(work / "in" / "recordings.jsonl"))
    segs = gss.manifests.load_segments(str(work / "in" / "segments.jsonl"))
    cfg = gss.scheduler.PipelineConfig(gss.stft.StftConfig(), gss.wpe.WpeConfig(4, 2, 1, 0, 1e-10), True, 3, 1.0, True,
                                       out_dir=str(work / "out_py"), max_batch_duration=5.0, workers=2)
    run = gss.scheduler.run_pipeline(recs, segs, cfg)
    cpp = json.load(open(work / "out_sync" / "summary.json"))
    assert run.failed_segments == 0 and len(run.json["outputs"]) == len(cpp["outputs"]) == 5
    for a, b in zip(run.json["outputs"], cpp["outputs"]):
        assert a["segment_id"] == b["segment_id"] and os.path.basename(a["path"]) == os.path.basename(b["path"])
        assert open(a["path"], "rb").read() == open(b["path"], "rb").read()
    for a, b in zip(run.json["batches"], cpp["batches"]):
        assert {k: a[k] for k in ("batch", "speaker", "frames", "segments", "ref_channel", "zeroed_bins")} == \
               {k: b[k] for k in ("batch", "speaker", "frames", "segments", "ref_channel", "zeroed_bins")}
        assert a["log_likelihood"] == b["log_likelihood"]
    assert list(run.json) == list(cpp) and list(run.json["config"]) == list(cpp["config"])
