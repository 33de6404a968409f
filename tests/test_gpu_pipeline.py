"""run_pipeline (scheduler.hpp:423-638) on the GPU executor: files, summary, failure isolation and the
worker-count / device-batch invariance of the written bytes (test_scheduler.cpp:278-407), plus parity of
the written waveforms with the CPU oracle run on the same assembled batches."""
import json
import os

import numpy as np
import pytest

from .gpu_util import sdr_db

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gss():
    from paper_2212_05271_b200 import gss as g
    g.default_context()
    return g


def fast_config(gss, out_dir, workers=0):  # test_scheduler.cpp:27-36
    sc = gss.scheduler
    return sc.PipelineConfig(gss.stft.StftConfig(), gss.wpe.WpeConfig(4, 2, 1, 0, 1e-10), True, 2, 1.0, True,
                             out_dir=out_dir, workers=workers)


def save_fixture(gss, root, name, duration, channels, seed, speakers):
    """A synthetic reverberant mixture as one WAV + its manifests (the role of synthbench::save_fixture)."""
    import synthbench as synth
    mf = gss.manifests
    os.makedirs(root, exist_ok=True)
    layout = [ivals for _, ivals in speakers]
    audio = synth.generate(duration, 16000, channels, seed, layout)
    path = os.path.join(root, name + ".wav")
    gss.wav.write(path, gss.stft.RealSignal(audio, 16000))
    rec = mf.Recording(name, [mf.Source(path, list(range(channels)))], 16000, duration)
    segs = [mf.Segment(name, spk, s, d, "%s-%s-%04d" % (name, spk, i))
            for spk, ivals in speakers for i, (s, d) in enumerate(ivals)]
    seg_path = os.path.join(root, name + ".segments.jsonl")
    mf.save_segments(seg_path, segs)
    return rec, seg_path


def test_run_pipeline_writes_outputs_and_a_faithful_summary(gss, oracle, tmp_path):
    rec, seg_path = save_fixture(gss, str(tmp_path / "in"), "rec0", 8.0, 2, 9,
                                 [("spk0", [(0.5, 3.0)]), ("spk1", [(4.0, 3.0)])])
    segs = gss.manifests.load_segments(seg_path)
    cfg = fast_config(gss, str(tmp_path / "out"))
    run = gss.scheduler.run_pipeline([rec], segs, cfg)
    j = run.json
    assert run.failed_segments == 0
    assert (j["num_recordings"], j["num_segments"], j["num_batches"], j["segments_written"]) == (1, 2, 2, 2)
    assert j["failures"] == [] and len(j["outputs"]) == 2
    for out in j["outputs"]:
        assert os.path.exists(out["path"]) and out["samples"] == 48000
        assert gss.wav.info(out["path"]).num_frames == 48000
    assert os.path.exists(cfg.out_dir + "/rec0-spk0-0000500_0003500.wav")
    assert os.path.exists(cfg.out_dir + "/rec0-spk1-0004000_0007000.wav")
    assert json.load(open(cfg.out_dir + "/summary.json")) == json.loads(json.dumps(j))
    echo = j["config"]
    assert echo["max-batch-duration"] == 50.0 and echo["context-duration"] == 1.0 and echo["bss-iterations"] == 2
    assert echo["no-wpe"] is False and echo["workers"] == 0 and echo["fft-size"] == 1024
    assert j["plan_cache"]["entries"] == j["plan_cache"]["computed"] and j["plan_cache"]["hits"] > 0
    assert j["stage_seconds"]["total"] > 0 and j["stage_seconds"]["mask"] > 0
    assert j["processed_audio_seconds"] > 0
    assert [b["segments"] for b in j["batches"]] == [1, 1] and all(b["frames"] > 0 for b in j["batches"])
    # the written waveforms are the oracle's, batch by batch
    plans = gss.scheduler.plan_batches(segs, cfg.max_batch_duration, cfg.mode)
    for plan, out, bj in zip(plans, j["outputs"], j["batches"]):
        ss = gss.scheduler.assemble(plan, rec, segs, cfg)
        want = oracle.enhance(ss.audio.channels, ss.activity.grid, ss.activity.target_index,
                              ss.activity.noise_index, [(p.sample_begin, p.sample_end) for p in ss.parts],
                              fft_size=cfg.stft.fft_size, shift=cfg.stft.shift, window=cfg.stft.window,
                              sample_rate=cfg.stft.sample_rate, enable_wpe=cfg.enable_wpe, taps=cfg.wpe.taps,
                              delay=cfg.wpe.delay, wpe_iterations=cfg.wpe.iterations,
                              psd_context=cfg.wpe.psd_context, regularization=cfg.wpe.regularization,
                              bss_iterations=cfg.bss_iterations, diag=True)
        got = gss.wav.read(out["path"]).channels[0]
        assert bj["ref_channel"] == want.ref_channel and bj["frames"] == want.frames
        assert len(got) == len(want.outputs[0]) and sdr_db(got, want.outputs[0]) >= 40.0
        assert abs(bj["log_likelihood"] - want.ll_final) <= 1e-4 * abs(want.ll_final)


def test_run_pipeline_records_load_failures_and_keeps_going(gss, tmp_path):  # test_scheduler.cpp:331-358
    mf = gss.manifests
    good, _ = save_fixture(gss, str(tmp_path / "in"), "good", 6.0, 2, 1, [("spk0", [(1.0, 2.0)])])
    bad = mf.Recording("bad", [mf.Source(str(tmp_path / "in" / "missing.wav"), [0, 1])], 16000, 6.0)
    segs = [mf.Segment("good", "spk0", 1.0, 2.0, "g-0"), mf.Segment("bad", "spk0", 1.0, 2.0, "b-0"),
            mf.Segment("bad", "spk0", 3.0, 1.0, "b-1")]
    cfg = fast_config(gss, str(tmp_path / "out"))
    run = gss.scheduler.run_pipeline([good, bad], segs, cfg)
    assert run.failed_segments == 2 and run.json["segments_written"] == 1
    assert [f["segment_id"] for f in run.json["failures"]] == ["b-0", "b-1"]
    assert os.path.exists(cfg.out_dir + "/good-spk0-0001000_0003000.wav")


def test_run_pipeline_rejects_segments_naming_unknown_recordings(gss, tmp_path):  # test_scheduler.cpp:360-374
    rec, _ = save_fixture(gss, str(tmp_path / "in"), "rec0", 4.0, 1, 2, [("spk0", [(1.0, 2.0)])])
    with pytest.raises(gss.ConfigError):
        gss.scheduler.run_pipeline([rec], [gss.manifests.Segment("ghost", "spk0", 1.0, 2.0, "x")],
                                   fast_config(gss, str(tmp_path / "out")))


def test_worker_count_and_device_batching_do_not_change_the_written_bytes(gss, tmp_path):
    # test_scheduler.cpp:376-407, extended by the knob the GPU executor adds (segments per device call)
    rec, seg_path = save_fixture(gss, str(tmp_path / "in"), "rec0", 8.0, 2, 31,
                                 [("spk0", [(0.5, 2.0), (5.0, 2.0)]), ("spk1", [(2.5, 2.5)])])
    segs = gss.manifests.load_segments(seg_path)
    runs = []
    for name, workers, gpu_batch in (("serial", 0, 16), ("threaded", 2, 16), ("single", 2, 1)):
        cfg = fast_config(gss, str(tmp_path / name), workers)
        cfg.max_batch_duration = 3.0  # three batches: spk0 twice, spk1 once
        runs.append(gss.scheduler.run_pipeline([rec], segs, cfg, gpu_batch=gpu_batch))
        assert runs[-1].failed_segments == 0
    a = runs[0].json["outputs"]
    assert len(a) == 3
    for other in runs[1:]:
        b = other.json["outputs"]
        assert [o["segment_id"] for o in a] == [o["segment_id"] for o in b]
        for oa, ob in zip(a, b):
            assert open(oa["path"], "rb").read() == open(ob["path"], "rb").read()
        assert [x["log_likelihood"] for x in runs[0].json["batches"]] == [x["log_likelihood"] for x in other.json["batches"]]
