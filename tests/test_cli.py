"""The `gss` command line (cli.hpp:320-404), case by case after the reference's tests/test_cli.cpp.
Argument handling, validate-manifests and trim-to-segments run on the CPU; enhance and bench run the device path."""
import json
import os

import pytest


def run(*args):
    from paper_2212_05271_b200.gss import cli
    return cli.run_cli([str(a) for a in args])


def make_fixture(root, channels=2):  # test_cli.cpp:45-57
    from synthbench import harness as hb
    spec = hb.MixtureSpec(8.0, 16000, channels, 13, [hb.SpeakerLayout("spk0", [(0.5, 3.0)]),
                                                      hb.SpeakerLayout("spk1", [(4.0, 3.0)])])
    mix = hb.generate(spec)
    return hb.save_fixture(mix, str(root), "rec0"), spec


def test_help_exits_cleanly_bad_usage_exits_2(capsys):  # test_cli.cpp:64-74
    assert run("--help") == 0
    assert run("enhance", "--help") == 0
    assert run() == 2
    assert run("frobnicate") == 2
    assert run("enhance") == 2
    assert run("enhance", "a.jsonl", "b.jsonl", "--bogus-flag") == 2
    assert run("enhance", "a.jsonl", "b.jsonl", "--segment-format", "xml") == 2


def test_missing_manifests_exit_2_and_name_the_path(tmp_path, capsys):  # test_cli.cpp:76-89
    present, absent = tmp_path / "present.jsonl", tmp_path / "absent.jsonl"
    present.write_text("")
    assert run("enhance", absent, present) == 2
    assert str(absent) in capsys.readouterr().err
    assert run("enhance", present, absent) == 2
    assert run("validate-manifests", absent, present) == 2
    assert run("trim-to-segments", absent, "--out", tmp_path / "out.jsonl") == 2
    assert run("bench", tmp_path / "absent.json") == 2
    assert "spec not found" in capsys.readouterr().err


def test_validate_manifests_distinguishes_clean_from_broken_inputs(tmp_path, capsys):  # test_cli.cpp:95-108
    paths, _ = make_fixture(tmp_path)
    assert run("validate-manifests", paths.recordings, paths.segments) == 0
    assert "1 recording(s), 2 segment(s), 0 skipped, 0 problem(s)" in capsys.readouterr().out
    bad = tmp_path / "bad_segments.jsonl"
    bad.write_text('{"id": "x", "recording_id": "ghost", "start": 0.0, "duration": 1.0, "speaker": "spk0"}\n')
    assert run("validate-manifests", paths.recordings, bad) == 1
    assert "unknown recording 'ghost'" in capsys.readouterr().err


def test_trim_to_segments_expands_supervision_arrays(tmp_path):  # test_cli.cpp:114-142
    from paper_2212_05271_b200.gss import manifests
    cuts = tmp_path / "cuts.jsonl"
    cuts.write_text('{"id": "meet01", "start": 0.0, "duration": 60.0, "supervisions": ['
                    '{"speaker": "alice", "start": 1.0, "duration": 2.0}, '
                    '{"speaker": "bob", "start": 4.0, "duration": 1.5}, '
                    '{"speaker": "alice", "start": 7.0, "duration": 0.5}]}\n')
    out = tmp_path / "segments.jsonl"
    assert run("trim-to-segments", cuts, "--out", out) == 0
    segs = manifests.load_segments(str(out))
    assert [s.id for s in segs] == ["meet01-alice-0000", "meet01-bob-0000", "meet01-alice-0001"]
    assert (segs[0].recording_id, segs[0].speaker, segs[0].start) == ("meet01", "alice", 1.0)
    out2 = tmp_path / "segments2.jsonl"
    assert run("trim-to-segments", out, "--out", out2) == 0   # a fixed point on its own output
    assert out2.read_bytes() == out.read_bytes()


def test_trim_to_segments_handles_empty_supervision_lists(tmp_path):  # test_cli.cpp:144-154
    cuts = tmp_path / "cuts.jsonl"
    cuts.write_text('{"id": "meet01", "duration": 60.0, "supervisions": []}\n')
    out = tmp_path / "segments.jsonl"
    assert run("trim-to-segments", cuts, "--out", out) == 0
    assert out.read_bytes() == b""


def test_trim_to_segments_cross_checks_recording_ids(tmp_path):  # test_cli.cpp:156-178
    paths, _ = make_fixture(tmp_path)
    cuts = tmp_path / "cuts.jsonl"
    cuts.write_text('{"id": "ghost", "supervisions": [{"speaker": "a", "start": 0.0, "duration": 1.0}]}\n')
    assert run("trim-to-segments", cuts, "--out", tmp_path / "out.jsonl", "--recordings", paths.recordings) == 1
    good = tmp_path / "good_cuts.jsonl"
    good.write_text('{"id": "rec0", "supervisions": [{"speaker": "a", "start": 0.0, "duration": 1.0}]}\n')
    assert run("trim-to-segments", good, "--out", tmp_path / "out.jsonl", "--recordings", paths.recordings) == 0
    nameless = tmp_path / "nameless.jsonl"
    nameless.write_text('{"start": 0.0, "duration": 1.0}\n')
    assert run("trim-to-segments", nameless, "--out", tmp_path / "out.jsonl") == 1


def test_pick_format_follows_the_extension():  # cli.hpp:32-41
    from paper_2212_05271_b200.gss import cli
    assert cli.pick_format("a.rttm", "auto") == "rttm" and cli.pick_format("a.rttm.gz", "auto") == "rttm"
    assert cli.pick_format("a.jsonl.gz", "auto") == "jsonl" and cli.pick_format("a.rttm", "jsonl") == "jsonl"


@pytest.mark.gpu
def test_enhance_writes_outputs_and_echoes_every_flag(tmp_path):  # test_cli.cpp:184-222
    paths, _ = make_fixture(tmp_path, 3)
    out_dir = str(tmp_path / "out")
    code = run("enhance", paths.recordings, paths.segments, "--out-dir", out_dir, "--segment-format", "jsonl",
               "--max-batch-duration", "30", "--context-duration", "1.5", "--bss-iterations", "2", "--no-wpe",
               "--channels", "0,2", "--one-per-batch", "--workers", "1", "--queue-capacity", "3", "--seed", "7")
    assert code == 0
    assert os.path.exists(out_dir + "/rec0-spk0-0000500_0003500.wav")
    assert os.path.exists(out_dir + "/rec0-spk1-0004000_0007000.wav")
    summary = json.load(open(out_dir + "/summary.json"))
    echo = summary["config"]
    want = {"max-batch-duration": 30.0, "context-duration": 1.5, "bss-iterations": 2, "no-wpe": True,
            "no-noise-class": False, "channels": [0, 2], "one-per-batch": True, "workers": 1, "queue-capacity": 3,
            "seed": 7, "out-dir": out_dir, "recordings": paths.recordings, "segments": paths.segments,
            "segment-format": "jsonl"}
    for k, v in want.items():
        assert echo[k] == v, k
    assert summary["segments_written"] == 2


@pytest.mark.gpu
def test_enhance_exits_1_when_segments_fail(tmp_path):  # test_cli.cpp:224-250
    paths, _ = make_fixture(tmp_path)
    recordings = tmp_path / "recordings2.jsonl"
    recordings.write_text(open(paths.recordings).read() +
                          '{"id": "broken", "sample_rate": 16000, "duration": 8.0, "sources": [{"path": "%s", '
                          '"channels": [0, 1]}]}\n' % (tmp_path / "missing.wav"))
    segments = tmp_path / "segments2.jsonl"
    segments.write_text(open(paths.segments).read() +
                        '{"id": "broken-0", "recording_id": "broken", "start": 1.0, "duration": 2.0, '
                        '"speaker": "spk0"}\n')
    code = run("enhance", recordings, segments, "--out-dir", tmp_path / "out", "--context-duration", "1",
               "--bss-iterations", "2")
    assert code == 1
    summary = json.load(open(tmp_path / "out" / "summary.json"))
    assert summary["segments_written"] == 2 and len(summary["failures"]) == 1


@pytest.mark.gpu
def test_bench_sweeps_the_grid_and_writes_a_csv(tmp_path):  # test_cli.cpp:256-300
    _, spec = make_fixture(tmp_path / "fx")
    spec_path = tmp_path / "spec.json"
    spec_path.write_text(json.dumps(spec.to_json()))
    assert run("bench", spec_path, "--out-dir", tmp_path / "bench", "--contexts", "1", "--iterations", "2",
               "--channels", "2") == 0
    lines = (tmp_path / "bench" / "results.csv").read_text().split("\n")
    assert lines[0] == "context_s,bss_iterations,channels,speaker,input_si_sdr_db,enhanced_si_sdr_db,improvement_db"
    rows = [r for r in lines[1:] if r]
    assert len(rows) == 2 and all(r.startswith("1,2,2,spk") for r in rows)
    (tmp_path / "broken.json").write_text("{ not json")
    assert run("bench", tmp_path / "broken.json") == 2
    (tmp_path / "empty_speakers.json").write_text('{"duration": 4.0, "speakers": []}')
    assert run("bench", tmp_path / "empty_speakers.json") == 2
