"""Manifest wire formats against the reference's golden files (tests/golden/, copied from the reference's
tests/data) and its test_manifests.cpp cases (CPU only; no device work)."""
import gzip
import os

import numpy as np
import pytest

from paper_2212_05271_b200.gss import ConfigError, IoError, ParseError, manifests as mf, wav
from paper_2212_05271_b200.gss.stft import RealSignal

DATA = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_recordings_golden_loads_with_stacked_sources():  # test_manifests.cpp:22-34
    recs = mf.load_recordings(DATA + "/recordings_golden.jsonl")
    assert len(recs) == 2
    assert recs[0].id == "meet01" and len(recs[0].sources) == 2 and recs[0].sources[0].channels == [0, 1]
    assert recs[0].channel_count() == 3 and recs[0].sample_rate == 16000 and recs[0].duration == 120.5
    assert recs[0].num_samples() == 1928000
    assert recs[1].channel_count() == 4


def test_recordings_serialization_round_trips(tmp_path):  # test_manifests.cpp:36-48
    recs = mf.load_recordings(DATA + "/recordings_golden.jsonl")
    path = str(tmp_path / "recordings_echo.jsonl")
    mf.save_recordings(path, recs)
    assert mf.load_recordings(path) == recs
    # nlohmann's dump(): insertion order, no spaces
    assert open(path).readline() == ('{"id":"meet01","sources":[{"path":"audio/meet01_a.wav","channels":[0,1]},'
                                     '{"path":"audio/meet01_b.wav","channels":[0]}],"sample_rate":16000,'
                                     '"duration":120.5}\n')


def test_recordings_loader_rejects_bad_manifests():  # test_manifests.cpp:50-62
    with pytest.raises(ParseError):
        mf.load_recordings(DATA + "/recordings_dup.jsonl")
    with pytest.raises(IoError):
        mf.load_recordings(DATA + "/missing.jsonl")
    with pytest.raises(ParseError) as e:  # malformed JSON carries path:line context
        mf.load_recordings(DATA + "/segments_broken.jsonl")
    assert "segments_broken.jsonl:1" in str(e.value)


def test_segments_golden_loads_in_order():  # test_manifests.cpp:68-82
    skipped = [-1]
    segs = mf.load_segments(DATA + "/segments_golden.jsonl", mf.JSONL, skipped)
    assert len(segs) == 4 and skipped == [0]
    s = segs[0]
    assert (s.id, s.recording_id, s.speaker, s.start, s.duration, s.end()) == ("meet01-alice-0000", "meet01",
                                                                               "alice", 1.5, 4.25, 5.75)
    assert segs[3].speaker == "carol"


def test_gzipped_segments_load_identically(tmp_path):  # test_manifests.cpp:84-100
    # the reference tree does not ship segments_golden.jsonl.gz: it is made from the .jsonl
    plain = mf.load_segments(DATA + "/segments_golden.jsonl")
    gz_path = str(tmp_path / "segments_golden.jsonl.gz")
    with gzip.open(gz_path, "wb") as f:
        f.write(open(DATA + "/segments_golden.jsonl", "rb").read())
    assert mf.load_segments(gz_path) == plain
    echo = str(tmp_path / "echo.jsonl.gz")  # writing through the gz path round trips too
    mf.save_segments(echo, plain)
    assert mf.load_segments(echo) == plain
    assert gzip.open(echo, "rb").read().decode() == mf.serialize_segments(plain)


def test_zero_or_negative_duration_segments_are_skipped_with_a_count():  # test_manifests.cpp:102-110
    skipped = []
    segs = mf.load_segments(DATA + "/segments_zero_duration.jsonl", mf.JSONL, skipped)
    assert [s.id for s in segs] == ["meet01-alice-0000", "meet01-bob-0001"] and skipped == [2]


def test_rttm_golden_maps_fields_and_synthesizes_ids():  # test_manifests.cpp:116-133
    skipped = []
    segs = mf.load_segments(DATA + "/segments_golden.rttm", mf.RTTM, skipped)
    assert len(segs) == 4 and skipped == [1]  # one zero-duration line dropped
    assert (segs[0].recording_id, segs[0].speaker, segs[0].start, segs[0].duration) == ("meet01", "alice", 1.5, 4.25)
    assert [s.id for s in segs] == ["meet01-alice-0000", "meet01-bob-0000", "meet01-alice-0001", "meet02-carol-0000"]
    # the RTTM and the JSONL goldens describe the same segments
    assert segs == mf.load_segments(DATA + "/segments_golden.jsonl")


def test_malformed_rttm_lines_raise_parse_error_with_location():  # test_manifests.cpp:135-146
    with pytest.raises(ParseError) as e:
        mf.load_segments(DATA + "/segments_malformed.rttm", mf.RTTM)
    assert ":2" in str(e.value)
    with pytest.raises(ParseError):
        mf.load_segments(DATA + "/segments_badnum.rttm", mf.RTTM)


def test_validate_flags_unknown_recordings_duplicates_and_overruns():  # test_manifests.cpp:152-166
    recs = mf.load_recordings(DATA + "/recordings_golden.jsonl")
    segs = mf.load_segments(DATA + "/segments_golden.jsonl")
    assert mf.validate(recs, segs) == []
    S = lambda i, r, sp, st, d: mf.Segment(r, sp, st, d, i)  # noqa: E731
    broken = segs + [S("dup", "meet01", "alice", 1.0, 1.0), S("dup", "meet01", "alice", 2.0, 1.0),
                     S("x1", "nope", "alice", 1.0, 1.0), S("x2", "meet02", "carol", 60.0, 10.0),
                     S("x3", "meet01", "bob", -0.5, 1.0)]
    assert len(mf.validate(recs, broken)) == 4


def test_load_audio_stacks_sources_and_honors_channel_subsets(tmp_path):  # test_manifests.cpp:221-258
    sr = 8000
    a, b = str(tmp_path / "srcA.wav"), str(tmp_path / "srcB.wav")
    wav.write(a, RealSignal(np.stack([np.full(800, 1.0, np.float32), np.full(800, 2.0, np.float32)]), sr))
    wav.write(b, RealSignal(np.arange(800, dtype=np.float32).reshape(1, -1), sr))
    rec = mf.Recording("r", [mf.Source(a, [0, 1]), mf.Source(b, [0])], sr, 0.1)
    full = mf.load_audio(rec, 100, 50)
    assert full.num_channels() == 3 and full.num_samples() == 50
    assert (full.channels[0][0], full.channels[1][0], full.channels[2][0]) == (1.0, 2.0, 100.0)
    subset = mf.load_audio(rec, 0, 10, [2, 0])
    assert subset.num_channels() == 2 and subset.channels[0][5] == 5.0 and subset.channels[1][5] == 1.0
    with pytest.raises(ConfigError):
        mf.load_audio(rec, 0, 10, [3])
    with pytest.raises(ConfigError):
        mf.load_audio(mf.Recording("r", rec.sources, 16000, 0.1), 0, 10)
    with pytest.raises(IoError):  # the file is shorter than the requested window
        mf.load_audio(rec, 790, 50)


def test_llround_matches_the_c_library():
    assert [mf.llround(x) for x in (0.5, 1.5, 2.5, -0.5, -2.5, 2.4999, 1e6 + 0.5)] == [1, 2, 3, -1, -3, 2, 1000001]
