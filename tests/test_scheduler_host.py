"""Batch planning and super-segment assembly (scheduler.hpp:101-275) against the reference's
test_scheduler.cpp cases. CPU only: the integer arithmetic runs in the library's host code, the audio is
read from WAV files written by the test."""
import numpy as np
import pytest

from paper_2212_05271_b200.gss import ShapeError, manifests as mf, scheduler as sc, stft, wav, wpe
from .refrng import Rng


def seg(i, r, sp, start, dur):
    return mf.Segment(r, sp, start, dur, i)


def ids(plans):
    return [[p.id for p in b.parts] for b in plans]


def test_plan_batches_packs_one_speaker_greedily():  # test_scheduler.cpp:49-62
    plans = sc.plan_batches([seg("s0", "r", "a", 0.0, 20.0), seg("s1", "r", "a", 30.0, 20.0),
                             seg("s2", "r", "a", 60.0, 20.0)], 50.0)
    assert ids(plans) == [["s0", "s1"], ["s2"]]


def test_plan_batches_round_robin_across_groups():  # test_scheduler.cpp:64-75
    plans = sc.plan_batches([seg("a0", "r", "a", 0.0, 10.0), seg("b0", "r", "b", 5.0, 10.0),
                             seg("a1", "r", "a", 40.0, 10.0)], 15.0)
    assert ids(plans) == [["a0"], ["b0"], ["a1"]]


def test_one_per_batch_never_merges():  # test_scheduler.cpp:77-90
    plans = sc.plan_batches([seg("a0", "r", "a", 0.0, 2.0), seg("a1", "r", "a", 3.0, 2.0),
                             seg("b0", "r", "b", 1.0, 2.0)], 50.0, sc.ONE_PER_BATCH)
    assert ids(plans) == [["a0"], ["b0"], ["a1"]]


def test_oversized_segments_stay_singletons():  # test_scheduler.cpp:92-102
    plans = sc.plan_batches([seg("big", "r", "a", 0.0, 60.0), seg("small", "r", "a", 70.0, 5.0)], 50.0)
    assert ids(plans) == [["big"], ["small"]]
    # a following short segment never joins an oversized singleton either way round
    plans = sc.plan_batches([seg("small", "r", "a", 0.0, 5.0), seg("big", "r", "a", 10.0, 60.0),
                             seg("tail", "r", "a", 80.0, 5.0)], 50.0)
    assert ids(plans) == [["small"], ["big"], ["tail"]]


def test_plan_batches_sorts_parts_temporally():  # test_scheduler.cpp:104-116
    plans = sc.plan_batches([seg("late", "r", "a", 12.0, 3.0), seg("early", "r", "a", 1.0, 3.0),
                             seg("mid", "r", "a", 6.0, 3.0)], 50.0)
    assert ids(plans) == [["early", "mid", "late"]]


def test_same_speaker_in_different_recordings_forms_separate_groups():  # test_scheduler.cpp:118-126
    plans = sc.plan_batches([seg("x0", "r1", "a", 0.0, 2.0), seg("x1", "r2", "a", 0.0, 2.0)], 50.0)
    assert [p.recording_id for p in plans] == ["r1", "r2"]


def fast_config(out_dir):  # test_scheduler.cpp:27-36: context 1 s, 2 iterations, default 1024/256 STFT
    return sc.PipelineConfig(stft.StftConfig(), wpe.WpeConfig(4, 2, 1, 0, 1e-10), True, 2, 1.0, True,
                             out_dir=out_dir)


def write_recording(tmp_path, name, seconds, channels, seed, sr=16000):
    rng = Rng(seed)
    x = np.array([[rng.uniform() * 2 - 1 for _ in range(int(seconds * sr))] for _ in range(channels)], np.float32)
    path = str(tmp_path / (name + ".wav"))
    wav.write(path, stft.RealSignal(x, sr))
    return mf.Recording(name, [mf.Source(path, list(range(channels)))], sr, float(seconds)), x


def test_assemble_concatenates_spans_and_maps_frame_centers(tmp_path):  # test_scheduler.cpp:132-201
    rec, src = write_recording(tmp_path, "rec", 8.0, 2, 3)
    segs = [seg("s-0", "rec", "s", 2.0, 3.0), seg("s-1", "rec", "s", 6.0, 1.0), seg("o-0", "rec", "o", 0.0, 1.5)]
    cfg = fast_config(str(tmp_path))
    ss = sc.assemble(sc.BatchPlan("rec", "s", [segs[0], segs[1]]), rec, segs, cfg)
    sr = 16000
    # spans: [1,2) ctx + [2,5) + [6,7) + [7,8) ctx, 6 s total, gap removed
    assert ss.audio.sample_rate == sr and ss.audio.num_channels() == 2 and ss.audio.num_samples() == 6 * sr
    assert ss.context_left == 1.0 and ss.context_right == 1.0
    assert [(p.sample_begin, p.sample_end) for p in ss.parts] == [(1 * sr, 4 * sr), (4 * sr, 5 * sr)]
    # the assembled waveform equals the source with [5,6) spliced out, sample for sample
    want = np.concatenate([src[:, 1 * sr:5 * sr], src[:, 6 * sr:8 * sr]], axis=1)
    assert ss.audio.channels.tobytes() == want.tobytes()
    # frame centers walk the spans in source coordinates
    frames = stft.frame_count(6 * sr, cfg.stft)
    fc = ss.frame_centers
    assert len(fc) == frames
    assert fc[0] == 1 * sr and fc[249] == 249 * 256 + sr and fc[250] == 6 * sr and fc[-1] == 8 * sr - 1
    # activity covers both speakers plus noise, pinned to the target
    act = ss.activity
    assert act.frames == frames and act.classes == ["o", "s", "noise"]
    assert act.classes[act.target_index] == "s" and act.noise_index == 2
    assert act.at(0, act.target_index) == 0 and act.at(100, act.target_index) == 1
    assert act.at(31, 0) == 1 and act.at(32, 0) == 0  # "o" is active only where source time < 1.5 s


def test_assemble_clips_context_at_the_recording_edges(tmp_path):  # test_scheduler.cpp:203-232
    rec, _ = write_recording(tmp_path, "rec", 4.0, 1, 5)
    segs = [seg("s-0", "rec", "s", 0.2, 1.0), seg("s-1", "rec", "s", 3.5, 0.5)]
    cfg = fast_config(str(tmp_path))
    a = sc.assemble(sc.BatchPlan("rec", "s", [segs[0]]), rec, segs, cfg)
    assert a.context_left == pytest.approx(0.2) and a.context_right == pytest.approx(1.0)
    b = sc.assemble(sc.BatchPlan("rec", "s", [segs[1]]), rec, segs, cfg)
    assert b.context_left == pytest.approx(1.0) and b.context_right == pytest.approx(0.0)


def test_assemble_overlapping_parts_are_longer_than_the_recording(tmp_path):
    # scheduler.hpp:196-222: spans are concatenated as they come, so overlapping parts of one speaker are
    # assembled twice and the right context starts at the LAST part's end (not the furthest end)
    st = stft.StftConfig()
    ap = sc.assemble_indices([(0.0, 40.0), (1.0, 1.0)], 16000, 41 * 16000, 15.0, st)
    sr = 16000
    assert ap.spans == [(0, 40 * sr), (1 * sr, 2 * sr), (2 * sr, 17 * sr)]
    assert ap.total == 56 * sr and len(ap.frame_centers) == stft.frame_count(56 * sr, st)
    assert list(ap.part_begin) == [0, 40 * sr] and list(ap.part_end) == [40 * sr, 41 * sr]
    assert ap.context_left == 0.0 and ap.context_right == 15.0
    # centres walk the spans in source time: the second span starts again at 1 s
    t = (40 * sr + st.shift - 1) // st.shift
    assert ap.frame_centers[t] == 1 * sr + (t * st.shift - 40 * sr)
    assert ap.frame_centers[-1] == 17 * sr - 1
    # the whole loader path
    rec, src = write_recording(tmp_path, "rec", 5.0, 1, 21)
    segs = [seg("a", "rec", "s", 0.5, 3.0), seg("b", "rec", "s", 1.0, 1.0)]
    ss = sc.assemble(sc.BatchPlan("rec", "s", segs), rec, segs, fast_config(str(tmp_path)))
    h = sr // 2
    want = np.concatenate([src[:, 0:h], src[:, h:7 * h], src[:, 2 * h:4 * h], src[:, 4 * h:6 * h]], axis=1)
    assert ss.audio.num_samples() == 11 * h > rec.num_samples() - 1 and ss.audio.channels.tobytes() == want.tobytes()


def test_assemble_rejects_empty_sample_ranges_and_honors_channel_subsets(tmp_path):
    rec, src = write_recording(tmp_path, "rec", 2.0, 3, 8)
    cfg = fast_config(str(tmp_path))
    with pytest.raises(ShapeError):  # scheduler.hpp:210-213: the segment starts past the recording's end
        sc.assemble(sc.BatchPlan("rec", "s", [seg("late", "rec", "s", 2.5, 0.5)]), rec, [], cfg)
    cfg.channels = [2, 0]
    one = seg("s-0", "rec", "s", 0.5, 1.0)
    ss = sc.assemble(sc.BatchPlan("rec", "s", [one]), rec, [one], cfg)
    assert ss.audio.num_channels() == 2 and ss.audio.channels.tobytes() == src[[2, 0]].tobytes()


def test_output_name_and_config_echo():  # scheduler.hpp:303-308, :60-81
    assert sc.output_name("rec", "s", 1.0, 3.0) == "rec-s-0001000_0003000.wav"
    assert sc.output_name("rec", "s", 3.5, 4.75) == "rec-s-0003500_0004750.wav"
    assert sc.output_name("r", "a", 0.0005, 0.0015) == "r-a-0000001_0000002.wav"  # llround, not banker's rounding
    echo = fast_config("o").echo()
    assert list(echo)[:5] == ["max-batch-duration", "context-duration", "bss-iterations", "no-wpe", "no-noise-class"]
    assert echo["max-batch-duration"] == 50.0 and echo["context-duration"] == 1.0 and echo["bss-iterations"] == 2
    assert echo["no-wpe"] is False and echo["workers"] == 0 and echo["fft-size"] == 1024


def test_ordered_queue_hands_out_plan_order():  # scheduler.hpp:383-412
    import threading
    q = sc.OrderedBatchQueue(2)
    got = []
    consumer = threading.Thread(target=lambda: got.extend(q.take().index for _ in range(4)))
    consumer.start()
    producers = [threading.Thread(target=q.put, args=(sc.LoadedBatch(i),)) for i in (1, 0, 3, 2)]
    for t in producers:
        t.start()
    for t in producers:
        t.join()
    consumer.join()
    assert got == [0, 1, 2, 3]


def test_ordered_queue_close_releases_blocked_loaders():
    import threading
    q = sc.OrderedBatchQueue(1)
    done = []
    t = threading.Thread(target=lambda: done.append(q.put(sc.LoadedBatch(5))))  # far ahead of the window: blocks
    t.start()
    t.join(0.1)
    assert t.is_alive()
    q.close()
    t.join(5)
    assert not t.is_alive() and done == [False]


@pytest.mark.parametrize("workers", [0, 3])
def test_run_pipeline_turns_a_device_failure_into_batch_failures(tmp_path, workers):
    # A call-level failure of the compute slot (here: a device that does not exist, on any box) must fail that
    # slot's batches and let the run finish with a summary, as the C++ mirror does, instead of escaping from
    # run_pipeline with the loader threads still blocked in the queue.
    import json
    import threading
    rec, _ = write_recording(tmp_path, "rec", 6.0, 2, 4)
    segs = [seg("s-%d" % i, "rec", "s", 0.5 + i, 0.8) for i in range(5)]
    cfg = fast_config(str(tmp_path / "out"))
    cfg.workers, cfg.queue_capacity, cfg.mode = workers, 1, sc.ONE_PER_BATCH
    before = threading.active_count()
    run = sc.run_pipeline([rec], segs, cfg, devices=[999], gpu_batch=2)
    assert run.failed_segments == 5 and run.json["segments_written"] == 0
    assert sorted(f["segment_id"] for f in run.json["failures"]) == [s.id for s in segs]
    assert all("Error" in f["error"] for f in run.json["failures"])
    assert json.load(open(cfg.out_dir + "/summary.json"))["failures"] == run.json["failures"]
    assert threading.active_count() == before  # loaders, writer and slot threads are gone
