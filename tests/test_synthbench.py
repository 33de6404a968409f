"""The synthbench harness (synthbench.hpp:68-726) and the C3 / C4 acceptance gates (acceptance.cpp:287-367).

CPU part: the cases of the reference's tests/test_synthbench.cpp that need no spectral operator (spec validation,
JSON round trip, generator properties, the SI-SDR metric, span cutting, fixture files). GPU part: the oracle-mask
MVDR ceiling, separation quality on the standard fixture (>= 10 dB SI-SDR improvement, <= 5 dB from the
oracle-mask MVDR) and the ablation orderings on the reverberant fixture, all through the product path."""
import json
import math
import statistics

import numpy as np
import pytest

from .refrng import Rng


@pytest.fixture(scope="module")
def hb():
    from synthbench import harness
    return harness


def tiny_spec(hb):  # test_synthbench.cpp:16-27
    return hb.MixtureSpec(8.0, 16000, 2, 11, [hb.SpeakerLayout("spk0", [(0.5, 3.0)]),
                                              hb.SpeakerLayout("spk1", [(4.0, 3.0)])], "delays", 0.0, 20.0)


def l2_rel_err(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def test_spec_validation_rejects_bad_layouts(hb):  # test_synthbench.cpp:35-58
    from synthbench import SpecError
    tiny_spec(hb).validate()
    for edit in (lambda s: s.speakers[0].segments.__setitem__(0, (6.0, 3.0)),
                 lambda s: s.speakers[0].segments.__setitem__(0, (-0.5, 1.0)),
                 lambda s: s.speakers[0].segments.__setitem__(0, (1.0, 0.0)),
                 lambda s: s.speakers.clear(),
                 lambda s: setattr(s, "reverb_t60", 2.5)):
        spec = tiny_spec(hb)
        edit(spec)
        with pytest.raises(SpecError):
            spec.validate()
        with pytest.raises(SpecError):
            hb.generate(spec)


def test_spec_survives_a_json_roundtrip(hb):  # test_synthbench.cpp:60-81
    from synthbench import SpecError
    spec = tiny_spec(hb)
    spec.reverb_t60, spec.steering, spec.noise_snr = 0.25, "random_phase", 15.0
    back = hb.MixtureSpec.from_json(json.loads(json.dumps(spec.to_json())))
    assert back == spec
    assert back.speakers[1].name == "spk1" and back.speakers[1].segments[0][0] == 4.0
    assert list(spec.to_json()) == ["duration", "sample_rate", "channels", "seed", "steering", "reverb_t60",
                                    "noise_snr", "speakers"]
    bad = spec.to_json()
    bad["steering"] = "sideways"
    with pytest.raises(SpecError):
        hb.MixtureSpec.from_json(bad)


def test_generate_is_bitwise_deterministic(hb):  # test_synthbench.cpp:93-107
    a, b = hb.generate(tiny_spec(hb)), hb.generate(tiny_spec(hb))
    assert a.mixture.channels.tobytes() == b.mixture.channels.tobytes()
    assert a.dry.tobytes() == b.dry.tobytes() and a.images0.tobytes() == b.images0.tobytes()


def test_single_anechoic_speaker_lands_on_channel_0_unchanged(hb):  # test_synthbench.cpp:109-116
    spec = tiny_spec(hb)
    spec.speakers, spec.noise_snr = [hb.SpeakerLayout("only", [(1.0, 5.0)])], 300.0
    mix = hb.generate(spec)
    assert l2_rel_err(mix.mixture.channels[0], mix.dry[0]) < 1e-6
    assert l2_rel_err(mix.images0[0], mix.dry[0]) < 1e-12


def test_channel_0_is_the_sum_of_the_speaker_images(hb):  # test_synthbench.cpp:118-127
    spec = tiny_spec(hb)
    spec.noise_snr = 300.0
    mix = hb.generate(spec)
    assert l2_rel_err(mix.mixture.channels[0], mix.images0.sum(axis=0, dtype=np.float32)) < 1e-6


def test_generate_emits_one_manifest_segment_per_layout_entry(hb):  # test_synthbench.cpp:129-138
    mix = hb.generate(tiny_spec(hb))
    assert [(s.id, s.speaker, s.start, s.duration) for s in mix.segments] == [("spk0-0000", "spk0", 0.5, 3.0),
                                                                             ("spk1-0000", "spk1", 4.0, 3.0)]
    assert mix.speaker_names == ["spk0", "spk1"]


def test_steering_delays_vanish_on_channel_0_and_stay_small():  # test_synthbench.cpp:140-149
    import synthbench
    lib = synthbench._load()
    for k in range(5):
        assert lib.gss_synth_steering_delay(k, 0) == 0
        assert all(1 <= lib.gss_synth_steering_delay(k, c) <= 9 for c in range(1, 8))


def test_reverberant_generation_adds_a_tail(hb):  # test_synthbench.cpp:151-168
    spec = tiny_spec(hb)
    spec.speakers, spec.noise_snr, spec.reverb_t60 = [hb.SpeakerLayout("only", [(0.5, 2.0)])], 300.0, 0.4
    mix = hb.generate(spec)
    lo, hi = int(2.6 * 16000), int(2.9 * 16000)
    assert float(np.sum(mix.dry[0][lo:hi].astype(np.float64) ** 2)) == 0.0
    assert float(np.sum(mix.images0[0][lo:hi].astype(np.float64) ** 2)) > 0.0


def test_si_sdr_caps_exact_and_scaled_matches(hb):  # test_synthbench.cpp:174-183
    ref = np.sin(2.0 * math.pi * 100.0 * np.arange(16000) / 16000.0).astype(np.float32)
    assert hb.si_sdr(ref, ref) == hb.SI_SDR_CAP
    assert hb.si_sdr(ref * np.float32(2.0), ref) == hb.SI_SDR_CAP


def test_si_sdr_of_reference_plus_equal_power_orthogonal_noise_is_0_db(hb):  # test_synthbench.cpp:185-195
    n = 16000
    s = np.sin(2.0 * math.pi * 100.0 * np.arange(n) / n)
    o = np.cos(2.0 * math.pi * 200.0 * np.arange(n) / n)
    assert abs(hb.si_sdr((s + o).astype(np.float32), s.astype(np.float32))) < 1e-4


def test_si_sdr_is_scale_invariant_and_decreases_with_noise(hb):  # test_synthbench.cpp:197-225
    from paper_2212_05271_b200.gss import DegenerateStatsError
    rng = Rng(5)
    n = 8000
    pairs = [(rng.gaussian(), rng.gaussian()) for _ in range(n)]
    ref = np.array([p[0] for p in pairs], np.float32)
    noise = np.array([p[1] for p in pairs], np.float32)

    def mixed(w):
        return ref + np.float32(w) * noise

    assert hb.si_sdr(mixed(0.1), ref) > hb.si_sdr(mixed(0.5), ref)
    base = hb.si_sdr(mixed(0.3), ref)
    assert abs(hb.si_sdr(mixed(0.3) * np.float32(0.3), ref) - base) < 1e-6
    zeros = np.zeros(n, np.float32)
    with pytest.raises(DegenerateStatsError):
        hb.si_sdr(ref, zeros)
    with pytest.raises(DegenerateStatsError):
        hb.si_sdr_best_shift(ref, zeros)


def test_si_sdr_best_shift_recovers_a_small_time_offset(hb):  # test_synthbench.cpp:227-244
    rng = Rng(8)
    n = 16000
    ref = np.array([rng.gaussian() for _ in range(n)], np.float32)
    delayed = np.zeros(n, np.float32)
    delayed[7:] = ref[:-7]
    assert hb.si_sdr(delayed, ref) < 5.0
    assert hb.si_sdr_best_shift(delayed, ref) == hb.SI_SDR_CAP
    assert hb.si_sdr_best_shift(ref, ref) == hb.SI_SDR_CAP
    noisy = ref + np.float32(0.2) * np.array([rng.gaussian() for _ in range(n)], np.float32)
    assert hb.si_sdr_best_shift(noisy, ref) >= hb.si_sdr(noisy, ref)


def test_si_sdr_matches_a_plain_double_loop(hb):
    # the metric as the reference writes it (synthbench.hpp:448-468), evaluated sample by sample
    rng = np.random.RandomState(3)
    ref = rng.randn(500).astype(np.float32)
    est = (0.7 * ref + 0.3 * rng.randn(500)).astype(np.float32)
    dot = sum(float(e) * float(r) for e, r in zip(est, ref))
    energy = sum(float(r) * float(r) for r in ref)
    alpha = dot / energy
    err = sum((alpha * float(r) - float(e)) ** 2 for e, r in zip(est, ref))
    assert abs(hb.si_sdr(est, ref) - 10.0 * math.log10(alpha * alpha * energy / err)) < 1e-9


def test_concat_spans_cuts_and_orders_the_speakers_samples(hb):  # test_synthbench.cpp:246-262
    from paper_2212_05271_b200.gss.manifests import Segment
    x = np.arange(10, dtype=np.float32)
    segs = [Segment("", "a", 3.0, 1.0), Segment("", "b", 0.0, 1.0), Segment("", "a", 1.0, 1.5)]
    assert hb.concat_spans(x, segs, "a", 2).tolist() == [2, 3, 4, 6, 7]
    assert len(hb.concat_spans(x, segs, "nobody", 2)) == 0


def test_save_fixture_writes_loadable_manifests(hb, tmp_path):  # test_synthbench.cpp:287-315
    from paper_2212_05271_b200.gss import manifests
    mix = hb.generate(tiny_spec(hb))
    paths = hb.save_fixture(mix, str(tmp_path / "synthfix"), "rec0")
    recs = manifests.load_recordings(paths.recordings)
    assert len(recs) == 1 and recs[0].id == "rec0" and recs[0].sample_rate == 16000
    assert recs[0].channel_count() == 2 and recs[0].duration == pytest.approx(8.0)
    skipped = [0]
    segs = manifests.load_segments(paths.segments, manifests.JSONL, skipped)
    assert len(segs) == 2 and skipped == [0] and segs[0].recording_id == "rec0"
    audio = manifests.load_audio(recs[0], 0, 16000)
    assert audio.channels.shape == (2, 16000)
    assert audio.channels[0].tobytes() == mix.mixture.channels[0][:16000].tobytes()  # float WAV is exact


def test_canned_fixtures_validate(hb):  # test_synthbench.cpp:317-324
    for spec in (hb.standard_fixture(), hb.reverberant_fixture(8), hb.ten_minute_fixture(), hb.fifty_segment_fixture()):
        spec.validate()
    assert len(hb.fifty_segment_fixture().speakers[0].segments) == 50
    assert hb.ten_minute_fixture().duration == 600.0
    assert hb.reverberant_fixture(8).channels == 8 and hb.reverberant_fixture().reverb_t60 == 0.3


# ---------------------------------------------------------------------------------------------------------------
# on the device
# ---------------------------------------------------------------------------------------------------------------
@pytest.mark.gpu
def test_oracle_beamformer_beats_the_best_input_channel(hb):  # test_synthbench.cpp:268-285
    from paper_2212_05271_b200 import gss
    spec = tiny_spec(hb)
    spec.channels = 4
    spec.speakers[0].segments = [(0.5, 5.0)]
    spec.speakers[1].segments = [(2.0, 5.0)]
    mix = hb.generate(spec)
    res = hb.oracle_mvdr(mix, gss.stft.StftConfig(sample_rate=spec.sample_rate))
    assert len(res.si_sdr_db) == 2 and len(res.enhanced) == 2
    for k in range(2):
        assert res.si_sdr_db[k] > hb.best_input_si_sdr(mix, k)


@pytest.mark.gpu
def test_oracle_mask_mvdr_matches_the_cpu_oracle_operators(hb, oracle):
    # the same ideal-ratio masks through the CPU oracle's stats / reference / MVDR / apply / iSTFT
    from paper_2212_05271_b200 import gss
    spec = tiny_spec(hb)
    spec.channels = 3
    spec.speakers[0].segments = [(0.5, 4.0)]
    spec.speakers[1].segments = [(2.0, 4.0)]
    mix = hb.generate(spec)
    cfg = gss.stft.StftConfig(sample_rate=16000)
    res = hb.oracle_mvdr(mix, cfg)
    ocfg = oracle.stft_cfg(cfg.fft_size, cfg.shift, cfg.window, cfg.sample_rate)
    y = oracle.stft(mix.mixture.channels, ocfg)
    residual = mix.mixture.channels[0].copy()
    for k in range(2):
        residual -= mix.images0[k]
    sp = oracle.stft(np.concatenate([mix.images0, residual[None]], 0), ocfg)
    p = np.abs(sp.astype(np.complex128)) ** 2
    tot = p.sum(axis=2, keepdims=True)
    gamma = np.where(tot > 0, p / np.where(tot > 0, tot, 1.0), np.array([0, 0, 1.0])).astype(np.float32)
    for k in range(2):
        tgt, bg = oracle.mvdr_stats(y, gamma, k)
        ref = oracle.select_reference(tgt, bg)
        h, _ = oracle.mvdr(tgt, bg, ref)
        want = oracle.istft(oracle.apply_filter(h, y), ocfg, mix.mixture.channels.shape[1])
        err = np.sum((res.enhanced[k].astype(np.float64) - want.reshape(-1)) ** 2)
        assert 10 * np.log10(np.sum(want.astype(np.float64) ** 2) / max(err, 1e-300)) >= 60.0


@pytest.mark.gpu
def test_separation_quality_on_the_standard_fixture(hb, tmp_path):  # acceptance.cpp:287-322 (criterion 3)
    from paper_2212_05271_b200 import gss
    spec = hb.standard_fixture()
    mix = hb.generate(spec)
    paths = hb.save_fixture(mix, str(tmp_path / "in"), "fix")
    cfg = gss.scheduler.PipelineConfig(out_dir=str(tmp_path / "out"))   # the reference defaults: 1024 / 256, WPE, 20 iters
    run = hb.run_fixture(mix, paths, cfg)
    ceiling = hb.oracle_mvdr(mix, gss.stft.StftConfig(sample_rate=spec.sample_rate))
    detail = []
    for k, name in enumerate(mix.speaker_names):
        improvement = run.speaker_si_sdr[k] - hb.best_input_si_sdr(mix, k)
        gap = ceiling.si_sdr_db[k] - run.speaker_si_sdr[k]
        detail.append("%s +%.1f dB (oracle gap %.1f dB)" % (name, improvement, gap))
        assert improvement >= 10.0 and gap <= 5.0, detail
    print("criterion 3:", ", ".join(detail), "; %.2f s" % run.wall_seconds)
    assert run.wall_seconds < 120.0


@pytest.mark.gpu
def test_ablation_orderings_on_the_reverberant_fixture(hb, tmp_path):  # acceptance.cpp:328-367 (criterion 4)
    from paper_2212_05271_b200 import gss
    mix = hb.generate(hb.reverberant_fixture(8))
    paths = hb.save_fixture(mix, str(tmp_path / "in"), "fix")

    def med(tag, channels, ctx, iters, wpe_on):
        cfg = gss.scheduler.PipelineConfig(out_dir=str(tmp_path / tag), context_duration=ctx, bss_iterations=iters,
                                           enable_wpe=wpe_on, channels=list(range(channels)))
        return statistics.median(hb.run_fixture(mix, paths, cfg).segment_si_sdr)

    base = med("base", 8, 15.0, 5, True)
    no_wpe = med("no_wpe", 8, 15.0, 5, False)
    ctx5 = med("ctx5", 8, 5.0, 5, True)
    it20 = med("it20", 8, 15.0, 20, True)
    ch2 = med("ch2", 2, 15.0, 5, True)
    ch4 = med("ch4", 4, 15.0, 5, True)
    print("criterion 4: median dB: wpe %.1f vs %.1f, ctx15 %.1f vs ctx5 %.1f, it5 %.1f vs it20 %.1f, ch2/4/8 "
          "%.1f/%.1f/%.1f" % (base, no_wpe, base, ctx5, base, it20, ch2, ch4, base))
    assert base > no_wpe
    assert base >= ctx5
    assert base >= it20 - 1.0
    assert ch2 <= ch4 <= base
