"""The reference's synthbench quality harness on the GPU path.

What the reference keeps in synthbench.hpp:68-176 (MixtureSpec / GeneratedMixture), :448-548 (SI-SDR metrics),
:560-623 (oracle-mask MVDR, the calibration ceiling), :628-726 (fixture writing + the four canned layouts), the
fixture runner of tests/acceptance.cpp:75-122 and cli.hpp:228-318 (`gss bench`, the ablation grid). Every
spectral operation here goes through the product's stage operators (`gss.stft.analyze`, `gss.beamform.*`,
`gss.scheduler.run_pipeline`), i.e. through libgss_b200.so on the GPU; the metrics are host-side double sums like
the reference's. Harness code: nothing under paper_2212_05271_b200/ imports it except the `bench` sub-command of
the CLI, lazily.
"""
from __future__ import annotations

import json
import math
import os
import time
from dataclasses import dataclass, field

import numpy as np

from paper_2212_05271_b200 import gss
from paper_2212_05271_b200.gss import manifests, scheduler, stft, wav
from paper_2212_05271_b200.gss.common import DegenerateStatsError

from . import SpecError, generate as _generate

SI_SDR_CAP = 100.0  # synthbench.hpp:444


def _llround(x: float) -> int:
    return manifests.llround(x)


# ---------------------------------------------------------------------------
# MixtureSpec / GeneratedMixture (synthbench.hpp:68-176)
# ---------------------------------------------------------------------------
@dataclass
class SpeakerLayout:
    name: str
    segments: list  # (start, duration) seconds


@dataclass
class MixtureSpec:
    duration: float = 40.0
    sample_rate: int = 16000
    channels: int = 4
    seed: int = 17
    speakers: list = field(default_factory=list)
    steering: str = "delays"
    reverb_t60: float = 0.0
    noise_snr: float = 20.0

    def validate(self) -> None:  # synthbench.hpp:89-109
        if self.duration <= 0 or self.sample_rate <= 0 or self.channels < 1:
            raise SpecError("mixture spec: duration, sample_rate, channels must be positive")
        if not self.speakers:
            raise SpecError("mixture spec: no speakers")
        for spk in self.speakers:
            if not spk.segments:
                raise SpecError("mixture spec: speaker '%s' has no segments" % spk.name)
            for start, dur in spk.segments:
                if start < 0 or dur <= 0 or start + dur > self.duration:
                    raise SpecError("mixture spec: segment [%g, %g) of '%s' outside [0, %g)"
                                    % (start, start + dur, spk.name, self.duration))
        if self.reverb_t60 < 0 or self.reverb_t60 > 2.0:
            raise SpecError("mixture spec: reverb_t60 must be in [0, 2]")
        if self.steering not in ("delays", "random_phase"):
            raise SpecError("mixture spec: unknown steering '%s'" % self.steering)

    @staticmethod
    def from_json(j: dict) -> "MixtureSpec":  # synthbench.hpp:111-137
        spec = MixtureSpec()
        for key in ("duration", "sample_rate", "channels", "seed", "reverb_t60", "noise_snr"):
            if key in j:
                setattr(spec, key, type(getattr(spec, key))(j[key]))
        if "steering" in j:
            if j["steering"] not in ("delays", "random_phase"):
                raise SpecError("mixture spec: unknown steering '%s'" % j["steering"])
            spec.steering = j["steering"]
        try:
            for spk in j["speakers"]:
                spec.speakers.append(SpeakerLayout(str(spk["name"]),
                                                   [(float(s[0]), float(s[1])) for s in spk["segments"]]))
        except (KeyError, IndexError, TypeError) as e:
            raise SpecError("mixture spec: malformed speakers (%s)" % e)
        spec.validate()
        return spec

    def to_json(self) -> dict:  # synthbench.hpp:139-163 (same key order)
        return {"duration": self.duration, "sample_rate": self.sample_rate, "channels": self.channels,
                "seed": self.seed, "steering": self.steering, "reverb_t60": self.reverb_t60,
                "noise_snr": self.noise_snr,
                "speakers": [{"name": s.name, "segments": [[a, b] for a, b in s.segments]} for s in self.speakers]}


@dataclass
class GeneratedMixture:  # synthbench.hpp:166-172
    mixture: stft.RealSignal
    dry: np.ndarray        # (K, N) anechoic, channel-0 aligned
    images0: np.ndarray    # (K, N) channel-0 image incl. reverb
    segments: list
    speaker_names: list


def generate(spec: MixtureSpec) -> GeneratedMixture:  # synthbench.hpp:323-438
    spec.validate()
    if spec.steering != "delays":
        raise SpecError("mixture spec: only 'delays' steering is generated here (random_phase places sources in "
                        "the STFT domain and is used by none of the fixtures, gates or BASELINE configs)")
    mix, dry, img = _generate(spec.duration, spec.sample_rate, spec.channels, spec.seed,
                              [s.segments for s in spec.speakers], spec.reverb_t60, spec.noise_snr, with_sources=True)
    segs = [manifests.Segment("", s.name, float(a), float(b), "%s-%04d" % (s.name, i))
            for s in spec.speakers for i, (a, b) in enumerate(s.segments)]
    return GeneratedMixture(stft.RealSignal(mix, spec.sample_rate), dry, img, segs, [s.name for s in spec.speakers])


# ---------------------------------------------------------------------------
# metrics (synthbench.hpp:444-548): double accumulation, 100 dB cap
# ---------------------------------------------------------------------------
def _si_sdr_core(est: np.ndarray, ref: np.ndarray) -> float:  # synthbench.hpp:448-468
    e = est.astype(np.float64)
    r = ref.astype(np.float64)
    ref_energy = float(np.dot(r, r))
    if ref_energy <= 0.0:
        raise DegenerateStatsError("si_sdr: reference signal is all zero")
    alpha = float(np.dot(e, r)) / ref_energy
    signal = alpha * alpha * ref_energy
    d = alpha * r - e
    error = float(np.dot(d, d))
    if error <= signal * 1e-10:
        return SI_SDR_CAP
    return min(SI_SDR_CAP, 10.0 * math.log10(signal / error))


def si_sdr(estimate, reference) -> float:  # synthbench.hpp:473-477: lengths trimmed to match
    est = np.asarray(estimate, dtype=np.float32).reshape(-1)
    ref = np.asarray(reference, dtype=np.float32).reshape(-1)
    n = min(len(est), len(ref))
    return _si_sdr_core(est[:n], ref[:n])


def si_sdr_best_shift(estimate, reference, max_shift: int = 16) -> float:  # synthbench.hpp:483-512
    est = np.asarray(estimate, dtype=np.float32).reshape(-1)
    ref = np.asarray(reference, dtype=np.float32).reshape(-1)
    best = None
    for s in range(-max_shift, max_shift + 1):
        e, r = (est[s:], ref) if s >= 0 else (est, ref[-s:])
        n = min(len(e), len(r))
        if n <= 0:
            continue
        try:
            v = _si_sdr_core(e[:n], r[:n])
        except DegenerateStatsError:
            continue  # a trimmed window may be silent even when the full reference is not
        best = v if best is None else max(best, v)
    if best is None:
        raise DegenerateStatsError("si_sdr: reference signal is all zero")
    return best


def concat_spans(x, segments, speaker: str, sr: int) -> np.ndarray:  # synthbench.hpp:516-534
    x = np.asarray(x).reshape(-1)
    mine = sorted((s for s in segments if s.speaker == speaker), key=lambda s: s.start)
    parts = []
    for s in mine:
        lo = _llround(s.start * sr)
        hi = min(_llround(s.end() * sr), len(x))
        parts.append(x[lo:max(lo, hi)])
    return np.concatenate(parts) if parts else np.zeros(0, dtype=x.dtype)


def best_input_si_sdr(mix: GeneratedMixture, speaker: int, channels: int | None = None) -> float:
    """synthbench.hpp:538-548 (all channels); cmd_bench restricts it to the first `channels` (cli.hpp:300-305)."""
    sr = mix.mixture.sample_rate
    name = mix.speaker_names[speaker]
    ref = concat_spans(mix.dry[speaker], mix.segments, name, sr)
    chans = mix.mixture.channels if channels is None else mix.mixture.channels[:channels]
    return max(si_sdr_best_shift(concat_spans(ch, mix.segments, name, sr), ref) for ch in chans)


# ---------------------------------------------------------------------------
# oracle-mask MVDR (synthbench.hpp:554-623): ideal-ratio masks from the true source images, then the product's
# own accumulate_stats / select_reference / mvdr / apply / synthesize on the GPU
# ---------------------------------------------------------------------------
@dataclass
class OracleResult:
    si_sdr_db: list
    enhanced: list


def oracle_mvdr(mix: GeneratedMixture, cfg: stft.StftConfig, ctx=None) -> OracleResult:
    k_count = len(mix.speaker_names)
    sr = mix.mixture.sample_rate
    y = stft.analyze(mix.mixture, cfg, ctx)
    # residual = channel 0 minus all source images, subtracted one speaker at a time in float like the reference
    residual = mix.mixture.channels[0].astype(np.float32).copy()
    for k in range(k_count):
        residual -= mix.images0[k]
    tracks = np.concatenate([mix.images0, residual[None, :]], axis=0).astype(np.float32)
    # the K + 1 mono transforms in one call: the STFT is per channel, so stacking them changes nothing
    spec = stft.analyze(stft.RealSignal(tracks, sr), cfg, ctx).data          # (F, T, K+1)
    p = spec.real.astype(np.float64) ** 2 + spec.imag.astype(np.float64) ** 2
    total = p.sum(axis=2, keepdims=True)
    fallback = np.zeros(k_count + 1)
    fallback[k_count] = 1.0
    gamma = np.where(total > 0.0, p / np.where(total > 0.0, total, 1.0), fallback).astype(np.float32)
    out = OracleResult([], [])
    for k in range(k_count):
        stats = gss.beamform.accumulate_stats(y, gamma, k, ctx)
        ref = gss.beamform.select_reference(stats, ctx)
        flt = gss.beamform.mvdr(stats, ref, ctx)
        enhanced = stft.synthesize(gss.beamform.apply(flt, y, ctx), ctx).channels[0]
        out.enhanced.append(enhanced)
        name = mix.speaker_names[k]
        out.si_sdr_db.append(si_sdr_best_shift(concat_spans(enhanced, mix.segments, name, sr),
                                               concat_spans(mix.dry[k], mix.segments, name, sr)))
    return out


# ---------------------------------------------------------------------------
# fixtures (synthbench.hpp:628-726)
# ---------------------------------------------------------------------------
@dataclass
class FixturePaths:
    recordings: str
    segments: str
    wav: str
    recording: manifests.Recording


def save_fixture(mix: GeneratedMixture, directory: str, rec_id: str) -> FixturePaths:  # synthbench.hpp:637-665
    os.makedirs(directory, exist_ok=True)
    wav_path = os.path.join(directory, rec_id + ".wav")
    wav.write(wav_path, mix.mixture)
    m, n = mix.mixture.channels.shape
    rec = manifests.Recording(rec_id, [manifests.Source(wav_path, list(range(m)))], mix.mixture.sample_rate,
                              n / mix.mixture.sample_rate)
    paths = FixturePaths(os.path.join(directory, "recordings.jsonl"), os.path.join(directory, "segments.jsonl"),
                         wav_path, rec)
    manifests.save_recordings(paths.recordings, [rec])
    manifests.save_segments(paths.segments, [manifests.Segment(rec_id, s.speaker, s.start, s.duration, s.id)
                                             for s in mix.segments])
    return paths


def standard_fixture() -> MixtureSpec:  # synthbench.hpp:668-680: two speakers, a third overlapped, anechoic
    return MixtureSpec(42.0, 16000, 4, 12345, [SpeakerLayout("spk0", [(2.0, 14.0), (22.0, 12.0)]),
                                               SpeakerLayout("spk1", [(10.0, 10.0), (28.0, 12.0)])],
                       "delays", 0.0, 20.0)


def reverberant_fixture(channels: int = 8) -> MixtureSpec:  # synthbench.hpp:684-690
    spec = standard_fixture()
    spec.channels, spec.seed, spec.reverb_t60 = channels, 54321, 0.3
    return spec


def ten_minute_fixture() -> MixtureSpec:  # synthbench.hpp:693-709
    a = SpeakerLayout("spk0", [(20.0 * i + 1.0, 8.5) for i in range(30)])
    b = SpeakerLayout("spk1", [(20.0 * i + 9.0, 10.0) for i in range(30)])
    return MixtureSpec(600.0, 16000, 4, 99991, [a, b], "delays", 0.15, 20.0)


def fifty_segment_fixture() -> MixtureSpec:  # synthbench.hpp:713-726
    a = SpeakerLayout("spk0", [(3.5 * i + 1.0, 2.0) for i in range(50)])
    return MixtureSpec(180.0, 16000, 4, 77777, [a], "delays", 0.0, 20.0)


# ---------------------------------------------------------------------------
# fixture runner (tests/acceptance.cpp:66-122) and the ablation grid (cli.hpp:218-318)
# ---------------------------------------------------------------------------
@dataclass
class FixtureRun:
    summary: scheduler.RunSummary
    segment_si_sdr: list
    speaker_si_sdr: list
    wall_seconds: float


def _segment_wav(out_dir: str, s) -> np.ndarray:
    return wav.read(os.path.join(out_dir, scheduler.output_name(s.recording_id, s.speaker, s.start, s.end()))).channels[0]


def run_fixture(mix: GeneratedMixture, paths: FixturePaths, cfg: scheduler.PipelineConfig, devices=None,
                gpu_batch: int = 16) -> FixtureRun:
    segs = manifests.load_segments(paths.segments, manifests.JSONL)
    t0 = time.perf_counter()
    summary = scheduler.run_pipeline([paths.recording], segs, cfg, devices=devices, gpu_batch=gpu_batch)
    wall = time.perf_counter() - t0
    if summary.failed_segments > 0:
        raise gss.common.GssError("%d segment(s) failed under %s" % (summary.failed_segments, cfg.out_dir))
    sr = mix.mixture.sample_rate
    run = FixtureRun(summary, [], [], wall)
    for s in segs:
        est = _segment_wav(cfg.out_dir, s)
        k = mix.speaker_names.index(s.speaker)
        lo = _llround(s.start * sr)
        run.segment_si_sdr.append(si_sdr_best_shift(est, mix.dry[k][lo:lo + len(est)]))
    for k, name in enumerate(mix.speaker_names):
        mine = sorted((s for s in segs if s.speaker == name), key=lambda s: s.start)
        est = np.concatenate([_segment_wav(cfg.out_dir, s) for s in mine])
        run.speaker_si_sdr.append(si_sdr_best_shift(est, concat_spans(mix.dry[k], mix.segments, name, sr)))
    return run


@dataclass
class BenchOptions:  # cli.hpp:218-226
    spec_path: str = ""
    out_dir: str = "gss-bench"
    contexts: list = field(default_factory=lambda: [5.0, 10.0, 15.0, 20.0])
    iterations: list = field(default_factory=lambda: [1, 5, 10, 20])
    channels: list = field(default_factory=list)  # counts to sweep; empty = all available
    no_wpe: bool = False
    max_batch_duration: float = 50.0


CSV_HEADER = "context_s,bss_iterations,channels,speaker,input_si_sdr_db,enhanced_si_sdr_db,improvement_db\n"


def bench_grid(spec: MixtureSpec, opt: BenchOptions, devices=None, gpu_batch: int = 16) -> str:
    """cli.hpp:246-313: generate the mixture, sweep (context x iterations x channel count) through run_pipeline,
    return the CSV text (also written to <out_dir>/results.csv)."""
    mix = generate(spec)
    rec = save_fixture(mix, os.path.join(opt.out_dir, "fixture"), "bench0").recording
    segments = [manifests.Segment(rec.id, s.speaker, s.start, s.duration, s.id) for s in mix.segments]
    counts = list(opt.channels) or [spec.channels]
    rows = [CSV_HEADER]
    sr = spec.sample_rate
    for ctx_s in opt.contexts:
        for iters in opt.iterations:
            for m in counts:
                if m < 1 or m > spec.channels:
                    raise gss.common.ConfigError("channel count %d outside 1..%d" % (m, spec.channels))
                cfg = scheduler.PipelineConfig(max_batch_duration=opt.max_batch_duration, context_duration=ctx_s,
                                               bss_iterations=iters, enable_wpe=not opt.no_wpe,
                                               channels=list(range(m)),
                                               out_dir="%s/run_ctx%g_it%d_ch%d" % (opt.out_dir, ctx_s, iters, m))
                summary = scheduler.run_pipeline([rec], segments, cfg, devices=devices, gpu_batch=gpu_batch)
                if summary.failed_segments > 0:
                    raise gss.common.GssError("%d segment(s) failed in %s" % (summary.failed_segments, cfg.out_dir))
                for k, name in enumerate(mix.speaker_names):
                    mine = sorted((s for s in segments if s.speaker == name), key=lambda s: s.start)
                    est = np.concatenate([_segment_wav(cfg.out_dir, s) for s in mine])
                    ref = concat_spans(mix.dry[k], mix.segments, name, sr)
                    enhanced = si_sdr_best_shift(est, ref)
                    inp = max(si_sdr_best_shift(concat_spans(mix.mixture.channels[c], mix.segments, name, sr), ref)
                              for c in range(m))
                    rows.append("%g,%d,%d,%s,%.4f,%.4f,%.4f\n" % (ctx_s, iters, m, name, inp, enhanced, enhanced - inp))
    text = "".join(rows)
    manifests.write_text(os.path.join(opt.out_dir, "results.csv"), text)
    return text


def cmd_bench(opt: BenchOptions, devices=None) -> int:  # cli.hpp:230-318: exit codes 0 / 1 / 2
    import sys
    if not os.path.exists(opt.spec_path):
        print("gss: spec not found: %s" % opt.spec_path, file=sys.stderr)
        return 2
    try:
        spec = MixtureSpec.from_json(json.loads(manifests.read_text(opt.spec_path)))
    except Exception as e:  # noqa: BLE001 - the reference maps every parse / validation failure to usage
        print("gss: bad mixture spec: %s" % e, file=sys.stderr)
        return 2
    try:
        bench_grid(spec, opt, devices)
        print("wrote %s/results.csv" % opt.out_dir)
        return 0
    except Exception as e:  # noqa: BLE001
        print("gss: bench failed: %s" % e, file=sys.stderr)
        return 1
