"""Synthetic multi-speaker reverberant mixtures and the BASELINE.json workloads (bench / test harness).

`generate` binds synthbench/gss_synth.cpp, a restatement of the input specification of the reference's
synthbench::generate (synthbench.hpp:323-438). Harness code (bench / tests / the ablation CLI): it lives outside
the product package, and the enhancement path never imports it. The SI-SDR metrics, oracle-mask MVDR, canned
fixtures and the ablation grid of synthbench.hpp:448-726 / cli.hpp:228-318 are in synthbench/harness.py.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

from paper_2212_05271_b200.capi import SpecError
from paper_2212_05271_b200.gss import manifests, scheduler, stft, wpe

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "libgss_synth.so")
_lib = None


def _load():
    global _lib
    if _lib is None:
        src = os.path.join(_HERE, "gss_synth.cpp")
        if not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(src):
            subprocess.run(["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-o", _LIB, src], check=True)
        _lib = C.CDLL(_LIB)
        _lib.gss_synth_last_error.restype = C.c_char_p
    return _lib


def generate(duration: float, sample_rate: int, channels: int, seed: int, speakers, reverb_t60: float = 0.3,
             noise_snr: float = 20.0, with_sources: bool = False):
    """speakers: list (one entry per speaker) of lists of (start, duration) seconds. Returns the (M, N) float32
    mixture; with `with_sources` also the per-speaker dry tracks and channel-0 images, both (K, N)
    (GeneratedMixture::dry / images0, synthbench.hpp:166-172)."""
    lib = _load()
    offs = [0]
    starts, durs = [], []
    for segs in speakers:
        for s, d in segs:
            starts.append(float(s))
            durs.append(float(d))
        offs.append(len(starts))
    n = int(math.floor(duration * sample_rate + 0.5))
    mix = np.zeros((channels, n), dtype=np.float32)
    dry = np.zeros((len(speakers), n), dtype=np.float32) if with_sources else None
    img = np.zeros((len(speakers), n), dtype=np.float32) if with_sources else None
    offs_a = np.array(offs, dtype=np.int32)
    st = np.array(starts, dtype=np.float64)
    du = np.array(durs, dtype=np.float64)
    rc = lib.gss_synth_generate(C.c_double(duration), C.c_int(sample_rate), C.c_int(channels), C.c_uint64(seed),
                                C.c_int(len(speakers)), offs_a.ctypes.data_as(C.c_void_p),
                                st.ctypes.data_as(C.c_void_p), du.ctypes.data_as(C.c_void_p),
                                C.c_double(reverb_t60), C.c_double(noise_snr), mix.ctypes.data_as(C.c_void_p),
                                dry.ctypes.data_as(C.c_void_p) if with_sources else None,
                                img.ctypes.data_as(C.c_void_p) if with_sources else None)
    if rc != 0:
        raise SpecError(lib.gss_synth_last_error().decode())
    return (mix, dry, img) if with_sources else mix


@dataclass
class Workload:
    name: str
    cfg: scheduler.PipelineConfig
    segments: list            # SuperSegments
    output_seconds: float     # sum of cut lengths (context excluded)
    assembled_seconds: float  # sum of window lengths (context included)


def _speaker_layout(n_speakers: int, window: float, target_start: float, target_dur: float, seed: int):
    """Deterministic talk pattern: the target speaks over [target_start, +target_dur) (plus one utterance in each
    context when there is room); the others overlap it partially, as in a meeting."""
    rng = np.random.RandomState(seed)
    spk = [[(target_start, target_dur)]]
    if target_start > 8.0:
        spk[0].append((1.0 + rng.uniform(0, 2), 4.0))
    if window - (target_start + target_dur) > 8.0:
        spk[0].append((target_start + target_dur + 2.0 + rng.uniform(0, 2), 4.0))
    for k in range(1, n_speakers):
        segs = []
        pos = rng.uniform(0.0, 3.0) + 1.5 * k
        while pos < window - 1.0:
            d = float(min(rng.uniform(3.0, 8.0), window - pos))
            if d >= 0.5:
                segs.append((float(pos), d))
            pos += d + rng.uniform(1.0, 6.0)
        if not segs:
            segs.append((0.0, min(2.0, window)))
        spk.append(segs)
    return [sorted(s) for s in spk]


def make_supersegment(seed: int, channels: int, n_speakers: int, target_dur: float, context: float,
                      cfg: scheduler.PipelineConfig, reverb_t60: float = 0.3, noise_snr: float = 20.0,
                      layout=None):
    """One SuperSegment: a window of context + target + context seconds cut around one target utterance."""
    sr = cfg.stft.sample_rate
    window = target_dur + 2 * context
    layout = layout or _speaker_layout(n_speakers, window, context, target_dur, seed)
    audio = generate(window, sr, channels, seed, layout, reverb_t60, noise_snr)
    n = audio.shape[1]
    segs = [manifests.Segment("rec", "spk%d" % k, s, d, "spk%d-%d" % (k, i))
            for k, ss in enumerate(layout) for i, (s, d) in enumerate(ss)]
    t = stft.frame_count(n, cfg.stft)
    centers = np.minimum(np.arange(t, dtype=np.int64) * cfg.stft.shift, n - 1)
    act = manifests.build_activity_at(segs, centers, sr, "spk0", cfg.noise_class)
    b = int(round(context * sr))
    e = min(n, int(round((context + target_dur) * sr)))
    part = scheduler.Part(manifests.Segment("rec", "spk0", context, target_dur, "tgt"), b, e)
    return scheduler.SuperSegment(stft.RealSignal(audio, sr), act, [part], "rec", "spk0", context, context, centers)


def _cfg(enable_wpe=True, delay=2, iters=20):
    return scheduler.PipelineConfig(stft.StftConfig(512, 128, 0, 16000), wpe.WpeConfig(10, delay, 3, 0, 1e-10),
                                    enable_wpe, iters)


def workload(name: str, n_segments: int | None = None, first: int = 0, threads: int = 8) -> Workload:
    """The BASELINE.json configs. `first`/`n_segments` select a shard."""
    if name == "cfg1":   # 2 speakers, 7 ch, 10 s, no WPE, context 0
        cfg = _cfg(False)
        total = 1
        layout = [[(0.5, 5.5)], [(4.0, 5.5)]]

        def mk(i):
            return make_supersegment(1001 + i, 7, 2, 10.0, 0.0, cfg, layout=layout)
    elif name == "cfg2":  # LibriCSS-shaped: 7 ch, 3 spk + noise, WPE, 15 s context, batch 16
        cfg = _cfg(True, 2)
        total = 16

        def mk(i):
            return make_supersegment(2000 + i, 7, 3, 10.0, 15.0, cfg)
    elif name == "cfg3":  # AMI-shaped: 8 ch, 4 spk + noise, WPE delay 3, batch 64
        cfg = _cfg(True, 3)
        total = 64

        def mk(i):
            return make_supersegment(3000 + i, 8, 4, 10.0, 15.0, cfg)
    elif name == "cfg4":  # AliMeeting-shaped: 8 ch, 4 spk, 30 s segments
        cfg = _cfg(True, 2)
        total = 4

        def mk(i):
            return make_supersegment(4000 + i, 8, 4, 30.0, 15.0, cfg)
    elif name == "tiny":  # fast smoke / test shape
        cfg = _cfg(True, 2, 5)
        total = 2

        def mk(i):
            return make_supersegment(7000 + i, 4, 2, 2.0, 1.0, cfg)
    else:
        raise ValueError("unknown workload " + name)
    n = total - first if n_segments is None else n_segments
    idx = [first + j for j in range(n)]
    _load()
    with ThreadPoolExecutor(max_workers=max(1, min(threads, len(idx)))) as ex:
        segs = list(ex.map(mk, idx))
    sr = cfg.stft.sample_rate
    out_s = sum((p.sample_end - p.sample_begin) / sr for s in segs for p in s.parts)
    asm_s = sum(s.audio.num_samples() / sr for s in segs)
    return Workload(name, cfg, segs, out_s, asm_s)


def sweep_params(total: int = 4096, seed: int = 5000):
    """BASELINE configs[4]: `total` segments, target durations U[2,12] s + 2 x 15 s context,
    2-8 channels, 2-4 speakers (+ noise class), 5/10/20/40 EM iterations, WPE on. Returns one
    (seed, channels, speakers, target seconds, iterations) tuple per segment; cheap, so every rank can draw the
    whole list and generate only the audio of the segments it owns."""
    rng = np.random.RandomState(seed)
    out = []
    for i in range(total):
        iters = int(rng.choice([5, 10, 20, 40]))
        out.append((seed + i, int(rng.randint(2, 9)), int(rng.randint(2, 5)), float(rng.uniform(2.0, 12.0)), iters))
    return out


def sweep_cfg(iters: int) -> scheduler.PipelineConfig:
    return _cfg(True, 2, iters)


def sweep_frames(target_dur: float, context: float = 15.0, cfg: scheduler.PipelineConfig | None = None) -> int:
    cfg = cfg or _cfg()
    n = int(math.floor((target_dur + 2 * context) * cfg.stft.sample_rate + 0.5))
    return stft.frame_count(n, cfg.stft)


def make_sweep_segments(params, threads: int = 8):
    """SuperSegments for a list of sweep_params() entries, generated on `threads` host threads."""
    _load()

    def mk(p):
        seed, m, k, dur, iters = p
        return make_supersegment(seed, m, k, dur, 15.0, sweep_cfg(iters))

    with ThreadPoolExecutor(max_workers=max(1, min(threads, len(params) or 1))) as ex:
        return list(ex.map(mk, params))
