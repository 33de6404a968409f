"""scheduler.hpp (hot-path part): PipelineConfig, SuperSegment, EnhancementResult, assemble's index
arithmetic, enhance_batch and its batched form enhance_batches."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from .. import capi
from .common import ConfigError, default_context
from .manifests import ActivityMatrix, Segment
from .stft import RealSignal, StftConfig
from .wpe import WpeConfig


@dataclass
class PipelineConfig:  # scheduler.hpp:30-44 (the fields enhance_batch reads)
    stft: StftConfig = field(default_factory=StftConfig)
    wpe: WpeConfig = field(default_factory=WpeConfig)
    enable_wpe: bool = True
    bss_iterations: int = 20
    context_duration: float = 15.0
    noise_class: bool = True

    def validate(self):  # scheduler.hpp:46-57
        if self.bss_iterations < 1:
            raise ConfigError("scheduler: bss_iterations must be >= 1")
        self.wpe.validate()
        self.stft.validate()

    def c(self) -> capi.PipelineConfig:
        return capi.PipelineConfig(self.stft.c(), self.wpe.c(), 1 if self.enable_wpe else 0, self.bss_iterations)


@dataclass
class Part:  # scheduler.hpp:168-172
    segment: Segment = field(default_factory=Segment)
    sample_begin: int = 0
    sample_end: int = 0


@dataclass
class SuperSegment:  # scheduler.hpp:165-180
    audio: RealSignal
    activity: ActivityMatrix
    parts: list
    recording_id: str = ""
    speaker: str = ""
    context_left: float = 0.0
    context_right: float = 0.0
    frame_centers: np.ndarray | None = None
    batch_index: int = 0


@dataclass
class EnhancementResult:  # scheduler.hpp:283-294 (paths are the caller's business)
    outputs: list            # one mono float32 array per part
    ll_final: float = 0.0
    zeroed_bins: int = 0
    ref_channel: int = 0
    frames: int = 0
    error: Exception | None = None
    mono: np.ndarray | None = None        # diagnostics (only when requested)
    posteriors: np.ndarray | None = None
    h: np.ndarray | None = None


@dataclass
class AssemblyPlan:
    spans: list
    part_begin: np.ndarray
    part_end: np.ndarray
    total: int
    frame_centers: np.ndarray
    context_left: float
    context_right: float


def output_name(recording_id: str, speaker: str, start: float, end: float) -> str:  # scheduler.hpp:303-308
    return "%s-%s-%07d_%07d.wav" % (recording_id, speaker, int(round(start * 1000)), int(round(end * 1000)))


def assemble_indices(parts_start_dur, sample_rate: int, rec_samples: int, context_duration: float,
                     stft: StftConfig) -> AssemblyPlan:  # scheduler.hpp:196-266
    lib = capi.load()
    n = len(parts_start_dur)
    starts = np.array([p[0] for p in parts_start_dur], dtype=np.float64)
    durs = np.array([p[1] for p in parts_start_dur], dtype=np.float64)
    spans = np.zeros(2 * (n + 2), dtype=np.int64)
    pb = np.zeros(max(n, 1), dtype=np.int64)
    pe = np.zeros(max(n, 1), dtype=np.int64)
    cap = int(rec_samples // max(stft.shift, 1) + 2 + 2 * n)
    centers = np.zeros(cap, dtype=np.int64)
    nsp, total, nc = C.c_int32(), C.c_int64(), C.c_int64()
    cl, cr = C.c_double(), C.c_double()
    capi.raise_for(lib.gss_b200_assemble_indices(
        C.c_int32(n), capi.ptr(starts), capi.ptr(durs), C.c_int32(sample_rate), C.c_int64(rec_samples),
        C.c_double(context_duration), C.c_int32(stft.fft_size), C.c_int32(stft.shift), capi.ptr(spans),
        C.byref(nsp), capi.ptr(pb), capi.ptr(pe), C.byref(total), capi.ptr(centers), C.c_int64(cap), C.byref(nc),
        C.byref(cl), C.byref(cr)))
    sp = [(int(spans[2 * i]), int(spans[2 * i + 1])) for i in range(nsp.value)]
    return AssemblyPlan(sp, pb[:n].copy(), pe[:n].copy(), int(total.value), centers[: nc.value].copy(), cl.value,
                        cr.value)


class _Marshalled:
    """Host buffers + descriptor array for a list of SuperSegments (kept alive for the call)."""

    def __init__(self, segments, cfg: PipelineConfig, diagnostics: bool, pinned: bool = False):
        self.n = len(segments)
        self.desc = (capi.SegmentDesc * max(self.n, 1))()
        self.diag = (capi.SegmentDiag * max(self.n, 1))()
        self.keep = []
        self.out_wave, self.out_len, self.mono, self.gamma, self.h = [], [], [], [], []
        self.h2d_bytes = 0
        self.d2h_bytes = 0
        f = cfg.stft.fft_size // 2 + 1

        def alloc(shape, dtype):
            if pinned:
                pb = capi.PinnedBuffer(shape, dtype)
                self.keep.append(pb)
                return pb.array
            return np.zeros(shape, dtype=dtype)

        for i, ss in enumerate(segments):
            audio = ss.audio.channels
            if pinned and not getattr(ss, "_pinned", False):
                buf = alloc(audio.shape, np.float32)
                buf[...] = audio
                audio = buf
            else:
                audio = np.ascontiguousarray(audio, dtype=np.float32)
            grid = np.ascontiguousarray(ss.activity.grid, dtype=np.uint8)
            m, n = audio.shape if audio.ndim == 2 else (0, 0)
            pb = np.array([p.sample_begin for p in ss.parts], dtype=np.int64)
            pe = np.array([p.sample_end for p in ss.parts], dtype=np.int64)
            cap = int(sum(max(0, min(e, n) - b) for b, e in zip(pb, pe)))
            ow = alloc((max(cap, 1),), np.float32)
            ol = np.zeros(max(len(pb), 1), dtype=np.int64)
            t, k = grid.shape
            mono = alloc((n,), np.float32) if diagnostics else None
            gam = np.zeros((f, t, k), dtype=np.float32) if diagnostics else None
            hh = np.zeros((f, m), dtype=np.complex128) if diagnostics else None
            self.keep += [audio, grid, pb, pe]
            self.out_wave.append(ow)
            self.out_len.append(ol)
            self.mono.append(mono)
            self.gamma.append(gam)
            self.h.append(hh)
            d = self.desc[i]
            d.audio = audio.ctypes.data
            d.channels, d.sample_rate, d.num_samples = m, int(ss.audio.sample_rate), n
            d.activity = grid.ctypes.data
            d.activity_frames, d.num_classes = t, k
            d.target_index, d.noise_index = int(ss.activity.target_index), int(ss.activity.noise_index)
            d.num_parts = len(pb)
            d.part_begin, d.part_end = pb.ctypes.data, pe.ctypes.data
            d.out_wave, d.out_lengths = ow.ctypes.data, ol.ctypes.data
            d.mono_out = mono.ctypes.data if mono is not None else None
            d.gamma_out = gam.ctypes.data if gam is not None else None
            d.h_out = hh.ctypes.data if hh is not None else None
            self.h2d_bytes += audio.nbytes + grid.nbytes
            self.d2h_bytes += cap * 4

    def results(self):
        res = []
        for i in range(self.n):
            dg = self.diag[i]
            if dg.status != 0:
                name = capi.error_from(dg.status, "segment %d failed with status %d" % (i, dg.status),
                                       dg.error_frequency)
                res.append(EnhancementResult([], error=name, frames=int(dg.frames)))
                continue
            outs, off = [], 0
            for ln in self.out_len[i][: self.desc[i].num_parts]:
                outs.append(np.array(self.out_wave[i][off: off + int(ln)], copy=True))
                off += int(ln)
            res.append(EnhancementResult(outs, float(dg.ll_final), int(dg.zeroed_bins), int(dg.ref_channel),
                                         int(dg.frames), None, self.mono[i], self.gamma[i], self.h[i]))
        return res


def enhance_batches(segments, cfg: PipelineConfig, ctx=None, diagnostics: bool = False):
    """scheduler::enhance_batch (scheduler.hpp:314-365) over a list of independent SuperSegments in one
    device batch. A failing segment carries its exception in `.error`; the others are unaffected."""
    ctx = ctx or default_context()
    cfg.validate()
    m = _Marshalled(segments, cfg, diagnostics)
    ccfg = cfg.c()
    ctx.check(ctx.lib.gss_b200_enhance_batch(ctx.handle, C.c_int32(m.n), m.desc, C.byref(ccfg), m.diag))
    return m.results()


def enhance_batch(ss: SuperSegment, cfg: PipelineConfig, ctx=None, diagnostics: bool = False) -> EnhancementResult:
    """The reference's signature: one SuperSegment; raises what the reference would throw."""
    r = enhance_batches([ss], cfg, ctx, diagnostics)[0]
    if r.error is not None:
        raise r.error
    return r


class ResidentBatch:
    """upload -> run (kernels only) -> fetch, for callers that keep a batch in HBM (bench.py's `value`)."""

    def __init__(self, segments, cfg: PipelineConfig, ctx=None, pinned: bool = True, diagnostics: bool = False):
        self.ctx = ctx or default_context()
        cfg.validate()
        self.m = _Marshalled(segments, cfg, diagnostics, pinned=pinned)
        self.ccfg = cfg.c()
        self.handle = None

    def upload(self):
        h = C.c_void_p()
        self.ctx.check(self.ctx.lib.gss_b200_batch_upload(self.ctx.handle, C.c_int32(self.m.n), self.m.desc,
                                                          C.byref(self.ccfg), C.byref(h)))
        self.handle = h
        return self

    def run(self):
        self.ctx.check(self.ctx.lib.gss_b200_batch_run(self.ctx.handle, self.handle))

    def fetch(self):
        self.ctx.check(self.ctx.lib.gss_b200_batch_fetch(self.ctx.handle, self.handle, self.m.diag))
        return self.m.results()

    def free(self):
        if self.handle is not None:
            self.ctx.lib.gss_b200_batch_free(self.ctx.handle, self.handle)
            self.handle = None

    def enhance(self):
        """The whole public call on host buffers: H2D + kernels + D2H."""
        self.ctx.check(self.ctx.lib.gss_b200_enhance_batch(self.ctx.handle, C.c_int32(self.m.n), self.m.desc,
                                                           C.byref(self.ccfg), self.m.diag))
        return self.m

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass
