"""stft.hpp: StftConfig, RealSignal, SpectrogramTensor, frame_count, frame_center, analyze, synthesize."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from .. import capi
from .common import ConfigError, default_context


@dataclass
class StftConfig:  # stft.hpp:16-36
    fft_size: int = 1024
    shift: int = 256
    window: int = 0  # 0 = hann, 1 = sqrt-hann
    sample_rate: int = 16000

    def num_bins(self) -> int:
        return self.fft_size // 2 + 1

    def validate(self):
        if self.fft_size <= 0 or self.shift <= 0:
            raise ConfigError("stft: fft_size and shift must be positive")
        if self.fft_size % self.shift != 0:
            raise ConfigError("stft: shift must divide fft_size for overlap-add")
        if self.sample_rate <= 0:
            raise ConfigError("stft: sample_rate must be positive")

    def c(self) -> capi.StftConfig:
        return capi.StftConfig(self.fft_size, self.shift, self.window, self.sample_rate)


@dataclass
class RealSignal:  # stft.hpp:39-47, channel-major (M, N) float32
    channels: np.ndarray
    sample_rate: int = 0

    def num_channels(self) -> int:
        return int(self.channels.shape[0]) if self.channels.ndim == 2 else 0

    def num_samples(self) -> int:
        return int(self.channels.shape[1]) if self.channels.ndim == 2 else 0


@dataclass
class SpectrogramTensor:  # stft.hpp:52-80, (F, T, M) complex64
    data: np.ndarray
    config: StftConfig = field(default_factory=StftConfig)
    origin_samples: int = 0
    num_samples: int = 0

    @property
    def num_bins(self):
        return int(self.data.shape[0])

    @property
    def num_frames(self):
        return int(self.data.shape[1])

    @property
    def num_channels(self):
        return int(self.data.shape[2])


def frame_count(num_samples: int, cfg: StftConfig) -> int:  # stft.hpp:120-124
    return int(capi.load().gss_b200_frame_count(int(num_samples), cfg.fft_size, cfg.shift))


def frame_center(t: int, cfg: StftConfig) -> int:  # stft.hpp:127-129
    return int(t) * cfg.shift


def analyze(signal: RealSignal, cfg: StftConfig, ctx=None) -> SpectrogramTensor:  # stft.hpp:131-175
    ctx = ctx or default_context()
    audio = np.ascontiguousarray(signal.channels, dtype=np.float32)
    if audio.ndim != 2:
        from .common import ShapeError
        raise ShapeError("stft.analyze: no channels")
    m, n = audio.shape
    t = frame_count(n, cfg) if cfg.shift > 0 and cfg.fft_size > 0 else 0
    out = np.empty((cfg.fft_size // 2 + 1 if cfg.fft_size > 0 else 0, max(t, 0), m), dtype=np.complex64)
    ccfg = cfg.c()
    ctx.check(ctx.lib.gss_b200_stft(ctx.handle, capi.ptr(audio), C.c_int32(m), C.c_int64(n),
                                    C.c_int32(signal.sample_rate), C.byref(ccfg), capi.ptr(out)))
    return SpectrogramTensor(out, cfg, -cfg.fft_size // 2, n)


def synthesize(spec: SpectrogramTensor, ctx=None) -> RealSignal:  # stft.hpp:179-229
    ctx = ctx or default_context()
    cfg = spec.config
    cfg.validate()
    data = capi.c64(spec.data)
    f, t, m = data.shape
    padded = (t - 1) * cfg.shift + cfg.fft_size
    out_len = spec.num_samples if spec.num_samples > 0 else max(0, padded - cfg.fft_size)
    out = np.zeros((m, out_len), dtype=np.float32)
    ccfg = cfg.c()
    ctx.check(ctx.lib.gss_b200_istft(ctx.handle, capi.ptr(data), C.c_int32(f), C.c_int64(t), C.c_int32(m),
                                     C.c_int64(spec.num_samples), C.byref(ccfg), capi.ptr(out)))
    return RealSignal(out, cfg.sample_rate)
