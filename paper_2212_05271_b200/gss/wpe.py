"""wpe.hpp: WpeConfig, dereverberate, unit_normalize."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, replace

import numpy as np

from .. import capi
from .common import ConfigError, default_context
from .stft import SpectrogramTensor


@dataclass
class WpeConfig:  # wpe.hpp:15-30
    taps: int = 10
    delay: int = 2
    iterations: int = 3
    psd_context: int = 0
    regularization: float = 1e-10

    def validate(self):
        if self.taps < 1 or self.delay < 1 or self.iterations < 1:
            raise ConfigError("wpe: taps, delay and iterations must be >= 1")
        if self.psd_context < 0 or self.regularization < 0.0:
            raise ConfigError("wpe: psd_context and regularization must be >= 0")

    def c(self) -> capi.WpeConfig:
        return capi.WpeConfig(self.taps, self.delay, self.iterations, self.psd_context, self.regularization)


def dereverberate(y: SpectrogramTensor, cfg: WpeConfig, ctx=None) -> SpectrogramTensor:  # wpe.hpp:105-120
    ctx = ctx or default_context()
    data = capi.c64(y.data)
    f, t, m = data.shape
    out = np.empty_like(data)
    ccfg = cfg.c()
    ctx.check(ctx.lib.gss_b200_wpe(ctx.handle, capi.ptr(data), C.c_int32(f), C.c_int64(t), C.c_int32(m),
                                   C.byref(ccfg), capi.ptr(out)))
    return replace(y, data=out)


def unit_normalize(y: SpectrogramTensor, ctx=None) -> SpectrogramTensor:  # wpe.hpp:124-140
    ctx = ctx or default_context()
    data = capi.c64(y.data)
    f, t, m = data.shape
    out = np.empty_like(data)
    ctx.check(ctx.lib.gss_b200_unit_normalize(ctx.handle, capi.ptr(data), C.c_int32(f), C.c_int64(t), C.c_int32(m),
                                              capi.ptr(out)))
    return replace(y, data=out)
