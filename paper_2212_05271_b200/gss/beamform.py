"""beamform.hpp: BeamformerStats, BeamformerFilter, accumulate_stats, select_reference, mvdr, apply."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, replace

import numpy as np

from .. import capi
from .common import ShapeError, default_context
from .stft import SpectrogramTensor


@dataclass
class BeamformerStats:  # beamform.hpp:18-24
    target: np.ndarray      # (F, M, M) complex128
    background: np.ndarray  # (F, M, M) complex128
    frame_count: int = 0

    @property
    def num_bins(self):
        return int(self.target.shape[0])

    @property
    def num_channels(self):
        return int(self.target.shape[1])


@dataclass
class BeamformerFilter:  # beamform.hpp:26-31
    h: np.ndarray  # (F, M) complex128
    ref_channel: int = 0
    zeroed_bins: int = 0

    @property
    def num_channels(self):
        return int(self.h.shape[1])


def accumulate_stats(y: SpectrogramTensor, gamma, target: int, ctx=None) -> BeamformerStats:  # beamform.hpp:35-85
    ctx = ctx or default_context()
    data = capi.c64(y.data)
    f, t, m = data.shape
    g = np.ascontiguousarray(gamma, dtype=np.float32)
    if g.ndim != 3 or g.shape[:2] != (f, t):
        raise ShapeError("accumulate_stats: posterior does not match tensor")
    k = g.shape[2]
    tgt = np.zeros((f, m, m), dtype=np.complex128)
    bg = np.zeros((f, m, m), dtype=np.complex128)
    ctx.check(ctx.lib.gss_b200_mvdr_stats(ctx.handle, capi.ptr(data), capi.ptr(g), C.c_int32(f), C.c_int64(t),
                                          C.c_int32(m), C.c_int32(k), C.c_int32(target), capi.ptr(tgt), capi.ptr(bg)))
    return BeamformerStats(tgt, bg, t)


def select_reference(stats: BeamformerStats, ctx=None) -> int:  # beamform.hpp:89-107
    ctx = ctx or default_context()
    tgt, bg = capi.c128(stats.target), capi.c128(stats.background)
    ref = C.c_int32()
    ctx.check(ctx.lib.gss_b200_select_reference(ctx.handle, capi.ptr(tgt), capi.ptr(bg), C.c_int32(tgt.shape[0]),
                                                C.c_int32(tgt.shape[1]), C.byref(ref)))
    return ref.value


def mvdr(stats: BeamformerStats, ref: int, ctx=None) -> BeamformerFilter:  # beamform.hpp:111-135
    ctx = ctx or default_context()
    tgt, bg = capi.c128(stats.target), capi.c128(stats.background)
    f, m = tgt.shape[0], tgt.shape[1]
    h = np.zeros((f, m), dtype=np.complex128)
    z = C.c_int64()
    ctx.check(ctx.lib.gss_b200_mvdr(ctx.handle, capi.ptr(tgt), capi.ptr(bg), C.c_int32(f), C.c_int32(m),
                                    C.c_int32(ref), capi.ptr(h), C.byref(z)))
    return BeamformerFilter(h, ref, z.value)


def apply(flt: BeamformerFilter, y: SpectrogramTensor, ctx=None) -> SpectrogramTensor:  # beamform.hpp:138-165
    ctx = ctx or default_context()
    data = capi.c64(y.data)
    f, t, m = data.shape
    h = capi.c128(flt.h)
    out = np.zeros((f, t, 1), dtype=np.complex64)
    ctx.check(ctx.lib.gss_b200_apply(ctx.handle, capi.ptr(h), C.c_int32(h.shape[0]), C.c_int32(h.shape[1]),
                                     capi.ptr(data), C.c_int32(f), C.c_int64(t), C.c_int32(m), capi.ptr(out)))
    return replace(y, data=out)
