"""cacgmm.hpp: CacgmmState, EmResult, cacg_log_pdf, time_varying_weights, em_fit, log_likelihood."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from .. import capi
from .common import default_context
from .manifests import ActivityMatrix
from .stft import SpectrogramTensor


@dataclass
class CacgmmState:  # cacgmm.hpp:22-49
    weights: np.ndarray  # (F, K) float64
    shapes: np.ndarray   # (F, K, M, M) complex128

    @staticmethod
    def uniform(bins: int, classes: int, channels: int) -> "CacgmmState":
        w = np.full((bins, classes), 1.0 / classes)
        s = np.broadcast_to(np.eye(channels, dtype=np.complex128), (bins, classes, channels, channels)).copy()
        return CacgmmState(w, s)


@dataclass
class EmResult:  # cacgmm.hpp:178-182
    state: CacgmmState
    posteriors: np.ndarray  # (F, T, K) float32
    likelihood_trace: list


def cacg_log_pdf(y, b) -> float:  # cacgmm.hpp:66-82
    y = capi.c128(y)
    b = capi.c128(b)
    if b.shape != (y.shape[0], y.shape[0]):
        raise capi.ShapeError("cacg_log_pdf: B does not match y")
    out = C.c_double()
    capi.raise_for(capi.load().gss_b200_cacg_log_pdf(C.c_int32(y.shape[0]), capi.ptr(y), capi.ptr(b), C.byref(out)))
    return out.value


def time_varying_weights(pi, activity, noise_index: int = -1):  # cacgmm.hpp:87-112
    pi = np.ascontiguousarray(pi, dtype=np.float64)
    act = np.ascontiguousarray(activity, dtype=np.uint8)
    if act.shape[0] != pi.shape[0]:
        raise capi.ShapeError("time_varying_weights: activity row does not match pi")
    out = np.zeros_like(pi)
    capi.raise_for(capi.load().gss_b200_time_varying_weights(C.c_int32(pi.shape[0]), capi.ptr(pi), capi.ptr(act),
                                                            C.c_int32(noise_index), capi.ptr(out)))
    return out


def em_fit(y: SpectrogramTensor, activity: ActivityMatrix, iterations: int = 20, ctx=None,
           want_posteriors: bool = True) -> EmResult:  # cacgmm.hpp:264-340
    ctx = ctx or default_context()
    data = capi.c64(y.data)
    f, t, m = data.shape
    grid = np.ascontiguousarray(activity.grid, dtype=np.uint8)
    k = grid.shape[1]
    gamma = np.zeros((f, t, k), dtype=np.float32) if want_posteriors else None
    pi = np.zeros((f, k), dtype=np.float64)
    shapes = np.zeros((f, k, m, m), dtype=np.complex128)
    trace = np.zeros(max(iterations, 0) + 1, dtype=np.float64)
    ctx.check(ctx.lib.gss_b200_em_fit(ctx.handle, capi.ptr(data), C.c_int32(f), C.c_int64(t), C.c_int32(m),
                                      capi.ptr(grid), C.c_int64(grid.shape[0]), C.c_int32(k),
                                      C.c_int32(activity.noise_index), C.c_int32(iterations), capi.ptr(gamma),
                                      capi.ptr(pi), capi.ptr(shapes), capi.ptr(trace)))
    return EmResult(CacgmmState(pi, shapes), gamma, [float(v) for v in trace])


def log_likelihood(y: SpectrogramTensor, state: CacgmmState, activity: ActivityMatrix, ctx=None) -> float:
    # cacgmm.hpp:343-370
    ctx = ctx or default_context()
    data = capi.c64(y.data)
    f, t, m = data.shape
    grid = np.ascontiguousarray(activity.grid, dtype=np.uint8)
    k = grid.shape[1]
    if grid.shape[0] != t or state.weights.shape != (f, k):
        raise capi.ShapeError("log_likelihood: inconsistent shapes")
    pi = np.ascontiguousarray(state.weights, dtype=np.float64)
    shapes = capi.c128(state.shapes)
    out = C.c_double()
    ctx.check(ctx.lib.gss_b200_log_likelihood(ctx.handle, capi.ptr(data), C.c_int32(f), C.c_int64(t), C.c_int32(m),
                                              capi.ptr(grid), C.c_int32(k), C.c_int32(activity.noise_index),
                                              capi.ptr(pi), capi.ptr(shapes), C.byref(out)))
    return out.value
