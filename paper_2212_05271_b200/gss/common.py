"""common.hpp: error classes, and the device context the operators run on."""
from __future__ import annotations

import ctypes as C
import threading

from .. import capi
from ..capi import (ConfigError, CudaError, DegenerateStatsError, EmptyTargetError, GssError,  # noqa: F401
                    InputTooShortError, IoError, ParseError, ShapeError, SingularMatrixError, SpecError,
                    UnsupportedError)


class Context:
    """One gss_b200_ctx: a device, a stream and its workspaces (one per host thread and device)."""

    def __init__(self, device: int = 0):
        lib = capi.load()
        h = C.c_void_p()
        capi.raise_for(lib.gss_b200_create(int(device), C.byref(h)))
        self.handle = h
        self.device = int(device)
        self.lib = lib

    def check(self, code: int):
        capi.raise_for(code, self.handle)

    @property
    def stream(self) -> int:
        return int(self.lib.gss_b200_stream(self.handle) or 0)

    @property
    def launch_count(self) -> int:
        return int(self.lib.gss_b200_launch_count(self.handle))

    @property
    def device_bytes(self) -> int:
        return int(self.lib.gss_b200_device_bytes(self.handle))

    def device_bytes_peak(self, reset: bool = False) -> int:
        """High-water mark of the workspaces since creation / the last reset."""
        return int(self.lib.gss_b200_device_bytes_peak(self.handle, C.c_int32(1 if reset else 0)))

    def stage_ms(self) -> dict:
        ms = (C.c_double * capi.NUM_STAGES)()
        self.check(self.lib.gss_b200_stage_ms(self.handle, ms))
        return dict(zip(capi.STAGE_NAMES, [float(v) for v in ms]))

    def profile(self, enable: bool = True):
        """Reset and (de)activate the per-kernel CUDA-event clocks."""
        self.check(self.lib.gss_b200_profile(self.handle, C.c_int32(1 if enable else 0)))

    def kernel_ms(self) -> dict:
        """{kernel class: (summed device ms, launches)} since the last profile() call."""
        ms = (C.c_double * capi.NUM_KERNELS)()
        n = (C.c_int64 * capi.NUM_KERNELS)()
        self.check(self.lib.gss_b200_kernel_ms(self.handle, ms, n))
        return {k: (float(ms[i]), int(n[i])) for i, k in enumerate(capi.KERNEL_NAMES)}

    def fp32_peak_tflops(self) -> float:
        v = C.c_double()
        self.check(self.lib.gss_b200_fp32_peak(self.handle, C.byref(v)))
        return v.value

    def close(self):
        if self.handle is not None:
            self.lib.gss_b200_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_tls = threading.local()


def default_context(device: int | None = None) -> Context:
    """The calling thread's context for `device` (created on first use)."""
    import os
    if device is None:
        device = int(os.environ.get("GSS_B200_DEVICE", os.environ.get("LOCAL_RANK", "0")))
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    if device not in ctxs:
        ctxs[device] = Context(device)
    return ctxs[device]
