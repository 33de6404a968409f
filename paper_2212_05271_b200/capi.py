"""ctypes binding of libgss_b200.so (include/gss_b200.h).

The shared library is the product; this module only marshals numpy arrays to
the C ABI. There is no Python or CPU implementation of any stage behind it: if
the library is missing or no B200 is visible, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# GSS_B200_LIB points at another build of the SAME library (kernel experiments: tools/variant.py)
LIB_PATH = os.environ.get("GSS_B200_LIB") or os.path.join(_HERE, "lib", "libgss_b200.so")

NUM_STAGES = 7
NUM_KERNELS = 11
KERNEL_NAMES = ("stft", "wpe_power", "wpe_gram", "wpe_solve", "wpe_apply", "em_pass", "em_update", "mvdr", "apply",
                "istft", "misc")
STAGE_NAMES = ("stft", "wpe", "mask", "beamform", "istft", "h2d", "d2h")


# --- the reference's exception hierarchy (common.hpp:17-79) -------------------
class GssError(RuntimeError):
    code = 100


class ShapeError(GssError):
    code = 1


class ConfigError(GssError):
    code = 2


class ParseError(GssError):
    code = 3


class IoError(GssError):
    code = 4


class SingularMatrixError(GssError):
    code = 5

    def __init__(self, msg, frequency=-1):
        super().__init__(msg)
        self._frequency = frequency

    def frequency(self):
        return self._frequency


class InputTooShortError(GssError):
    code = 6


class EmptyTargetError(GssError):
    code = 7


class DegenerateStatsError(GssError):
    code = 8


class SpecError(GssError):
    code = 9


class CudaError(GssError):
    code = 101


class UnsupportedError(GssError):
    code = 102


_BY_CODE = {c.code: c for c in (ShapeError, ConfigError, ParseError, IoError, SingularMatrixError,
                                InputTooShortError, EmptyTargetError, DegenerateStatsError, SpecError,
                                CudaError, UnsupportedError)}


def error_from(code: int, msg: str, frequency: int = -1) -> GssError:
    cls = _BY_CODE.get(code, GssError)
    if cls is SingularMatrixError:
        return SingularMatrixError(msg, frequency)
    return cls(msg)


class StftConfig(C.Structure):
    _fields_ = [("fft_size", C.c_int32), ("shift", C.c_int32), ("window", C.c_int32), ("sample_rate", C.c_int32)]


class WpeConfig(C.Structure):
    _fields_ = [("taps", C.c_int32), ("delay", C.c_int32), ("iterations", C.c_int32), ("psd_context", C.c_int32),
                ("regularization", C.c_double)]


class PipelineConfig(C.Structure):
    _fields_ = [("stft", StftConfig), ("wpe", WpeConfig), ("enable_wpe", C.c_int32), ("bss_iterations", C.c_int32)]


class SegmentDesc(C.Structure):
    _fields_ = [("audio", C.c_void_p), ("channels", C.c_int32), ("sample_rate", C.c_int32),
                ("num_samples", C.c_int64), ("activity", C.c_void_p), ("activity_frames", C.c_int64),
                ("num_classes", C.c_int32), ("target_index", C.c_int32), ("noise_index", C.c_int32),
                ("num_parts", C.c_int32), ("part_begin", C.c_void_p), ("part_end", C.c_void_p),
                ("out_wave", C.c_void_p), ("out_lengths", C.c_void_p), ("mono_out", C.c_void_p),
                ("gamma_out", C.c_void_p), ("h_out", C.c_void_p)]


class SegmentDiag(C.Structure):
    _fields_ = [("status", C.c_int32), ("ref_channel", C.c_int32), ("error_frequency", C.c_int64),
                ("zeroed_bins", C.c_int64), ("frames", C.c_int64), ("ll_final", C.c_double)]


EXPORTS = [
    "gss_b200_default_stft_config", "gss_b200_default_wpe_config", "gss_b200_default_pipeline_config",
    "gss_b200_create", "gss_b200_destroy", "gss_b200_last_error", "gss_b200_last_error_frequency",
    "gss_b200_stream", "gss_b200_launch_count", "gss_b200_device_bytes", "gss_b200_device_bytes_peak", "gss_b200_host_alloc",
    "gss_b200_host_free", "gss_b200_stft", "gss_b200_istft", "gss_b200_wpe", "gss_b200_unit_normalize",
    "gss_b200_em_fit", "gss_b200_log_likelihood", "gss_b200_mvdr_stats", "gss_b200_select_reference",
    "gss_b200_mvdr", "gss_b200_apply", "gss_b200_enhance_batch", "gss_b200_batch_upload", "gss_b200_batch_run",
    "gss_b200_batch_fetch", "gss_b200_batch_free", "gss_b200_stage_ms", "gss_b200_profile", "gss_b200_kernel_ms", "gss_b200_fp32_peak", "gss_b200_frame_count",
    "gss_b200_build_activity_at", "gss_b200_assemble_indices", "gss_b200_cacg_log_pdf",
    "gss_b200_time_varying_weights",
    "gss_b200_stft_dev", "gss_b200_istft_dev", "gss_b200_wpe_dev", "gss_b200_unit_normalize_dev", "gss_b200_apply_dev",
    "gss_b200_enhance_batch_dev", "gss_b200_nvtx_range_count",
]

_lib = None


def load():
    """dlopen libgss_b200.so. Raises if it has not been built (python -m paper_2212_05271_b200.build)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2212_05271_b200.build` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    lib.gss_b200_last_error.restype = C.c_char_p
    lib.gss_b200_last_error.argtypes = [C.c_void_p]
    lib.gss_b200_last_error_frequency.restype = C.c_int64
    lib.gss_b200_last_error_frequency.argtypes = [C.c_void_p]
    lib.gss_b200_stream.restype = C.c_void_p
    lib.gss_b200_stream.argtypes = [C.c_void_p]
    lib.gss_b200_launch_count.restype = C.c_int64
    lib.gss_b200_launch_count.argtypes = [C.c_void_p]
    lib.gss_b200_device_bytes.restype = C.c_int64
    lib.gss_b200_device_bytes.argtypes = [C.c_void_p]
    lib.gss_b200_nvtx_range_count.restype = C.c_int64
    lib.gss_b200_nvtx_range_count.argtypes = [C.c_void_p]
    lib.gss_b200_device_bytes_peak.restype = C.c_int64
    lib.gss_b200_device_bytes_peak.argtypes = [C.c_void_p, C.c_int32]
    lib.gss_b200_frame_count.restype = C.c_int64
    lib.gss_b200_frame_count.argtypes = [C.c_int64, C.c_int32, C.c_int32]
    lib.gss_b200_create.argtypes = [C.c_int, C.POINTER(C.c_void_p)]
    lib.gss_b200_destroy.argtypes = [C.c_void_p]
    lib.gss_b200_destroy.restype = None
    lib.gss_b200_host_alloc.argtypes = [C.c_int64, C.POINTER(C.c_void_p)]
    lib.gss_b200_host_free.argtypes = [C.c_void_p]
    lib.gss_b200_host_free.restype = None
    lib.gss_b200_batch_free.argtypes = [C.c_void_p, C.c_void_p]
    lib.gss_b200_batch_free.restype = None
    _lib = lib
    return lib


def ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def c64(a):
    return np.ascontiguousarray(a, dtype=np.complex64)


def c128(a):
    return np.ascontiguousarray(a, dtype=np.complex128)


def raise_for(code: int, ctx=None):
    if code == 0:
        return
    lib = load()
    msg = lib.gss_b200_last_error(ctx).decode(errors="replace")
    freq = int(lib.gss_b200_last_error_frequency(ctx))
    raise error_from(code, msg, freq)


class PinnedBuffer:
    """Page-locked host memory from gss_b200_host_alloc, exposed as a numpy array."""

    def __init__(self, shape, dtype):
        self.shape = tuple(int(s) for s in np.atleast_1d(shape))
        self.dtype = np.dtype(dtype)
        nbytes = int(np.prod(self.shape)) * self.dtype.itemsize
        p = C.c_void_p()
        raise_for(load().gss_b200_host_alloc(C.c_int64(max(nbytes, 1)), C.byref(p)))
        self._p = p
        buf = (C.c_char * max(nbytes, 1)).from_address(p.value)
        self.array = np.frombuffer(buf, dtype=self.dtype, count=int(np.prod(self.shape))).reshape(self.shape)

    def free(self):
        if self._p is not None:
            self.array = None
            load().gss_b200_host_free(self._p)
            self._p = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass
