"""ctypes binding of the CPU ORACLE (oracle/gss_oracle.hpp).

TEST INFRASTRUCTURE ONLY. Importable from tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs; the product package
(paper_2212_05271_b200) must never import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")

ERR_NAMES = {
    0: "ok", 1: "ShapeError", 2: "ConfigError", 3: "ParseError", 4: "IoError",
    5: "SingularMatrixError", 6: "InputTooShortError", 7: "EmptyTargetError",
    8: "DegenerateStatsError", 9: "SpecError", 100: "InternalError",
}


class OracleError(RuntimeError):
    def __init__(self, code, msg, frequency=-1):
        super().__init__(f"{ERR_NAMES.get(code, code)}: {msg}")
        self.code = code
        self.kind = ERR_NAMES.get(code, str(code))
        self.frequency = frequency


def build(march: str | None = None, out_dir: str | None = None, vector_gram: bool = False) -> str:
    """Compile liboracle.so (g++). Returns the path of the built library. `vector_gram` builds the timing-only
    variant whose Gram dot products run on SIMD partial sums (-DGSS_ORACLE_VECTOR_GRAM; needs `out_dir`)."""
    env = dict(os.environ)
    args = ["make", "-C", _HERE]
    if march:
        args.append(f"ORACLE_MARCH={march}")
    if out_dir:
        os.makedirs(out_dir, exist_ok=True)
        out = os.path.join(out_dir, "liboracle.so")
        cmd = ["g++", "-O3", f"-march={march or 'x86-64-v3'}", "-std=c++17", "-fPIC", "-pthread",
               "-shared", "-o", out, os.path.join(_HERE, "oracle_capi.cpp")]
        if vector_gram:
            cmd.insert(1, "-DGSS_ORACLE_VECTOR_GRAM")
        subprocess.run(cmd, check=True, env=env)
        return out
    subprocess.run(args, check=True, env=env, stdout=subprocess.DEVNULL)
    return _LIB_PATH


_lib = None


def load(path: str | None = None):
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = path or _LIB_PATH
    if not os.path.exists(p):
        build()
    lib = C.CDLL(p)
    lib.oracle_last_error.restype = C.c_char_p
    lib.oracle_last_error_frequency.restype = C.c_long
    lib.oracle_frame_count.restype = C.c_int64
    lib.oracle_frame_count.argtypes = [C.c_int64, C.c_int, C.c_int]
    _lib = lib
    return lib


def _check(code):
    if code != 0:
        lib = load()
        raise OracleError(code, lib.oracle_last_error().decode(), lib.oracle_last_error_frequency())


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _c128(a):
    return np.ascontiguousarray(a, dtype=np.complex128)


def _c64(a):
    return np.ascontiguousarray(a, dtype=np.complex64)


class StftCfg(C.Structure):
    _fields_ = [("fft_size", C.c_int), ("shift", C.c_int), ("window", C.c_int), ("sample_rate", C.c_int)]


class WpeCfg(C.Structure):
    _fields_ = [("taps", C.c_int), ("delay", C.c_int), ("iterations", C.c_int), ("psd_context", C.c_int),
                ("regularization", C.c_double)]


class EnhanceCfg(C.Structure):
    _fields_ = [("fft_size", C.c_int), ("shift", C.c_int), ("window", C.c_int), ("sample_rate", C.c_int),
                ("enable_wpe", C.c_int), ("taps", C.c_int), ("delay", C.c_int), ("wpe_iterations", C.c_int),
                ("psd_context", C.c_int), ("regularization", C.c_double), ("bss_iterations", C.c_int)]


def stft_cfg(fft_size=1024, shift=256, window=0, sample_rate=16000):
    return StftCfg(fft_size, shift, window, sample_rate)


def wpe_cfg(taps=10, delay=2, iterations=3, psd_context=0, regularization=1e-10):
    return WpeCfg(taps, delay, iterations, psd_context, regularization)


def set_threads(n: int):
    load().oracle_set_threads(int(n))


def hardware_threads() -> int:
    return int(load().oracle_hardware_threads())


# --------------------------------------------------------------------------- numerics
def hermitize(a):
    a = _c128(a)
    out = np.empty((a.shape[0], a.shape[0]), np.complex128)
    _check(load().oracle_hermitize(a.shape[0], a.shape[1], _p(a), _p(out)))
    return out


def regularize(a, eps=1e-10):
    a = _c128(a)
    out = np.empty_like(a)
    _check(load().oracle_regularize(a.shape[0], _p(a), C.c_double(eps), _p(out)))
    return out


def hermitian_solve(a, b, frequency=-1):
    a, b = _c128(a), _c128(b)
    x = np.empty_like(b)
    _check(load().oracle_hermitian_solve(a.shape[0], b.shape[1], _p(a), _p(b), C.c_long(frequency), _p(x)))
    return x


def hermitian_inverse_logdet(a):
    a = _c128(a)
    inv = np.empty_like(a)
    ld = C.c_double()
    _check(load().oracle_hermitian_inverse_logdet(a.shape[0], _p(a), _p(inv), C.byref(ld)))
    return inv, ld.value


def hermitian_eig(a):
    a = _c128(a)
    vecs = np.empty_like(a)
    vals = np.empty(a.shape[0], np.float64)
    _check(load().oracle_hermitian_eig(a.shape[0], _p(a), _p(vecs), _p(vals)))
    return vals, vecs


def weighted_gram(a, w=None, chunk=2048):
    a = _c64(a)
    rows, cols = a.shape
    wv = None if w is None else np.ascontiguousarray(w, np.float32)
    out = np.empty((cols, cols), np.complex128)
    _check(load().oracle_weighted_gram(_p(a), C.c_int64(rows), cols, _p(wv), C.c_int64(chunk), _p(out)))
    return out


# --------------------------------------------------------------------------- stft
def make_window(fft_size, window=0):
    out = np.empty(fft_size, np.float64)
    _check(load().oracle_make_window(fft_size, window, _p(out)))
    return out


def frame_count(n, fft_size=1024, shift=256):
    return int(load().oracle_frame_count(int(n), fft_size, shift))


def stft(audio, cfg: StftCfg, signal_rate=None):
    audio = np.ascontiguousarray(audio, np.float32)
    if audio.ndim == 1:
        audio = audio[None]
    m, n = audio.shape
    f = cfg.fft_size // 2 + 1
    t = max(frame_count(n, cfg.fft_size, max(cfg.shift, 1)), 0) if cfg.shift > 0 else 0
    out = np.empty((f, t, m), np.complex64)
    sr = cfg.sample_rate if signal_rate is None else signal_rate
    _check(load().oracle_stft(_p(audio), m, C.c_int64(n), sr, C.byref(cfg), _p(out)))
    return out


def istft(spec, cfg: StftCfg, num_samples=0):
    spec = _c64(spec)
    if spec.ndim == 2:
        spec = spec[:, :, None]
    f, t, m = spec.shape
    out_len = num_samples if num_samples > 0 else max(0, (t - 1) * cfg.shift)
    out = np.zeros((m, out_len), np.float32)
    _check(load().oracle_istft(_p(spec), f, C.c_int64(t), m, C.c_int64(num_samples), C.byref(cfg), _p(out)))
    return out


def wpe(y, cfg: WpeCfg):
    y = _c64(y)
    f, t, m = y.shape
    out = np.empty_like(y)
    _check(load().oracle_wpe(_p(y), f, C.c_int64(t), m, C.byref(cfg), _p(out)))
    return out


def unit_normalize(y):
    y = _c64(y)
    f, t, m = y.shape
    out = np.empty_like(y)
    _check(load().oracle_unit_normalize(_p(y), f, C.c_int64(t), m, _p(out)))
    return out


# --------------------------------------------------------------------------- cacgmm
def cacg_log_pdf(y, b):
    y, b = _c128(y), _c128(b)
    out = C.c_double()
    _check(load().oracle_cacg_log_pdf(y.shape[0], _p(y), _p(b), C.byref(out)))
    return out.value


def time_varying_weights(pi, act, noise_index=-1):
    pi = np.ascontiguousarray(pi, np.float64)
    act = np.ascontiguousarray(act, np.uint8)
    if act.shape[0] != pi.shape[0]:
        # let the oracle raise its ShapeError through the same path
        pass
    out = np.empty_like(pi)
    if act.shape[0] != pi.shape[0]:
        raise OracleError(1, "time_varying_weights: activity row does not match pi")
    _check(load().oracle_time_varying_weights(pi.shape[0], _p(pi), _p(act), noise_index, _p(out)))
    return out


@dataclass
class EmResult:
    gamma: np.ndarray   # (F,T,K) float32
    pi: np.ndarray      # (F,K) float64
    shapes: np.ndarray  # (F,K,M,M) complex128
    trace: np.ndarray   # (iters+1,) float64


def em_fit(yn, act, target=0, noise=-1, iterations=20, precise_quad=False) -> EmResult:
    yn = _c64(yn)
    act = np.ascontiguousarray(act, np.uint8)
    f, t, m = yn.shape
    act_frames, k = act.shape
    gamma = np.zeros((f, t, k), np.float32)
    pi = np.zeros((f, k), np.float64)
    shapes = np.zeros((f, k, m, m), np.complex128)
    trace = np.zeros(max(iterations, 0) + 1, np.float64)
    _check(load().oracle_em_fit(_p(yn), f, C.c_int64(t), m, _p(act), C.c_int64(act_frames), k, target, noise,
                                iterations, int(precise_quad), _p(gamma), _p(pi), _p(shapes), _p(trace)))
    return EmResult(gamma, pi, shapes, trace)


def log_likelihood(yn, act, pi, shapes, noise=-1):
    yn = _c64(yn)
    act = np.ascontiguousarray(act, np.uint8)
    f, t, m = yn.shape
    k = act.shape[1]
    pi = np.ascontiguousarray(pi, np.float64)
    shapes = _c128(shapes)
    out = C.c_double()
    _check(load().oracle_log_likelihood(_p(yn), f, C.c_int64(t), m, _p(act), k, noise, _p(pi), _p(shapes),
                                        C.byref(out)))
    return out.value


# --------------------------------------------------------------------------- beamform
def mvdr_stats(y, gamma, target):
    y = _c64(y)
    gamma = np.ascontiguousarray(gamma, np.float32)
    f, t, m = y.shape
    k = gamma.shape[2]
    if gamma.shape[:2] != (f, t):
        raise OracleError(1, "accumulate_stats: posterior does not match tensor")
    tgt = np.empty((f, m, m), np.complex128)
    bg = np.empty((f, m, m), np.complex128)
    _check(load().oracle_mvdr_stats(_p(y), _p(gamma), f, C.c_int64(t), m, k, target, _p(tgt), _p(bg)))
    return tgt, bg


def select_reference(tgt, bg):
    tgt, bg = _c128(tgt), _c128(bg)
    ref = C.c_int()
    _check(load().oracle_select_reference(_p(tgt), _p(bg), tgt.shape[0], tgt.shape[1], C.byref(ref)))
    return ref.value


def mvdr(tgt, bg, ref):
    tgt, bg = _c128(tgt), _c128(bg)
    f, m = tgt.shape[0], tgt.shape[1]
    h = np.zeros((f, m), np.complex128)
    zeroed = C.c_int64()
    _check(load().oracle_mvdr(_p(tgt), _p(bg), f, m, ref, _p(h), C.byref(zeroed)))
    return h, zeroed.value


def apply_filter(h, y):
    h, y = _c128(h), _c64(y)
    f, t, m = y.shape
    out = np.empty((f, t), np.complex64)
    _check(load().oracle_apply(_p(h), h.shape[0], h.shape[1], _p(y), f, C.c_int64(t), m, _p(out)))
    return out


# --------------------------------------------------------------------------- guide / indexing
@dataclass
class Activity:
    grid: np.ndarray  # (T,K) uint8
    classes: list
    target_index: int
    noise_index: int


def build_activity_at(segments, centers, sample_rate, target, noise_class=True) -> Activity:
    """segments: iterable of (speaker, start, duration)."""
    segs = list(segments)
    n = len(segs)
    spk = (C.c_char_p * max(n, 1))(*[s[0].encode() for s in segs])
    starts = np.array([s[1] for s in segs], np.float64)
    durs = np.array([s[2] for s in segs], np.float64)
    centers = np.ascontiguousarray(centers, np.int64)
    kmax = len({s[0] for s in segs} | {target}) + 1
    grid = np.zeros(centers.shape[0] * kmax, np.uint8)
    nk, ti, ni = C.c_int(), C.c_int(), C.c_int()
    labels = C.create_string_buffer(65536)
    _check(load().oracle_build_activity_at(n, spk, _p(starts), _p(durs), _p(centers), C.c_int64(centers.shape[0]),
                                           sample_rate, target.encode(), int(noise_class), _p(grid),
                                           C.c_int64(grid.size), C.byref(nk), C.byref(ti), C.byref(ni), labels,
                                           65536))
    k = nk.value
    return Activity(grid[: centers.shape[0] * k].reshape(centers.shape[0], k).copy(),
                    labels.value.decode().split("\n"), ti.value, ni.value)


@dataclass
class Assembly:
    spans: np.ndarray        # (n_spans,2) int64 source [begin,end)
    part_begin: np.ndarray
    part_end: np.ndarray
    total: int
    frame_centers: np.ndarray
    context_left: float
    context_right: float


def assemble_indices(parts, sr, rec_samples, context, fft_size=1024, shift=256) -> Assembly:
    """parts: iterable of (start, duration) in temporal order."""
    parts = list(parts)
    n = len(parts)
    starts = np.array([p[0] for p in parts], np.float64)
    durs = np.array([p[1] for p in parts], np.float64)
    spans = np.zeros((n + 2, 2), np.int64)
    pb = np.zeros(n, np.int64)
    pe = np.zeros(n, np.int64)
    cap = int(rec_samples // shift + 8)
    centers = np.zeros(cap, np.int64)
    nsp, total, ncen = C.c_int(), C.c_int64(), C.c_int64()
    cl, cr = C.c_double(), C.c_double()
    _check(load().oracle_assemble_indices(n, _p(starts), _p(durs), sr, C.c_int64(rec_samples), C.c_double(context),
                                          fft_size, shift, _p(spans), C.byref(nsp), _p(pb), _p(pe), C.byref(total),
                                          _p(centers), C.c_int64(cap), C.byref(ncen), C.byref(cl), C.byref(cr)))
    return Assembly(spans[: nsp.value].copy(), pb, pe, total.value, centers[: ncen.value].copy(), cl.value, cr.value)


# --------------------------------------------------------------------------- enhance
@dataclass
class EnhanceResult:
    outputs: list
    ll_final: float
    zeroed_bins: int
    ref_channel: int
    frames: int
    stage_seconds: np.ndarray
    mono: np.ndarray | None = None
    gamma: np.ndarray | None = None
    h: np.ndarray | None = None


def enhance(audio, act, target, noise, parts, *, fft_size=1024, shift=256, window=0, sample_rate=16000,
            enable_wpe=True, taps=10, delay=2, wpe_iterations=3, psd_context=0, regularization=1e-10,
            bss_iterations=20, diag=False) -> EnhanceResult:
    """parts: list of (sample_begin, sample_end) inside the assembled audio."""
    audio = np.ascontiguousarray(audio, np.float32)
    act = np.ascontiguousarray(act, np.uint8)
    m, n = audio.shape
    t_act, k = act.shape
    pb = np.array([p[0] for p in parts], np.int64)
    pe = np.array([p[1] for p in parts], np.int64)
    cfg = EnhanceCfg(fft_size, shift, window, sample_rate, int(enable_wpe), taps, delay, wpe_iterations,
                     psd_context, regularization, bss_iterations)
    cap = int(np.sum(np.maximum(np.minimum(pe, n) - pb, 0)))
    out = np.zeros(max(cap, 1), np.float32)
    lens = np.zeros(len(parts), np.int64)
    f = fft_size // 2 + 1
    t = frame_count(n, fft_size, shift) if shift > 0 and fft_size > 0 else 0
    mono = np.zeros(n, np.float32) if diag else None
    gamma = np.zeros((f, t, k), np.float32) if diag else None
    h = np.zeros((f, m), np.complex128) if diag else None
    ll, zeroed, ref, frames = C.c_double(), C.c_int64(), C.c_int(), C.c_int64()
    secs = np.zeros(5, np.float64)
    _check(load().oracle_enhance(_p(audio), m, C.c_int64(n), _p(act), C.c_int64(t_act), k, target, noise,
                                 len(parts), _p(pb), _p(pe), C.byref(cfg), _p(out), _p(lens), _p(mono), _p(gamma),
                                 _p(h), C.byref(ll), C.byref(zeroed), C.byref(ref), C.byref(frames), _p(secs)))
    outs, off = [], 0
    for ln in lens:
        outs.append(out[off: off + ln].copy())
        off += int(ln)
    return EnhanceResult(outs, ll.value, zeroed.value, ref.value, frames.value, secs, mono, gamma, h)
