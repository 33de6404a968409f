"""manifests.hpp (hot-path part): Segment, ActivityMatrix, build_activity_at, build_activity."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from .. import capi


@dataclass
class Segment:  # manifests.hpp:42-51
    recording_id: str = ""
    speaker: str = ""
    start: float = 0.0
    duration: float = 0.0
    id: str = ""

    def end(self) -> float:
        return self.start + self.duration


@dataclass
class ActivityMatrix:  # manifests.hpp:58-68, frame-major (T, K) uint8
    grid: np.ndarray
    classes: list = field(default_factory=list)
    target_index: int = 0
    noise_index: int = -1

    @property
    def frames(self) -> int:
        return int(self.grid.shape[0])

    def num_classes(self) -> int:
        return int(self.grid.shape[1])

    def at(self, t, k):
        return int(self.grid[t, k])


def build_activity_at(segments, frame_center_samples, sample_rate: int, target: str,
                      noise_class: bool) -> ActivityMatrix:  # manifests.hpp:372-414
    lib = capi.load()
    n = len(segments)
    spk = (C.c_char_p * max(n, 1))(*[s.speaker.encode() for s in segments])
    starts = np.array([s.start for s in segments], dtype=np.float64)
    durs = np.array([s.duration for s in segments], dtype=np.float64)
    centers = np.ascontiguousarray(frame_center_samples, dtype=np.int64)
    kmax = len({s.speaker for s in segments} | {target}) + 1
    grid = np.zeros((len(centers), kmax), dtype=np.uint8)
    nk, ti, ni = C.c_int32(), C.c_int32(), C.c_int32()
    labels = C.create_string_buffer(64 * kmax + sum(len(s.speaker) for s in segments) + len(target) + 16)
    code = lib.gss_b200_build_activity_at(C.c_int32(n), spk, capi.ptr(starts), capi.ptr(durs), capi.ptr(centers),
                                          C.c_int64(len(centers)), C.c_int32(sample_rate), target.encode(),
                                          C.c_int32(1 if noise_class else 0), capi.ptr(grid),
                                          C.c_int64(grid.size), C.byref(nk), C.byref(ti), C.byref(ni), labels,
                                          C.c_int32(len(labels)))
    capi.raise_for(code)
    k = nk.value
    g = grid.reshape(-1)[: len(centers) * k].reshape(len(centers), k).copy()
    return ActivityMatrix(g, labels.value.decode().split("\n"), ti.value, ni.value)


def build_activity(segments, frame_begin: int, frame_end: int, target: str, cfg, noise_class: bool):
    # manifests.hpp:419-433
    if frame_end < frame_begin:
        raise capi.ShapeError("build_activity: frame window is inverted")
    centers = np.arange(frame_begin, frame_end, dtype=np.int64) * cfg.shift
    return build_activity_at(segments, centers, cfg.sample_rate, target, noise_class)
