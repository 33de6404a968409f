"""manifests.hpp: Recording / Segment manifests (JSONL, gzip-transparent; RTTM), cross-manifest validation,
the activity guide (build_activity_at, build_activity) and multi-source audio loading (load_audio)."""
from __future__ import annotations

import ctypes as C
import gzip
import json
import math
from dataclasses import dataclass, field

import numpy as np

from .. import capi
from ..capi import ConfigError, IoError, ParseError


def llround(x: float) -> int:
    """std::llround: halves away from zero (Python's round() rounds halves to even)."""
    return int(math.floor(abs(x) + 0.5)) * (1 if x >= 0 else -1)


@dataclass
class Source:  # manifests.hpp:22-25
    path: str = ""
    channels: list = field(default_factory=list)


@dataclass
class Recording:  # manifests.hpp:27-40
    id: str = ""
    sources: list = field(default_factory=list)
    sample_rate: int = 0
    duration: float = 0.0

    def channel_count(self) -> int:
        return sum(len(s.channels) for s in self.sources)

    def num_samples(self) -> int:
        return llround(self.duration * self.sample_rate)


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


# ---------------------------------------------------------------------------
# file reading (gzip-transparent by extension), manifests.hpp:79-114
# ---------------------------------------------------------------------------
def read_text(path: str) -> str:
    try:
        if path.endswith(".gz"):
            with gzip.open(path, "rb") as f:
                return f.read().decode("utf-8")
        with open(path, "rb") as f:
            return f.read().decode("utf-8")
    except FileNotFoundError:
        raise IoError("cannot open file: " + path)
    except (OSError, EOFError) as e:
        raise IoError(("gzip read failed: " if path.endswith(".gz") else "cannot open file: ") + path + " (%s)" % e)


def write_text(path: str, content: str) -> None:
    try:
        if path.endswith(".gz"):
            with gzip.open(path, "wb") as f:
                f.write(content.encode("utf-8"))
        else:
            with open(path, "wb") as f:
                f.write(content.encode("utf-8"))
    except OSError:
        raise IoError("cannot create file: " + path)


def _for_each_jsonl(path: str, fn):  # manifests.hpp:120-142: failures carry the 1-based line number
    for line_no, line in enumerate(read_text(path).split("\n"), 1):
        if not line.strip(" \t\r"):
            continue
        try:
            j = json.loads(line)
        except ValueError as e:
            raise ParseError("%s:%d: invalid JSON: %s" % (path, line_no, e))
        try:
            fn(j, line_no)
        except (KeyError, TypeError, ValueError) as e:
            raise ParseError("%s:%d: %s" % (path, line_no, e))


def _typed(j, key, kind):
    """j.at(key).get<kind>() of the reference: missing key or wrong JSON type is a (line-numbered) parse error."""
    if not isinstance(j, dict) or key not in j:
        raise KeyError("key '%s' not found" % key)
    v = j[key]
    if kind is float:
        if isinstance(v, bool) or not isinstance(v, (int, float)):
            raise TypeError("type must be number, but is %s" % type(v).__name__)
        return float(v)
    if kind is int:
        if isinstance(v, bool) or not isinstance(v, (int, float)):
            raise TypeError("type must be number, but is %s" % type(v).__name__)
        return int(v)
    if not isinstance(v, kind):
        raise TypeError("type must be %s, but is %s" % (kind.__name__, type(v).__name__))
    return v


def load_recordings(path: str) -> list:  # manifests.hpp:150-192
    out, seen = [], set()

    def one(j, line_no):
        r = Recording(_typed(j, "id", str), [], _typed(j, "sample_rate", int), _typed(j, "duration", float))
        for sj in _typed(j, "sources", list):
            chans = _typed(sj, "channels", list)
            if any(isinstance(c, bool) or not isinstance(c, int) for c in chans):
                raise TypeError("type must be number, but is not")
            r.sources.append(Source(_typed(sj, "path", str), list(chans)))
        if r.id in seen:
            raise ParseError("%s:%d: duplicate recording id '%s'" % (path, line_no, r.id))
        seen.add(r.id)
        if r.duration <= 0.0:
            raise ParseError("%s:%d: recording '%s' has duration %g" % (path, line_no, r.id, r.duration))
        if r.sample_rate <= 0:
            raise ParseError("%s:%d: recording '%s' has sample_rate %d" % (path, line_no, r.id, r.sample_rate))
        for src in r.sources:
            if len(set(src.channels)) != len(src.channels):
                raise ParseError("%s:%d: recording '%s' repeats a channel index" % (path, line_no, r.id))
        if r.channel_count() < 1:
            raise ParseError("%s:%d: recording '%s' has no channels" % (path, line_no, r.id))
        out.append(r)

    _for_each_jsonl(path, one)
    return out


def _dump(obj) -> str:  # nlohmann dump(): no spaces, insertion order
    return json.dumps(obj, separators=(",", ":"), ensure_ascii=False)


def serialize_recordings(recs) -> str:  # manifests.hpp:194-217
    return "".join(_dump({"id": r.id, "sources": [{"path": s.path, "channels": list(s.channels)} for s in r.sources],
                          "sample_rate": r.sample_rate, "duration": r.duration}) + "\n" for r in recs)


def save_recordings(path: str, recs) -> None:
    write_text(path, serialize_recordings(recs))


def serialize_segments(segs) -> str:  # manifests.hpp:222-243
    return "".join(_dump({"id": s.id, "recording_id": s.recording_id, "speaker": s.speaker, "start": s.start,
                          "duration": s.duration}) + "\n" for s in segs)


def save_segments(path: str, segs) -> None:
    write_text(path, serialize_segments(segs))


JSONL, RTTM = "jsonl", "rttm"  # SegmentFormat (manifests.hpp:53)


def _load_segments_jsonl(path, skipped):  # manifests.hpp:253-272
    out = []

    def one(j, line_no):
        s = Segment(_typed(j, "recording_id", str), _typed(j, "speaker", str), _typed(j, "start", float),
                    _typed(j, "duration", float), _typed(j, "id", str))
        if s.duration <= 0.0:
            skipped[0] += 1  # the reference logs a warning and drops the entry
            return
        out.append(s)

    _for_each_jsonl(path, one)
    return out


def _load_segments_rttm(path, skipped):  # manifests.hpp:274-318
    out, counters = [], {}
    for line_no, line in enumerate(read_text(path).split("\n"), 1):
        fields = line.split()
        if not fields or fields[0] != "SPEAKER":
            continue  # other record types are legal
        if len(fields) < 9:
            raise ParseError("%s:%d: RTTM SPEAKER line has %d fields, need 9+" % (path, line_no, len(fields)))
        try:
            start, duration = _stod(fields[3]), _stod(fields[4])
        except ValueError:
            raise ParseError("%s:%d: RTTM line has non-numeric start/duration" % (path, line_no))
        if duration <= 0.0:
            skipped[0] += 1
            continue
        key = (fields[1], fields[7])
        n = counters.get(key, 0)
        counters[key] = n + 1
        out.append(Segment(fields[1], fields[7], start, duration, "%s-%s-%04d" % (fields[1], fields[7], n)))
    return out


def _stod(tok: str) -> float:
    """std::stod with the whole token consumed (no surrounding space, no '_' digit separators)."""
    if tok != tok.strip() or "_" in tok:
        raise ValueError(tok)
    return float(tok)


def load_segments(path: str, fmt: str = JSONL, skipped: list | None = None) -> list:  # manifests.hpp:322-331
    """Segments of a JSONL or RTTM manifest; entries with duration <= 0 are dropped and counted in skipped[0]."""
    count = [0]
    out = _load_segments_jsonl(path, count) if fmt == JSONL else _load_segments_rttm(path, count)
    if skipped is not None:
        skipped[:] = [count[0]]
    return out


def validate(recordings, segments) -> list:  # manifests.hpp:334-361
    """Cross-manifest validation; human-readable problems (empty = OK)."""
    problems, by_id, seg_ids = [], {r.id: r for r in recordings}, set()
    for s in segments:
        if s.id in seg_ids:
            problems.append("duplicate segment id '%s'" % s.id)
        seg_ids.add(s.id)
        rec = by_id.get(s.recording_id)
        if rec is None:
            problems.append("segment '%s' references unknown recording '%s'" % (s.id, s.recording_id))
            continue
        if s.start < 0.0:
            problems.append("segment '%s' starts at %g" % (s.id, s.start))
        if s.end() > rec.duration + 1e-6:
            problems.append("segment '%s' ends at %g, past recording end %g" % (s.id, s.end(), rec.duration))
    return problems


def load_audio(rec: Recording, start_sample: int, count: int, channel_subset=()):  # manifests.hpp:442-479
    """[start_sample, start_sample + count) across all sources of a recording, channels stacked in source
    order; channel_subset selects stacked indices (empty = all)."""
    from . import wav
    from .stft import RealSignal
    rows = []
    for src in rec.sources:
        part = wav.read(src.path, start_sample, count)
        if part.sample_rate != rec.sample_rate:
            raise ConfigError("recording '%s': %s is %d Hz, manifest says %d" % (rec.id, src.path, part.sample_rate,
                                                                                  rec.sample_rate))
        if part.num_samples() < count:
            raise IoError("recording '%s': %s has %d samples at offset %d, need %d"
                          % (rec.id, src.path, part.num_samples(), start_sample, count))
        for c in src.channels:
            if c < 0 or c >= part.num_channels():
                raise ConfigError("recording '%s': %s has no channel %d" % (rec.id, src.path, c))
            rows.append(part.channels[c])
    if channel_subset:
        for c in channel_subset:
            if c < 0 or c >= len(rows):
                raise ConfigError("channel subset index %d out of range [0, %d)" % (c, len(rows)))
        rows = [rows[c] for c in channel_subset]
    data = np.ascontiguousarray(np.stack(rows), dtype=np.float32) if rows else np.zeros((0, 0), np.float32)
    return RealSignal(data, rec.sample_rate)
