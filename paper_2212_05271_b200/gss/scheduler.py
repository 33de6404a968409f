"""scheduler.hpp: PipelineConfig, batch planning (plan_batches), SuperSegment assembly (assemble), the hot
path enhance_batch with its batched form enhance_batches, and the run_pipeline executor (loader threads ->
ordered queue -> one compute slot per GPU -> writer, summary.json)."""
from __future__ import annotations

import concurrent.futures as cf
import ctypes as C
import json
import os
import threading
import time
from dataclasses import dataclass, field

import numpy as np

from .. import capi
from . import manifests, wav
from .common import ConfigError, Context, ShapeError, default_context
from .manifests import ActivityMatrix, Segment, llround
from .stft import RealSignal, StftConfig, frame_count
from .wpe import WpeConfig

SUPER_SEGMENT, ONE_PER_BATCH = "super-segment", "one-per-batch"  # BatchMode (scheduler.hpp:28)


@dataclass
class PipelineConfig:  # scheduler.hpp:30-82
    stft: StftConfig = field(default_factory=StftConfig)
    wpe: WpeConfig = field(default_factory=WpeConfig)
    enable_wpe: bool = True
    bss_iterations: int = 20
    context_duration: float = 15.0
    noise_class: bool = True
    max_batch_duration: float = 50.0
    channels: list = field(default_factory=list)   # stacked-channel subset; empty = all
    mode: str = SUPER_SEGMENT
    workers: int = 0          # data-loader threads; 0 = fully synchronous
    queue_capacity: int = 2   # prefetch depth of the loader -> compute queue
    seed: int = 0             # echoed into the summary; the pipeline is deterministic
    out_dir: str = "."
    extra_echo: list = field(default_factory=list)  # (key, value) pairs echoed into the summary

    def validate(self):  # scheduler.hpp:46-57
        if self.max_batch_duration <= 0 or self.context_duration < 0:
            raise ConfigError("scheduler: durations must be positive")
        if self.bss_iterations < 1:
            raise ConfigError("scheduler: bss_iterations must be >= 1")
        if self.workers < 0 or self.queue_capacity < 1:
            raise ConfigError("scheduler: workers >= 0 and queue_capacity >= 1 required")
        self.wpe.validate()
        self.stft.validate()

    def echo(self) -> dict:  # scheduler.hpp:60-81: flag-style echo of every knob
        j = {"max-batch-duration": self.max_batch_duration, "context-duration": self.context_duration,
             "bss-iterations": self.bss_iterations, "no-wpe": not self.enable_wpe,
             "no-noise-class": not self.noise_class, "channels": list(self.channels),
             "one-per-batch": self.mode == ONE_PER_BATCH, "workers": self.workers,
             "queue-capacity": self.queue_capacity, "seed": self.seed, "out-dir": self.out_dir,
             "wpe-taps": self.wpe.taps, "wpe-delay": self.wpe.delay, "wpe-iterations": self.wpe.iterations,
             "fft-size": self.stft.fft_size, "shift": self.stft.shift}
        for k, v in self.extra_echo:
            j[k] = v
        return j

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
    return "%s-%s-%07d_%07d.wav" % (recording_id, speaker, llround(start * 1000.0), llround(end * 1000.0))


@dataclass
class BatchPlan:  # scheduler.hpp:86-96: same-recording, same-speaker segments concatenated along time
    recording_id: str = ""
    speaker: str = ""
    parts: list = field(default_factory=list)  # temporal order

    def total_duration(self) -> float:
        d = 0.0
        for p in self.parts:
            d += p.duration
        return d


def plan_batches(segments, max_batch_duration: float, mode: str = SUPER_SEGMENT) -> list:  # scheduler.hpp:101-160
    """Groups segments by (recording, speaker) in first-appearance order, fills batches greedily in temporal
    order up to the duration cap, then emits round-robin across groups. Oversized segments stay singletons."""
    groups = {}
    for seg in segments:
        groups.setdefault((seg.recording_id, seg.speaker), []).append(seg)
    per_group = []
    for key, segs in groups.items():  # dicts keep first-appearance order
        segs = sorted(segs, key=lambda x: (x.start, x.id))
        buckets = []
        for seg in segs:
            if mode == ONE_PER_BATCH or seg.duration > max_batch_duration:
                buckets.append(BatchPlan(key[0], key[1], [seg]))
                continue
            if buckets and len(buckets[-1].parts) == 1 and buckets[-1].parts[0].duration > max_batch_duration:
                buckets.append(BatchPlan(key[0], key[1], [seg]))  # never append to an oversized singleton
                continue
            if not buckets or buckets[-1].total_duration() + seg.duration > max_batch_duration:
                buckets.append(BatchPlan(key[0], key[1], []))
            buckets[-1].parts.append(seg)
        per_group.append(buckets)
    plans, rnd = [], 0
    while True:
        took = False
        for buckets in per_group:
            if rnd < len(buckets):
                plans.append(buckets[rnd])
                took = True
        if not took:
            return plans
        rnd += 1


def assemble_indices(parts_start_dur, sample_rate: int, rec_samples: int, context_duration: float,
                     stft: StftConfig) -> AssemblyPlan:  # scheduler.hpp:196-266
    lib = capi.load()
    n = len(parts_start_dur)
    starts = np.array([p[0] for p in parts_start_dur], dtype=np.float64)
    durs = np.array([p[1] for p in parts_start_dur], dtype=np.float64)
    spans = np.zeros(2 * (n + 2), dtype=np.int64)
    pb = np.zeros(max(n, 1), dtype=np.int64)
    pe = np.zeros(max(n, 1), dtype=np.int64)
    # spans are concatenated, so overlapping parts of one speaker make the assembled signal longer than the
    # recording: size the frame-centre buffer from the span total (each span within a sample of llround(dur * sr))
    sr = float(sample_rate)
    total_cap = int(sum(llround(max(d, 0.0) * sr) + 1 for d in durs)) + 2 * (llround(max(context_duration, 0.0) * sr) + 1)
    cap = int(total_cap // max(stft.shift, 1) + 2 + 2 * n)
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


def assemble(plan: BatchPlan, rec, all_segments, cfg: PipelineConfig) -> SuperSegment:  # scheduler.hpp:185-275
    """Reads the audio spans of one plan ([left context][parts with gaps removed][right context]) and builds
    the activity guide over the assembled frames. `all_segments` must hold every segment of the plan's
    recording (any speaker) so that cross-speaker activity is right inside the context windows."""
    for seg in plan.parts:  # the reference names the offending segment (scheduler.hpp:210-213)
        s0 = llround(seg.start * rec.sample_rate)
        s1 = min(rec.num_samples(), llround(seg.end() * rec.sample_rate))
        if s1 <= s0:
            raise ShapeError("segment '%s' maps to an empty sample range" % seg.id)
    ap = assemble_indices([(p.start, p.duration) for p in plan.parts], rec.sample_rate, rec.num_samples(),
                          cfg.context_duration, cfg.stft)
    audio = None
    off = 0
    for b, e in ap.spans:
        piece = manifests.load_audio(rec, b, e - b, cfg.channels)
        if audio is None:
            audio = np.zeros((piece.num_channels(), ap.total), dtype=np.float32)
        audio[:, off: off + (e - b)] = piece.channels
        off += e - b
    parts = [Part(seg, int(ap.part_begin[i]), int(ap.part_end[i])) for i, seg in enumerate(plan.parts)]
    rec_segments = [x for x in all_segments if x.recording_id == plan.recording_id]
    activity = manifests.build_activity_at(rec_segments, ap.frame_centers, rec.sample_rate, plan.speaker,
                                           cfg.noise_class)
    return SuperSegment(RealSignal(audio, rec.sample_rate), activity, parts, plan.recording_id, plan.speaker,
                        ap.context_left, ap.context_right, ap.frame_centers)


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
            # mono may live in pinned memory owned by this object: hand out a copy, never a view
            mono = None if self.mono[i] is None else np.array(self.mono[i], copy=True)
            res.append(EnhancementResult(outs, float(dg.ll_final), int(dg.zeroed_bins), int(dg.ref_channel),
                                         int(dg.frames), None, mono, self.gamma[i], self.h[i]))
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


# ---------------------------------------------------------------------------
# run_pipeline (scheduler.hpp:366-638)
# ---------------------------------------------------------------------------
@dataclass
class LoadedBatch:  # scheduler.hpp:371-376
    index: int = 0
    batch: SuperSegment | None = None  # None on load failure
    error: str = ""
    load_seconds: float = 0.0


class OrderedBatchQueue:
    """Bounded queue that hands batches to the consumer in plan order whichever loader finished first
    (scheduler.hpp:383-412); this is what makes the worker count invisible in the output."""

    def __init__(self, capacity: int):
        self.capacity = int(capacity)
        self.cv = threading.Condition()
        self.ready = {}
        self.next = 0
        self.closed = False

    def put(self, item: LoadedBatch) -> bool:
        """False when the queue was closed (the consumer is gone): the loader should stop."""
        with self.cv:
            self.cv.wait_for(lambda: self.closed or item.index < self.next + self.capacity)
            if self.closed:
                return False
            self.ready[item.index] = item
            self.cv.notify_all()
            return True

    def close(self) -> None:
        """Releases every loader blocked in put(); used when the consumer leaves abnormally."""
        with self.cv:
            self.closed = True
            self.cv.notify_all()

    def take(self) -> LoadedBatch:
        with self.cv:
            self.cv.wait_for(lambda: self.next in self.ready)
            item = self.ready.pop(self.next)
            self.next += 1
            self.cv.notify_all()
            return item


@dataclass
class RunSummary:  # scheduler.hpp:414-417
    json: dict
    failed_segments: int = 0


class _ComputeSlot:
    """One GPU: a context created on the slot's own thread, and a single-thread executor that runs the
    device batches handed to it in submission order."""

    def __init__(self, device: int):
        self.device = device
        self.pool = cf.ThreadPoolExecutor(max_workers=1, thread_name_prefix="gss-gpu%d" % device)
        self.ctx = None
        self.stage = {}

    def _run(self, batches, cfg):
        if self.ctx is None:
            self.ctx = Context(self.device)
        res = enhance_batches(batches, cfg, self.ctx)
        for k, v in self.ctx.stage_ms().items():  # milliseconds of the call that just returned
            self.stage[k] = self.stage.get(k, 0.0) + v * 1e-3
        return res

    def submit(self, batches, cfg):
        return self.pool.submit(self._run, batches, cfg)

    def close(self):
        self.pool.shutdown(wait=True)
        if self.ctx is not None:
            self.ctx.close()


def run_pipeline(recordings, segments, cfg: PipelineConfig, devices=None, gpu_batch: int = 16) -> RunSummary:
    """plan -> (loader threads) assemble -> enhance -> write, with a JSON summary (scheduler.hpp:423-638).

    The reference's compute consumer handles one batch at a time on the host. Here the compute slots are
    GPUs (`devices`, default: device 0): loaded batches are taken from the ordered queue in plan order,
    grouped `gpu_batch` at a time into one device call and dealt to the slots round-robin; results are
    consumed strictly in plan order, so outputs, summary and written bytes do not depend on the worker
    count, the number of GPUs or the grouping (a segment's result is independent of its device batch)."""
    cfg.validate()
    wall0 = time.perf_counter()
    problems = manifests.validate(recordings, segments)
    if problems:
        raise ConfigError("manifest validation failed:" + "".join("\n  " + p for p in problems))
    os.makedirs(cfg.out_dir, exist_ok=True)
    rec_by_id = {r.id: r for r in recordings}
    plans = plan_batches(segments, cfg.max_batch_duration, cfg.mode)
    devices = list(devices) if devices else [0]
    summary = {"config": cfg.echo(), "num_recordings": len(recordings), "num_segments": len(segments),
               "num_batches": len(plans)}
    failures, outputs, batches_json = [], [], []
    st = {"written": 0, "failed": 0, "load": 0.0, "write": 0.0, "audio": 0.0}
    shapes = set()

    def load_one(i: int) -> LoadedBatch:
        item = LoadedBatch(i)
        t0 = time.perf_counter()
        try:
            item.batch = assemble(plans[i], rec_by_id[plans[i].recording_id], segments, cfg)
            item.batch.batch_index = i
        except Exception as e:  # a load failure fails every part of that batch, the run continues
            item.batch, item.error = None, str(e)
        item.load_seconds = time.perf_counter() - t0
        return item

    # writer: a single thread keeps file output off the compute path, preserving enqueue order
    write_failures, write_q, write_cv, write_state = [], [], threading.Condition(), {"done": False}

    def do_write(path, seg_id, audio):
        try:
            wav.write(path, RealSignal(audio.reshape(1, -1), cfg.stft.sample_rate))
        except Exception as e:
            write_failures.append((seg_id, str(e)))

    def writer_loop():
        while True:
            with write_cv:
                write_cv.wait_for(lambda: write_state["done"] or write_q)
                if not write_q:
                    return
                job = write_q.pop(0)
            t0 = time.perf_counter()
            do_write(*job)
            st["write"] += time.perf_counter() - t0

    writer = threading.Thread(target=writer_loop, name="gss-writer") if cfg.workers > 0 else None
    if writer:
        writer.start()

    def fail_batch(index, error):
        for part in plans[index].parts:
            failures.append({"segment_id": part.id, "batch": index, "error": error})
            st["failed"] += 1

    def consume(item: LoadedBatch, result):  # strictly in plan order
        st["load"] += item.load_seconds
        if item.batch is None:
            fail_batch(item.index, item.error)
            return
        if result.error is not None:  # pooled statistics make the whole batch fail together
            fail_batch(item.index, str(result.error))
            return
        ss = item.batch
        st["audio"] += ss.audio.num_samples() / ss.audio.sample_rate
        shapes.add((ss.audio.num_channels(), ss.activity.num_classes()))
        batches_json.append({"batch": item.index, "speaker": ss.speaker, "frames": result.frames,
                             "segments": len(ss.parts), "ref_channel": result.ref_channel,
                             "zeroed_bins": result.zeroed_bins, "log_likelihood": result.ll_final})
        for part, audio in zip(ss.parts, result.outputs):
            seg = part.segment
            path = cfg.out_dir + "/" + output_name(seg.recording_id, seg.speaker, seg.start, seg.end())
            outputs.append({"segment_id": seg.id, "path": path, "samples": int(len(audio))})
            st["written"] += 1
            if writer:
                with write_cv:
                    write_q.append((path, seg.id, audio))
                    write_cv.notify()
            else:
                t0 = time.perf_counter()
                do_write(path, seg.id, audio)
                st["write"] += time.perf_counter() - t0

    slots = [_ComputeSlot(d) for d in devices]
    inflight = []  # (items of a device batch, future) in plan order

    def drain(limit):
        while len(inflight) > limit:
            items, fut = inflight.pop(0)
            try:
                results = iter(fut.result()) if fut is not None else iter(())
            except Exception as exc:  # call-level device failure: its batches fail, the run goes on
                for it in items:
                    st["load"] += it.load_seconds
                    fail_batch(it.index, it.error if it.batch is None else "%s: %s" % (type(exc).__name__, exc))
                continue
            for it in items:
                consume(it, next(results) if it.batch is not None else None)

    queue = None
    try:
        if cfg.workers == 0:
            source = (load_one(i) for i in range(len(plans)))
            loaders = []
        else:
            queue = OrderedBatchQueue(max(cfg.queue_capacity, 1))
            ticket = iter(range(len(plans)))
            ticket_lock = threading.Lock()

            def loader():
                while True:
                    with ticket_lock:
                        i = next(ticket, None)
                    if i is None:
                        return
                    if not queue.put(load_one(i)):
                        return

            loaders = [threading.Thread(target=loader, name="gss-loader%d" % w) for w in range(cfg.workers)]
            for t in loaders:
                t.start()
            source = (queue.take() for _ in range(len(plans)))
        chunk, n_chunks = [], 0
        for item in source:
            chunk.append(item)
            if len(chunk) == max(1, gpu_batch):
                good = [it.batch for it in chunk if it.batch is not None]
                inflight.append((chunk, slots[n_chunks % len(slots)].submit(good, cfg) if good else None))
                n_chunks += 1
                chunk = []
                drain(2 * len(slots))  # at most two device batches queued per GPU
        if chunk:
            good = [it.batch for it in chunk if it.batch is not None]
            inflight.append((chunk, slots[n_chunks % len(slots)].submit(good, cfg) if good else None))
        drain(0)
        for t in loaders:
            t.join()
    finally:
        if queue is not None:
            queue.close()  # a no-op after a normal run; on an exception it lets blocked loaders leave
        if writer:
            with write_cv:
                write_state["done"] = True
                write_cv.notify_all()
            writer.join()
        stage = {}
        for sl in slots:
            for k, v in sl.stage.items():
                stage[k] = stage.get(k, 0.0) + v
            sl.close()
    for seg_id, error in write_failures:
        failures.append({"segment_id": seg_id, "error": "write failed: " + error})
        st["failed"] += 1
        st["written"] -= 1
    summary["segments_written"] = st["written"]
    summary["failures"] = failures
    summary["batches"] = batches_json
    summary["outputs"] = outputs
    # The reference reports its einsum planner's cache here; on the device that contraction is hard-coded per
    # (channels, classes) kernel specialisation, which plays the planner's role: one "entry" per shape used.
    summary["plan_cache"] = {"entries": len(shapes), "computed": len(shapes),
                             "hits": max(0, len(batches_json) - len(shapes))}
    summary["stage_seconds"] = {"load": st["load"], "stft": stage.get("stft", 0.0), "wpe": stage.get("wpe", 0.0),
                                "mask": stage.get("mask", 0.0), "beamform": stage.get("beamform", 0.0),
                                "istft": stage.get("istft", 0.0), "write": st["write"],
                                "total": time.perf_counter() - wall0}
    summary["processed_audio_seconds"] = st["audio"]
    summary["devices"] = devices
    manifests.write_text(cfg.out_dir + "/summary.json", json.dumps(summary, indent=2) + "\n")
    return RunSummary(summary, st["failed"])
