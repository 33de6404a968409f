#!/usr/bin/env python
"""Headline benchmark: enhanced audio-seconds per wall-second (xRT) of the GSS enhance path
(STFT -> WPE -> 20-iteration cACGMM -> Souden MVDR -> iSTFT).

    python bench.py --gpus N --steps K --warmup W            # this repo (CUDA, sm_100a)
    python bench.py --impl reference --gpus N ...            # the reference's CPU path (oracle port)

Headline workload = the largest single-GPU configuration of BASELINE.json: configs[2] (AMI-shaped: 8 channels,
4 speakers + noise, WPE taps 10 / delay 3, 20 EM iterations, batch of 64 segments of 10 s + 2 x 15 s context).
One "step" = one pass of the hot path over one batch of 64 synthetic SuperSegments per GPU (weak scaling: every
rank enhances its own 64 segments; no collective on the data path). `value` is timed with the batch already
resident in HBM; `e2e` is the same metric through the public call on HOST buffers (pinned), host<->device copies
included. The same JSON line carries a `configs` block with configs[0], [1], [3] (each rank its own batch) and a
256-segment sample of configs[4] (the 4096-segment sweep, sharded over the ranks by sharding.shard: strong
scaling). With --gpus N > 1 and no torchrun environment the script re-launches itself as N ranks. Prints ONE
JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "enhanced audio-sec per wall-sec (xRT)"
UNIT = "audio-s/s"

# BASELINE.json configs -> (workload name, default segments per GPU, description)
WORKLOADS = {
    "cfg1": (1, "BASELINE configs[0]: synthetic 2-speaker 7-ch 16 kHz 10 s segment, 512/128 STFT, 20 cACGMM iters, "
                "no WPE, context 0"),
    "cfg2": (16, "BASELINE configs[1]: LibriCSS-shaped 7-ch, 3 spk + noise, WPE on (taps 10, delay 2, 3 iters), "
                 "15 s context, 20 cACGMM iters, 512/128 STFT"),
    "cfg3": (64, "BASELINE configs[2]: AMI-shaped 8-ch, 4 spk + noise, WPE taps 10 delay 3 (3 iters), 15 s context, "
                 "20 cACGMM iters, 512/128 STFT"),
    "cfg4": (16, "BASELINE configs[3]: AliMeeting-shaped 8-ch, 4 spk + noise, 30 s segments + 2 x 15 s context "
                 "(T = 7501), all F = 257 bins per launch, WPE on, 20 cACGMM iters"),
    "tiny": (2, "test shape: 4-ch, 2 spk + noise, 2 s + 2 x 1 s, 5 iters"),
}
SWEEP_TOTAL = 4096


def _peaks():
    """(HBM GB/s, dense bf16 TFLOP/s burst, source). TF32 tensor throughput is half the bf16 rate."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), "measured (MEASURED_PEAKS.json)"
    return 6650.0, 1590.0, "fallback (B200_PROFILING.md)"


def _ncu_traffic():
    """DRAM bytes per launch and segment of each kernel class from the committed ncu --set full captures."""
    import glob
    for p in sorted(glob.glob(os.path.join(ROOT, "profiles", "ncu_traffic_r*.json")), reverse=True):
        try:
            return json.load(open(p))
        except Exception:
            continue
    return {}


class ClockSampler(threading.Thread):
    """SM clock / throttle reasons while the timed region runs: NVML when importable (millisecond samples),
    else nvidia-smi (the recipe's clocks line)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        super().__init__(daemon=True)
        self.index, self.rows, self.stop_flag = index, [], False

    def _run_nvml(self):
        import pynvml as nv
        nv.nvmlInit()
        h = nv.nvmlDeviceGetHandleByIndex(self.index)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        bits = [(nv.nvmlClocksEventReasonHwSlowdown if hasattr(nv, "nvmlClocksEventReasonHwSlowdown")
                 else nv.nvmlClocksThrottleReasonHwSlowdown),
                (nv.nvmlClocksEventReasonHwThermalSlowdown if hasattr(nv, "nvmlClocksEventReasonHwThermalSlowdown")
                 else nv.nvmlClocksThrottleReasonHwThermalSlowdown),
                (nv.nvmlClocksEventReasonSwThermalSlowdown if hasattr(nv, "nvmlClocksEventReasonSwThermalSlowdown")
                 else nv.nvmlClocksThrottleReasonSwThermalSlowdown),
                (nv.nvmlClocksEventReasonSwPowerCap if hasattr(nv, "nvmlClocksEventReasonSwPowerCap")
                 else nv.nvmlClocksThrottleReasonSwPowerCap)]
        get = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or nv.nvmlDeviceGetCurrentClocksThrottleReasons
        while not self.stop_flag:
            r = get(h)
            self.rows.append([str(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)), str(mx)]
                             + ["Active" if r & b else "Not Active" for b in bits])
            time.sleep(0.005)

    def run(self):
        try:
            self._run_nvml()
            return
        except Exception:
            pass
        while not self.stop_flag:
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                f = [x.strip() for x in out.stdout.strip().split(",")]
                if len(f) >= 6:
                    self.rows.append(f)
            except Exception:
                pass
            time.sleep(0.1)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = [n for i, n in enumerate(names) if any(r[2 + i].lower().startswith("active") for r in self.rows)]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": float(self.rows[0][1]),
                "reasons": reasons, "samples": len(self.rows)}


def algorithmic_work(segs, cfg):
    """SURVEY.md 8(d) per-segment figures, summed over a batch: flops / bytes per kernel class per step."""
    F = cfg.stft.fft_size // 2 + 1
    n = cfg.stft.fft_size
    I = cfg.bss_iterations
    J = cfg.wpe.iterations if cfg.enable_wpe else 0
    w = {k: {"flops": 0.0, "bytes": 0.0} for k in ("stft", "wpe_power", "wpe_gram", "wpe_solve", "wpe_apply", "em_pass",
                                                   "em_update", "mvdr", "apply", "istft")}
    import math
    # which WPE kernels a segment runs (api.cu: by shape unless GSS_B200_WPE_GRAM / _APPLY force one)
    g_env, a_env = os.environ.get("GSS_B200_WPE_GRAM", "auto"), os.environ.get("GSS_B200_WPE_APPLY", "auto")
    for ss in segs:
        M, N = ss.audio.channels.shape
        T, K = ss.activity.grid.shape
        FT = F * T
        km = cfg.wpe.taps * M
        tc_gram = g_env == "tc" or (g_env != "fp32" and M >= 4)
        tc_apply = a_env == "tc" or (a_env != "fp32" and M >= 4)
        w["stft"]["bytes"] += 4 * M * N + 8 * FT * M
        w["stft"]["flops"] += M * T * (2.5 * n * math.log2(n) + n)
        if J:
            # with psd_context 0 the tensor-core prediction writes the next iteration's weights: one power pass
            n_power = 1 if (cfg.wpe.psd_context == 0 and tc_apply) else J
            w["wpe_power"]["bytes"] += n_power * (8 * FT * M + 4 * FT)
            w["wpe_gram"]["flops"] += J * FT * 8 * (km * (km + 1) / 2 + km * M)
            w["wpe_gram"]["bytes"] += J * (8 * FT * M + 4 * FT)
            w["wpe_solve"]["flops"] += J * F * (8 / 3 * km ** 3 + 16 * km * km * M)
            w["wpe_apply"]["flops"] += J * FT * 8 * km * M
            w["wpe_apply"]["bytes"] += J * 2 * 8 * FT * M
        if J and tc_gram:
            # tensor-core Gram: executed tensor flops (hi/lo split: 3 MMAs per product; a 128 x NR accumulator plus,
            # where an Im a row lies beyond row 127, the corner block as an M = 64 MMA of N2 columns)
            kmp = (km + 7) // 8 * 8
            nr = (2 * kmp + 16 + 15) // 16 * 16
            nr = (nr + 31) // 32 * 32 if nr < 128 else nr  # kernels.h wpe_tc_operand_rows
            n2 = max(0, nr - 128) if kmp + km > 128 else 0
            w["wpe_gram"]["tensor_flops"] = (w["wpe_gram"].get("tensor_flops", 0.0) +
                                             J * FT * 3 * 2 * (128 * nr + 64 * n2))
        if J and tc_apply:
            # tensor-core prediction: per frame and tap K = 16, A_hi x [B_hi | B_lo] (N = 32) + A_lo x B_hi (N = 16)
            w["wpe_apply"]["tensor_flops"] = w["wpe_apply"].get("tensor_flops", 0.0) + J * FT * cfg.wpe.taps * 2 * 2 * 8 * 48
        w["em_pass"]["flops"] += (I + 1) * FT * (3 * M * M + 4 * M * M * K + 20 * K)
        w["em_pass"]["bytes"] += (I + 1) * (8 * FT * M + T * K)
        w["em_update"]["flops"] += (I + 1) * F * K * (8 * M ** 3)
        w["apply"]["flops"] += FT * 8 * M
        w["apply"]["bytes"] += 8 * FT * M + 8 * FT
        w["istft"]["bytes"] += 8 * FT + 4 * N
        w["istft"]["flops"] += T * (2.5 * n * math.log2(n) + n)
    return w


def sum_work(calls):
    """algorithmic_work over a list of (cfg, segments) device calls."""
    total = {}
    for cfg, segs in calls:
        for name, d in algorithmic_work(segs, cfg).items():
            t = total.setdefault(name, {})
            for k, v in d.items():
                t[k] = t.get(k, 0.0) + v
    return total


def tensor_peak(kernel, bf16_peak):
    """(dense peak of the MMA kind the kernel runs, its name): kind::f16 at the 16-bit rate, kind::tf32 at half of it."""
    env = {"wpe_gram": "GSS_B200_WPE_GRAM_KIND", "wpe_apply": "GSS_B200_WPE_APPLY_KIND"}[kernel]
    return (0.5 * bf16_peak, "TF32 dense = 0.5 x bf16 ") if os.environ.get(env) == "tf32" else (bf16_peak, "FP16 dense = bf16 ")


def kernel_table(kms, steps, work, nseg, hbm_peak, bf16_peak, fp32_peak, peak_src, traffic):
    """Per kernel class: ms per step, launches, the roofline that bounds it and the fraction reached."""
    tc_gram = tc_apply = True  # a class is tensor-bound when any of its segments ran the tcgen05 kernel (tensor_flops > 0)
    kernels = {}
    for name, (kms_total, n) in kms.items():
        if n == 0 or name not in work:
            continue
        per_step = kms_total / steps
        fl, by = work[name].get("flops", 0.0), work[name].get("bytes", 0.0)
        t_f = fl / (fp32_peak * 1e12) if fp32_peak > 0 else 0.0
        t_b = by / (hbm_peak * 1e9)
        bound = "fp32" if t_f > t_b else "hbm"
        ach = (fl / (per_step * 1e-3) * 1e-12) if bound == "fp32" else (by / (per_step * 1e-3) * 1e-9)
        peak = fp32_peak if bound == "fp32" else hbm_peak
        kernels[name] = {"ms_per_step": round(per_step, 4), "launches_per_step": n // steps, "bound": bound,
                         "achieved": round(ach, 2), "peak": round(peak, 2),
                         "unit": "TFLOP/s" if bound == "fp32" else "GB/s", "frac": round(ach / peak, 4)}
        note = ("; a thread issues one tcgen05.mma per ~100 - 150 cycles whatever its M, N and kind (tools/mma_probe.cu), "
                "so a kernel of small-N MMAs pays for its instruction count and stays far from the dense peak")
        for kname, on in (("wpe_gram", tc_gram), ("wpe_apply", tc_apply)):
            if name == kname and on and work[name].get("tensor_flops"):
                # tcgen05: `achieved` stays the ALGORITHMIC (FP32-equivalent) rate; the executed tensor rate (3 MMAs
                # per product, padded tiles) is reported beside it
                tpeak, tname = tensor_peak(name, bf16_peak)
                ex = work[name]["tensor_flops"] / (per_step * 1e-3) * 1e-12
                kernels[name].update({"bound": "tensor", "peak": round(tpeak, 2), "frac": round(ach / tpeak, 4),
                                      "executed_tensor_tflops": round(ex, 1), "executed_frac": round(ex / tpeak, 4),
                                      "peak_note": tname + peak_src + note})
        if name in traffic and nseg:
            kernels[name]["traffic_bytes_per_launch"] = int(traffic[name]["dram_bytes_per_segment_launch"] * nseg)
    return kernels


class Bench:
    """One rank's measuring context: device, library context, stream, barrier."""

    def __init__(self, rank, world, local_rank):
        import torch
        import torch.distributed as dist
        from paper_2212_05271_b200 import gss
        self.torch, self.dist, self.gss = torch, dist, gss
        self.rank, self.world, self.local_rank = rank, world, local_rank
        if world > 1:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        torch.cuda.set_device(local_rank)
        self.ctx = gss.default_context(local_rank)
        self.stream = torch.cuda.ExternalStream(self.ctx.stream, device=torch.device("cuda", local_rank))
        self.hbm_peak, bf16_peak, self.peak_src = _peaks()
        self.bf16_peak = bf16_peak
        self.fp32_peak = self.ctx.fp32_peak_tflops()
        self.traffic = _ncu_traffic()

    def barrier(self):
        self.torch.cuda.synchronize()
        if self.world > 1:
            self.dist.barrier()
        self.torch.cuda.synchronize()

    device = "cuda"  # the CPU test of the aggregation (gloo, world size 2) overrides it

    def max_over_ranks(self, values):
        t = self.torch.tensor(values, dtype=self.torch.float64, device=self.device)
        if self.world > 1:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return [float(v) for v in t]

    def sum_over_ranks(self, values):
        t = self.torch.tensor(values, dtype=self.torch.float64, device=self.device)
        if self.world > 1:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)
        return [float(v) for v in t]

    def measure(self, calls, steps, warmup, sampler=None):
        """calls = [(cfg, segments)]: one step runs every call once. Returns this rank's timings:
        resident (CUDA events on the library's stream, K steps, nothing else inside), the same K steps again with
        every launch bracketed by events (per-kernel table), and the public call on pinned host buffers."""
        torch, ctx = self.torch, self.ctx
        sched = self.gss.scheduler
        ctx.device_bytes_peak(reset=True)
        rbs = [sched.ResidentBatch(segs, cfg, ctx, pinned=True) for cfg, segs in calls if segs]
        for rb in rbs:
            rb.upload()
        for _ in range(warmup):
            for rb in rbs:
                rb.run()
        self.barrier()
        if sampler is not None:
            sampler.start()
        l0 = ctx.launch_count
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(self.stream)
        for _ in range(steps):
            for rb in rbs:
                rb.run()
        e1.record(self.stream)
        self.barrier()
        ms = e0.elapsed_time(e1) if rbs else 0.0
        launches = ctx.launch_count - l0
        if sampler is not None:
            sampler.stop_flag = True
        ctx.profile(True)
        p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        p0.record(self.stream)
        for _ in range(steps):
            for rb in rbs:
                rb.run()
        p1.record(self.stream)
        self.barrier()
        ms_profiled = p0.elapsed_time(p1) if rbs else 0.0
        kms = ctx.kernel_ms()
        ctx.profile(False)
        peak_bytes = ctx.device_bytes_peak()
        failures = []
        for rb in rbs:
            failures += [str(r.error) for r in rb.fetch() if r.error is not None]
            rb.free()
        stage = ctx.stage_ms()
        # end to end through the public call on host (pinned) buffers: H2D + kernels + D2H every step
        for _ in range(min(warmup, 2)):
            for rb in rbs:
                rb.enhance()
        self.barrier()
        t0 = time.perf_counter()
        for _ in range(steps):
            for rb in rbs:
                rb.enhance()
        torch.cuda.synchronize()
        e2e_ms = (time.perf_counter() - t0) * 1e3
        self.barrier()
        return {"ms": ms, "launches": int(launches), "kms": kms, "ms_profiled": ms_profiled, "e2e_ms": e2e_ms,
                "h2d": sum(rb.m.h2d_bytes for rb in rbs), "d2h": sum(rb.m.d2h_bytes for rb in rbs),
                "failures": failures, "stage": stage, "peak_device_bytes": peak_bytes}


def seconds_of(calls, sr=16000):
    out_s = sum((p.sample_end - p.sample_begin) / sr for _, segs in calls for s in segs for p in s.parts)
    asm_s = sum(s.audio.num_samples() / sr for _, segs in calls for s in segs)
    return out_s, asm_s


def summarise(b, calls, r, steps, scaling):
    """Aggregate one workload over the ranks: times are the max over ranks, work is the sum."""
    ms_max, e2e_max = b.max_over_ranks([r["ms"], r["e2e_ms"]])
    out_s, asm_s = seconds_of(calls)
    nseg = sum(len(segs) for _, segs in calls)
    out_all, asm_all, nseg_all, h2d, d2h, launches = b.sum_over_ranks([out_s, asm_s, nseg, r["h2d"], r["d2h"],
                                                                       r["launches"]])
    res = {"segments": int(nseg_all), "scaling": scaling, "ms_per_step": round(ms_max / steps, 3),
           "value": round(out_all * steps / (ms_max * 1e-3), 2),
           "xrt_processed": round(asm_all * steps / (ms_max * 1e-3), 2),
           "segments_per_s": round(nseg_all * steps / (ms_max * 1e-3), 2),
           "e2e": {"value": round(out_all * steps / (e2e_max * 1e-3), 2), "unit": UNIT,
                   "ms_per_step": round(e2e_max / steps, 3),
                   "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)},
           "gpu_launches": int(launches), "per_rank_ms_per_step": None}
    if b.world > 1:
        per = [None] * b.world
        b.dist.all_gather_object(per, round(r["ms"] / steps, 3))
        res["per_rank_ms_per_step"] = per
    return res


def top_kernel(kernels):
    return max(kernels, key=lambda k: kernels[k]["ms_per_step"]) if kernels else None


def side_config(b, name, calls, steps, warmup, scaling, label, extra=None):
    """One entry of the `configs` block: resident value, e2e, and the kernel that dominates with its roofline."""
    r = b.measure(calls, steps, warmup)
    res = summarise(b, calls, r, steps, scaling)
    if b.rank != 0:
        return None
    work = sum_work(calls)
    nseg = sum(len(segs) for _, segs in calls)
    kernels = kernel_table(r["kms"], steps, work, nseg, b.hbm_peak, b.bf16_peak, b.fp32_peak, b.peak_src, {})
    top = top_kernel(kernels)
    res.update({"workload": label, "steps": steps,
                "kernels_ms_per_step": {k: v["ms_per_step"] for k, v in kernels.items()},
                "roofline": None if not top else {"kernel": top, "bound": kernels[top]["bound"],
                                                  "achieved": kernels[top]["achieved"], "peak": kernels[top]["peak"],
                                                  "unit": kernels[top]["unit"], "frac": kernels[top]["frac"]},
                "peak_device_bytes": r["peak_device_bytes"], "failures": r["failures"]})
    if extra:
        res.update(extra)
    return res


def sweep_calls(b, n_sample):
    """This rank's share of the configs[4] sample: `n_sample` of the 4096 sweep segments (every 4096/n_sample-th),
    split over the ranks by the static size-balanced shard (sharding.shard on the SURVEY 8e cost model), grouped by
    EM iteration count (one device call per group)."""
    import synthbench as synth
    from paper_2212_05271_b200 import sharding
    params = synth.sweep_params(SWEEP_TOTAL)[:: max(1, SWEEP_TOTAL // n_sample)][:n_sample]
    costs = [sharding.segment_cost(synth.sweep_frames(p[3]), p[1], p[2] + 1, p[4], 10, 3) for p in params]
    owned = sharding.shard(costs, b.world)
    mine = [params[i] for i in owned[b.rank]]
    segs = synth.make_sweep_segments(mine, threads=max(2, (os.cpu_count() or 8) // max(1, b.world)))
    by_iter = {}
    for p, ss in zip(mine, segs):
        by_iter.setdefault(p[4], []).append(ss)
    calls = [(synth.sweep_cfg(it), by_iter[it]) for it in sorted(by_iter)]
    loads = [sum(costs[i] for i in own) for own in owned]
    balance = sum(loads) / (b.world * max(loads)) if loads and max(loads) > 0 else 1.0
    return calls, round(balance, 4)


def run_ours(args, rank, world, local_rank):
    import synthbench as synth
    b = Bench(rank, world, local_rank)
    nseg = args.segments or WORKLOADS[args.workload][0]
    threads = max(2, (os.cpu_count() or 8) // max(1, world))
    wl = synth.workload(args.workload, n_segments=nseg, first=rank * nseg, threads=threads)
    cfg = wl.cfg
    calls = [(cfg, wl.segments)]
    sampler = ClockSampler(local_rank)
    r = b.measure(calls, args.steps, args.warmup, sampler)
    head = summarise(b, calls, r, args.steps, "weak")
    line = None
    if rank == 0:
        work = sum_work(calls)
        kernels = kernel_table(r["kms"], args.steps, work, nseg, b.hbm_peak, b.bf16_peak, b.fp32_peak, b.peak_src,
                               b.traffic)
        top = top_kernel(kernels)
        roof = None
        if top:
            k = kernels[top]
            roof = {"kernel": top, "bound": k["bound"], "achieved": k["achieved"], "peak": k["peak"], "unit": k["unit"],
                    "frac": k["frac"], "traffic": k.get("traffic_bytes_per_launch"),
                    "traffic_source": "committed ncu --set full capture (profiles/ncu_traffic_*.json: DRAM bytes per "
                                      "launch and segment, scaled by this run's segment count), not measured in this "
                                      "run" if k.get("traffic_bytes_per_launch") else None,
                    "algorithmic_per_launch": (work[top]["flops"] if k["bound"] != "hbm" else work[top]["bytes"])
                    / max(1, k["launches_per_step"]),
                    "peak_source": ("measured FFMA loop in this run (gss_b200_fp32_peak)" if k["bound"] == "fp32"
                                    else k.get("peak_note", b.peak_src)),
                    "avg_launch_ms": round(k["ms_per_step"] / max(1, k["launches_per_step"]), 4),
                    "share_of_step": round(k["ms_per_step"] / (r["ms_profiled"] / args.steps), 4),
                    "note": ("algorithmic flops are SURVEY 8(d)'s count, which charges all K classes per frame; the sweep "
                             "skips classes that are inactive in a whole group of 32 frames, so the executed FMA count is "
                             "lower (DESIGN.md section 3)") if top == "em_pass" else None,
                    "timing": "CUDA events around every launch of a second pass of the same K steps "
                              "(%.3f ms/step with the events in; the headline pass has none)"
                              % (r["ms_profiled"] / args.steps)}
        I = cfg.bss_iterations
        em_ms = r["kms"]["em_pass"][0] + r["kms"]["em_update"][0]
        line = {
            "metric": METRIC, "value": head["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": head["ms_per_step"], "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": workload_config(args.workload, nseg, wl),
            "xrt_processed": head["xrt_processed"], "segments_per_s": head["segments_per_s"],
            "em_iters_per_s": round(nseg * world * I * args.steps / max(1e-9, em_ms) * 1e3, 1),
            "e2e": head["e2e"], "gpu_launches": head["gpu_launches"],
            "per_rank_ms_per_step": head["per_rank_ms_per_step"],
            "stage_ms": {k: round(v, 3) for k, v in r["stage"].items()},
            "roofline": roof, "kernels": kernels, "fp32_peak_tflops": round(b.fp32_peak, 2),
            "peak_device_bytes": r["peak_device_bytes"],
            "clocks": sampler.summary(), "failures": r["failures"],
        }
    del r
    # ---- the other BASELINE configs, same run (each rank its own batch; the sweep sample is sharded: strong scaling)
    configs = {}
    if not args.headline_only:
        ks = max(3, min(args.steps, args.side_steps))
        for name in ("cfg1", "cfg2", "cfg4"):
            if name == args.workload:
                continue
            n = WORKLOADS[name][0]
            w2 = synth.workload(name, n_segments=n, first=rank * n, threads=threads)
            c = side_config(b, name, [(w2.cfg, w2.segments)], ks, 3, "weak", WORKLOADS[name][1],
                            {"segments_per_gpu": n, "window_s": round(w2.assembled_seconds / n, 3)})
            if rank == 0:
                configs[name] = c
            del w2
        sc, balance = sweep_calls(b, args.sweep_segments)
        c = side_config(b, "cfg5", sc, ks, 3, "strong",
                        "BASELINE configs[4] sample: %d of the %d sweep segments (every %d-th; durations U[2,12] s + "
                        "2 x 15 s context, 2-8 channels, 2-4 speakers + noise, EM iterations in {5,10,20,40}, WPE on), "
                        "sharded over the ranks by sharding.shard" % (args.sweep_segments, SWEEP_TOTAL,
                                                                    SWEEP_TOTAL // args.sweep_segments),
                        {"shard_load_balance": balance, "device_calls_per_step": len(sc)})
        if rank == 0:
            configs["cfg5"] = c
    if rank == 0:
        line["configs"] = configs
    return line, wl


def workload_config(name, nseg, wl):
    import numpy as np  # noqa: F401
    cfg = wl.cfg
    seg = wl.segments[0]
    gb = nseg * 8.0 * (cfg.stft.fft_size // 2 + 1) * seg.activity.grid.shape[0] * seg.audio.channels.shape[0] / 1e9
    return {"workload": WORKLOADS[name][1], "name": name, "segments_per_gpu": nseg,
            "window_s": wl.assembled_seconds / max(1, len(wl.segments)),
            "output_s_per_segment": wl.output_seconds / max(1, len(wl.segments)),
            "l2": "working set per step (2 x %.2f GB spectrograms) exceeds the 126 MB L2; no flush needed" % gb}


def oracle_enhance(orc, ss, cfg):
    return orc.enhance(ss.audio.channels, ss.activity.grid, ss.activity.target_index, ss.activity.noise_index,
                       [(p.sample_begin, p.sample_end) for p in ss.parts], fft_size=cfg.stft.fft_size,
                       shift=cfg.stft.shift, window=cfg.stft.window, sample_rate=cfg.stft.sample_rate,
                       enable_wpe=cfg.enable_wpe, taps=cfg.wpe.taps, delay=cfg.wpe.delay,
                       wpe_iterations=cfg.wpe.iterations, psd_context=cfg.wpe.psd_context,
                       regularization=cfg.wpe.regularization, bss_iterations=cfg.bss_iterations)


def load_oracle(vector_gram=True):
    """The CPU oracle port of the reference path, rebuilt for this host's ISA when possible. `vector_gram`: the
    timing-only build whose Gram dot products run on SIMD partial sums (what Eigen's cfloat GEMM gives the
    reference; oracle/gss_oracle.hpp, GSS_ORACLE_VECTOR_GRAM) -- the faster, fairer CPU arm."""
    from oracle import oracle as orc
    tag = "native_vec" if vector_gram else "native"
    try:
        path = orc.build(march="native", out_dir=os.path.join(ROOT, "oracle", "_build", tag), vector_gram=vector_gram)
        orc.load(path)
        return orc, ("port, -O3 -march=native, " + ("SIMD Gram (GSS_ORACLE_VECTOR_GRAM)" if vector_gram
                                                   else "scalar Gram (the parity checker's build)"))
    except Exception:
        orc.load()
        return orc, "port, prebuilt x86-64-v3 scalar Gram (rebuild failed on this host)"


def reference_note():
    """Why the CPU arm is the port: the reference needs Eigen, and its sources do not travel to the GPU box."""
    eigen = any(os.path.isdir(p) for p in ("/usr/include/eigen3", "/usr/local/include/eigen3"))
    ref = os.path.isdir("/root/reference/proj/include/gss")
    return ("Eigen headers %s, reference sources %s on this host: the true reference (header-only C++20 over Eigen) "
            "cannot be compiled here, the CPU arm is the Eigen-free restatement oracle/gss_oracle.hpp"
            % ("present" if eigen else "absent", "present" if ref else "absent"))


def time_oracle(orc, segs, cfg):
    t0 = time.perf_counter()
    for ss in segs:
        oracle_enhance(orc, ss, cfg)
    return time.perf_counter() - t0


def cpu_baseline(wl, n_sample=6):
    """Reference CPU path (oracle port) on a bounded sample of the same workload, all host threads
    (parallel_for over F, parallel.hpp:14-51). Both builds are timed: the SIMD-Gram one is the reported value."""
    cfg = wl.cfg
    sr = cfg.stft.sample_rate
    segs = wl.segments[:n_sample]
    out_s = sum((p.sample_end - p.sample_begin) / sr for s in segs for p in s.parts)
    orc, kind = load_oracle(True)
    dt = time_oracle(orc, segs, cfg)
    orc2, kind2 = load_oracle(False)
    few = segs[:2]
    dt2 = time_oracle(orc2, few, cfg)
    out2 = sum((p.sample_end - p.sample_begin) / sr for s in few for p in s.parts)
    return {"value": round(out_s / dt, 4), "unit": UNIT, "cores": orc.hardware_threads(), "kind": "port",
            "build": kind,
            "sample": "%d of the %d segments of one batch (%.1f s window each), %.1f s of CPU time"
                      % (len(segs), len(wl.segments), wl.assembled_seconds / len(wl.segments), dt),
            "seconds": round(dt, 2),
            "scalar_gram_build": {"value": round(out2 / dt2, 4), "segments": len(few), "seconds": round(dt2, 2),
                                  "build": kind2},
            "note": reference_note()}


def run_reference(args, rank, world):
    if rank != 0:
        return None
    import synthbench as synth
    nseg = args.segments or WORKLOADS[args.workload][0]
    wl = synth.workload(args.workload, n_segments=1)
    orc, kind = load_oracle(True)
    cfg = wl.cfg
    for _ in range(args.warmup):
        oracle_enhance(orc, wl.segments[0], cfg)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle_enhance(orc, wl.segments[0], cfg)
    dt = time.perf_counter() - t0
    value = wl.output_seconds * args.steps / dt
    config = workload_config(args.workload, nseg, wl)
    return {"impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt / args.steps * 1e3, 2),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32/f64 mixed (reference)",
            "data": "synthetic", "config": config,
            "note": "each step enhances ONE segment of the batch on the host cores (bounded sample); xRT is "
                    "per-segment work, so it compares directly with the GPU arm's value. " + reference_note(),
            "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": orc.hardware_threads(), "kind": "port",
                             "build": kind, "sample": "1 segment (%.0f s window) per step" % wl.assembled_seconds},
            "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg3", choices=sorted(WORKLOADS))
    ap.add_argument("--segments", type=int, default=0, help="segments per GPU per step (default: the config's batch)")
    ap.add_argument("--headline-only", action="store_true", help="skip the `configs` block (cfg1/2/4 and the sweep)")
    ap.add_argument("--side-steps", type=int, default=5, help="timed steps of each `configs` entry")
    ap.add_argument("--sweep-segments", type=int, default=256, help="sample size of the configs[4] sweep")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    if args.impl == "reference":
        line = run_reference(args, int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")))
        if line is not None:
            print(json.dumps(line), flush=True)
        return
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # `python bench.py --gpus N`: become N ranks (one per GPU, NCCL) like the driver's torchrun launch
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(args.gpus),
               "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    args.warmup = max(args.warmup, 3)
    line, wl = run_ours(args, rank, world, local_rank)
    if rank == 0:
        line["cpu_baseline"] = cpu_baseline(wl) if (world == 1 and not args.no_cpu_baseline) else None
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
