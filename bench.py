#!/usr/bin/env python
"""Headline benchmark: enhanced audio-seconds per wall-second (xRT) of the GSS enhance path
(STFT -> WPE -> 20-iteration cACGMM -> Souden MVDR -> iSTFT) on BASELINE.json configs[1]
(LibriCSS-shaped: 7 channels, 3 speakers + noise, WPE on, 15 s context, batch of 16 segments).

    python bench.py --gpus N --steps K --warmup W            # this repo (CUDA, sm_100a)
    python bench.py --impl reference --gpus N ...            # the reference's CPU path (oracle port)

One "step" = one pass of the hot path over one batch of 16 synthetic SuperSegments per GPU (weak scaling:
every rank enhances its own 16 segments; no collective on the data path). `value` is timed with the batch
already resident in HBM; `e2e` is the same metric through the public call on HOST buffers (pinned),
host<->device copies included. Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
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


def _peaks():
    """(HBM GB/s, dense bf16 TFLOP/s burst, source). TF32 tensor throughput is half the bf16 rate."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), "measured (MEASURED_PEAKS.json)"
    return 6650.0, 1590.0, "fallback (B200_PROFILING.md)"


def _ncu_traffic():
    """DRAM bytes per launch and segment of each kernel class from the committed ncu --set full captures."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic_r01.json")
    try:
        return json.load(open(p))
    except Exception:
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
    for ss in segs:
        M, N = ss.audio.channels.shape
        T, K = ss.activity.grid.shape
        FT = F * T
        km = cfg.wpe.taps * M
        w["stft"]["bytes"] += 4 * M * N + 8 * FT * M
        w["stft"]["flops"] += M * T * (2.5 * n * math.log2(n) + n)
        if J:
            # with psd_context 0 the tensor-core prediction writes the next iteration's weights: one power pass
            n_power = 1 if (cfg.wpe.psd_context == 0 and os.environ.get("GSS_B200_WPE_APPLY") != "fp32") else J
            w["wpe_power"]["bytes"] += n_power * (8 * FT * M + 4 * FT)
            w["wpe_gram"]["flops"] += J * FT * 8 * (km * (km + 1) / 2 + km * M)
            w["wpe_gram"]["bytes"] += J * (8 * FT * M + 4 * FT)
            w["wpe_solve"]["flops"] += J * F * (8 / 3 * km ** 3 + 16 * km * km * M)
            w["wpe_apply"]["flops"] += J * FT * 8 * km * M
            w["wpe_apply"]["bytes"] += J * 2 * 8 * FT * M
        if J:
            # tensor-core Gram: executed TF32 flops (3xTF32 split; a 128 x NR accumulator plus the corner block as
            # an M = 64 MMA of N2 columns; the tensor core's cost floor is that of M = 128 for either)
            kmp = (km + 7) // 8 * 8
            nr = (2 * kmp + 16 + 15) // 16 * 16
            n2 = max(0, nr - 128)
            w["wpe_gram"]["tensor_flops"] = (w["wpe_gram"].get("tensor_flops", 0.0) +
                                             J * FT * 3 * 2 * (128 * nr + 64 * n2))
            # tensor-core prediction: per frame and tap 2 k-steps of 8, A_hi x [B_hi | B_lo] (N = 32) + A_lo x B_hi (N = 16)
            w["wpe_apply"]["tensor_flops"] = w["wpe_apply"].get("tensor_flops", 0.0) + J * FT * cfg.wpe.taps * 2 * 2 * 8 * 48
        w["em_pass"]["flops"] += (I + 1) * FT * (3 * M * M + 4 * M * M * K + 20 * K)
        w["em_pass"]["bytes"] += (I + 1) * (8 * FT * M + T * K)
        w["em_update"]["flops"] += (I + 1) * F * K * (8 * M ** 3)
        w["apply"]["flops"] += FT * 8 * M
        w["apply"]["bytes"] += 8 * FT * M + 8 * FT
        w["istft"]["bytes"] += 8 * FT + 4 * N
        w["istft"]["flops"] += T * (2.5 * n * math.log2(n) + n)
    return w


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_2212_05271_b200 import gss
    import synthbench as synth

    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    torch.cuda.set_device(local_rank)
    ctx = gss.default_context(local_rank)
    nseg = args.segments
    wl = synth.workload(args.workload, n_segments=nseg, first=rank * nseg)
    cfg = wl.cfg
    rb = gss.scheduler.ResidentBatch(wl.segments, cfg, ctx, pinned=True)
    rb.upload()
    stream = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", local_rank))

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        rb.run()
    barrier()
    # ---- the timed region: exactly K steps, device-timed on the launching stream, no per-kernel events inside
    sampler = ClockSampler(local_rank)
    sampler.start()
    l0 = ctx.launch_count
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        rb.run()
    e1.record(stream)
    barrier()
    ms = e0.elapsed_time(e1)
    launches = ctx.launch_count - l0
    sampler.stop_flag = True
    # ---- the same K steps again with every launch bracketed by CUDA events: the per-kernel table / roofline
    ctx.profile(True)
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    for _ in range(args.steps):
        rb.run()
    p1.record(stream)
    barrier()
    ms_profiled = p0.elapsed_time(p1)
    kms = ctx.kernel_ms()
    ctx.profile(False)
    res = rb.fetch()
    stage = ctx.stage_ms()
    failures = [str(r.error) for r in res if r.error is not None]
    rb.free()

    # end to end through the public call on host (pinned) buffers: H2D + kernels + D2H every step
    for _ in range(min(args.warmup, 2)):
        rb.enhance()
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        rb.enhance()
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    barrier()

    t = torch.tensor([ms, e2e_s * 1e3], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max, e2e_ms_max = float(t[0]), float(t[1])
    out_s = wl.output_seconds * world      # weak scaling: every rank processes the same amount
    asm_s = wl.assembled_seconds * world
    value = out_s * args.steps / (ms_max * 1e-3)
    line = None
    if rank == 0:
        hbm_peak, bf16_peak, peak_src = _peaks()
        tf32_peak = 0.5 * bf16_peak
        fp32_peak = ctx.fp32_peak_tflops()
        work = algorithmic_work(wl.segments, cfg)
        traffic = _ncu_traffic()
        tc_gram = os.environ.get("GSS_B200_WPE_GRAM", "tc") != "fp32"
        tc_apply = os.environ.get("GSS_B200_WPE_APPLY", "tc") != "fp32"
        kernels = {}
        for name, (kms_total, n) in kms.items():
            if n == 0 or name not in work:
                continue
            per_step = kms_total / args.steps
            fl, by = work[name]["flops"], work[name]["bytes"]
            t_f = fl / (fp32_peak * 1e12) if fp32_peak > 0 else 0.0
            t_b = by / (hbm_peak * 1e9)
            bound = "fp32" if t_f > t_b else "hbm"
            ach = (fl / (per_step * 1e-3) * 1e-12) if bound == "fp32" else (by / (per_step * 1e-3) * 1e-9)
            peak = fp32_peak if bound == "fp32" else hbm_peak
            kernels[name] = {"ms_per_step": round(per_step, 4), "launches_per_step": n // args.steps, "bound": bound,
                             "achieved": round(ach, 2), "peak": round(peak, 2),
                             "unit": "TFLOP/s" if bound == "fp32" else "GB/s", "frac": round(ach / peak, 4)}
            if name == "wpe_gram" and tc_gram and "tensor_flops" in work[name]:
                # tcgen05 kind::tf32: `achieved` stays the ALGORITHMIC (FP32-equivalent) rate; the executed tensor
                # rate (3 MMAs per product, padded tiles) is reported beside it
                ex = work[name]["tensor_flops"] / (per_step * 1e-3) * 1e-12
                kernels[name].update({"bound": "tensor", "peak": round(tf32_peak, 2), "frac": round(ach / tf32_peak, 4),
                                      "executed_tensor_tflops": round(ex, 1),
                                      "executed_frac": round(ex / tf32_peak, 4),
                                      "peak_note": "TF32 dense = 0.5 x bf16 " + peak_src})
            if name == "wpe_apply" and tc_apply and "tensor_flops" in work[name]:
                ex = work[name]["tensor_flops"] / (per_step * 1e-3) * 1e-12
                kernels[name].update({"bound": "tensor", "peak": round(tf32_peak, 2), "frac": round(ach / tf32_peak, 4),
                                      "executed_tensor_tflops": round(ex, 1),
                                      "executed_frac": round(ex / tf32_peak, 4),
                                      "peak_note": "TF32 dense = 0.5 x bf16 " + peak_src + "; N = 16-32 MMAs re-stream "
                                                   "their 128 x 8 A tile from shared memory, which is what bounds them"})
            if name in traffic:
                kernels[name]["traffic_bytes_per_launch"] = int(traffic[name]["dram_bytes_per_segment_launch"] * nseg)
        top = max(kernels, key=lambda k: kernels[k]["ms_per_step"]) if kernels else None
        roof = None
        if top:
            k = kernels[top]
            roof = {"kernel": top, "bound": k["bound"], "achieved": k["achieved"], "peak": k["peak"], "unit": k["unit"],
                    "frac": k["frac"], "traffic": k.get("traffic_bytes_per_launch"),
                    "algorithmic_per_launch": (work[top]["flops"] if k["bound"] != "hbm" else work[top]["bytes"])
                    / max(1, k["launches_per_step"]),
                    "peak_source": ("measured FFMA loop in this run (gss_b200_fp32_peak)" if k["bound"] == "fp32"
                                    else k.get("peak_note", peak_src)),
                    "avg_launch_ms": round(k["ms_per_step"] / max(1, k["launches_per_step"]), 4),
                    "share_of_step": round(k["ms_per_step"] / (ms_profiled / args.steps), 4),
                    "timing": "CUDA events around every launch of a second pass of the same K steps "
                              "(%.3f ms/step with the events in; the headline pass has none)" % (ms_profiled / args.steps)}
        I = cfg.bss_iterations
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "BASELINE configs[1]: LibriCSS-shaped 7-ch, 3 spk + noise, WPE on "
                                   "(taps 10, delay 2, 3 iters), 15 s context, 20 cACGMM iters, 512/128 STFT",
                       "name": args.workload, "segments_per_gpu": nseg, "window_s": wl.assembled_seconds / nseg,
                       "output_s_per_segment": wl.output_seconds / nseg,
                       "l2": "working set per step (2 x %.2f GB spectrograms) exceeds the 126 MB L2; no flush needed"
                             % (sum(8.0 * (cfg.stft.fft_size // 2 + 1) * s.activity.grid.shape[0]
                                    * s.audio.channels.shape[0] for s in wl.segments) / 1e9)},
            "xrt_processed": round(asm_s * args.steps / (ms_max * 1e-3), 2),
            "segments_per_s": round(nseg * world * args.steps / (ms_max * 1e-3), 2),
            "em_iters_per_s": round(nseg * world * I * args.steps / max(1e-9, kms["em_pass"][0] + kms["em_update"][0])
                                    * 1e3, 1),
            "e2e": {"value": round(out_s * args.steps / (e2e_ms_max * 1e-3), 2), "unit": UNIT,
                    "ms_per_step": round(e2e_ms_max / args.steps, 3),
                    "h2d_bytes_per_step": rb.m.h2d_bytes, "d2h_bytes_per_step": rb.m.d2h_bytes},
            "gpu_launches": int(launches),
            "stage_ms": {k: round(v, 3) for k, v in stage.items()},
            "roofline": roof, "kernels": kernels, "fp32_peak_tflops": round(fp32_peak, 2),
            "clocks": sampler.summary(), "failures": failures,
        }
    return line, wl


def oracle_enhance(orc, ss, cfg):
    return orc.enhance(ss.audio.channels, ss.activity.grid, ss.activity.target_index, ss.activity.noise_index,
                       [(p.sample_begin, p.sample_end) for p in ss.parts], fft_size=cfg.stft.fft_size,
                       shift=cfg.stft.shift, window=cfg.stft.window, sample_rate=cfg.stft.sample_rate,
                       enable_wpe=cfg.enable_wpe, taps=cfg.wpe.taps, delay=cfg.wpe.delay,
                       wpe_iterations=cfg.wpe.iterations, psd_context=cfg.wpe.psd_context,
                       regularization=cfg.wpe.regularization, bss_iterations=cfg.bss_iterations)


def load_oracle():
    """The CPU oracle port of the reference path, rebuilt for this host's ISA when possible."""
    from oracle import oracle as orc
    try:
        path = orc.build(march="native", out_dir=os.path.join(ROOT, "oracle", "_build", "native"))
        orc.load(path)
    except Exception:
        orc.load()
    return orc


def cpu_baseline(wl, n_sample=8):
    """Reference CPU path (oracle port; the reference itself needs Eigen and cannot be built) on a bounded
    sample of the same workload, all host threads (parallel_for over F, parallel.hpp:14-51)."""
    orc = load_oracle()
    cfg = wl.cfg
    segs = wl.segments[:n_sample]
    t0 = time.perf_counter()
    for ss in segs:
        oracle_enhance(orc, ss, cfg)
    dt = time.perf_counter() - t0
    sr = cfg.stft.sample_rate
    out_s = sum((p.sample_end - p.sample_begin) / sr for s in segs for p in s.parts)
    return {"value": round(out_s / dt, 4), "unit": UNIT, "cores": orc.hardware_threads(), "kind": "port",
            "sample": "%d of the %d segments of one batch (%.1f s window each), %.1f s of CPU time"
                      % (len(segs), len(wl.segments), wl.assembled_seconds / len(wl.segments), dt),
            "seconds": round(dt, 2)}


def run_reference(args, rank, world):
    if rank != 0:
        return None
    import synthbench as synth
    wl = synth.workload(args.workload, n_segments=1)
    orc = load_oracle()
    cfg = wl.cfg
    for _ in range(args.warmup):
        oracle_enhance(orc, wl.segments[0], cfg)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle_enhance(orc, wl.segments[0], cfg)
    dt = time.perf_counter() - t0
    value = wl.output_seconds * args.steps / dt
    return {"impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt / args.steps * 1e3, 2),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32/f64 mixed (reference)",
            "data": "synthetic",
            "config": {"workload": "BASELINE configs[1]: LibriCSS-shaped 7-ch, 3 spk + noise, WPE on "
                                   "(taps 10, delay 2, 3 iters), 15 s context, 20 cACGMM iters, 512/128 STFT",
                       "name": args.workload, "segments_per_step": 1,
                       "note": "each step enhances ONE segment of the batch on the host cores (bounded sample); "
                               "xRT is per-segment work, so it compares directly with the GPU arm's value"},
            "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": orc.hardware_threads(), "kind": "port",
                             "sample": "1 segment (%.0f s window) per step" % wl.assembled_seconds},
            "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg2")
    ap.add_argument("--segments", type=int, default=16, help="segments per GPU per step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    if args.impl == "reference":
        line = run_reference(args, rank, world)
        if line is not None:
            print(json.dumps(line), flush=True)
        return
    args.warmup = max(args.warmup, 3)
    line, wl = run_ours(args, rank, world, local_rank)
    if rank == 0:
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(wl)
        else:
            line["cpu_baseline"] = None
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
