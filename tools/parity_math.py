#!/usr/bin/env python
"""How much of the device-vs-oracle mask difference is fast math, and how much is summation order?

    python tools/parity_math.py cfg1 cfg2                       # the loaded library (GSS_B200_LIB selects a variant)
    python tools/parity_math.py --oracle-orders cfg1 cfg2       # CPU only: two builds of the ORACLE against each other

For one segment of each workload prints max / 99.9th percentile / relative-Frobenius mask difference, the filter
difference and the waveform SDR against the scalar-Gram oracle. Run once with the product library and once with
the accurate-math variant (tools/variant.py accurate -DGSS_ACCURATE_MATH=1: IEEE reciprocal / square root,
log2f / exp2f, double soft-max sum). `--oracle-orders` compares the oracle with its own SIMD-Gram build
(-DGSS_ORACLE_VECTOR_GRAM: same arithmetic, another float summation order inside a 2048-row chunk), i.e. what two
FP32 CPU implementations of the same algorithm differ by. Test infrastructure, not product code."""
import os
import sys
import tempfile

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as orc  # noqa: E402
import synthbench as synth  # noqa: E402


def oracle_run(ss, cfg):
    return orc.enhance(ss.audio.channels, ss.activity.grid, ss.activity.target_index, ss.activity.noise_index,
                       [(p.sample_begin, p.sample_end) for p in ss.parts], fft_size=cfg.stft.fft_size,
                       shift=cfg.stft.shift, enable_wpe=cfg.enable_wpe, taps=cfg.wpe.taps, delay=cfg.wpe.delay,
                       wpe_iterations=cfg.wpe.iterations, bss_iterations=cfg.bss_iterations, diag=True)


def report(tag, name, gamma, h, mono, want):
    dg = np.abs(gamma - want.gamma)
    err = np.sum((mono.astype(np.float64) - want.mono) ** 2)
    sdr = 10 * np.log10(np.sum(want.mono.astype(np.float64) ** 2) / max(err, 1e-300))
    per_bin = dg.reshape(dg.shape[0], -1).max(axis=1)
    print(f"[{tag}] {name}: max|dgamma|={dg.max():.2e} p99.9={np.percentile(dg, 99.9):.2e} "
          f"p99.99={np.percentile(dg, 99.99):.2e} rel(gamma)={np.linalg.norm(gamma - want.gamma) / np.linalg.norm(want.gamma):.2e} "
          f"rel(h)={np.linalg.norm(h - want.h) / np.linalg.norm(want.h):.2e} SDR={sdr:.1f} dB "
          f"bins with max|dgamma| > 1e-2: {int((per_bin > 1e-2).sum())}/{len(per_bin)}", flush=True)


def main():
    args = sys.argv[1:]
    orders = "--oracle-orders" in args
    names = [a for a in args if not a.startswith("--")] or ["cfg1"]
    for name in names:
        w = synth.workload(name, n_segments=1)
        ss, cfg = w.segments[0], w.cfg
        orc.load(orc._LIB_PATH)
        want = oracle_run(ss, cfg)
        if orders:
            orc.load(orc.build(out_dir=os.path.join(tempfile.gettempdir(), "gss_oracle_vec"), vector_gram=True))
            other = oracle_run(ss, cfg)
            orc.load(orc._LIB_PATH)
            report("oracle, SIMD-Gram build vs scalar-Gram build", name, other.gamma, other.h, other.mono, want)
            continue
        from paper_2212_05271_b200 import capi, gss
        r = gss.scheduler.enhance_batch(ss, cfg, diagnostics=True)
        assert r.ref_channel == want.ref_channel
        report(os.path.basename(capi.LIB_PATH), name, r.posteriors, r.h, r.mono, want)


if __name__ == "__main__":
    main()
