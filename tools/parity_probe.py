"""Stage-by-stage parity probe against the CPU oracle (diagnostic; run on the GPU box).

    python tools/parity_probe.py [tiny|cfg1|cfg2]

For one segment of the workload prints the relative error each device stage adds when fed the ORACLE's
output of the previous stage, then the end-to-end figures. Test infrastructure, not product code."""
import sys
import os
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as orc  # noqa: E402
from paper_2212_05271_b200 import gss  # noqa: E402
import synthbench as synth  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-30))


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "tiny"
    if name.startswith("custom:"):  # custom:<channels>,<speakers>,<iterations>[,<target seconds>,<context seconds>]
        from paper_2212_05271_b200.gss import scheduler, stft as st_, wpe as wp_
        v = [float(x) for x in name.split(":")[1].split(",")]
        cfg = scheduler.PipelineConfig(st_.StftConfig(512, 128, 0, 16000), wp_.WpeConfig(10, 2, 3, 0, 1e-10), True, int(v[2]))
        ss = synth.make_supersegment(5000 + 10 * int(v[0]) + int(v[1]), int(v[0]), int(v[1]),
                                     v[3] if len(v) > 3 else 2.0, v[4] if len(v) > 4 else 1.5, cfg)
    else:
        w = synth.workload(name, n_segments=1)
        ss, cfg = w.segments[0], w.cfg
    ocfg = orc.stft_cfg(cfg.stft.fft_size, cfg.stft.shift, cfg.stft.window, cfg.stft.sample_rate)
    t0 = time.time()
    y_o = orc.stft(ss.audio.channels, ocfg)
    y_g = gss.stft.analyze(ss.audio, cfg.stft).data
    print(f"[{name}] stft rel={rel(y_g, y_o):.2e}  per-bin max rel={np.max(np.linalg.norm(y_g - y_o, axis=(1, 2)) / np.linalg.norm(y_o, axis=(1, 2))):.2e}")
    d_o = y_o
    if cfg.enable_wpe:
        wc = cfg.wpe
        d_o = orc.wpe(y_o, orc.wpe_cfg(wc.taps, wc.delay, wc.iterations, wc.psd_context, wc.regularization))
        d_g = gss.wpe.dereverberate(gss.stft.SpectrogramTensor(y_o, cfg.stft), wc).data
        pb = np.linalg.norm(d_g - d_o, axis=(1, 2)) / np.linalg.norm(d_o, axis=(1, 2))
        print(f"[{name}] wpe (oracle input) rel={rel(d_g, d_o):.2e} per-bin max rel={pb.max():.2e} at f={pb.argmax()}")
    yn_o = orc.unit_normalize(d_o)
    act = ss.activity
    em_o = orc.em_fit(yn_o, act.grid, act.target_index, act.noise_index, cfg.bss_iterations)
    em_g = gss.cacgmm.em_fit(gss.stft.SpectrogramTensor(yn_o, cfg.stft), act, cfg.bss_iterations)
    dg = np.abs(em_g.posteriors - em_o.gamma)
    print(f"[{name}] em (oracle input, stage API) rel(gamma)={rel(em_g.posteriors, em_o.gamma):.2e} "
          f"p99.99={np.percentile(dg, 99.99):.2e} max={dg.max():.2e} rel(B)={rel(em_g.state.shapes, em_o.shapes):.2e}")
    for it in (1, 2, 5, 10):
        if it < cfg.bss_iterations:
            a = orc.em_fit(yn_o, act.grid, act.target_index, act.noise_index, it)
            b = gss.cacgmm.em_fit(gss.stft.SpectrogramTensor(yn_o, cfg.stft), act, it)
            d = np.abs(b.posteriors - a.gamma)
            print(f"    after {it:2d} iterations: max|dgamma|={d.max():.2e} p99.99={np.percentile(d, 99.99):.2e}")
    st_o = orc.mvdr_stats(d_o, em_o.gamma, act.target_index)
    st_g = gss.beamform.accumulate_stats(gss.stft.SpectrogramTensor(d_o, cfg.stft), em_o.gamma, act.target_index)
    print(f"[{name}] stats (oracle input) rel(target)={rel(st_g.target, st_o[0]):.2e} rel(bg)={rel(st_g.background, st_o[1]):.2e}")
    r = gss.scheduler.enhance_batch(ss, cfg, diagnostics=True)
    want = orc.enhance(ss.audio.channels, act.grid, act.target_index, act.noise_index,
                       [(p.sample_begin, p.sample_end) for p in ss.parts], fft_size=cfg.stft.fft_size,
                       shift=cfg.stft.shift, enable_wpe=cfg.enable_wpe, taps=cfg.wpe.taps, delay=cfg.wpe.delay,
                       wpe_iterations=cfg.wpe.iterations, bss_iterations=cfg.bss_iterations, diag=True)
    dg = np.abs(r.posteriors - want.gamma)
    err = np.sum((r.mono.astype(np.float64) - want.mono) ** 2)
    sdr = 10 * np.log10(np.sum(want.mono.astype(np.float64) ** 2) / max(err, 1e-300))
    print(f"[{name}] end to end: ref {r.ref_channel}/{want.ref_channel} rel(gamma)={rel(r.posteriors, want.gamma):.2e} "
          f"p99.9={np.percentile(dg, 99.9):.2e} p99.99={np.percentile(dg, 99.99):.2e} max={dg.max():.2e} "
          f"rel(h)={rel(r.h, want.h):.2e} SDR={sdr:.1f} dB rel(ll)={abs(r.ll_final - want.ll_final) / abs(want.ll_final):.2e} "
          f"({time.time() - t0:.0f} s)")
    # which bins carry the largest mask / filter differences (a diverging bin shows up here)
    pb = dg.reshape(dg.shape[0], -1).max(axis=1)
    hb = np.linalg.norm(r.h - want.h, axis=1) / np.maximum(np.linalg.norm(want.h, axis=1), 1e-30)
    worst = np.argsort(-pb)[:5]
    print("    worst bins (f, max|dgamma|, rel h): " + ", ".join(f"({f}, {pb[f]:.1e}, {hb[f]:.1e})" for f in worst)
          + f"; bins with max|dgamma| > 1e-2: {int((pb > 1e-2).sum())} of {len(pb)}")


if __name__ == "__main__":
    main()
