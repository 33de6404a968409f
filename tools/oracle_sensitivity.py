"""How far the CPU oracle's own masks move under FP32-level perturbations (CPU only; no GPU, no product code).

    python tools/oracle_sensitivity.py [cfg1|cfg2|cfg3]

Runs the oracle's em_fit on one segment of the workload three times: as is, with the quadratic form evaluated
in double instead of float (precise_quad), and with the input multiplied by (1 + 1e-7 N(0,1)). Bins whose
masks flip under such a perturbation are bins where 20 EM iterations are chaotic in FP32 for ANY
implementation; the device-vs-oracle parity gates (percentiles, relative Frobenius) are set with that in mind.
Test infrastructure."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as orc  # noqa: E402
import synthbench as synth  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
    w = synth.workload(name, n_segments=1)
    ss, cfg = w.segments[0], w.cfg
    ocfg = orc.stft_cfg(cfg.stft.fft_size, cfg.stft.shift, cfg.stft.window, cfg.stft.sample_rate)
    y = orc.stft(ss.audio.channels, ocfg)
    if cfg.enable_wpe:
        wc = cfg.wpe
        y = orc.wpe(y, orc.wpe_cfg(wc.taps, wc.delay, wc.iterations, wc.psd_context, wc.regularization))
    yn = orc.unit_normalize(y)
    act = ss.activity
    base = orc.em_fit(yn, act.grid, act.target_index, act.noise_index, cfg.bss_iterations)
    rng = np.random.default_rng(0)
    pert = (yn * (1.0 + 1e-7 * rng.standard_normal(yn.shape))).astype(np.complex64)
    for label, other in (("precise_quad", orc.em_fit(yn, act.grid, act.target_index, act.noise_index,
                                                     cfg.bss_iterations, precise_quad=True)),
                         ("input x (1 + 1e-7 N)", orc.em_fit(pert, act.grid, act.target_index, act.noise_index,
                                                             cfg.bss_iterations))):
        d = np.abs(other.gamma - base.gamma)
        pb = d.reshape(d.shape[0], -1).max(axis=1)
        worst = np.argsort(-pb)[:5]
        print(f"[{name}] oracle vs oracle ({label}): max={d.max():.2e} mean={d.mean():.2e} "
              f"p99.99={np.percentile(d, 99.99):.2e} rel={np.linalg.norm(other.gamma - base.gamma) / np.linalg.norm(base.gamma):.2e}; "
              f"bins with max|dgamma| > 1e-2: {int((pb > 1e-2).sum())} of {len(pb)}; worst bins "
              + ", ".join(f"({f}, {pb[f]:.1e})" for f in worst))


if __name__ == "__main__":
    main()
