"""GPU parity of every stage operator against the CPU oracle, through the C ABI of libgss_b200.so.

Tolerances (BASELINE.json north_star): masks and beamformer weights within 1e-3 in FP32, waveform SDR
>= 40 dB, integer results exact. Each test names the reference test it mirrors where one exists.
"""
import numpy as np
import pytest

from .gpu_util import cgauss_tensor, random_activity, rel_fro, sdr_db

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gss():
    from paper_2212_05271_b200 import gss as g
    g.default_context()  # fails loudly when there is no B200 / library
    return g


def spec(gss, data, cfg=None, num_samples=0):
    return gss.stft.SpectrogramTensor(np.ascontiguousarray(data, np.complex64), cfg or gss.stft.StftConfig(),
                                      0, num_samples)


# --------------------------------------------------------------------------- STFT
@pytest.mark.parametrize("fft,shift,m,n", [(512, 128, 3, 5000), (1024, 256, 7, 4097), (512, 128, 8, 512),
                                           (256, 64, 1, 3000), (512, 256, 2, 16000)])
def test_stft_matches_oracle(gss, oracle, fft, shift, m, n):
    rng = np.random.RandomState(fft + m + n)
    audio = (rng.randn(m, n) * 0.1).astype(np.float32)
    cfg = gss.stft.StftConfig(fft, shift, 0, 16000)
    got = gss.stft.analyze(gss.stft.RealSignal(audio, 16000), cfg)
    want = oracle.stft(audio, oracle.stft_cfg(fft, shift, 0, 16000))
    assert got.data.shape == want.shape
    assert got.origin_samples == -fft // 2 and got.num_samples == n  # test_stft.cpp:90-99
    err = np.abs(got.data - want).max() / np.abs(want).max()
    assert err < 2e-6, err


def test_stft_dc_bin_and_sqrt_hann(gss, oracle):
    # test_stft.cpp:120-131: DC bin of an all-ones signal = sum(window) = fft/2
    cfg = gss.stft.StftConfig()
    got = gss.stft.analyze(gss.stft.RealSignal(np.ones((1, 8192), np.float32), 16000), cfg)
    assert abs(got.data[0, 4, 0] - 512.0) < 1e-2
    cfg2 = gss.stft.StftConfig(512, 128, 1, 16000)
    rng = np.random.RandomState(5)
    audio = rng.randn(2, 4000).astype(np.float32)
    got = gss.stft.analyze(gss.stft.RealSignal(audio, 0), cfg2)
    want = oracle.stft(audio, oracle.stft_cfg(512, 128, 1, 16000))
    assert np.abs(got.data - want).max() / np.abs(want).max() < 2e-6


def test_stft_errors(gss):
    # test_stft.cpp:101-118
    a = np.zeros((2, 100), np.float32)
    with pytest.raises(gss.InputTooShortError):
        gss.stft.analyze(gss.stft.RealSignal(a, 16000), gss.stft.StftConfig())
    with pytest.raises(gss.ConfigError):
        gss.stft.analyze(gss.stft.RealSignal(np.zeros((1, 4096), np.float32), 8000), gss.stft.StftConfig())
    with pytest.raises(gss.ConfigError):
        gss.stft.analyze(gss.stft.RealSignal(np.zeros((1, 4096), np.float32), 16000),
                         gss.stft.StftConfig(1024, 300))


@pytest.mark.parametrize("n,fft,shift,window", [(4096, 1024, 256, 0), (50000, 1024, 256, 0), (4097, 1024, 256, 0),
                                                (1024, 1024, 256, 0), (8000, 512, 128, 1), (6000, 512, 128, 0)])
def test_istft_round_trip_and_oracle(gss, oracle, n, fft, shift, window):
    # test_stft.cpp:149-172 (round trip <= 1e-6) and parity with the oracle's synthesize
    rng = np.random.RandomState(n)
    audio = (rng.randn(2, n) * 0.3).astype(np.float32)
    cfg = gss.stft.StftConfig(fft, shift, window, 16000)
    sp = gss.stft.analyze(gss.stft.RealSignal(audio, 16000), cfg)
    back = gss.stft.synthesize(sp)
    assert back.channels.shape == audio.shape
    assert np.abs(back.channels - audio).max() < 2e-6
    want = oracle.istft(sp.data, oracle.stft_cfg(fft, shift, window, 16000), n)
    assert np.abs(back.channels - want).max() < 2e-6
    # num_samples == 0: length (T-1)*shift
    sp0 = gss.stft.SpectrogramTensor(sp.data, cfg, 0, 0)
    b0 = gss.stft.synthesize(sp0)
    w0 = oracle.istft(sp.data, oracle.stft_cfg(fft, shift, window, 16000), 0)
    assert b0.channels.shape == w0.shape
    assert np.abs(b0.channels - w0).max() < 2e-6


def test_istft_random_spectrum_matches_oracle(gss, oracle):
    # arbitrary (non-STFT-consistent) spectra, incl. imaginary DC/Nyquist parts that the real inverse ignores
    x = cgauss_tensor(3, 257, 37, 2)
    cfg = gss.stft.StftConfig(512, 128, 0, 16000)
    got = gss.stft.synthesize(gss.stft.SpectrogramTensor(x, cfg, 0, 4000)).channels
    want = oracle.istft(x, oracle.stft_cfg(512, 128), 4000)
    assert np.abs(got - want).max() / np.abs(want).max() < 2e-6


# --------------------------------------------------------------------------- WPE
def test_unit_normalize(gss, oracle):
    # test_wpe.cpp:163-182
    y = cgauss_tensor(1, 9, 50, 5)
    y[2, 3, :] = 0
    got = gss.wpe.unit_normalize(spec(gss, y)).data
    want = oracle.unit_normalize(y)
    assert np.abs(got - want).max() < 1e-6
    assert np.all(got[2, 3] == 0)
    nz = np.linalg.norm(got, axis=2)
    nz[2, 3] = 1
    assert np.abs(nz - 1).max() < 1e-5


def test_wpe_pass_through_and_config(gss):
    # test_wpe.cpp:58-76
    y = cgauss_tensor(2, 4, 12, 3)
    out = gss.wpe.dereverberate(spec(gss, y), gss.wpe.WpeConfig(10, 2, 3)).data
    assert out.tobytes() == y.tobytes()
    with pytest.raises(gss.ConfigError):
        gss.wpe.dereverberate(spec(gss, y), gss.wpe.WpeConfig(0, 2, 3))


@pytest.mark.parametrize("f,t,m,taps,delay,iters,ctx", [(6, 600, 4, 8, 2, 3, 0), (5, 700, 7, 10, 2, 3, 0),
                                                        (4, 640, 8, 10, 3, 2, 0), (5, 300, 2, 5, 1, 3, 2),
                                                        (3, 1300, 3, 10, 2, 1, 0), (3, 200, 1, 4, 2, 2, 0),
                                                        (3, 400, 5, 6, 2, 2, 0), (3, 400, 6, 7, 2, 2, 1)])
def test_wpe_matches_oracle(gss, oracle, f, t, m, taps, delay, iters, ctx):
    # white input (test_wpe.cpp:101-110 shape) plus a synthetic echo (test_wpe.cpp:112-146)
    rng = np.random.RandomState(f * t + m)
    s = (rng.randn(f, t, m) + 1j * rng.randn(f, t, m)).astype(np.complex64)
    y = s.copy()
    y[:, 3:, :] += 0.7 * s[:, :-3, :]
    y[:, 5:, :] += 0.4 * np.roll(s, 1, axis=2)[:, :-5, :]
    cfg = gss.wpe.WpeConfig(taps, delay, iters, ctx, 1e-10)
    got = gss.wpe.dereverberate(spec(gss, y), cfg).data
    want = oracle.wpe(y, oracle.wpe_cfg(taps, delay, iters, ctx, 1e-10))
    err = rel_fro(got, want)
    assert err < 1e-4, err
    # determinism (test_wpe.cpp:88-95)
    again = gss.wpe.dereverberate(spec(gss, y), cfg).data
    assert again.tobytes() == got.tobytes()


@pytest.mark.parametrize("m,taps,delay", [(3, 10, 120), (7, 10, 119), (4, 4, 130), (8, 3, 126)])
def test_wpe_long_prediction_delay(gss, oracle, m, taps, delay):
    # history H = delay + taps - 1 around the 128 slab rows the tensor-core prediction can stage beside a tile:
    # H <= 128 stays on tcgen05, H > 128 must take the FP32 kernel (it once read unstaged shared memory)
    rng = np.random.RandomState(m * 1000 + delay)
    f, t = 3, 900
    s = (rng.randn(f, t, m) + 1j * rng.randn(f, t, m)).astype(np.complex64)
    y = s.copy()
    y[:, delay:, :] += 0.6 * s[:, :-delay, :]
    y[:, delay + 2:, :] += 0.3 * np.roll(s, 1, axis=2)[:, :-(delay + 2), :]
    cfg = gss.wpe.WpeConfig(taps, delay, 2, 0, 1e-10)
    got = gss.wpe.dereverberate(spec(gss, y), cfg).data
    want = oracle.wpe(y, oracle.wpe_cfg(taps, delay, 2, 0, 1e-10))
    assert rel_fro(got, want) < 1e-4, rel_fro(got, want)
    # the echo is predictable from the delayed taps: the output must be closer to the dry signal than the input
    assert np.linalg.norm(got - s) < 0.8 * np.linalg.norm(y - s)  # the oracle itself: 0.62 - 0.73


def test_wpe_eigen_floor_fallback(gss, oracle):
    # numerics.hpp:58-73, 90-93 through the WPE solve: a silent channel and regularization 0 make R exactly
    # singular, the Cholesky pivot is 0, and the solve must fall back to the eigenvalue floor like the oracle
    rng = np.random.RandomState(12)
    f, t, m, taps = 3, 400, 3, 4
    s = (rng.randn(f, t, m) + 1j * rng.randn(f, t, m)).astype(np.complex64)
    y = s.copy()
    y[:, 2:, :] += 0.5 * s[:, :-2, :]
    y[:, :, 1] = 0
    cfg = gss.wpe.WpeConfig(taps, 2, 2, 0, 0.0)
    got = gss.wpe.dereverberate(spec(gss, y), cfg).data
    want = oracle.wpe(y, oracle.wpe_cfg(taps, 2, 2, 0, 0.0))
    assert np.isfinite(got).all()
    assert np.all(got[:, :, 1] == 0)
    assert rel_fro(got, want) < 1e-4, rel_fro(got, want)


def test_wpe_tensor_core_kernels_match_the_fp32_kernels_at_full_width(gss):
    # 257 bins x 40 frame tiles keep several blocks per SM busy at once: the tcgen05 Gram and prediction must
    # agree with the FP32-FMA kernels they replace (a race between a block's workers shows up here, not on the
    # small shapes above)
    import os
    rng = np.random.RandomState(3)
    f, t, m = 257, 5001, 7
    s = (rng.randn(f, t, m) + 1j * rng.randn(f, t, m)).astype(np.complex64)
    y = s.copy()
    y[:, 3:, :] += 0.5 * s[:, :-3, :]
    cfg = gss.wpe.WpeConfig(10, 2, 2, 0, 1e-10)
    got = gss.wpe.dereverberate(spec(gss, y), cfg).data
    old = {k: os.environ.get(k) for k in ("GSS_B200_WPE_APPLY", "GSS_B200_WPE_GRAM")}
    os.environ["GSS_B200_WPE_APPLY"] = os.environ["GSS_B200_WPE_GRAM"] = "fp32"
    try:
        ctx = gss.Context(0)  # the switches are read when a context is created
        want = gss.wpe.dereverberate(spec(gss, y), cfg, ctx).data
        ctx.close()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    assert rel_fro(got, want) < 1e-5, rel_fro(got, want)
    assert np.abs(got - want).max() < 1e-3 * np.abs(want).max()


@pytest.mark.gpu
@pytest.mark.parametrize("m", [8, 5])
def test_wpe_tensor_core_prediction_over_a_wide_dynamic_range(gss, m):
    # The FP16-kind prediction scales a 140-frame tile by one power of two. Quiet frames far below the loudest frame of
    # their tile keep fewer bits (FP32-level down to -100 dB, 2^-17 at -140 dB), so the check is
    # per frame, relative to that frame: the tensor-core kernels against the FP32-FMA kernels on the same input.
    import os
    rng = np.random.RandomState(40 + m)
    f, t = 5, 900
    s = (rng.randn(f, t, m) + 1j * rng.randn(f, t, m)).astype(np.complex64)
    y = s.copy()
    y[:, 3:, :] += 0.5 * s[:, :-3, :]
    env = np.ones(t, np.float32)
    env[100:130] = 1e3      # a burst ...
    env[130:400] = 1e-4     # ... followed by 140 dB less, first inside the burst's tile, then in tiles of its own
    env[500:540] = 0.0      # digital silence
    env[600:] *= np.exp(2 * rng.randn(t - 600)).astype(np.float32)
    y *= env[None, :, None]
    y[0] *= 1e-5
    y[4] *= 1e4
    cfg = gss.wpe.WpeConfig(10, 2, 1, 0, 1e-10)  # one iteration, FP32 Gram in both runs: the filters are the same bits
    old = {k: os.environ.get(k) for k in ("GSS_B200_WPE_APPLY", "GSS_B200_WPE_GRAM")}
    res = {}
    try:
        for kind in ("tc", "fp32"):
            os.environ["GSS_B200_WPE_GRAM"] = "fp32"
            os.environ["GSS_B200_WPE_APPLY"] = kind
            ctx = gss.Context(0)  # the switches are read when a context is created
            res[kind] = gss.wpe.dereverberate(spec(gss, y), cfg, ctx).data
            ctx.close()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    got, want = res["tc"], res["fp32"]
    assert np.isfinite(got).all()
    # Y_t = obs_t - sum over the window: where a quiet frame follows a burst the difference cancels, and any FP32
    # evaluation is only good relative to the window's largest frame. That is the scale an error is measured on.
    h = cfg.delay + cfg.taps - 1
    fn = np.sqrt((np.abs(y) ** 2).sum(2))                       # (f, t) frame norms of the input
    pad = np.concatenate([np.zeros((f, h), fn.dtype), fn], 1)
    scale = np.max(np.stack([pad[:, u: u + t] for u in range(h + 1)]), 0)  # largest of frames t-h .. t
    num = np.sqrt((np.abs(got - want) ** 2).sum(2))
    live = scale > 0
    assert np.array_equal(got[~live], want[~live])              # silent stretches stay exactly silent
    worst = (num[live] / scale[live]).max()
    print(f"[prediction dynamic range M={m}] worst per-frame difference relative to its window {worst:.2e}, "
          f"overall {rel_fro(got, want):.2e}")
    assert worst < 2e-5, worst  # measured 2.2e-6 (M = 8), 9.6e-7 (M = 5)
    assert rel_fro(got, want) < 1e-5


def _gram_float64(y, taps, delay, floor=1e-10):
    """R = sum_t w_t a_t a_t^H and P = sum_t w_t a_t y_t^H in float64, weights as the device forms them (wpe.hpp:40-89)."""
    f, t, m = y.shape
    km, h = taps * m, delay + taps - 1
    R = np.zeros((f, km, km), np.complex128)
    P = np.zeros((f, km, m), np.complex128)
    for ff in range(f):
        yf = y[ff].astype(np.complex128)
        pw = (np.abs(y[ff]) ** 2).astype(np.float32).sum(1)
        lam = np.maximum(np.float32(floor), (pw.astype(np.float64) / m).astype(np.float32))
        w = (np.float32(1.0) / lam).astype(np.float64)
        pad = np.vstack([np.zeros((h, m), np.complex128), yf])
        A = np.stack([pad[tt: tt + taps].reshape(-1) for tt in range(t)])
        R[ff] = (A.T * w) @ A.conj()
        P[ff] = (A.T * w) @ yf.conj()
    return R, P


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["f16", "tf32"])
@pytest.mark.parametrize("m, t", [(8, 700), (4, 333), (5, 1000), (1, 300), (2, 350), (3, 400), (6, 500), (7, 450)])
def test_wpe_tensor_core_gram_over_a_wide_dynamic_range(gss, kind, m, t):
    # The FP16 kind scales every 128-frame stage by a power of two; loud bursts next to near-silence, exact zeros
    # and very small / very large overall levels are where a fixed-range format would lose the Gram. Both kinds must
    # stay at FP32-sum accuracy against a float64 evaluation.
    import ctypes as C
    import os
    from paper_2212_05271_b200 import capi
    rng = np.random.RandomState(m * 1000 + t)
    f, taps, delay = 3, 10, 2
    y = (rng.randn(f, t, m) + 1j * rng.randn(f, t, m)).astype(np.complex64)
    y[:, 3:] += 0.6 * y[:, :-3]
    env = np.ones(t, np.float32)
    env[40:60] = 1e3        # a burst
    env[60:200] = 1e-4      # near-silence right after it (its history holds the burst)
    env[260:300] = 0.0      # digital silence: the power floor is the weight
    env[300:] *= np.exp(rng.randn(t - 300)).astype(np.float32)
    y *= env[None, :, None]
    y[0] *= 1e-6            # overall level per bin
    y[2] *= 1e4
    old = os.environ.get("GSS_B200_WPE_GRAM_KIND")
    os.environ["GSS_B200_WPE_GRAM_KIND"] = kind
    os.environ["GSS_B200_WPE_GRAM"] = "tc"
    try:
        ctx = gss.Context(0)  # the switches are read when a context is created
        cfg = capi.WpeConfig(taps, delay, 1, 0, 1e-10)
        km = taps * m
        out = np.zeros((f, km * km + km * m), np.complex128)
        ctx.check(ctx.lib.gss_b200_debug_wpe_gram(ctx.handle, capi.ptr(y), C.c_int32(f), C.c_int64(t), C.c_int32(m),
                                                  C.byref(cfg), capi.ptr(out)))
        ctx.close()
    finally:
        os.environ.pop("GSS_B200_WPE_GRAM", None)
        if old is None:
            os.environ.pop("GSS_B200_WPE_GRAM_KIND", None)
        else:
            os.environ["GSS_B200_WPE_GRAM_KIND"] = old
    R = out[:, : km * km].reshape(f, km, km)
    P = out[:, km * km:].reshape(f, km, m)
    Rr, Pr = _gram_float64(y, taps, delay)
    for ff in range(f):
        # the regularisation the solve adds is not part of the dumped Gram; compare bin by bin (levels differ by 1e10)
        assert rel_fro(R[ff], Rr[ff]) < 3e-6, (kind, ff, rel_fro(R[ff], Rr[ff]))
        assert rel_fro(P[ff], Pr[ff]) < 3e-6, (kind, ff, rel_fro(P[ff], Pr[ff]))
        # entry-wise against the diagonal scale: no row or column loses its small entries
        d = np.sqrt(np.abs(np.diag(Rr[ff])).clip(1e-300))
        assert (np.abs(R[ff] - Rr[ff]) / np.outer(d, d)).max() < 1e-5, (kind, ff)


def test_wpe_eigen_floor_fallback_many_bins_at_once(gss, oracle):
    # every one of 48 bins (more than the 32 scratch slots of a launch) needs the fallback with a 40 x 40
    # system: the blocks queue for slots instead of failing, and the block-parallel Jacobi keeps it quick
    import time
    rng = np.random.RandomState(13)
    f, t, m, taps = 48, 300, 4, 10
    s = (rng.randn(f, t, m) + 1j * rng.randn(f, t, m)).astype(np.complex64)
    y = s.copy()
    y[:, 3:, :] += 0.4 * s[:, :-3, :]
    y[:, :, 2] = 0
    cfg = gss.wpe.WpeConfig(taps, 2, 1, 0, 0.0)
    gss.wpe.dereverberate(spec(gss, y), cfg)  # warm-up (allocations, module load)
    t0 = time.perf_counter()
    got = gss.wpe.dereverberate(spec(gss, y), cfg).data
    dt = time.perf_counter() - t0
    want = oracle.wpe(y, oracle.wpe_cfg(taps, 2, 1, 0, 0.0))
    assert np.isfinite(got).all() and np.all(got[:, :, 2] == 0)
    assert rel_fro(got, want) < 1e-4, rel_fro(got, want)
    assert dt < 0.5, dt  # one thread per bin took about 60 ms per 40 x 40 bin


# --------------------------------------------------------------------------- cACGMM
def _em_problem(seed, f, t, m, k, noise=True):
    rng = np.random.RandomState(seed)
    act = random_activity(seed, t, k, noise)
    # class-dependent spatial structure so the fit is not degenerate
    steer = (rng.randn(k, m) + 1j * rng.randn(k, m))
    y = np.zeros((f, t, m), np.complex64)
    for ff in range(f):
        lab = np.array([rng.choice(np.flatnonzero(act[tt])) for tt in range(t)])
        sig = (rng.randn(t) + 1j * rng.randn(t))[:, None] * steer[lab]
        y[ff] = (sig + 0.3 * (rng.randn(t, m) + 1j * rng.randn(t, m))).astype(np.complex64)
    return y, act


@pytest.mark.parametrize("m,k,noise", [(4, 3, True), (7, 3, True), (7, 4, True), (8, 5, True), (2, 2, True),
                                       (3, 2, False), (5, 4, True), (6, 6, True), (8, 7, True), (1, 2, True),
                                       (7, 8, True), (5, 6, False),
                                       # every class tier of the row-owner sweep (cacgmm_pass3.cuh: M = 7, 8)
                                       (7, 2, True), (7, 5, True), (7, 6, False), (8, 2, True), (8, 3, True), (8, 4, False),
                                       (8, 6, True), (8, 8, True)])
def test_em_fit_matches_oracle(gss, oracle, m, k, noise):
    f, t, iters = 6, 520, 8
    y, act = _em_problem(100 * m + k, f, t, m, k, noise)
    yn = oracle.unit_normalize(y)
    am = gss.manifests.ActivityMatrix(act, ["c%d" % i for i in range(k)], 0, k - 1 if noise else -1)
    got = gss.cacgmm.em_fit(spec(gss, yn), am, iters)
    want = oracle.em_fit(yn, act, 0, k - 1 if noise else -1, iters)
    assert len(got.likelihood_trace) == iters + 1
    # inactive posteriors exactly zero, rows sum to one (test_cacgmm.cpp:224-278)
    assert np.all(got.posteriors[:, act == 0] == 0)
    assert np.abs(got.posteriors.sum(2) - 1).max() < 1e-5
    d_gamma = np.abs(got.posteriors - want.gamma).max()
    assert d_gamma < 1e-3, d_gamma
    assert np.abs(got.state.weights - want.pi).max() < 1e-4
    for ff in range(f):
        for kk in range(k):
            e = rel_fro(got.state.shapes[ff, kk], want.shapes[ff, kk])
            assert e < 1e-3, (ff, kk, e)
    tr = np.abs(np.array(got.likelihood_trace) - want.trace) / np.abs(want.trace)
    assert tr.max() < 1e-5, tr
    # log_likelihood(state) == last trace entry (test_cacgmm.cpp:280-301)
    ll = gss.cacgmm.log_likelihood(spec(gss, yn), got.state, am)
    assert abs(ll - got.likelihood_trace[-1]) / abs(ll) < 1e-6


def test_em_first_iteration_closed_form(gss):
    # test_cacgmm.cpp:165-182: with B = I and unit-norm frames, LL_0 = F*T*c0(M) when all classes are active
    import math
    f, t, m, k = 5, 300, 4, 3
    y = cgauss_tensor(9, f, t, m)
    y /= np.linalg.norm(y, axis=2, keepdims=True)
    act = np.ones((t, k), np.uint8)
    am = gss.manifests.ActivityMatrix(act, ["a", "b", "c"], 0, -1)
    res = gss.cacgmm.em_fit(spec(gss, y), am, 1)
    c0 = -m * math.log(2 * math.pi) + math.lgamma(m)
    assert abs(c0 - (-5.559748796409327)) < 1e-12
    assert abs(res.likelihood_trace[0] - f * t * c0) / abs(f * t * c0) < 1e-6


def test_em_dead_class_and_errors(gss, oracle):
    # test_cacgmm.cpp:303-335: a class that is never active keeps B = I and pi = 1e-10
    f, t, m, k = 3, 200, 3, 3
    y = cgauss_tensor(4, f, t, m)
    yn = oracle.unit_normalize(y)
    act = np.ones((t, k), np.uint8)
    act[:, 1] = 0
    am = gss.manifests.ActivityMatrix(act, ["a", "b", "n"], 0, 2)
    res = gss.cacgmm.em_fit(spec(gss, yn), am, 3)
    assert np.all(res.posteriors[:, :, 1] == 0)
    assert np.allclose(res.state.weights[:, 1], 1e-10)
    assert np.abs(res.state.shapes[:, 1] - np.eye(m)).max() < 1e-12
    with pytest.raises(gss.ConfigError):
        gss.cacgmm.em_fit(spec(gss, yn), am, 0)
    bad = gss.manifests.ActivityMatrix(act[:-1], ["a", "b", "n"], 0, 2)
    with pytest.raises(gss.ShapeError):
        gss.cacgmm.em_fit(spec(gss, yn), bad, 2)


@pytest.mark.parametrize("m", [2, 4, 7, 8])
def test_em_shape_matrices_cholesky_rejects_take_the_eigenvalue_floor(gss, oracle, m):
    # cacgmm.hpp:134-140 / numerics.hpp:103-122: an indefinite or rank-deficient shape matrix is inverted through
    # the eigenvalue floor (1e-10 * lambda_max). On the device that is a warp-parallel Jacobi; it must agree with
    # the oracle's fallback through the likelihood and the posteriors' normaliser.
    f, t, k = 9, 300, 3
    y, act = _em_problem(31 + m, f, t, m, k, True)
    yn = oracle.unit_normalize(y)
    rng = np.random.RandomState(m)
    shapes = np.zeros((f, k, m, m), np.complex128)
    for ff in range(f):
        for kk in range(k):
            q, _ = np.linalg.qr(rng.randn(m, m) + 1j * rng.randn(m, m))
            w = rng.uniform(0.5, 2.0, m)
            kind = (ff + kk) % 3
            if kind == 0 and m > 1:
                w[rng.randint(m)] = -0.3            # indefinite
            elif kind == 1:
                w[: max(1, m // 2)] = -1e-7         # rank-deficient up to rounding (an exact zero pivot may come
                #                                     out as +-1e-17 and pass one Cholesky but not the other)
            b = (q * w) @ q.conj().T                # kind 2: positive definite (the Cholesky path, same launch)
            shapes[ff, kk] = 0.5 * (b + b.conj().T)
    pi = rng.uniform(0.2, 1.0, (f, k))
    am = gss.manifests.ActivityMatrix(act, ["c%d" % i for i in range(k)], 0, k - 1)
    got = gss.cacgmm.log_likelihood(spec(gss, yn), gss.cacgmm.CacgmmState(pi, shapes), am)
    want = oracle.log_likelihood(yn, act, pi, shapes, k - 1)
    assert np.isfinite(got) and abs(got - want) / abs(want) < 2e-5, (got, want)


def test_em_degenerate_frames_without_noise_class(gss, oracle):
    # frames with no active class: uniform over all classes (cacgmm.hpp:217-226)
    f, t, m, k = 3, 260, 4, 3
    y, _ = _em_problem(77, f, t, m, k, True)
    yn = oracle.unit_normalize(y)
    act = random_activity(5, t, k, noise=False, holes=True)
    assert (act.sum(1) == 0).any()
    am = gss.manifests.ActivityMatrix(act, ["a", "b", "c"], 0, -1)
    got = gss.cacgmm.em_fit(spec(gss, yn), am, 4)
    want = oracle.em_fit(yn, act, 0, -1, 4)
    assert np.abs(got.posteriors - want.gamma).max() < 1e-3
    assert np.abs(np.array(got.likelihood_trace) - want.trace).max() / np.abs(want.trace).max() < 1e-5


# --------------------------------------------------------------------------- beamformer
@pytest.mark.parametrize("m,k", [(2, 2), (4, 3), (7, 4), (8, 5), (3, 6), (5, 2), (6, 8), (1, 2)])
def test_mvdr_chain_matches_oracle(gss, oracle, m, k):
    f, t = 9, 333
    rng = np.random.RandomState(m * 10 + k)
    y = cgauss_tensor(m + k, f, t, m, 3.0)
    g = rng.rand(f, t, k).astype(np.float32)
    g /= g.sum(2, keepdims=True)
    target = k // 2
    st = gss.beamform.accumulate_stats(spec(gss, y), g, target)
    wt, wb = oracle.mvdr_stats(y, g, target)
    assert rel_fro(st.target, wt) < 1e-5 and rel_fro(st.background, wb) < 1e-5
    ref = gss.beamform.select_reference(st)
    assert ref == oracle.select_reference(wt, wb)
    flt = gss.beamform.mvdr(st, ref)
    wh, wz = oracle.mvdr(wt, wb, ref)
    assert flt.zeroed_bins == wz
    assert rel_fro(flt.h, wh) < 1e-4
    out = gss.beamform.apply(flt, spec(gss, y)).data
    want = oracle.apply_filter(wh, y)
    assert out.shape == (f, t, 1)
    assert rel_fro(out[:, :, 0], want) < 1e-4


def test_mvdr_frozen_vector_and_edge_cases(gss):
    # test_beamform.cpp:127-145: frozen h = [0.8+0.04i, -0.08-0.2i]
    tgt = np.array([[[2, 0.5j], [-0.5j, 1]]], np.complex128)
    bg = np.array([[[1, 0.2], [0.2, 2]]], np.complex128)
    st = gss.beamform.BeamformerStats(tgt, bg, 1)
    flt = gss.beamform.mvdr(st, 0)
    c = np.linalg.solve(bg[0], tgt[0])
    want = c[:, 0] / np.trace(c)
    assert np.abs(flt.h[0] - want).max() < 1e-9
    # ties -> lowest index (test_beamform.cpp:100-121)
    eye = np.tile(np.eye(3, dtype=np.complex128), (4, 1, 1))
    assert gss.beamform.select_reference(gss.beamform.BeamformerStats(eye, eye, 1)) == 0
    t2 = eye.copy()
    t2[:, 2, 2] = 5
    assert gss.beamform.select_reference(gss.beamform.BeamformerStats(t2, eye, 1)) == 2
    # zero target -> trace 0 -> zeroed bins counted (test_beamform.cpp:190-205)
    z = gss.beamform.mvdr(gss.beamform.BeamformerStats(np.zeros_like(eye), eye, 1), 0)
    assert z.zeroed_bins == 4 and np.all(z.h == 0)
    with pytest.raises(gss.ShapeError):
        gss.beamform.mvdr(gss.beamform.BeamformerStats(eye, eye, 1), 3)
    # all-zero target mask -> DegenerateStatsError (test_beamform.cpp:88-94)
    y = cgauss_tensor(1, 4, 50, 3)
    g = np.zeros((4, 50, 2), np.float32)
    g[:, :, 1] = 1
    with pytest.raises(gss.DegenerateStatsError):
        gss.beamform.accumulate_stats(spec(gss, y), g, 0)


def test_numerics_rank_deficient_background_uses_eigen_floor(gss, oracle):
    # test_numerics.cpp:130-138 through the MVDR solve: rank-1 background is repaired by the eigenvalue floor
    v = np.array([1, 1j, 1 + 1j])
    bg = np.outer(v, v.conj())[None].astype(np.complex128)
    tgt = np.eye(3, dtype=np.complex128)[None]
    flt = gss.beamform.mvdr(gss.beamform.BeamformerStats(tgt, bg, 1), 0)
    wh, wz = oracle.mvdr(tgt, bg, 0)
    assert np.isfinite(flt.h).all() and flt.zeroed_bins == wz
    assert rel_fro(flt.h, wh) < 1e-3
    # indefinite background: Cholesky fails, the device runs the Jacobi eigenvalue-floor fallback
    # (numerics.hpp:58-73, 90-93) and must agree with the oracle's fallback
    rng = np.random.RandomState(3)
    for m in (2, 4, 7, 8):
        q, _ = np.linalg.qr(rng.randn(m, m) + 1j * rng.randn(m, m))
        lam = np.linspace(-1.0, 3.0, m)
        bg = ((q * lam) @ q.conj().T)[None]
        bg = 0.5 * (bg + bg.conj().transpose(0, 2, 1))
        r = rng.randn(m, m) + 1j * rng.randn(m, m)
        tgt = (r @ r.conj().T)[None]
        flt = gss.beamform.mvdr(gss.beamform.BeamformerStats(tgt, bg, 1), 1 % m)
        wh, wz = oracle.mvdr(tgt, bg, 1 % m)
        assert flt.zeroed_bins == wz
        assert rel_fro(flt.h, wh) < 1e-6, (m, rel_fro(flt.h, wh))
    # no positive eigenvalue at all -> SingularMatrixError carrying the bin (test_numerics.cpp:140-148)
    bad = np.zeros((40, 3, 3), np.complex128)
    bad[:] = np.eye(3)
    bad[37] = -np.eye(3)
    with pytest.raises(gss.SingularMatrixError) as e:
        gss.beamform.mvdr(gss.beamform.BeamformerStats(bad, bad, 1), 0)
    assert e.value.frequency() == 37
