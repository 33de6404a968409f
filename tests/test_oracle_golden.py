"""Pins the CPU oracle against every frozen known-answer value and property the
reference's own test-suite holds for the hot path.

Each test cites the reference test it restates (paths under
/root/reference/proj/tests/). These run on CPU (`-m "not gpu"`).
"""
import math

import numpy as np
import pytest

from .refrng import Rng


def rel_err(got, want):  # test_util.hpp:35-37
    return abs(got - want) / max(1.0, abs(want))


def random_hermitian_pd(rng, m, shift):
    r = np.array([[rng.cgaussian() for _ in range(m)] for _ in range(m)])
    return r @ r.conj().T + shift * np.eye(m)


# --------------------------------------------------------------------------- numerics
def test_hermitize_and_regularize(oracle):
    # test_numerics.cpp:93-115
    rng = Rng(11)
    a = np.array([[rng.cgaussian() for _ in range(3)] for _ in range(3)])
    h = oracle.hermitize(a)
    assert np.abs(h - h.conj().T).max() < 1e-14
    assert np.abs(h - 0.5 * (a + a.conj().T)).max() < 1e-14
    with pytest.raises(oracle.OracleError) as e:
        oracle.hermitize(np.zeros((2, 3), complex))
    assert e.value.kind == "ShapeError"
    r = oracle.regularize(np.eye(2) * 4.0, 0.5)
    assert r[0, 0].real == pytest.approx(6.0) and r[1, 1].real == pytest.approx(6.0)
    rz = oracle.regularize(np.zeros((2, 2)), 0.25)
    assert rz[0, 0].real == pytest.approx(0.25)


def test_hermitian_solve_matches_lu(oracle):
    # test_numerics.cpp:117-128
    rng = Rng(21)
    for m in (1, 2, 4, 6):
        r = np.array([[rng.cgaussian() for _ in range(m)] for _ in range(m)])
        a = r @ r.conj().T + m * np.eye(m)
        b = np.array([[rng.cgaussian() for _ in range(2)] for _ in range(m)])
        x = oracle.hermitian_solve(a, b)
        want = np.linalg.solve(a, b)
        assert np.linalg.norm(x - want) / np.linalg.norm(want) < 1e-10


def test_hermitian_solve_rank_deficient_and_zero(oracle):
    # test_numerics.cpp:130-148
    v = np.array([1, 1j, 1 + 1j])
    x = oracle.hermitian_solve(np.outer(v, v.conj()), np.eye(3))
    assert np.isfinite(x).all()
    # eigen-floor semantics: eigenvalues floored at 1e-10 * lambda_max
    lam = np.linalg.eigvalsh(np.outer(v, v.conj())).max()
    assert np.abs(x).max() == pytest.approx(1.0 / (1e-10 * lam) * (2.0 / 3.0), rel=1e-3) or np.abs(x).max() > 1e8
    with pytest.raises(oracle.OracleError) as e:
        oracle.hermitian_solve(np.zeros((2, 2)), np.eye(2), 37)
    assert e.value.kind == "SingularMatrixError" and e.value.frequency == 37


def test_hermitian_eig_matches_numpy(oracle):
    rng = Rng(5)
    for m in (2, 3, 5, 8, 20):
        a = random_hermitian_pd(rng, m, 0.0)
        vals, vecs = oracle.hermitian_eig(a)
        assert np.allclose(np.sort(vals), np.linalg.eigvalsh(a), rtol=1e-10, atol=1e-10)
        assert np.abs(vecs @ np.diag(vals) @ vecs.conj().T - a).max() < 1e-9 * np.abs(a).max()


def test_inverse_logdet_frozen(oracle):
    # test_numerics.cpp:150-160
    b = np.array([[2, 1j], [-1j, 2]])
    inv, ld = oracle.hermitian_inverse_logdet(b)
    assert ld == pytest.approx(1.0986122886681096, rel=1e-12)
    want = np.array([[2 / 3, -1j / 3], [1j / 3, 2 / 3]])
    assert np.abs(inv - want).max() < 1e-12


def test_weighted_gram_frozen_and_chunking(oracle):
    # test_numerics.cpp:166-211
    rows = np.array([[1, 1j], [2, 0]], np.complex64)
    phi = oracle.weighted_gram(rows, np.array([0.5, 2.0], np.float32))
    want = np.array([[8.5, -0.5j], [0.5j, 0.5]])
    assert np.abs(phi - want).max() < 1e-6
    rng = Rng(31)
    a = rng.ctensor(777, 3)
    w = np.array([rng.uniform() for _ in range(777)], np.float32)
    ad = a.astype(np.complex128)
    naive = np.einsum("t,tm,tn->mn", w.astype(np.float64), ad, ad.conj())
    g_def = oracle.weighted_gram(a, w)
    g_small = oracle.weighted_gram(a, w, 64)
    assert np.linalg.norm(g_def - naive) / np.linalg.norm(naive) < 1e-6
    assert np.linalg.norm(g_small - g_def) / np.linalg.norm(g_def) < 1e-6
    g_unit = oracle.weighted_gram(a, None)
    naive_unit = np.einsum("tm,tn->mn", ad, ad.conj())
    assert np.linalg.norm(g_unit - naive_unit) / np.linalg.norm(naive_unit) < 1e-6


# --------------------------------------------------------------------------- stft
def test_hann_window_frozen(oracle):
    # test_stft.cpp:43-73
    want = [0.0, 0.1464466094067262, 0.5, 0.8535533905932737, 1.0, 0.8535533905932738, 0.5, 0.14644660940672632]
    w = oracle.make_window(8, 0)
    assert np.allclose(w, want, rtol=1e-12, atol=1e-15)
    ws = oracle.make_window(8, 1)
    assert np.allclose(ws, np.sqrt(want), rtol=1e-12, atol=1e-15)
    w = oracle.make_window(1024, 0)
    for n in range(256):
        assert sum(w[n + 256 * k] ** 2 for k in range(4)) == pytest.approx(1.5, rel=1e-12)


def test_frame_geometry(oracle):
    # test_stft.cpp:79-99
    assert oracle.frame_count(1024) == 5
    assert oracle.frame_count(1025) == 5
    assert oracle.frame_count(1279) == 5
    assert oracle.frame_count(1280) == 6
    rng = np.random.default_rng(101)
    s = rng.uniform(-1, 1, (3, 5000)).astype(np.float32)
    spec = oracle.stft(s, oracle.stft_cfg())
    assert spec.shape == (513, oracle.frame_count(5000), 3)


def test_stft_errors(oracle):
    # test_stft.cpp:101-118
    cfg = oracle.stft_cfg()
    with pytest.raises(oracle.OracleError) as e:
        oracle.stft(np.zeros((1, 512), np.float32), cfg)
    assert e.value.kind == "InputTooShortError"
    with pytest.raises(oracle.OracleError) as e:
        oracle.stft(np.zeros((1, 4000), np.float32), cfg, signal_rate=8000)
    assert e.value.kind == "ConfigError"
    with pytest.raises(oracle.OracleError) as e:
        oracle.stft(np.zeros((1, 4000), np.float32), oracle.stft_cfg(shift=300))
    assert e.value.kind == "ConfigError"


def test_dc_bin_of_ones(oracle):
    # test_stft.cpp:120-131
    spec = oracle.stft(np.ones((1, 2048), np.float32), oracle.stft_cfg())
    v = spec[0, 4, 0]
    assert abs(v) == pytest.approx(512.0, rel=1e-5)
    assert abs(v.imag) < 1e-4


def test_stft_matches_numpy_fft(oracle):
    # independent evaluation of stft.hpp:131-175 semantics with numpy
    rng = np.random.default_rng(7)
    x = rng.standard_normal(3000).astype(np.float32)
    cfg = oracle.stft_cfg(512, 128)
    spec = oracle.stft(x[None], cfg)
    pad = 256
    padded = np.concatenate([x[pad:0:-1], x, x[-2:-pad - 2:-1]]).astype(np.float64)
    w = 0.5 * (1 - np.cos(2 * np.pi * np.arange(512) / 512))
    for t in (0, 1, 7, spec.shape[1] - 1):
        want = np.fft.rfft(padded[t * 128: t * 128 + 512] * w)
        assert np.abs(spec[:, t, 0] - want).max() < 1e-4 * max(1, np.abs(want).max())


@pytest.mark.parametrize("seed,m,n,window", [(201, 1, 4096, 0), (202, 3, 50000, 0), (203, 2, 4097, 0),
                                             (204, 1, 1024, 0), (205, 2, 30000, 1)])
def test_round_trip(oracle, seed, m, n, window):
    # test_stft.cpp:149-162
    rng = np.random.default_rng(seed)
    s = rng.uniform(-1, 1, (m, n)).astype(np.float32)
    cfg = oracle.stft_cfg(window=window)
    back = oracle.istft(oracle.stft(s, cfg), cfg, n)
    assert back.shape == s.shape
    for c in range(m):
        err = np.linalg.norm(back[c].astype(np.float64) - s[c]) / np.linalg.norm(s[c])
        assert err < 1e-6


def test_synthesize_rejects_mismatch(oracle):
    # test_stft.cpp:174-179
    spec = oracle.stft(np.zeros((1, 4000), np.float32) + 0.1, oracle.stft_cfg())
    with pytest.raises(oracle.OracleError) as e:
        oracle.istft(spec, oracle.stft_cfg(fft_size=512, shift=128), 4000)
    assert e.value.kind == "ConfigError"


# --------------------------------------------------------------------------- wpe
def test_wpe_config_and_passthrough(oracle):
    # test_wpe.cpp:58-76
    y = Rng(5).ctensor(33, 12, 2)
    for bad in (dict(taps=0), dict(delay=0), dict(iterations=0)):
        with pytest.raises(oracle.OracleError) as e:
            oracle.wpe(y, oracle.wpe_cfg(**bad))
        assert e.value.kind == "ConfigError"
    out = oracle.wpe(y, oracle.wpe_cfg())  # T == taps+delay -> bit-identical pass-through
    assert out.tobytes() == y.tobytes()


def test_wpe_deterministic_and_white(oracle):
    # test_wpe.cpp:88-110
    y = Rng(7).ctensor(9, 120, 2)
    a = oracle.wpe(y, oracle.wpe_cfg())
    b = oracle.wpe(y, oracle.wpe_cfg())
    assert a.tobytes() == b.tobytes()
    y = Rng(8).ctensor(12, 600, 2)
    out = oracle.wpe(y, oracle.wpe_cfg(taps=8))
    l2 = np.linalg.norm(out.astype(np.complex128) - y) / np.linalg.norm(y)
    assert l2 < 0.25


def test_wpe_removes_late_echo(oracle):
    # test_wpe.cpp:112-146
    clean = Rng(9).ctensor(6, 700, 2)
    echo = clean.copy()
    echo[:, 3:, :] += np.float32(0.9) * clean[:, :-3, :]
    out = oracle.wpe(echo, oracle.wpe_cfg(taps=8, delay=2))

    def l2(a, b):
        return np.linalg.norm(a.astype(np.complex128) - b) / np.linalg.norm(b)

    before, after = l2(echo, clean), l2(out, clean)
    assert before > 0.8
    assert after < 0.5 * before
    assert np.sum(np.abs(out) ** 2) < np.sum(np.abs(echo) ** 2)


def test_wpe_psd_context_finite(oracle):
    # test_wpe.cpp:148-157
    y = Rng(10).ctensor(8, 200, 2)
    out = oracle.wpe(y, oracle.wpe_cfg(psd_context=2))
    assert np.isfinite(out.view(np.float32)).all()
    assert not np.array_equal(out, oracle.wpe(y, oracle.wpe_cfg()))


def test_wpe_matches_numpy_double(oracle):
    # independent double-precision evaluation of wpe.hpp:61-98
    rng = np.random.default_rng(3)
    F, T, M, taps, delay = 3, 150, 2, 4, 2
    s = (rng.standard_normal((F, T, M)) + 1j * rng.standard_normal((F, T, M))).astype(np.complex64)
    y = s.copy()
    y[:, 4:, :] += np.complex64(0.6) * s[:, :-4, :]
    out = oracle.wpe(y, oracle.wpe_cfg(taps=taps, delay=delay, iterations=2))
    for f in range(F):
        obs = y[f].astype(np.complex128)
        km = taps * M
        hist = np.zeros((T, km), complex)
        for t in range(T):
            for k in range(taps):
                src = t - delay - k
                if src >= 0:
                    hist[t, k * M:(k + 1) * M] = obs[src]
        cur = obs.copy()
        for _ in range(2):
            lam = np.maximum(1e-10, np.mean(np.abs(cur) ** 2, axis=1))
            w = 1.0 / lam
            R = np.einsum("t,ti,tj->ij", w, hist, hist.conj())
            P = np.einsum("t,ti,tj->ij", w, hist, obs.conj())
            R = 0.5 * (R + R.conj().T)
            R = R + 1e-10 * (np.trace(R).real / km) * np.eye(km)
            G = np.linalg.solve(R, P)
            cur = obs - hist @ G.conj()
        assert np.abs(out[f] - cur).max() < 2e-4 * np.abs(cur).max()


def test_unit_normalize(oracle):
    # test_wpe.cpp:163-182
    y = Rng(11).ctensor(5, 40, 3)
    out = oracle.unit_normalize(y)
    assert np.allclose(np.sqrt(np.sum(np.abs(out.astype(np.complex128)) ** 2, axis=2)), 1.0, atol=1e-5)
    y = np.zeros((2, 3, 2), np.complex64)
    y[1, 1, 0] = 3 + 4j
    out = oracle.unit_normalize(y)
    assert out[0, 0, 0] == 0 and out[0, 0, 1] == 0
    assert abs(out[1, 1, 0]) == pytest.approx(1.0, rel=1e-5)


# --------------------------------------------------------------------------- cacgmm
def test_cacg_log_pdf_frozen(oracle):
    # test_cacgmm.cpp:53-79
    assert oracle.cacg_log_pdf([1], np.eye(1)) == pytest.approx(-1.8378770664093453, rel=1e-12)
    assert oracle.cacg_log_pdf([1, 0], np.eye(2)) == pytest.approx(-3.6757541328186907, rel=1e-12)
    assert oracle.cacg_log_pdf([1, 0], np.diag([2, 0.5])) == pytest.approx(-2.2894597716988, rel=1e-12)
    b = np.array([[2, 0.3 + 0.4j], [0.3 - 0.4j, 1]])
    yd = np.array([0.6 + 0.2j, -0.5 + 0.1j])
    assert oracle.cacg_log_pdf(yd, b) == pytest.approx(-3.5072719119712183, rel=1e-11)


def test_cacg_log_pdf_vs_lu_and_scale(oracle):
    # test_cacgmm.cpp:81-110
    rng = Rng(17)
    for m in (1, 2, 4):
        for _ in range(100):
            r = np.array([[rng.cgaussian() for _ in range(m)] for _ in range(m)])
            b = r @ r.conj().T + 0.1 * m * np.eye(m)
            y = np.array([rng.cgaussian() for _ in range(m)])
            y = y / np.linalg.norm(y)
            q = (y.conj() @ np.linalg.inv(b) @ y).real
            want = -m * math.log(2 * math.pi) + math.lgamma(m) - math.log(abs(np.linalg.det(b))) - m * math.log(q)
            assert rel_err(oracle.cacg_log_pdf(y, b), want) < 1e-8
    rng = Rng(18)
    r = np.array([[rng.cgaussian() for _ in range(3)] for _ in range(3)])
    b = r @ r.conj().T + np.eye(3)
    y = np.array([rng.cgaussian() for _ in range(3)])
    y /= np.linalg.norm(y)
    assert oracle.cacg_log_pdf(y, b) == pytest.approx(oracle.cacg_log_pdf(y, 7.5 * b), rel=1e-9)


def test_time_varying_weights_frozen(oracle):
    # test_cacgmm.cpp:116-137
    w = oracle.time_varying_weights([0.2, 0.3, 0.5], [1, 0, 1], 2)
    assert w[0] == pytest.approx(0.28571428571428575)
    assert w[1] == 0.0
    assert w[2] == pytest.approx(0.7142857142857143)
    assert w.sum() == pytest.approx(1.0)
    n = oracle.time_varying_weights([0.2, 0.3, 0.5], [0, 0, 0], 2)
    assert list(n) == [0.0, 0.0, 1.0]
    u = oracle.time_varying_weights([0.2, 0.3, 0.5], [0, 0, 0], -1)
    assert np.allclose(u, 1 / 3)


def _all_on(frames, k):
    return np.ones((frames, k), np.uint8)


def test_first_iteration_likelihood_closed_form(oracle):
    # test_cacgmm.cpp:165-182
    rng = Rng(23)
    y = oracle.unit_normalize(rng.ctensor(4, 30, 4))
    res = oracle.em_fit(y, _all_on(30, 1), target=0, noise=0, iterations=1)
    c0 = -4 * math.log(2 * math.pi) + math.lgamma(4)
    assert c0 == pytest.approx(-5.559748796409327, rel=1e-12)
    assert res.trace[0] == pytest.approx(4 * 30 * c0, rel=1e-6)


def test_em_separates_two_classes(oracle):
    # test_cacgmm.cpp:184-222
    rng = Rng(29)
    bins, frames = 5, 120
    y = np.zeros((bins, frames, 2), np.complex64)
    for f in range(bins):
        for t in range(frames):
            first = t < frames // 2
            main, leak = rng.cgaussian(), 0.05 * rng.cgaussian()
            y[f, t, 0 if first else 1] = main
            y[f, t, 1 if first else 0] = leak
    y = oracle.unit_normalize(y)
    act = _all_on(frames, 2)
    margin = frames // 10
    act[:margin, 1] = 0
    act[frames - margin:, 0] = 0
    res = oracle.em_fit(y, act, target=0, noise=-1, iterations=15)
    want = (np.arange(margin, frames - margin) >= frames // 2).astype(int)
    got = (res.gamma[:, margin:frames - margin, 0] <= 0.5).astype(int)
    assert (got == want[None]).mean() > 0.95


def test_activity_pins_classes(oracle):
    # test_cacgmm.cpp:224-278
    rng = Rng(31)
    bins, frames = 3, 80
    y = np.zeros((bins, frames, 2), np.complex64)
    for f in range(bins):
        for t in range(frames):
            first = t < frames // 2
            y[f, t, 0 if first else 1] = rng.cgaussian()
            y[f, t, 1 if first else 0] = 0.05 * rng.cgaussian()
    y = oracle.unit_normalize(y)
    act = np.zeros((frames, 3), np.uint8)
    act[:frames // 2, 0] = 1
    act[frames // 2:, 1] = 1
    act[:, 2] = 1
    res = oracle.em_fit(y, act, target=0, noise=2, iterations=10)
    assert (res.gamma[:, :frames // 2, 1] == 0.0).all()
    assert (res.gamma[:, frames // 2:, 0] == 0.0).all()
    assert np.abs(res.gamma.astype(np.float64).sum(axis=2) - 1.0).max() < 1e-6
    assert res.gamma[:, :frames // 2, 0].mean() > 0.8


def test_likelihood_trace_monotone_and_consistent(oracle):
    # test_cacgmm.cpp:280-301
    y = oracle.unit_normalize(Rng(37).ctensor(6, 90, 3))
    act = _all_on(90, 3)
    res = oracle.em_fit(y, act, target=0, noise=2, iterations=12)
    assert len(res.trace) == 13
    for prev, cur in zip(res.trace[:-1], res.trace[1:]):
        assert cur >= prev - 1e-5 * abs(prev)
    ll = oracle.log_likelihood(y, act, res.pi, res.shapes, noise=2)
    assert ll == pytest.approx(res.trace[-1], rel=1e-9)


def test_dead_class_keeps_shape(oracle):
    # test_cacgmm.cpp:303-327
    y = oracle.unit_normalize(Rng(41).ctensor(2, 50, 2))
    act = np.zeros((50, 2), np.uint8)
    act[:, 1] = 1
    res = oracle.em_fit(y, act, target=1, noise=1, iterations=3)
    for f in range(2):
        assert res.pi[f, 0] == pytest.approx(1e-10)
        assert np.linalg.norm(res.shapes[f, 0] - np.eye(2)) < 1e-12
    assert (res.gamma[:, :, 0] == 0.0).all()


def test_em_fit_validates(oracle):
    # test_cacgmm.cpp:329-335
    y = np.zeros((2, 10, 2), np.complex64)
    with pytest.raises(oracle.OracleError) as e:
        oracle.em_fit(y, _all_on(9, 1), 0, 0, 5)
    assert e.value.kind == "ShapeError"
    with pytest.raises(oracle.OracleError) as e:
        oracle.em_fit(y, _all_on(10, 1), 0, 0, 0)
    assert e.value.kind == "ConfigError"


def test_em_health_acceptance_c2(oracle):
    # acceptance.cpp:221-281 (8 of the 50 seeded problems; all 50 run in the reference)
    bins, frames, ch, k = 16, 200, 4, 3
    for problem in range(8):
        rng = Rng(500 + problem)
        y = oracle.unit_normalize(rng.ctensor(bins, frames, ch))
        act = np.zeros((frames, k), np.uint8)
        for t in range(frames):
            for c in range(k):
                act[t, c] = rng.next() % 3 != 0
            if not act[t].any():
                act[t, 2] = 1
        res = oracle.em_fit(y, act, 0, 2, 20)
        for prev, cur in zip(res.trace[:-1], res.trace[1:]):
            assert prev - cur <= 1e-5 * abs(prev)
        assert (res.gamma[:, act == 0] == 0).all()
        assert np.abs(res.gamma.sum(axis=2, dtype=np.float32) - 1.0).max() <= 1e-6


# --------------------------------------------------------------------------- beamform
def test_stats_two_frames(oracle):
    # test_beamform.cpp:45-59
    y = np.zeros((1, 2, 2), np.complex64)
    y[0, 0, 0] = 1
    y[0, 1, 1] = 1
    g = np.array([[[1, 0], [0, 1]]], np.float32)
    tgt, bg = oracle.mvdr_stats(y, g, 0)
    assert abs(tgt[0, 0, 0] - 0.5) < 1e-12 and abs(tgt[0, 1, 1]) < 1e-12
    assert abs(bg[0, 1, 1] - 0.5) < 1e-12 and abs(bg[0, 0, 0]) < 1e-12


def test_background_sums_non_target(oracle):
    # test_beamform.cpp:61-86
    rng = Rng(3)
    y = rng.ctensor(2, 40, 2)
    g = np.array([rng.uniform() for _ in range(2 * 40 * 3)], np.float32).reshape(2, 40, 3)
    tgt, bg = oracle.mvdr_stats(y, g, 1)
    yd = y.astype(np.complex128)
    for f in range(2):
        outer = np.einsum("tm,tn->tmn", yd[f], yd[f].conj())
        wt = np.einsum("t,tmn->mn", g[f, :, 1].astype(np.float64), outer) / 40
        wb = np.einsum("t,tmn->mn", (g[f, :, 0] + g[f, :, 2]).astype(np.float64), outer) / 40
        assert np.linalg.norm(tgt[f] - wt) / np.linalg.norm(wt) < 1e-6
        assert np.linalg.norm(bg[f] - wb) / np.linalg.norm(wb) < 1e-6


def test_degenerate_stats(oracle):
    # test_beamform.cpp:88-94
    y = np.ones((1, 4, 2), np.complex64)
    g = np.zeros((1, 4, 2), np.float32)
    g[0, :, 1] = 1
    with pytest.raises(oracle.OracleError) as e:
        oracle.mvdr_stats(y, g, 0)
    assert e.value.kind == "DegenerateStatsError"


def test_select_reference(oracle):
    # test_beamform.cpp:100-121
    t0 = np.diag([1.0, 3.0]).astype(complex)
    b0 = np.diag([2.0, 1.0]).astype(complex)
    assert oracle.select_reference(np.stack([t0, t0]), np.stack([b0, b0])) == 1
    eye = np.eye(2, dtype=complex)
    assert oracle.select_reference(np.stack([eye, eye]), np.stack([eye, eye])) == 0


def test_mvdr_frozen(oracle):
    # test_beamform.cpp:127-145
    t = np.array([[1, 0.5j], [-0.5j, 0.5]])
    b = np.array([[1, 0.2], [0.2, 2]], complex)
    h, zeroed = oracle.mvdr(t[None], b[None], 0)
    assert zeroed == 0
    assert abs(h[0, 0] - (0.8 + 0.04j)) < 1e-6
    assert abs(h[0, 1] - (-0.08 - 0.2j)) < 1e-6


def test_mvdr_vs_inverse_nulling_zeroed(oracle):
    # test_beamform.cpp:147-205
    rng = Rng(7)
    for _ in range(50):
        m = 2 + rng.next() % 3
        t = random_hermitian_pd(rng, m, 0.05 * m)
        b = random_hermitian_pd(rng, m, 0.05 * m)
        ref = rng.next() % m
        h, _ = oracle.mvdr(t[None], b[None], ref)
        reg = 0.5 * (b + b.conj().T)
        reg = reg + 1e-10 * np.trace(reg).real / m * np.eye(m)
        c = np.linalg.inv(reg) @ t
        want = c[:, ref] / np.trace(c)
        assert np.linalg.norm(h[0] - want) / np.linalg.norm(want) < 1e-6
    d1 = np.array([1, 1]) / math.sqrt(2)
    d2 = np.array([1, -1]) / math.sqrt(2)
    h, _ = oracle.mvdr(np.outer(d1, d1)[None].astype(complex), (np.outer(d2, d2) + 1e-4 * np.eye(2))[None].astype(complex), 0)
    assert abs(np.vdot(h[0], d2)) < 1e-3 and abs(np.vdot(h[0], d1)) > 0.5
    z, eye = np.zeros((2, 2), complex), np.eye(2, dtype=complex)
    h, zeroed = oracle.mvdr(np.stack([z, eye, z]), np.stack([eye, eye, eye]), 0)
    assert zeroed == 2
    assert np.linalg.norm(h[0]) == 0 and np.linalg.norm(h[1]) > 0 and np.linalg.norm(h[2]) == 0


def test_apply(oracle):
    # test_beamform.cpp:211-237
    y = np.zeros((2, 3, 2), np.complex64)
    for t in range(3):
        y[0, t, 0] = t + 1
        y[0, t, 1] = 1j * (t + 1)
        y[1, t, 0] = 1 + 1j
        y[1, t, 1] = 2
    h = np.array([[1, 0], [0, 1j]])
    out = oracle.apply_filter(h, y)
    assert abs(out[0, 1] - 2) < 1e-6
    assert abs(out[1, 0] - (-2j)) < 1e-6
    with pytest.raises(oracle.OracleError) as e:
        oracle.apply_filter(h[:1], y)
    assert e.value.kind == "ShapeError"


# --------------------------------------------------------------------------- guide + indexing (bit-exact)
def test_activity_grid_boundaries(oracle):
    # test_manifests.cpp:167-189
    segs = [("alice", 0.5, 1.0), ("bob", 0.75, 0.5)]
    centers = [0, 8000, 12000, 19999, 20000, 23999, 24000]
    act = oracle.build_activity_at(segs, centers, 16000, "alice", True)
    assert act.classes == ["alice", "bob", "noise"]
    assert (act.target_index, act.noise_index) == (0, 2)
    assert act.grid[:, 0].tolist() == [0, 1, 1, 1, 1, 1, 0]
    assert act.grid[:, 1].tolist() == [0, 0, 1, 1, 0, 0, 0]
    assert act.grid[:, 2].tolist() == [1] * 7


def test_activity_no_noise_and_empty_target(oracle):
    # test_manifests.cpp:191-206
    act = oracle.build_activity_at([("zed", 0.0, 1.0), ("amy", 0.5, 1.0)], [4000, 12000], 16000, "zed", False)
    assert act.classes == ["amy", "zed"] and act.noise_index == -1 and act.target_index == 1
    with pytest.raises(oracle.OracleError) as e:
        oracle.build_activity_at([("alice", 0.5, 1.0)], [100000, 200000], 16000, "alice", True)
    assert e.value.kind == "EmptyTargetError"


def test_assemble_indices(oracle):
    # test_scheduler.cpp:132-201 (index arithmetic; the audio splice is I/O)
    sr = 16000
    a = oracle.assemble_indices([(2.0, 3.0), (6.0, 1.0)], sr, 8 * sr, 1.0)
    assert a.spans.tolist() == [[1 * sr, 2 * sr], [2 * sr, 5 * sr], [6 * sr, 7 * sr], [7 * sr, 8 * sr]]
    assert a.total == 6 * sr
    assert a.context_left == pytest.approx(1.0) and a.context_right == pytest.approx(1.0)
    assert a.part_begin.tolist() == [1 * sr, 4 * sr]
    assert a.part_end.tolist() == [4 * sr, 5 * sr]
    frames = oracle.frame_count(6 * sr)
    assert len(a.frame_centers) == frames
    assert a.frame_centers[0] == 1 * sr
    assert a.frame_centers[249] == 249 * 256 + sr
    assert a.frame_centers[250] == 6 * sr
    assert a.frame_centers[-1] == 8 * sr - 1
    segs = [("s", 2.0, 3.0), ("s", 6.0, 1.0), ("o", 0.0, 1.5)]
    act = oracle.build_activity_at(segs, a.frame_centers, sr, "s", True)
    tgt = act.target_index
    assert act.classes[tgt] == "s" and act.noise_index >= 0 and len(act.classes) == 3
    assert act.grid[0, tgt] == 0 and act.grid[100, tgt] == 1
    o = act.classes.index("o")
    assert act.grid[31, o] == 1 and act.grid[32, o] == 0


def test_assemble_clips_context(oracle):
    # test_scheduler.cpp:203-232
    sr = 16000
    a = oracle.assemble_indices([(0.2, 1.0)], sr, 4 * sr, 1.0)
    assert a.context_left == pytest.approx(0.2) and a.context_right == pytest.approx(1.0)
    b = oracle.assemble_indices([(3.5, 0.5)], sr, 4 * sr, 1.0)
    assert b.context_left == pytest.approx(1.0) and b.context_right == pytest.approx(0.0)


def test_vector_gram_variant_agrees(oracle, tmp_path):
    """bench.py times the oracle built with -DGSS_ORACLE_VECTOR_GRAM (SIMD partial sums in the Gram, what Eigen's
    cfloat GEMM gives the reference). Same chunks, same double accumulation across chunks; only the float
    summation order inside a chunk differs, so the two builds agree to float rounding."""
    rng = np.random.RandomState(7)
    a = (rng.randn(5000, 11) + 1j * rng.randn(5000, 11)).astype(np.complex64)
    w = rng.rand(5000).astype(np.float32)
    want = oracle.weighted_gram(a, w)
    want_unit = oracle.weighted_gram(a[:37, :3])
    try:
        oracle.load(oracle.build(out_dir=str(tmp_path), vector_gram=True))
        got = oracle.weighted_gram(a, w)
        got_unit = oracle.weighted_gram(a[:37, :3])
    finally:
        oracle.load(oracle._LIB_PATH)
    assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-6
    assert np.linalg.norm(got_unit - want_unit) / np.linalg.norm(want_unit) < 1e-6
    assert np.allclose(got, got.conj().T)
