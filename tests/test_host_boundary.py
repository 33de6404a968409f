"""CPU checks of the drop-in boundary: the C ABI library loads and exports every symbol declared in
include/gss_b200.h, fails loudly without a device, and its host-only (integer / scalar) entry points are
bit-exact with the oracle and with the reference's frozen vectors. No compute kernels run here."""
import ctypes as C
import math
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def gss():
    from paper_2212_05271_b200 import build
    build.build(verbose=False)
    from paper_2212_05271_b200 import gss as g
    return g


def test_library_exports_every_declared_symbol(gss):
    from paper_2212_05271_b200 import capi
    lib = capi.load()
    header = open(os.path.join(ROOT, "include", "gss_b200.h")).read()
    declared = sorted(set(re.findall(r"\b(gss_b200_[a-z0-9_]+)\s*\(", header)))
    assert len(declared) >= 30
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(capi.EXPORTS) == declared


def test_struct_layouts_match_header(gss):
    from paper_2212_05271_b200 import capi
    assert C.sizeof(capi.StftConfig) == 16
    assert C.sizeof(capi.WpeConfig) == 24
    assert C.sizeof(capi.PipelineConfig) == 48
    assert C.sizeof(capi.SegmentDesc) == 112
    assert C.sizeof(capi.SegmentDiag) == 40
    cfg = capi.PipelineConfig()
    capi.load().gss_b200_default_pipeline_config(C.byref(cfg))
    # stft.hpp:17-21, wpe.hpp:16-20, scheduler.hpp:31-41 defaults
    assert (cfg.stft.fft_size, cfg.stft.shift, cfg.stft.window, cfg.stft.sample_rate) == (1024, 256, 0, 16000)
    assert (cfg.wpe.taps, cfg.wpe.delay, cfg.wpe.iterations, cfg.wpe.psd_context) == (10, 2, 3, 0)
    assert cfg.wpe.regularization == 1e-10 and cfg.enable_wpe == 1 and cfg.bss_iterations == 20


def test_no_cpu_fallback(gss):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    with pytest.raises(gss.common.CudaError) as e:
        gss.Context(0)
    assert "no CPU fallback" in str(e.value)


def test_product_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2212_05271_b200")
    for dp, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".cpp", ".h", ".inc", ".hpp")):
                src = open(os.path.join(dp, fn), errors="replace").read()
                assert "gss_oracle" not in src and "liboracle" not in src, fn
                assert not re.search(r"^\s*(from|import)\s+oracle\b", src, re.M), fn


def test_frame_geometry(gss, oracle):
    # test_stft.cpp:79-88
    cfg = gss.stft.StftConfig()
    assert gss.stft.frame_count(1024, cfg) == 5 and gss.stft.frame_count(1280, cfg) == 6
    assert gss.stft.frame_center(3, cfg) == 768
    for n in list(range(512, 2000, 37)) + [160000, 640000, 960000]:
        assert gss.stft.frame_count(n, gss.stft.StftConfig(512, 128)) == oracle.frame_count(n, 512, 128)


def test_activity_grid_boundaries(gss):
    # test_manifests.cpp:167-189: half-open boundaries at 19999/20000 and 23999/24000
    S = gss.manifests.Segment
    segs = [S("r", "alice", 0.5, 1.0), S("r", "bob", 0.75, 0.5)]
    act = gss.manifests.build_activity_at(segs, [0, 8000, 12000, 19999, 20000, 23999, 24000], 16000, "alice", True)
    assert act.classes == ["alice", "bob", "noise"]
    assert (act.target_index, act.noise_index) == (0, 2)
    assert act.grid[:, 0].tolist() == [0, 1, 1, 1, 1, 1, 0]
    assert act.grid[:, 1].tolist() == [0, 0, 1, 1, 0, 0, 0]
    assert act.grid[:, 2].tolist() == [1] * 7
    # test_manifests.cpp:191-206
    act = gss.manifests.build_activity_at([S("r", "zed", 0.0, 1.0), S("r", "amy", 0.5, 1.0)], [4000, 12000], 16000,
                                          "zed", False)
    assert act.classes == ["amy", "zed"] and act.noise_index == -1 and act.target_index == 1
    with pytest.raises(gss.EmptyTargetError):
        gss.manifests.build_activity_at([S("r", "alice", 0.5, 1.0)], [100000, 200000], 16000, "alice", True)


def test_activity_bit_exact_vs_oracle(gss, oracle):
    rng = np.random.RandomState(3)
    S = gss.manifests.Segment
    for trial in range(20):
        nseg = rng.randint(1, 12)
        spk = ["s%d" % rng.randint(0, 5) for _ in range(nseg)]
        st = rng.uniform(0, 30, nseg).round(3)
        du = rng.uniform(0.01, 8, nseg).round(3)
        centers = np.sort(rng.randint(0, 40 * 16000, 400)).astype(np.int64)
        target = spk[0]
        noise = bool(trial % 2)
        try:
            want = oracle.build_activity_at(list(zip(spk, st, du)), centers, 16000, target, noise)
        except oracle.OracleError as e:
            assert e.kind == "EmptyTargetError"
            with pytest.raises(gss.EmptyTargetError):
                gss.manifests.build_activity_at([S("r", a, b, c) for a, b, c in zip(spk, st, du)], centers, 16000,
                                                target, noise)
            continue
        got = gss.manifests.build_activity_at([S("r", a, b, c) for a, b, c in zip(spk, st, du)], centers, 16000,
                                              target, noise)
        assert got.classes == want.classes
        assert (got.target_index, got.noise_index) == (want.target_index, want.noise_index)
        assert got.grid.tobytes() == want.grid.tobytes()


def test_assemble_indices(gss, oracle):
    # test_scheduler.cpp:132-232
    sr = 16000
    cfg = gss.stft.StftConfig()
    a = gss.scheduler.assemble_indices([(2.0, 3.0), (6.0, 1.0)], sr, 8 * sr, 1.0, cfg)
    assert a.spans == [(1 * sr, 2 * sr), (2 * sr, 5 * sr), (6 * sr, 7 * sr), (7 * sr, 8 * sr)]
    assert a.total == 6 * sr
    assert a.part_begin.tolist() == [1 * sr, 4 * sr] and a.part_end.tolist() == [4 * sr, 5 * sr]
    assert len(a.frame_centers) == gss.stft.frame_count(6 * sr, cfg)
    assert a.frame_centers[0] == sr and a.frame_centers[249] == 249 * 256 + sr
    assert a.frame_centers[250] == 6 * sr and a.frame_centers[-1] == 8 * sr - 1
    b = gss.scheduler.assemble_indices([(0.2, 1.0)], sr, 4 * sr, 1.0, cfg)
    assert b.context_left == pytest.approx(0.2) and b.context_right == pytest.approx(1.0)
    b = gss.scheduler.assemble_indices([(3.5, 0.5)], sr, 4 * sr, 1.0, cfg)
    assert b.context_left == pytest.approx(1.0) and b.context_right == pytest.approx(0.0)
    rng = np.random.RandomState(8)
    for _ in range(30):  # bit-exact against the oracle on random plans
        n = rng.randint(1, 6)
        starts = np.sort(rng.uniform(0, 50, n)).round(4)
        durs = rng.uniform(0.05, 3, n).round(4)
        for i in range(n - 1):
            durs[i] = min(durs[i], max(0.01, starts[i + 1] - starts[i]))
        ctx = float(rng.choice([0.0, 0.5, 15.0]))
        parts = list(zip(starts.tolist(), durs.tolist()))
        try:
            want = oracle.assemble_indices(parts, sr, 55 * sr, ctx, 512, 128)
        except oracle.OracleError:
            with pytest.raises(gss.ShapeError):
                gss.scheduler.assemble_indices(parts, sr, 55 * sr, ctx, gss.stft.StftConfig(512, 128))
            continue
        got = gss.scheduler.assemble_indices(parts, sr, 55 * sr, ctx, gss.stft.StftConfig(512, 128))
        assert got.spans == [tuple(x) for x in want.spans.tolist()]
        assert got.part_begin.tolist() == want.part_begin.tolist()
        assert got.part_end.tolist() == want.part_end.tolist()
        assert got.total == want.total
        assert got.frame_centers.tobytes() == want.frame_centers.tobytes()
        assert got.context_left == want.context_left and got.context_right == want.context_right


def test_scalar_known_answers(gss, oracle):
    # test_cacgmm.cpp:53-79 frozen pdf values
    pdf = gss.cacgmm.cacg_log_pdf
    assert pdf([1.0], [[1.0]]) == pytest.approx(-1.8378770664093453, abs=1e-12)
    assert pdf([1.0, 0.0], np.eye(2)) == pytest.approx(-3.6757541328186907, abs=1e-12)
    assert pdf([1.0, 0.0], np.diag([2.0, 0.5])) == pytest.approx(-2.2894597716988, abs=1e-10)
    assert pdf([1j, 1.0], [[2, 1j], [-1j, 2]]) == pytest.approx(oracle.cacg_log_pdf([1j, 1.0], [[2, 1j], [-1j, 2]]),
                                                                abs=1e-12)
    rng = np.random.RandomState(2)
    for m in (1, 2, 3, 5, 8):
        r = rng.randn(m, m) + 1j * rng.randn(m, m)
        b = r @ r.conj().T + 0.1 * np.eye(m)
        y = rng.randn(m) + 1j * rng.randn(m)
        assert pdf(y, b) == pytest.approx(oracle.cacg_log_pdf(y, b), abs=1e-9)
    with pytest.raises(gss.ShapeError):
        pdf([1.0, 2.0], np.eye(3))
    # test_cacgmm.cpp:116-137 frozen weights + fallbacks
    tvw = gss.cacgmm.time_varying_weights
    w = tvw([0.2, 0.3, 0.5], [1, 0, 1])
    assert w.tolist() == pytest.approx([0.2857142857142857, 0.0, 0.7142857142857143])
    assert tvw([0.2, 0.3, 0.5], [0, 0, 0], 2).tolist() == [0.0, 0.0, 1.0]
    assert tvw([0.2, 0.3, 0.5], [0, 0, 0], -1).tolist() == pytest.approx([1 / 3] * 3)
    with pytest.raises(gss.ShapeError):
        tvw([0.5, 0.5], [1, 1, 1])
    assert math.isfinite(pdf([0.0, 0.0], np.eye(2)))  # quadratic-form floor 1e-10
