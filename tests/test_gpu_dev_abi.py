"""The device-pointer (`_dev`) entry points of the C ABI (include/gss_b200.h) and the NVTX ranges.

Tensors live in HBM (torch tensors here, raw cudaMalloc'ed pointers to the library), the caller's stream orders the
calls, and the results must be the same bits the host-pointer entry points return."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch
    from paper_2212_05271_b200 import capi, gss
    ctx = gss.default_context()
    return torch, capi, gss, ctx


def dptr(t):
    return C.c_void_p(t.data_ptr())


def test_stage_operators_on_device_tensors_match_the_host_entry_points(env):
    torch, capi, gss, ctx = env
    lib = ctx.lib
    rng = np.random.RandomState(5)
    m, n = 4, 20000
    cfg = gss.stft.StftConfig(512, 128, 0, 16000)
    audio = (rng.randn(m, n) * 0.1).astype(np.float32)
    want_spec = gss.stft.analyze(gss.stft.RealSignal(audio, 16000), cfg)
    f, t = want_spec.data.shape[:2]
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        d_audio = torch.from_numpy(audio).cuda(non_blocking=True)      # queued on the caller's stream ...
        d_spec = torch.empty((f, t, m, 2), dtype=torch.float32, device="cuda")
        ccfg = cfg.c()
        # ... and consumed by the library without any host synchronisation in between
        ctx.check(lib.gss_b200_stft_dev(ctx.handle, dptr(d_audio), C.c_int32(m), C.c_int64(n), C.c_int32(16000),
                                        C.byref(ccfg), dptr(d_spec), C.c_void_p(side.cuda_stream)))
        got_spec = torch.view_as_complex(d_spec).cpu().numpy()          # ordered after the call by the stream
    assert got_spec.tobytes() == want_spec.data.tobytes()

    wcfg = gss.wpe.WpeConfig(6, 2, 2, 0, 1e-10)
    want_wpe = gss.wpe.dereverberate(want_spec, wcfg).data
    want_norm = gss.wpe.unit_normalize(gss.stft.SpectrogramTensor(want_wpe, cfg)).data
    with torch.cuda.stream(side):
        d_wpe = torch.empty_like(d_spec)
        d_norm = torch.empty_like(d_spec)
        cw = wcfg.c()
        ctx.check(lib.gss_b200_wpe_dev(ctx.handle, dptr(d_spec), C.c_int32(f), C.c_int64(t), C.c_int32(m), C.byref(cw),
                                       dptr(d_wpe), C.c_void_p(side.cuda_stream)))
        ctx.check(lib.gss_b200_unit_normalize_dev(ctx.handle, dptr(d_wpe), C.c_int32(f), C.c_int64(t), C.c_int32(m),
                                                  dptr(d_norm), C.c_void_p(side.cuda_stream)))
        got_wpe = torch.view_as_complex(d_wpe).cpu().numpy()
        got_norm = torch.view_as_complex(d_norm).cpu().numpy()
    assert got_wpe.tobytes() == want_wpe.tobytes()
    assert got_norm.tobytes() == want_norm.tobytes()

    h = (rng.randn(f, m) + 1j * rng.randn(f, m)).astype(np.complex128)
    want_x = gss.beamform.apply(gss.beamform.BeamformerFilter(h), gss.stft.SpectrogramTensor(want_wpe, cfg))
    want_wave = gss.stft.synthesize(gss.stft.SpectrogramTensor(want_x.data, cfg, 0, n)).channels
    with torch.cuda.stream(side):
        d_x = torch.empty((f, t, 2), dtype=torch.float32, device="cuda")
        d_wave = torch.empty((1, n), dtype=torch.float32, device="cuda")
        ctx.check(lib.gss_b200_apply_dev(ctx.handle, capi.ptr(h), C.c_int32(f), C.c_int32(m), dptr(d_wpe), C.c_int32(f),
                                         C.c_int64(t), C.c_int32(m), dptr(d_x), C.c_void_p(side.cuda_stream)))
        ctx.check(lib.gss_b200_istft_dev(ctx.handle, dptr(d_x), C.c_int32(f), C.c_int64(t), C.c_int32(1), C.c_int64(n),
                                         C.byref(ccfg), dptr(d_wave), C.c_void_p(side.cuda_stream)))
        got_wave = d_wave.cpu().numpy()
    assert got_wave.tobytes() == np.ascontiguousarray(want_wave).tobytes()


def test_enhance_batch_on_device_audio_matches_the_host_call_and_opens_nvtx_ranges(env):
    torch, capi, gss, ctx = env
    import synthbench as synth
    w = synth.workload("tiny", n_segments=2)
    want = gss.scheduler.enhance_batches(w.segments, w.cfg, ctx)
    m = gss.scheduler._Marshalled(w.segments, w.cfg, diagnostics=False)
    keep = []
    for i, ss in enumerate(w.segments):
        d_audio = torch.from_numpy(np.ascontiguousarray(ss.audio.channels, np.float32)).cuda()
        d_out = torch.zeros(max(1, len(m.out_wave[i])), dtype=torch.float32, device="cuda")
        keep += [d_audio, d_out]
        m.desc[i].audio = d_audio.data_ptr()
        m.desc[i].out_wave = d_out.data_ptr()
    torch.cuda.synchronize()
    ranges0 = int(ctx.lib.gss_b200_nvtx_range_count(ctx.handle))
    ccfg = w.cfg.c()
    ctx.check(ctx.lib.gss_b200_enhance_batch_dev(ctx.handle, C.c_int32(m.n), m.desc, C.byref(ccfg), m.diag,
                                                 C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    for i, r in enumerate(want):
        assert m.diag[i].status == 0 and m.diag[i].ref_channel == r.ref_channel and m.diag[i].frames == r.frames
        got = keep[2 * i + 1].cpu().numpy()[: len(r.outputs[0])]
        assert got.tobytes() == r.outputs[0].tobytes()
    # one range for the call, one per stage (stft, wpe per upload wave; mask, beamform, istft, d2h)
    assert int(ctx.lib.gss_b200_nvtx_range_count(ctx.handle)) - ranges0 >= 7
