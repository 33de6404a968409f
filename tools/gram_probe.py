"""Compares the WPE Gram (R, P) of the device kernels with a float64 numpy evaluation (diagnostic).
   GSS_B200_WPE_GRAM=fp32 selects the FP32-FMA kernel, default is the tcgen05 kernel."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2212_05271_b200 import capi, gss  # noqa: E402


def reference(y, taps, delay):
    f, t, m = y.shape
    km = taps * m
    h = delay + taps - 1
    R = np.zeros((f, km, km), np.complex128)
    P = np.zeros((f, km, m), np.complex128)
    y64 = y.astype(np.complex128)
    for ff in range(f):
        yf = y64[ff]
        s = (np.abs(y[ff]) ** 2).astype(np.float32).sum(1)
        lam = np.maximum(1e-10, s.astype(np.float64) / m).astype(np.float32)
        w = (np.float32(1.0) / lam).astype(np.float64)
        pad = np.vstack([np.zeros((h, m), np.complex128), yf])
        # window of frame t: frames t-h .. t-h+taps-1 (reverse tap order) = pad[t : t+taps]
        A = np.stack([pad[tt: tt + taps].reshape(-1) for tt in range(t)])
        R[ff] = (A.T * w) @ A.conj()
        P[ff] = (A.T * w) @ yf.conj()
    return R, P


def main():
    ctx = gss.default_context()
    lib = capi.load()
    for (f, t, m, taps, delay) in [(3, 200, 7, 10, 2), (2, 333, 8, 10, 3), (2, 100, 2, 5, 1), (2, 150, 4, 8, 2),
                                   (2, 64, 1, 4, 2), (2, 97, 5, 10, 2), (513, 79, 3, 10, 2), (4, 5001, 7, 10, 2)]:
        rng = np.random.RandomState(t)
        y = (rng.randn(f, t, m) + 1j * rng.randn(f, t, m)).astype(np.complex64)
        y[:, 3:] += 0.6 * y[:, :-3]
        cfg = capi.WpeConfig(taps, delay, 1, 0, 1e-10)
        km = taps * m
        out = np.zeros((f, km * km + km * m), np.complex128)
        ctx.check(lib.gss_b200_debug_wpe_gram(ctx.handle, capi.ptr(y), C.c_int32(f), C.c_int64(t), C.c_int32(m),
                                              C.byref(cfg), capi.ptr(out)))
        R = out[:, : km * km].reshape(f, km, km)
        P = out[:, km * km:].reshape(f, km, m)
        Rr, Pr = reference(y, taps, delay)
        eR = np.linalg.norm(R - Rr) / np.linalg.norm(Rr)
        eP = np.linalg.norm(P - Pr) / np.linalg.norm(Pr)
        print(f"F={f} T={t} M={m} taps={taps} delay={delay}: rel(R)={eR:.2e} rel(P)={eP:.2e} "
              f"max|R-Rr|/max|Rr|={np.abs(R - Rr).max() / np.abs(Rr).max():.2e}")


if __name__ == "__main__":
    main()
