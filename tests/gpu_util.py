"""Shared helpers for the GPU parity tests (test infrastructure)."""
import numpy as np

from .refrng import Rng


def cgauss_tensor(seed, f, t, m, scale=1.0):
    rng = np.random.RandomState(seed)
    return ((rng.randn(f, t, m) + 1j * rng.randn(f, t, m)) * scale).astype(np.complex64)


def random_activity(seed, t, k, noise=True, holes=False):
    """Speaker-like on/off runs; last class is the always-on noise class when noise=True."""
    rng = np.random.RandomState(seed)
    act = np.zeros((t, k), np.uint8)
    nspk = k - 1 if noise else k
    for c in range(nspk):
        pos = int(rng.randint(0, max(1, t // 4)))
        while pos < t:
            ln = int(rng.randint(t // 8 + 1, t // 2 + 2))
            act[pos:pos + ln, c] = 1
            pos += ln + int(rng.randint(1, t // 4 + 2))
    if noise:
        act[:, k - 1] = 1
    elif not holes:
        dead = act.sum(1) == 0
        act[dead, 0] = 1
    return act


def rel_fro(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-30))


def sdr_db(est, ref):
    est = np.asarray(est, np.float64)
    ref = np.asarray(ref, np.float64)
    err = np.sum((est - ref) ** 2)
    return float(10 * np.log10(np.sum(ref ** 2) / max(err, 1e-300)))


__all__ = ["Rng", "cgauss_tensor", "random_activity", "rel_fro", "sdr_db"]
