"""The reference test-suite's deterministic generator (tests/test_util.hpp:13-33),
restated so the seeded inputs of its random cases can be regenerated here."""
import math

import numpy as np

MASK = (1 << 64) - 1


class Rng:
    def __init__(self, seed):
        self.state = seed & MASK

    def next(self):
        self.state = (self.state + 0x9E3779B97F4A7C15) & MASK
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
        return z ^ (z >> 31)

    def uniform(self):
        return (self.next() >> 11) * 2.0 ** -53

    def gaussian(self):
        u1, u2 = self.uniform(), self.uniform()
        if u1 < 1e-300:
            u1 = 1e-300
        return math.sqrt(-2.0 * math.log(u1)) * math.cos(6.283185307179586 * u2)

    def cgaussian(self):
        re = self.gaussian() * math.sqrt(0.5)
        im = self.gaussian() * math.sqrt(0.5)
        return complex(re, im)

    def ctensor(self, *shape):
        """cfloat tensor filled in row-major order like `for (auto& v : t.data) v = cfloat(cgaussian())`."""
        n = int(np.prod(shape))
        out = np.empty(n, np.complex64)
        for i in range(n):
            out[i] = self.cgaussian()
        return out.reshape(shape)
