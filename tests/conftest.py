import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu on the GPU box)")


GOLDEN = os.path.join(ROOT, "tests", "golden")


@pytest.fixture(scope="session")
def small_golden():
    return np.load(os.path.join(GOLDEN, "small.npz"))


@pytest.fixture(scope="session")
def cfg_golden():
    return np.load(os.path.join(GOLDEN, "configs.npz"))


def rand_tensor_ref(stream, m, n, p):
    """The reference tests' rand_tensor (test_tproduct.cpp:14-19): with one Rng,
    t1 entries then t2 entries, each rand_cx = {sym(), sym()} (test_util.hpp:46).
    `stream` is a callable returning the next k sym() draws."""
    t1 = stream(2 * m * n * p).view(np.complex128).reshape(p, m, n).copy()
    t2 = stream(2 * m * n * p).view(np.complex128).reshape(p, m, n).copy()
    return t1, t2


class RefRng:
    """Replays the reference's Rng(seed) (rng.hpp:18-30): sym() and next_u64()
    interleaved in call order, via the oracle's mt19937_64 stream."""

    def __init__(self, seed):
        self._seed = seed
        self._u = np.empty(0, np.uint64)
        self._i = 0
        self._ensure(1 << 16)

    def _ensure(self, k):
        if self._i + k > self._u.size:
            import oracle as O
            self._u = O.rng_u64(self._seed, max(2 * self._u.size, self._i + k + (1 << 16)))

    def next_u64(self):
        self._ensure(1)
        v = int(self._u[self._i])
        self._i += 1
        return v

    def sym(self, k=None):
        if k is None:
            return 2.0 * ((self.next_u64() >> 11) * 2.0 ** -53) - 1.0
        self._ensure(k)
        raw = self._u[self._i:self._i + k]
        self._i += k
        return 2.0 * ((raw >> np.uint64(11)).astype(np.float64) * 2.0 ** -53) - 1.0

    def tensor(self, m, n, p):
        return rand_tensor_ref(lambda k: self.sym(k), m, n, p)
