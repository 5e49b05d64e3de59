"""The five BASELINE.json configurations and their seeded input generators
(SURVEY.md §8(d)).

Seeds mirror run_bench (/root/reference/proj/src/bench.cpp:66-69): base seed
S = 42 (bench.hpp:19); config c uses seedA = derive_seed(S, 2(c-1)) and
seedB = derive_seed(S, 2(c-1)+1).  The datasets are synthetic by definition
(BASELINE.json describes distributions, not files).

This module is standalone (no package import, no library): bench.py's
reference arm loads it by path so that arm never loads the product library.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

BASE_SEED = 42
_M64 = (1 << 64) - 1


def derive_seed(base: int, stream: int) -> int:
    """derive_seed of rng.cpp:15-19 (splitmix64 chain), restated; equal to
    qt_derive_seed (tests/test_abi.py)."""
    state, out = base & _M64, 0
    for _ in range(stream + 1):
        state = (state + 0x9E3779B97F4A7C15) & _M64
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
        out = z ^ (z >> 31)
    return out


@dataclass(frozen=True)
class Config:
    idx: int
    name: str
    m: int
    n: int
    s: int
    p: int
    dist_a: int
    scale_a: float
    dist_b: int
    scale_b: float
    note: str

    def seeds(self):
        return derive_seed(BASE_SEED, 2 * (self.idx - 1)), derive_seed(BASE_SEED, 2 * (self.idx - 1) + 1)

    # algorithmic work; the same figures the roofline uses
    @property
    def flops_gemm(self) -> float:
        return 32.0 * self.m * self.n * self.s * self.p

    @property
    def flops_fft(self) -> float:
        lg = math.log2(self.p) if self.p > 1 else 0.0
        return 10.0 * (self.m * self.n + self.n * self.s + self.m * self.s) * self.p * lg

    @property
    def flops_eff(self) -> float:
        return self.flops_gemm + self.flops_fft

    def bytes_tensor(self, rows: int, cols: int) -> int:
        return 32 * rows * cols * self.p  # both CD planes, 16 B per complex

    @property
    def bytes_fft_fwd(self) -> int:   # K1: read A, B; write Â, B̂
        return 2 * (self.bytes_tensor(self.m, self.n) + self.bytes_tensor(self.n, self.s))

    @property
    def bytes_fft_inv(self) -> int:   # K3: read Ĉ, write C
        return 2 * self.bytes_tensor(self.m, self.s)

    @property
    def bytes_gemm(self) -> int:      # K2: read Â, B̂ once, write Ĉ
        return self.bytes_tensor(self.m, self.n) + self.bytes_tensor(self.n, self.s) + self.bytes_tensor(self.m, self.s)


U, N, P = 0, 1, 2  # QT_DIST_UNIFORM_SYM, QT_DIST_NORMAL, QT_DIST_PURE_UNIT (include/qtensor_b200.h)

CONFIGS = {
    1: Config(1, "cfg1_32x32x32_p16", 32, 32, 32, 16, U, 1.0, U, 1.0,
              "uniform[-1,1) all 4 components; definitional-oracle case"),
    2: Config(2, "cfg2_256x256x256_p64", 256, 256, 256, 64, N, 1.0, N, 1.0,
              "N(0,1) all 4 components; balanced FFT/GEMM"),
    3: Config(3, "cfg3_16x16x16_p4096", 16, 16, 16, 4096, U, 1.0, U, 1.0,
              "FFT-dominated long tubes"),
    4: Config(4, "cfg4_video_1080x1920x64_p64", 1080, 1920, 64, 64, P, 1.0, N, 1.0 / math.sqrt(1920.0),
              "A pure quaternion RGB U[0,1); B N(0,1/1920)"),
    5: Config(5, "cfg5_2048x2048x2048_p32", 2048, 2048, 2048, 32, U, 1.0, U, 1.0,
              "GEMM-dominated; the 1/2/4/8-GPU scaling case"),
}


def make_inputs(cfg: Config):
    """Host CdTensor3 pair (A, B) for a config, deterministic from the seeds."""
    from .tproduct import gen_tensor
    sa, sb = cfg.seeds()
    a = gen_tensor(cfg.m, cfg.n, cfg.p, sa, cfg.dist_a, cfg.scale_a)
    b = gen_tensor(cfg.n, cfg.s, cfg.p, sb, cfg.dist_b, cfg.scale_b)
    return a, b
