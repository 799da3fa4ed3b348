"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO ambiguity-function arithmetic: it only draws waveforms
(complex64 sample vectors) and states the five BASELINE.json workloads as plain
numbers.  It is the one module both `oracle/` (through `tests/`) and the product
path (`bench.py`, `__graft_entry__.smoke`) may import (task rule ③).

Recipe (SURVEY.md §8(d) "Synthetic inputs"):
  * splitmix64, state seeded as seed(c, b) = 1_000_000*(c-1) + b for config c
    (1-based) and waveform b, so config 1's single waveform is "seed 0".
  * u = (x >> 11) * 2**-53  (53-bit uniform in [0, 1)).
  * Gaussian by Box-Muller on consecutive uniform pairs: cos branch first,
    then sin branch.
  * Draw order per waveform: per-waveform parameters, then phases for
    n = 0..N-1, then amplitude ripple for n = 0..N-1.
  * Everything computed in float64 then rounded to nearest complex64.

The paper's own workload is random-start phase-coded waveforms of N = 256
(§7.1); it uses no dataset, so every input here is synthetic.
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "SplitMix64", "CONFIGS", "config_waveforms", "waveform", "random_phase",
    "complex_gaussian", "barker13", "lfm", "frank", "p4", "qpsk",
]

_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


class SplitMix64:
    """Counter-based splitmix64 stream (vectorised with wrapping uint64)."""

    def __init__(self, seed: int):
        self.state = np.uint64(seed & 0xFFFFFFFFFFFFFFFF)
        self.pos = 0  # number of outputs already drawn

    def u64(self, n: int) -> np.ndarray:
        i = np.arange(self.pos + 1, self.pos + n + 1, dtype=np.uint64)
        self.pos += n
        with np.errstate(over="ignore"):
            z = self.state + i * _GAMMA
            z = (z ^ (z >> np.uint64(30))) * _M1
            z = (z ^ (z >> np.uint64(27))) * _M2
            z = z ^ (z >> np.uint64(31))
        return z

    def uniform(self, n: int) -> np.ndarray:
        return (self.u64(n) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)

    def gaussian(self, n: int) -> np.ndarray:
        pairs = (n + 1) // 2
        u = self.uniform(2 * pairs).reshape(pairs, 2)
        r = np.sqrt(-2.0 * np.log1p(-u[:, 0]))  # 1-u in (0,1]: never log(0)
        z = np.empty((pairs, 2))
        z[:, 0] = r * np.cos(2.0 * np.pi * u[:, 1])
        z[:, 1] = r * np.sin(2.0 * np.pi * u[:, 1])
        return z.reshape(-1)[:n]


def _c64(re_im_phase: np.ndarray, amp: np.ndarray | float = 1.0) -> np.ndarray:
    return (amp * np.exp(1j * re_im_phase)).astype(np.complex64)


# --------------------------------------------------------------------------
# Waveform families (textbook definitions; SURVEY.md §8(c) reading #17)
# --------------------------------------------------------------------------
def random_phase(rng: SplitMix64, n: int, ripple_sigma: float = 0.0) -> np.ndarray:
    theta = 2.0 * np.pi * rng.uniform(n)
    amp = 1.0 + ripple_sigma * rng.gaussian(n) if ripple_sigma else 1.0
    return _c64(theta, amp)


def complex_gaussian(rng: SplitMix64, n: int) -> np.ndarray:
    z = rng.gaussian(2 * n).reshape(n, 2)
    return (z[:, 0] + 1j * z[:, 1]).astype(np.complex64)


def lfm(n: int, beta: float) -> np.ndarray:
    k = np.arange(n, dtype=np.float64)
    return _c64(np.pi * beta * k * k / n)


def frank(n: int) -> np.ndarray:
    L = int(round(np.sqrt(n)))
    if L * L != n:
        raise ValueError("Frank code needs N = L^2")
    p, q = np.divmod(np.arange(n), L)
    # phase 2*pi*p*q/L reduced exactly on integers first
    return _c64(2.0 * np.pi * ((p * q) % L) / L)


def p4(n: int) -> np.ndarray:
    k = np.arange(n, dtype=np.int64)
    num = (k * k - k * n) % (2 * n)          # exact integer phase numerator
    return _c64(np.pi * num / n)


def qpsk(rng: SplitMix64, n: int) -> np.ndarray:
    q = np.floor(4.0 * rng.uniform(n)).astype(np.int64) % 4
    lut = np.array([1, 1j, -1, -1j], dtype=np.complex64)   # j**q, exact
    return lut[q]


def barker13() -> np.ndarray:
    return np.array([1, 1, 1, 1, 1, -1, -1, 1, 1, -1, 1, -1, 1], dtype=np.complex64)


# --------------------------------------------------------------------------
# The five BASELINE.json workloads, as plain numbers.
# Loss-region fields: k_max, d_max (|k| <= k_max, |d| <= d_max with d the
# fftshift-centred Doppler index), mainlobe (ml_k, ml_d) excluded.
# --------------------------------------------------------------------------
CONFIGS = {
    1: dict(name="c1", B=1, N=64, M=64, family="random_phase",
            surface="c64", layout="centered",
            loss=dict(k_max=63, d_max=32, ml_k=0, ml_d=0, lambda_isl=1.0,
                      lambda_psl=0.0, temperature=0.01, normalize=1)),
    2: dict(name="c2", B=256, N=256, M=256, family="random_phase",
            surface=None, layout="centered",
            loss=dict(k_max=64, d_max=32, ml_k=0, ml_d=0, lambda_isl=1.0,
                      lambda_psl=0.0, temperature=0.01, normalize=1)),
    3: dict(name="c3", B=1024, N=1024, M=1024, family="mixed",
            surface="abs", layout="centered",
            loss=dict(k_max=1023, d_max=512, ml_k=0, ml_d=0, lambda_isl=1.0,
                      lambda_psl=0.0, temperature=0.01, normalize=1)),
    4: dict(name="c4", B=64, N=4096, M=8192, family="ripple",
            surface=None, layout="centered",
            loss=dict(k_max=512, d_max=256, ml_k=0, ml_d=1, lambda_isl=1.0,
                      lambda_psl=1.0, temperature=0.01, normalize=1)),
    5: dict(name="c5", B=8, N=16384, M=16384, family="random_phase",
            surface=None, layout="centered",
            loss=dict(k_max=16383, d_max=8192, ml_k=0, ml_d=0, lambda_isl=1.0,
                      lambda_psl=1.0, temperature=0.01, normalize=1)),
}


def seed_of(config: int, b: int) -> int:
    return 1_000_000 * (config - 1) + b


def waveform(config: int, b: int, n: int | None = None) -> np.ndarray:
    """Waveform b of config `config` (complex64, length N or override n)."""
    cfg = CONFIGS[config]
    n = cfg["N"] if n is None else n
    rng = SplitMix64(seed_of(config, b))
    fam = cfg["family"]
    if fam == "random_phase":
        return random_phase(rng, n)
    if fam == "ripple":
        return random_phase(rng, n, ripple_sigma=0.05)
    if fam == "mixed":                       # SURVEY §8(c) reading #16
        f = b % 3
        if f == 0:
            beta = 0.5 + 1.5 * rng.uniform(1)[0]
            return lfm(n, beta)
        if f == 1:
            return frank(n) if (b // 3) % 2 == 0 else p4(n)
        return qpsk(rng, n)
    raise ValueError(fam)


def lfm_beta(config: int, b: int) -> float:
    """The LFM sweep factor drawn for waveform b of the mixed family."""
    rng = SplitMix64(seed_of(config, b))
    return 0.5 + 1.5 * rng.uniform(1)[0]


def config_waveforms(config: int, batch: int | None = None, start: int = 0,
                     n: int | None = None) -> np.ndarray:
    """[batch, N] complex64 array of waveforms start..start+batch-1."""
    cfg = CONFIGS[config]
    batch = cfg["B"] if batch is None else batch
    return np.stack([waveform(config, start + b, n) for b in range(batch)])
