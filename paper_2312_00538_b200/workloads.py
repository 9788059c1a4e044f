"""Seeded synthetic stand-ins for the BASELINE.json configurations.

The public datasets the paper uses (cod-rna, HIGGS, SUSY) are
not in this image; these generators reproduce the *shapes, sizes and value
distributions* BASELINE.json names, with fixed seeds
(1001..1005). Features are min-max scaled per column to [-1/4, 1/4] where the
config says so. Windows, weights (eta = 1/P, P:src/pipeline.cpp:241) and
length scales (1) follow the configs; fit_fraction is 1.0 for the matvec-only
configs 2 and 4 and 1/1.2 for the training-path configs 1, 3, 5
(P:src/pipeline.cpp:202).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class Workload:
    name: str
    points: np.ndarray      # n x d, row-major float64
    windows: list
    fit_fraction: float
    v: np.ndarray           # the input vector x ~ N(0, 1)
    labels: np.ndarray | None = None

    @property
    def n(self) -> int:
        return int(self.points.shape[0])

    @property
    def d(self) -> int:
        return int(self.points.shape[1])

    @property
    def D(self) -> int:
        return sum(len(w) for w in self.windows)

    def hbm_bytes(self, word: int = 8) -> int:
        """Algorithmic HBM bytes per matvec, B = w n (2 D + 2)."""
        return word * self.n * (2 * self.D + 2)

    def fma_count(self, m: int = 4) -> int:
        """Algorithmic FP64 FMAs per matvec, F = 2 n sum_l (2m)^{d_l}."""
        return 2 * self.n * sum((2 * m) ** len(w) for w in self.windows)


def minmax_quarter(x: np.ndarray) -> np.ndarray:
    lo = x.min(axis=0, keepdims=True)
    hi = x.max(axis=0, keepdims=True)
    span = np.where(hi > lo, hi - lo, 1.0)
    return (x - lo) / span * 0.5 - 0.25


def _triples(d_cont: int) -> list:
    return [[3 * i, 3 * i + 1, 3 * i + 2] for i in range(d_cont // 3)]


def config1(n: int = 2000, seed: int = 1001) -> Workload:
    rng = np.random.default_rng(seed)
    x = minmax_quarter(rng.standard_normal((n, 6)))
    w = rng.standard_normal(6)
    eps = rng.standard_normal(n)
    y = np.where(x @ w + 0.1 * eps >= 0.0, 1.0, -1.0)  # sign(0) = +1 (P:src/ipm.cpp:295)
    return Workload("cfg1 n=2000 d=6 windows(3,3) ipm-path", x, [[0, 1, 2], [3, 4, 5]], 1.0 / 1.2,
                    rng.standard_normal(n), y)


def config2(n: int = 60000, seed: int = 1002) -> Workload:
    rng = np.random.default_rng(seed)
    x = rng.uniform(-0.25, 0.25, size=(n, 8))
    return Workload("cfg2 n=60000 d=8 windows(3,3,2) matvec", x, [[0, 1, 2], [3, 4, 5], [6, 7]], 1.0,
                    rng.standard_normal(n))


def config3(n: int = 100000, seed: int = 1003) -> Workload:
    rng = np.random.default_rng(seed)
    u = rng.standard_normal(22)
    u /= np.linalg.norm(u)
    y = np.where(rng.uniform(size=n) < 0.5, 1.0, -1.0)
    x = minmax_quarter(rng.standard_normal((n, 22)) + 0.5 * y[:, None] * u[None, :])
    return Workload("cfg3 n=100000 d=22 windows(7x3,1) ipm-path", x, _triples(21) + [[21]], 1.0 / 1.2,
                    rng.standard_normal(n), y)


def config4(n: int = 500000, seed: int = 1004) -> Workload:
    rng = np.random.default_rng(seed)
    cont = rng.standard_normal((n, 10))
    binr = (rng.uniform(size=(n, 44)) < 0.1).astype(np.float64)
    x = minmax_quarter(np.concatenate([cont, binr], axis=1))
    return Workload("cfg4 n=500000 d=54 windows(18x3) matvec", x, _triples(54), 1.0,
                    rng.standard_normal(n))


def config5(n: int = 10_000_000, seed: int = 1005) -> Workload:
    rng = np.random.default_rng(seed)
    base = rng.standard_normal((n, 21))
    pairs = rng.integers(0, 21, size=(7, 2))
    derived = np.empty((n, 7))
    for k, (a, b) in enumerate(pairs):
        derived[:, k] = base[:, a] * base[:, b] if k % 2 == 0 else np.abs(base[:, a])
    x = np.concatenate([base, derived], axis=1)
    w1 = rng.standard_normal((28, 16)) / np.sqrt(28)
    w2 = rng.standard_normal(16) / 4.0
    y = np.where(np.tanh(x @ w1) @ w2 >= 0.0, 1.0, -1.0)
    x = minmax_quarter(x)
    return Workload("cfg5 n=10000000 d=28 windows(9x3,1) ipm-path", x, _triples(27) + [[27]], 1.0 / 1.2,
                    rng.standard_normal(n), y)


CONFIGS = {1: config1, 2: config2, 3: config3, 4: config4, 5: config5}


def make(cfg: int, n: int | None = None) -> Workload:
    f = CONFIGS[cfg]
    return f() if n is None else f(n=n)
