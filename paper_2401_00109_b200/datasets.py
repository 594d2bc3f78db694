"""Seeded synthetic inputs with the shapes of BASELINE.json's five configs.

The reference's benchmarks use synthetic generators too (bench.hpp:27-86);
BASELINE.json's configs name no public dataset, so these numpy generators
stand in. They are NOT the reference's exact draw sequence:
parity is always checked by feeding the SAME generated array to the oracle
and to the GPU path, never by regenerating.

``scale`` shrinks a config (fewer series / shorter series) for tests while
keeping its layout, tolerances and digitization parameters.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
from scipy.signal import lfilter

# layouts (core.hpp:55)
UNIVARIATE_PARTITIONED, MULTIVARIATE, COLLECTION = 0, 1, 2


@dataclass
class Workload:
    name: str
    values: np.ndarray            # all series concatenated (float64)
    series_lengths: np.ndarray    # samples per series (int64)
    layout: int
    parts: int                    # partitions per series
    cfg: dict = field(default_factory=dict)  # jb_config overrides

    @property
    def n_points(self) -> int:
        return int(self.values.size)


def _znorm_rows(x: np.ndarray) -> np.ndarray:
    mu = x.mean(axis=-1, keepdims=True)
    sd = x.std(axis=-1, keepdims=True)
    sd[sd == 0] = 1.0
    return (x - mu) / sd


def _walks(rng, n_series, length):
    x = np.zeros((n_series, length))
    x[:, 1:] = np.cumsum(rng.standard_normal((n_series, length - 1)), axis=1)
    return _znorm_rows(x)


def _sines(rng, n_series, length):
    t = np.arange(length, dtype=np.float64)
    out = np.empty((n_series, length))
    for i in range(n_series):
        P = rng.uniform(20, 500, 3)
        A = rng.uniform(0.5, 2.0, 3)
        ph = rng.uniform(0, 2 * np.pi, 3)
        s = (A[:, None] * np.sin(2 * np.pi * t[None, :] / P[:, None] + ph[:, None])).sum(0)
        out[i] = s + rng.normal(0.0, 0.1, length)
    return _znorm_rows(out)


def config1(scale: float = 1.0) -> Workload:
    """64 z-normed random walks x 2000, tol .05, svq k=50 r=.5 (PR1 workload)."""
    rng = np.random.default_rng(0)
    ns = max(1, int(round(64 * scale)))
    x = _walks(rng, ns, 2000)
    return Workload("cfg1", x.reshape(-1), np.full(ns, 2000, np.int64), COLLECTION, 1,
                    dict(tol=0.05, backend="svq", k=50, r=0.5, seed=0, scl=1.0))


def config2(scale: float = 1.0) -> Workload:
    """1000 x 10000 3-sinusoid + noise, tol .1, GA alpha .1 two-norm, 4 parts."""
    rng = np.random.default_rng(2)
    ns = max(1, int(round(1000 * scale)))
    x = _sines(rng, ns, 10000)
    return Workload("cfg2", x.reshape(-1), np.full(ns, 10000, np.int64), COLLECTION, 4,
                    dict(tol=0.1, backend="ga", alpha=0.1, sort_key=1, early_stop=1, scl=1.0))


def config3(scale: float = 1.0) -> Workload:
    """1000 samples x 64 AR(1) channels x 4096 (shared-factor corr .5), joint
    fit over all channels; tol .05, svq k=100 r=.3."""
    rng = np.random.default_rng(3)
    ns = max(1, int(round(1000 * scale)))
    length = 4096
    out = np.empty((ns, 64, length))
    for s in range(ns):
        f = rng.standard_normal(length)
        e = np.sqrt(0.5) * f[None, :] + np.sqrt(0.5) * rng.standard_normal((64, length))
        out[s] = _znorm_rows(lfilter([1.0], [1.0, -0.95], e, axis=-1))
    return Workload("cfg3", out.reshape(-1), np.full(ns * 64, length, np.int64), COLLECTION, 1,
                    dict(tol=0.05, backend="svq", k=100, r=0.3, seed=0, scl=1.0))


def config4(scale: float = 1.0, partitions: int | None = None) -> Workload:
    """One random walk of 1e9 samples with N(0,5) level shifts at Poisson
    times (mean gap 1e6), 10,000 partitions; tol .1, svq k=200 r=.1."""
    rng = np.random.default_rng(4)
    n = max(1000, int(round(1e9 * scale)))
    m = partitions if partitions is not None else max(1, int(round(10000 * scale)))
    steps = rng.standard_normal(n - 1)
    gap = 1e6 * max(scale, 1e-3)
    t = 0.0
    while True:
        t += rng.exponential(gap)
        if t >= n - 1:
            break
        steps[int(t)] += rng.normal(0.0, 5.0)
    x = np.empty(n)
    x[0] = 0.0
    np.cumsum(steps, out=x[1:])
    return Workload("cfg4", x, np.array([n], np.int64), UNIVARIATE_PARTITIONED, m,
                    dict(tol=0.1, backend="svq", k=200, r=0.1, seed=0, scl=1.0))


def config5(scale: float = 1.0) -> Workload:
    """10,000 x 100,000, 50/50 z-normed walks and noisy 3-sinusoids, 8 parts
    per series; tol .05, svq k=500 r=.2."""
    rng = np.random.default_rng(5)
    ns = max(2, int(round(10000 * scale)))
    length = 100000
    out = np.empty((ns, length))
    for i in range(ns):
        out[i] = (_walks(rng, 1, length) if i % 2 == 0 else _sines(rng, 1, length))[0]
    return Workload("cfg5", out.reshape(-1), np.full(ns, length, np.int64), COLLECTION, 8,
                    dict(tol=0.05, backend="svq", k=500, r=0.2, seed=0, scl=1.0))


CONFIGS = {1: config1, 2: config2, 3: config3, 4: config4, 5: config5}


def small(cfg_id: int, seed_scale: float | None = None) -> Workload:
    """Oracle-sized variants (finish in seconds on the CPU oracle)."""
    if cfg_id == 1:
        return config1(1.0)
    if cfg_id == 2:
        return config2(0.02)
    if cfg_id == 3:
        return config3(0.001)
    if cfg_id == 4:
        return config4(2e-4)
    if cfg_id == 5:
        w = config5(2e-4)
        return w
    raise ValueError(cfg_id)
