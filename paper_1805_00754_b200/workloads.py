"""Seeded synthetic workloads of BASELINE.json's configs.

There is no public dataset for this path (the paper's UCI Activity / Gas /
London series are absent and not needed); these generators stand in with the
shapes, sizes and value distributions BASELINE.json names.  numpy PCG64 with a
recorded seed, fp64, row-major t x c.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    t: int
    c: int
    b: int
    k: int
    seed: int


CONFIGS = {
    "cfg1": Config("cfg1", 100_000, 16, 1_000, 10, 1),
    "cfg2": Config("cfg2", 1_000_000, 64, 2_000, 20, 2),
    "cfg3": Config("cfg3", 4_000_000, 256, 4_000, 30, 3),
    "cfg4": Config("cfg4", 10_000_000, 32, 1_000, 10, 4),
    "cfg5": Config("cfg5", 2_000_000, 1024, 8_192, 64, 5),
}


def _sinusoid_mix(rng, t0: int, t: int, nf: int, c: int, pmin: float, pmax: float, log_periods=False):
    if log_periods:
        periods = np.exp(rng.uniform(np.log(pmin), np.log(pmax), nf))
    else:
        periods = rng.uniform(pmin, pmax, nf)
    phases = rng.uniform(0.0, 2.0 * np.pi, nf)
    load = rng.standard_normal((nf, c))
    return periods, phases, load


def generate(name: str, rows: int | None = None, seed: int | None = None) -> np.ndarray:
    """First ``rows`` rows (default: all t) of config ``name``."""
    cfg = CONFIGS[name]
    t = cfg.t if rows is None else int(rows)
    rng = np.random.default_rng(cfg.seed if seed is None else seed)
    tt = np.arange(t, dtype=np.float64)[:, None]
    c = cfg.c
    if name in ("cfg1", "cfg4"):
        nf, noise = (5, 0.1) if name == "cfg1" else (6, 0.1)
        periods, phases, load = _sinusoid_mix(rng, 0, t, nf, c, 50.0, 5000.0)
        x = np.sin(2 * np.pi * tt / periods[None, :] + phases[None, :]) @ load
        x += noise * rng.standard_normal((t, c))
    elif name == "cfg2":
        # per-series Gaussian random walk (sigma 0.01) + 8 shared seasonal sinusoids
        # (periods 24..10,000) with random loadings + N(0, 0.05^2)
        periods, phases, load = _sinusoid_mix(rng, 0, t, 8, c, 24.0, 10_000.0, log_periods=True)
        x = np.cumsum(0.01 * rng.standard_normal((t, c)), axis=0)
        x += np.sin(2 * np.pi * tt / periods[None, :] + phases[None, :]) @ load
        x += 0.05 * rng.standard_normal((t, c))
    elif name == "cfg3":
        periods, phases, load = _sinusoid_mix(rng, 0, t, 20, c, 50.0, 20_000.0, log_periods=True)
        x = np.sin(2 * np.pi * tt / periods[None, :] + phases[None, :]) @ load
        x += 0.1 * rng.standard_t(3.0, (t, c))
    elif name == "cfg5":
        periods, phases, load = _sinusoid_mix(rng, 0, t, 50, c, 50.0, 50_000.0, log_periods=True)
        x = np.sin(2 * np.pi * tt / periods[None, :] + phases[None, :]) @ load
        x += 0.2 * rng.standard_normal((t, c))
    else:
        raise KeyError(name)
    return np.ascontiguousarray(x, dtype=np.float64)


def query_lengths(name: str):
    """Query length sets of SURVEY §8(d)."""
    if name == "cfg2":
        return [10_000 * 2 ** j for j in range(6)]
    if name == "cfg3":
        return [320_000]
    if name == "cfg5":
        return [10_000 * 2 ** j for j in range(8)]
    return [10_000, 50_000]


def query_offsets(total_rows: int, length: int, n: int, seed: int = 42) -> np.ndarray:
    """cmd_bench protocol (commands.hpp:253-266): one seeded offset sequence,
    reused for every length, uniform in [0, total_rows - length]."""
    rng = np.random.default_rng(seed)
    return rng.integers(0, total_rows - length + 1, size=n)
