"""Seeded synthetic agent populations for the five BASELINE.json configs.

This module is shared by the oracle side (tests, bench cpu_baseline) and the
product side (bench, smoke).  It holds NO arithmetic of the method (no grid, no
force, no displacement): it only draws positions and diameters.

Counter-based uniform generator.  For (seed, id, stream):
    h = splitmix64_finalizer(seed * 0x9E3779B97F4A7C15 + (4*id + stream))  (mod 2^64)
    u = (h >> 11) * 2^-53                      in [0, 1)
    v = lo + (hi - lo) * u                     (one rounded multiply, one rounded add)
streams 0,1,2 = x,y,z and stream 3 = diameter.  The CUDA library carries its own
implementation of the same generator (kernel K0, ``bdm_generate_uniform``) so
that cfg4/cfg5 can be generated on the device; the two are compared bit for bit
in tests/test_gpu_parity.py.

Workload recipes (DESIGN.md §"Inputs"):
  cfg1  BASELINE.json configs[0]: N=4096, U[0,160)^3 um, D ~ U[8,12)          seed 1
  cfg2  configs[1]: 100^3 lattice of 10 um spacing, id=(i*100+j)*100+k,
        jitter U[-2,2) per component, D ~ U[9,11)                               seed 2
  cfg3  configs[2]: N=2e7, Gaussian N(0, sigma^2 I), sigma = 992.2 um
        (core density 1.3e-3 um^-3, reading R19), D = exp(ln 10 + 0.15 Z)
        clipped to [6,16]; numpy default_rng(3)                                 seed 3
  cfg4  configs[3]: N=2e8 uniform in [0,8a)x[0,a)x[0,a), a=(N/1e-3/8)^(1/3)     seed 4
  cfg5  configs[4]: N=1e9 uniform in [0,1e4)^3                                  seed 5
"""
from __future__ import annotations

import math

import numpy as np

MASK64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
TWO_M53 = 2.0 ** -53

CFG_N = {1: 4096, 2: 1_000_000, 3: 20_000_000, 4: 200_000_000, 5: 1_000_000_000}
CFG_STEPS = {1: 1, 2: 10, 3: 10, 4: 20, 5: 5}
CFG3_SIGMA = 992.2
DENSITY = 1.0e-3  # agents per um^3 (cfg2 lattice: one agent per 10^3 um^3)


def splitmix64(z: np.ndarray) -> np.ndarray:
    """SplitMix64 finalizer on uint64 arrays (wrapping arithmetic)."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def uniform01(seed: int, ids: np.ndarray, stream: int) -> np.ndarray:
    ids = np.asarray(ids, dtype=np.uint64)
    base = np.uint64((seed * GOLDEN) & MASK64)
    with np.errstate(over="ignore"):
        h = splitmix64(base + ids * np.uint64(4) + np.uint64(stream))
    return (h >> np.uint64(11)).astype(np.float64) * TWO_M53


def uniform(seed: int, ids: np.ndarray, stream: int, lo: float, hi: float) -> np.ndarray:
    u = uniform01(seed, ids, stream)
    return np.float64(lo) + np.float64(hi - lo) * u


def cfg4_side(n: int = CFG_N[4]) -> float:
    return (n / DENSITY / 8.0) ** (1.0 / 3.0)


def box_of(cfg: int, n: int | None = None):
    """(lo, hi) bounds per axis of the counter-hash configs (1, 4, 5)."""
    if cfg == 1:
        return (0.0, 0.0, 0.0), (160.0, 160.0, 160.0)
    if cfg == 4:
        a = cfg4_side(n if n is not None else CFG_N[4])
        return (0.0, 0.0, 0.0), (8.0 * a, a, a)
    if cfg == 5:
        return (0.0, 0.0, 0.0), (1.0e4, 1.0e4, 1.0e4)
    raise ValueError(cfg)


def uniform_population(seed: int, ids, lo3, hi3, dlo: float, dhi: float):
    ids = np.asarray(ids, dtype=np.uint64)
    pos = np.empty((ids.size, 3), dtype=np.float64)
    for ax in range(3):
        pos[:, ax] = uniform(seed, ids, ax, lo3[ax], hi3[ax])
    diam = uniform(seed, ids, 3, dlo, dhi)
    return pos, diam


def lattice_population(seed: int = 2, side: int = 100, spacing: float = 10.0,
                       jitter: float = 2.0, dlo: float = 9.0, dhi: float = 11.0):
    """cfg2: id = (i*side + j)*side + k at 10*(i,j,k) plus U[-2,2) jitter."""
    n = side ** 3
    ids = np.arange(n, dtype=np.uint64)
    i = (ids // np.uint64(side * side)).astype(np.float64)
    j = ((ids // np.uint64(side)) % np.uint64(side)).astype(np.float64)
    k = (ids % np.uint64(side)).astype(np.float64)
    pos = np.empty((n, 3), dtype=np.float64)
    for ax, c in enumerate((i, j, k)):
        pos[:, ax] = c * spacing + uniform(seed, ids, ax, -jitter, jitter)
    diam = uniform(seed, ids, 3, dlo, dhi)
    return pos, diam


def gaussian_population(n: int = CFG_N[3], seed: int = 3, sigma: float = CFG3_SIGMA):
    """cfg3: Gaussian cluster, log-normal diameters clipped to [6, 16]."""
    rng = np.random.default_rng(seed)
    pos = rng.standard_normal((n, 3)) * sigma
    z = rng.standard_normal(n)
    diam = np.clip(np.exp(math.log(10.0) + 0.15 * z), 6.0, 16.0)
    return np.ascontiguousarray(pos), np.ascontiguousarray(diam)


def make_config(cfg: int, n: int | None = None):
    """Host arrays (pos[n,3], diam[n]) for a config; n overrides N where meaningful."""
    if cfg == 1:
        n = CFG_N[1] if n is None else n
        lo, hi = box_of(1)
        return uniform_population(1, np.arange(n), lo, hi, 8.0, 12.0)
    if cfg == 2:
        side = 100 if n is None else int(round(n ** (1.0 / 3.0)))
        return lattice_population(2, side)
    if cfg == 3:
        return gaussian_population(CFG_N[3] if n is None else n)
    if cfg in (4, 5):
        n = CFG_N[cfg] if n is None else n
        lo, hi = box_of(cfg, n)
        return uniform_population(cfg, np.arange(n), lo, hi, 8.0, 12.0)
    raise ValueError(cfg)


def random_instance(seed: int, n: int, side: float, dlo: float = 8.0, dhi: float = 12.0):
    """Small random instances for oracle cross-checks (varied density)."""
    rng = np.random.default_rng(seed)
    pos = rng.uniform(-0.5 * side, 0.5 * side, size=(n, 3))
    diam = rng.uniform(dlo, dhi, size=n)
    return pos, diam
