"""Seeded synthetic workloads with the shapes of BASELINE.json's configs.

BASELINE.json names no public dataset (the paper's UCI Adult / Medical-Cost
tables are absent and are not reconstructed), so these seeded generators stand
in for every config:

  C1  4096 x U[0.01, 1]  -> crypto_invsqrt, degree 15 / 2 iters and 511 / 6
  C2  32768 x N(50, 10^2) -> znorm, B = 100 (also B = 20)
  C3  32768 x N(0, 1) and 32768 x LogNormal(0, 0.5) -> skewness + kurtosis, B = 20
  C4  8 x 32768, pairwise rho = 0.6, unit variance -> 28 pearson pairs, B = 20

Uniforms use the reference's platform-stable construction (mt19937_64,
``(r >> 11) * 2^-53``, data.hpp:148-160) through whichever ``uniform(seed, n,
lo, hi)`` the caller passes (the product's ``synthetic_uniform`` or an
oracle's).  Normals are Box-Muller over that stream with Python's ``math``
(libm), never numpy's ziggurat, so one seed gives one input everywhere the
same libm runs.
"""
from __future__ import annotations

import math
from typing import Callable, Optional, Tuple

import numpy as np

Uniform = Callable[[int, int, float, float], np.ndarray]


def box_muller(uniform: Uniform, seed: int, n: int) -> np.ndarray:
    """n standard normals from the mt19937_64 stream of ``seed``."""
    m = (n + 1) // 2
    u = uniform(seed, 2 * m, 0.0, 1.0)
    out = np.empty(2 * m)
    two_pi = 2.0 * math.pi
    for i in range(m):
        r = math.sqrt(-2.0 * math.log(1.0 - u[2 * i]))
        t = two_pi * u[2 * i + 1]
        out[2 * i] = r * math.cos(t)
        out[2 * i + 1] = r * math.sin(t)
    return out[:n]


def normal(uniform: Uniform, seed: int, n: int, mu: float, sigma: float) -> np.ndarray:
    return mu + sigma * box_muller(uniform, seed, n)


def lognormal(uniform: Uniform, seed: int, n: int, mu: float, sigma: float) -> np.ndarray:
    z = box_muller(uniform, seed, n)
    return np.array([math.exp(mu + sigma * v) for v in z])


def correlated_table(uniform: Uniform, seed: int, cols: int, n: int, rho: float) -> np.ndarray:
    """cols x n, x_k = sqrt(rho) z + sqrt(1 - rho) e_k (pairwise rho, unit variance)."""
    z = box_muller(uniform, seed, n)
    a, b = math.sqrt(rho), math.sqrt(1.0 - rho)
    return np.stack([a * z + b * box_muller(uniform, seed + 1 + k, n) for k in range(cols)])


DEFAULT_CFG = dict(n=2, cheb_degree=511, newton_iters=6, baseline_mode=False, baseline_iters=0)

# api / kwargs follow tests/oracle_abi.py (which: 0 invsqrt; stat 4 znorm 5 kurt 6 skew 8 pearson)
CONFIG_CASES = {
    "C1_d15": dict(api="invroot", params=dict(slot_count=4096), gen=("uniform", 11, 4096, 0.01, 1.0),
                   kwargs=dict(which=0, lx=11, S=1.0, n_valid=4096,
                               cfg=dict(DEFAULT_CFG, cheb_degree=15, newton_iters=2))),
    "C1_d511": dict(api="invroot", params=dict(slot_count=4096), gen=("uniform", 11, 4096, 0.01, 1.0),
                    kwargs=dict(which=0, lx=11, S=1.0, n_valid=4096, cfg=dict(DEFAULT_CFG))),
    "C2_B100": dict(api="stat", params=dict(slot_count=32768), gen=("normal", 21, 32768, 50.0, 10.0),
                    kwargs=dict(which=4, B=100.0, cfg=dict(DEFAULT_CFG))),
    "C2_B20": dict(api="stat", params=dict(slot_count=32768), gen=("normal", 21, 32768, 50.0, 10.0),
                   kwargs=dict(which=4, B=20.0, cfg=dict(DEFAULT_CFG))),
    "C3_skew_normal": dict(api="stat", params=dict(slot_count=32768), gen=("normal", 31, 32768, 0.0, 1.0),
                           kwargs=dict(which=6, B=20.0, cfg=dict(DEFAULT_CFG))),
    "C3_kurt_normal": dict(api="stat", params=dict(slot_count=32768), gen=("normal", 31, 32768, 0.0, 1.0),
                           kwargs=dict(which=5, B=20.0, cfg=dict(DEFAULT_CFG))),
    "C3_skew_lognormal": dict(api="stat", params=dict(slot_count=32768), gen=("lognormal", 32, 32768, 0.0, 0.5),
                              kwargs=dict(which=6, B=20.0, cfg=dict(DEFAULT_CFG))),
    "C3_kurt_lognormal": dict(api="stat", params=dict(slot_count=32768), gen=("lognormal", 32, 32768, 0.0, 0.5),
                              kwargs=dict(which=5, B=20.0, cfg=dict(DEFAULT_CFG))),
}
C4_SEED, C4_COLS, C4_ROWS, C4_RHO = 41, 8, 32768, 0.6
C4_PAIRS = [(i, j) for i in range(C4_COLS) for j in range(i + 1, C4_COLS)]
for _i, _j in C4_PAIRS:
    CONFIG_CASES[f"C4_p{_i}{_j}"] = dict(api="stat", params=dict(slot_count=32768), gen=("table", _i, _j),
                                          kwargs=dict(which=8, B=20.0, cfg=dict(DEFAULT_CFG)))

_table_cache = {}


def c4_table(uniform: Uniform) -> np.ndarray:
    key = id(uniform)
    if key not in _table_cache:
        _table_cache[key] = correlated_table(uniform, C4_SEED, C4_COLS, C4_ROWS, C4_RHO)
    return _table_cache[key]


def make_inputs(spec: dict, uniform: Uniform) -> Tuple[np.ndarray, Optional[np.ndarray]]:
    g = spec["gen"]
    if g[0] == "uniform":
        return uniform(g[1], g[2], g[3], g[4]), None
    if g[0] == "normal":
        return normal(uniform, g[1], g[2], g[3], g[4]), None
    if g[0] == "lognormal":
        return lognormal(uniform, g[1], g[2], g[3], g[4]), None
    if g[0] == "table":
        t = c4_table(uniform)
        return t[g[1]].copy(), t[g[2]].copy()
    raise ValueError(g)
