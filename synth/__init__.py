"""Seeded synthetic input generators shared by tests, smoke() and bench.py.

Holds NONE of the method's arithmetic (no factorisation, solve, stencil or
time step): only the input recipes of DESIGN.md §5, each a numpy PCG64 stream
with a stated seed, so the CUDA path and the CPU oracle see identical bytes
(SURVEY §8(c) reading r17: "generate inputs on the host once").
"""
from __future__ import annotations

import math
import numpy as np


def rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


# --------------------------------------------------------------- banded LHS
def dd_penta(n: int, count: int = 1, seed: int = 1):
    """Random diagonally-dominant pentadiagonal diagonals (cfg1 recipe):
    a,b,d,e ~ U(-1,1), c = |a|+|b|+|d|+|e| + U(0.5,1.5).  Arrays of n*count,
    interleaved [i*count + s]."""
    g = rng(seed)
    a, b, d, e = (g.uniform(-1.0, 1.0, size=n * count) for _ in range(4))
    c = np.abs(a) + np.abs(b) + np.abs(d) + np.abs(e) + g.uniform(0.5, 1.5, size=n * count)
    return a, b, c, d, e


def dd_tri(n: int, count: int = 1, seed: int = 11):
    g = rng(seed)
    a, c = (g.uniform(-1.0, 1.0, size=n * count) for _ in range(2))
    b = np.abs(a) + np.abs(c) + g.uniform(0.5, 1.5, size=n * count)
    return a, b, c


def const_penta(n: int, a: float, b: float, c: float, d: float, e: float):
    """Constant diagonals (the CN / ADI hyperdiffusion matrix of P:1486 has
    (sigma, -4 sigma, 1 + 6 sigma, -4 sigma, sigma))."""
    return tuple(np.full(n, v, dtype=np.float64) for v in (a, b, c, d, e))


def const_tri(n: int, a: float, b: float, c: float):
    return tuple(np.full(n, v, dtype=np.float64) for v in (a, b, c))


def hyper_sigma(dx: float, dt: float, D: float = 1.0, gamma: float = 0.01) -> float:
    """sigma of the ADI operator L_x = I + 2/3 D gamma dt d_xxxx."""
    return (2.0 / 3.0) * D * gamma * dt / dx ** 4


# thesis statistics grid spacing: dx = 2 pi / 256, dt = 0.1 dx
DX_STATS = 2.0 * math.pi / 256.0
SIGMA_STATS = hyper_sigma(DX_STATS, 0.1 * DX_STATS)  # = 45.09, kappa = 1 + 16 sigma = 722


# --------------------------------------------------------------- right-hand sides
def rhs_uniform(n: int, m: int, seed: int = 2, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    return rng(seed).uniform(lo, hi, size=n * m)


def rhs_normal(n: int, m: int, seed: int = 1) -> np.ndarray:
    return rng(seed).standard_normal(size=n * m)


# --------------------------------------------------------------- Cahn–Hilliard states
def ch_ic_random(sims: int, n: int, seed: int = 3, lo: float = -0.1, hi: float = 0.1) -> np.ndarray:
    """U(lo, hi) quench (symmetric +-0.1 P:1167/4213; asymmetric 0.4..0.6 P:3960);
    simulation k uses seed + k (r17).  Shape (sims, n, n), row-major [j][i]."""
    out = np.empty((sims, n, n))
    for k in range(sims):
        out[k] = rng(seed + k).uniform(lo, hi, size=(n, n))
    return out


def ch_ic_tanh(n: int, L: float = 2 * math.pi, eps: float = 1e-6) -> np.ndarray:
    """Table 3.1 IC eps*tanh(r - pi), r measured from the domain centre (r10):
    x, y = -L/2 + i dx, dx = L/n (r1)."""
    dx = L / n
    x = -L / 2 + dx * np.arange(n)
    X, Y = np.meshgrid(x, x, indexing="xy")  # X varies along i (columns)
    return eps * np.tanh(np.sqrt(X ** 2 + Y ** 2) - math.pi)


def ch_ic_cos1d(n: int, L: float = 2 * math.pi, eps: float = 1e-6, k: int = 5) -> np.ndarray:
    """Table 6.1 IC eps*cos(5x), x = i dx (r11)."""
    x = (L / n) * np.arange(n)
    return eps * np.cos(k * x)


def ch_dt(n: int, L: float) -> float:
    """dt = 0.1 dx with dx = L/n (r1, r2)."""
    return 0.1 * L / n


def ch_nsteps(T: float, dt: float) -> int:
    """ceil(T/dt) steps (r3), guarded against round-off just above an integer."""
    q = T / dt
    r = round(q)
    return int(r) if abs(q - r) < 1e-9 * max(1.0, q) else int(math.ceil(q))
