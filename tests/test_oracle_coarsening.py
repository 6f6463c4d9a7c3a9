"""Pins of the oracle's coarsening-statistics functions:
free energy F (reading r24), growth rate beta (r27), the
Cahn–Hilliard–Cook noise (r25/r26).  Closed forms, exact
discrete identities and moments -- none re-derives the oracle's own loop."""
import math

import numpy as np
import pytest

import oracle
import synth


def test_free_energy_constant_state():
    """C = c everywhere: no gradient, F = 1/4 (c^2 - 1)^2 |Omega| (reading r24)."""
    for c, L in ((0.5, 1.0), (-0.25, 4 * math.pi), (1.0, 2.0)):
        F = oracle.ch_free_energy(np.full((1, 16, 16), c), L=L, gamma=0.01)
        assert F[0] == pytest.approx(0.25 * (c * c - 1) ** 2 * L * L, rel=1e-14, abs=1e-15)


@pytest.mark.parametrize("axis", [0, 1])
def test_free_energy_single_mode_closed_form(axis):
    """C = eps cos(2 pi k i / n) along x (or y): sum cos^2 = n/2, sum cos^4 = 3n/8
    (0 < 4k < n) and sum (cos th_{i+1} - cos th_i)^2 = 2 n sin^2(pi k / n), so
    F = dx^2 n^2/4 (1 - eps^2 + 3 eps^4 / 8) + gamma eps^2 n^2 sin^2(pi k/n)."""
    n, k, eps, L, gam = 32, 3, 0.3, 2.0, 0.07
    dx = L / n
    m = eps * np.cos(2 * math.pi * k * np.arange(n) / n)
    c = np.tile(m, (n, 1)) if axis == 0 else np.tile(m[:, None], (1, n))
    F = oracle.ch_free_energy(c[None], L=L, gamma=gam)[0]
    exact = dx * dx * n * n / 4 * (1 - eps ** 2 + 3 * eps ** 4 / 8) + gam * eps ** 2 * n * n * math.sin(math.pi * k / n) ** 2
    assert F == pytest.approx(exact, rel=1e-13)


def test_free_energy_batch_and_decrease_along_adi():
    """Batch entries are independent; F decreases along the scheme (P:822-824:
    the decay is what fixes the bulk coefficient 1/4 of reading r24) in the
    regime of test_ch_free_energy_decreases (n = 32, L = 4 pi, 6 x 20 steps)."""
    n, L = 32, 4 * math.pi
    dt = synth.ch_dt(n, L)
    c0 = synth.ch_ic_random(2, n, seed=6)
    F0 = oracle.ch_free_energy(c0, L=L, gamma=0.01)
    assert F0[1] == pytest.approx(oracle.ch_free_energy(c0[1:], L=L, gamma=0.01)[0], rel=1e-15)
    cn, cm, prev = c0, c0, F0
    for _ in range(6):
        cn, cm = oracle.ch_adi_steps(cn, cm, 20, dt=dt, D=1.0, gamma=0.01, L=L)
        F = oracle.ch_free_energy(cn, L=L, gamma=0.01)
        assert np.all(F <= prev + 1e-12)
        prev = F
    assert np.all(prev < 0.9 * F0)


def test_beta_closed_forms():
    """F = 10 - t: central differences are exact, beta = t / (10 - t).
    F = t^(-p): the central difference is F' + F'(3) h^2/6 + O(h^4), so inside
    beta_h = p + p(p+1)(p+2) h^2 / (6 t^2) + O(h^4); one-sided ends O(h)."""
    t = np.linspace(1.0, 3.0, 41)
    F = np.stack([10.0 - t, t ** (-1.0 / 3.0)], axis=1)
    beta = oracle.coarsening_beta(t, F)
    assert np.allclose(beta[:, 0], t / (10 - t), rtol=1e-13)
    p, h = 1.0 / 3.0, t[1] - t[0]
    lead = p + p * (p + 1) * (p + 2) * h * h / (6 * t[1:-1] ** 2)
    assert np.max(np.abs(beta[1:-1, 1] - lead)) < 2e-6
    assert np.max(np.abs(beta[[0, -1], 1] - 1.0 / 3.0)) < 2e-2


def test_cook_rho_moments_and_determinism():
    """(rho_x, rho_y) are independent N(0,1): mean, variance, correlation and
    kurtosis over 2e5 cells; the same counter gives the same pair."""
    rx = np.empty(200000)
    ry = np.empty(200000)
    for k in range(rx.size):
        rx[k], ry[k] = oracle.cook_rho(7, 3, 1, k)
    for r in (rx, ry):
        assert abs(r.mean()) < 0.01 and abs(r.var() - 1) < 0.015
        assert abs(np.mean(r ** 4) / r.var() ** 2 - 3) < 0.05
    assert abs(np.corrcoef(rx, ry)[0, 1]) < 0.01
    assert oracle.cook_rho(7, 3, 1, 12345) == (rx[12345], ry[12345])
    assert oracle.cook_rho(7, 4, 1, 12345) != (rx[12345], ry[12345])
    assert oracle.cook_rho(7, 3, 2, 12345) != (rx[12345], ry[12345])


def test_cook_noise_structure():
    """eta = amp div rho: sums to 0 on the periodic grid; Var = amp^2 / dx^2
    (four independent normals / (2 dx)); correlation -1/4 at distance 2 along
    x or y, 0 at distance 1 (the central-difference stencil); eta scales as
    sqrt(sigma) with the same draws."""
    sims, n, L, dt, sigma = 2, 128, 2.0, 1e-3, 1e-14
    dx = L / n
    eta = oracle.cook_noise(sims, n, dt=dt, L=L, sigma=sigma, seed=5, step=9)
    amp2 = sigma / (dx * dx * dt)
    for s in range(sims):
        assert abs(eta[s].sum()) <= 1e-12 * np.abs(eta[s]).sum()
    v = eta.var() / (amp2 / dx ** 2)
    assert abs(v - 1) < 0.03
    e = eta / math.sqrt(amp2 / dx ** 2)
    for ax in (1, 2):
        c2 = np.mean(e * np.roll(e, 2, axis=ax))
        c1 = np.mean(e * np.roll(e, 1, axis=ax))
        assert abs(c2 + 0.25) < 0.02 and abs(c1) < 0.02
    eta4 = oracle.cook_noise(sims, n, dt=dt, L=L, sigma=4 * sigma, seed=5, step=9)
    assert np.allclose(eta4, 2 * eta, rtol=1e-15, atol=0)


def test_cook_adi_reduces_and_conserves():
    """sigma = 0 is the plain scheme bitwise; with noise (IC 0) the mass
    stays 0 to rounding and the field grows from the fluctuations only."""
    n, L = 64, 64 * synth.DX_STATS
    dt = synth.ch_dt(n, L)
    c0 = synth.ch_ic_random(1, n, seed=12)
    a = oracle.ch_adi_steps(c0, c0, 3, dt=dt, D=1.0, gamma=0.01, L=L)
    b = oracle.ch_adi_steps_cook(c0, c0, 3, dt=dt, D=1.0, gamma=0.01, L=L, sigma=0.0, seed=1)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    z = np.zeros((1, n, n))
    cn, cm = oracle.ch_adi_steps_cook(z, z, 5, dt=dt, D=1.0, gamma=0.01, L=L, sigma=1e-14, seed=3)
    assert np.max(np.abs(cn)) > 0
    assert abs(cn.sum()) <= 1e-13 * np.abs(cn).sum()
