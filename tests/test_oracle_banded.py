"""Pins for the oracle's banded solvers (penta LR, Navon cyclic, Thomas, Sherman–Morrison).

Every pin compares against something the oracle does not compute itself:
dense LU (numpy.linalg.solve), the L*R product, circulant eigenvalues (FFT),
manufactured solutions, the row-sum identity and the hand value of SPEC S:74.
"""
import numpy as np
import pytest

import oracle
import synth


def dense_penta(a, b, c, d, e, periodic):
    n = c.size
    A = np.zeros((n, n))
    for i in range(n):
        for off, v in ((-2, a[i]), (-1, b[i]), (0, c[i]), (1, d[i]), (2, e[i])):
            j = i + off
            if periodic:
                A[i, j % n] += v
            elif 0 <= j < n:
                A[i, j] = v
    return A


def dense_tri(a, b, c, periodic):
    n = b.size
    A = np.zeros((n, n))
    for i in range(n):
        for off, v in ((-1, a[i]), (0, b[i]), (1, c[i])):
            j = i + off
            if periodic:
                A[i, j % n] += v
            elif 0 <= j < n:
                A[i, j] = v
    return A


def relerr(x, ref):
    return np.max(np.abs(x - ref)) / np.max(np.abs(ref))


# ------------------------------------------------------------------ penta LR
@pytest.mark.parametrize("n", [5, 6, 7, 8, 13, 32, 64])
def test_penta_factor_reconstructs_A(n):
    a, b, c, d, e = synth.dd_penta(n, 1, seed=100 + n)
    al, be, ga, de, ep = oracle.penta_factor(a, b, c, d, e)
    L = np.diag(al) + np.diag(be[1:], -1) + np.diag(ep[2:], -2)
    R = np.eye(n) + np.diag(ga[:-1], 1) + np.diag(de[:-2], 2)
    A = dense_penta(a, b, c, d, e, periodic=False)
    assert np.max(np.abs(L @ R - A)) <= 1e-12 * np.max(np.abs(A))


@pytest.mark.parametrize("n", [5, 9, 16, 64])
def test_penta_solve_vs_dense_lu(n):
    m = 7
    a, b, c, d, e = synth.dd_penta(n, m, seed=n)
    f = synth.rhs_normal(n, m, seed=n + 1)
    x = oracle.penta_batch_solve(a, b, c, d, e, f, n=n, m=m)
    for s in range(m):
        A = dense_penta(a[s::m], b[s::m], c[s::m], d[s::m], e[s::m], periodic=False)
        ref = np.linalg.solve(A, f[s::m])
        assert relerr(x[s::m], ref) <= 1e-13


def test_penta_identity_and_manufactured():
    n, m = 40, 3
    z = np.zeros(n)
    x = oracle.penta_batch_solve(z, z, np.ones(n), z, z, np.arange(n * m, dtype=float), n=n, m=m)
    assert np.array_equal(x, np.arange(n * m, dtype=float))
    a, b, c, d, e = synth.dd_penta(n, 1, seed=5)
    xt = synth.rhs_normal(n, 1, seed=6)
    A = dense_penta(a, b, c, d, e, periodic=False)
    x = oracle.penta_batch_solve(a, b, c, d, e, A @ xt, n=n, m=1)
    assert relerr(x, xt) <= 1e-13


def test_penta_layouts_agree_and_shared_lhs():
    n, m = 33, 5
    a, b, c, d, e = synth.dd_penta(n, 1, seed=8)
    f = synth.rhs_normal(n, m, seed=9)  # interleaved
    xi = oracle.penta_batch_solve(a, b, c, d, e, f, n=n, m=m, layout="interleaved")
    fc = f.reshape(n, m).T.reshape(-1)  # contiguous copy
    xc = oracle.penta_batch_solve(a, b, c, d, e, fc, n=n, m=m, layout="contiguous")
    assert np.array_equal(xc.reshape(m, n).T.reshape(-1), xi)
    # shared LHS == per-system LHS with identical copies (regime equivalence)
    rep = [np.repeat(v, m) for v in (a, b, c, d, e)]
    xp = oracle.penta_batch_solve(*rep, f, n=n, m=m)
    assert np.array_equal(xp, xi)


def test_penta_zero_pivot():
    n = 8
    a, b, c, d, e = synth.dd_penta(n, 1, seed=3)
    c = c.copy()
    c[0] = 0.0
    with pytest.raises(oracle.OracleError) as ei:
        oracle.penta_factor(a, b, c, d, e)
    assert ei.value.code == oracle.EZEROPIVOT and ei.value.row == 0


# ------------------------------------------------------------------ cyclic penta (Navon)
@pytest.mark.parametrize("n", [7, 8, 12, 31, 64])
def test_cyclic_penta_vs_dense_lu(n):
    m = 4
    a, b, c, d, e = synth.dd_penta(n, m, seed=200 + n)
    f = synth.rhs_normal(n, m, seed=300 + n)
    x = oracle.penta_batch_solve(a, b, c, d, e, f, n=n, m=m, periodic=True)
    for s in range(m):
        A = dense_penta(a[s::m], b[s::m], c[s::m], d[s::m], e[s::m], periodic=True)
        assert relerr(x[s::m], np.linalg.solve(A, f[s::m])) <= 1e-12


@pytest.mark.parametrize("n,sigma", [(12, 0.1), (64, 45.09), (256, synth.SIGMA_STATS), (128, 2886.0)])
def test_cyclic_penta_circulant_closed_form(n, sigma):
    """Constant coefficients => circulant; x = IFFT(FFT(f)/lambda_k) with
    lambda_k = sum_o c_o exp(2 pi i o k/N) = 1 + 16 sigma sin^4(pi k/N)."""
    a, b, c, d, e = synth.const_penta(n, sigma, -4 * sigma, 1 + 6 * sigma, -4 * sigma, sigma)
    f = synth.rhs_uniform(n, 1, seed=n)
    x = oracle.penta_batch_solve(a, b, c, d, e, f, n=n, m=1, periodic=True)
    k = np.arange(n)
    lam = 1 + 16 * sigma * np.sin(np.pi * k / n) ** 4
    ref = np.real(np.fft.ifft(np.fft.fft(f) / lam))
    kappa = 1 + 16 * sigma
    assert relerr(x, ref) <= 2e-16 * kappa * 10


def test_cyclic_penta_rowsum_identity():
    """CN hyperdiffusion rows sum to 1, so A*1 = 1 and rhs = 1 gives x = 1."""
    n, s = 50, 5.2429e-3
    a, b, c, d, e = synth.const_penta(n, s, -4 * s, 1 + 6 * s, -4 * s, s)
    x = oracle.penta_batch_solve(a, b, c, d, e, np.ones(n), n=n, m=1, periodic=True)
    assert np.max(np.abs(x - 1)) <= 1e-14


def test_cyclic_penta_trivial_wrap():
    n = 20
    z = np.zeros(n)
    f = synth.rhs_normal(n, 1, seed=4)
    x = oracle.penta_batch_solve(z, z, np.ones(n), z, z, f, n=n, m=1, periodic=True)
    assert np.array_equal(x, f)


# ------------------------------------------------------------------ Thomas + Sherman–Morrison
def test_thomas_hand_value():
    """diffusion row a=c=-0.25, b=1.5 => chat_1 = -1/6."""
    a, b, c = synth.const_tri(6, -0.25, 1.5, -0.25)
    ch = oracle.tri_factor(a, b, c)
    assert ch[0] == pytest.approx(-1.0 / 6.0, abs=1e-16)


@pytest.mark.parametrize("n", [3, 6, 17, 64])
def test_thomas_vs_dense(n):
    m = 5
    a, b, c = synth.dd_tri(n, m, seed=n)
    f = synth.rhs_normal(n, m, seed=n + 7)
    x = oracle.tri_batch_solve(a, b, c, f, n=n, m=m)
    for s in range(m):
        A = dense_tri(a[s::m], b[s::m], c[s::m], periodic=False)
        assert relerr(x[s::m], np.linalg.solve(A, f[s::m])) <= 1e-13


@pytest.mark.parametrize("n", [3, 8, 64])
def test_sherman_morrison_vs_dense(n):
    m = 3
    a, b, c = synth.dd_tri(n, m, seed=40 + n)
    f = synth.rhs_normal(n, m, seed=41 + n)
    x = oracle.tri_batch_solve(a, b, c, f, n=n, m=m, periodic=True)
    for s in range(m):
        A = dense_tri(a[s::m], b[s::m], c[s::m], periodic=True)
        assert relerr(x[s::m], np.linalg.solve(A, f[s::m])) <= 1e-12


def test_sherman_morrison_closed_form():
    """CN diffusion: circulant, lambda_k = b + 2a cos(2 pi k/N)."""
    n, sx = 128, 0.25
    a, b, c = synth.const_tri(n, -sx, 1 + 2 * sx, -sx)
    f = synth.rhs_uniform(n, 1, seed=12)
    x = oracle.tri_batch_solve(a, b, c, f, n=n, m=1, periodic=True)
    lam = (1 + 2 * sx) - 2 * sx * np.cos(2 * np.pi * np.arange(n) / n)
    assert relerr(x, np.real(np.fft.ifft(np.fft.fft(f) / lam))) <= 1e-14
    # sin recovery: rhs = A sin(2 pi i/N)
    s = np.sin(2 * np.pi * np.arange(n) / n)
    A = dense_tri(a, b, c, periodic=True)
    assert np.max(np.abs(oracle.tri_batch_solve(a, b, c, A @ s, n=n, m=1, periodic=True) - s)) <= 1e-13
