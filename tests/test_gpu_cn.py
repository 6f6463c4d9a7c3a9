"""GPU tests of the thesis's Crank–Nicolson benchmark problems composed from the
library calls (stencil_apply for the explicit half, the batched banded solve
for the implicit half), and of the solver regimes around them:

* hyperdiffusion CN (§4.2, eq:1d_hyper_scheme) — validation of
  P:1736-1765: C(x,0) = cos(4 pi x), gamma = D = L = 1, dt = 1e-8, T = 1e-4;
  eps_N(T) of eq:myerr against the exact e^{-k^4 t} cos(kx) must reproduce
  the CPU values of SURVEY §8(c) and the N^-2 slope (paper: -2.0162);
* periodic CN diffusion with the tridiagonal solver (§5.3) — the
  exact per-mode amplification (1 - 4 s S^2) / (1 + 4 s S^2), S = sin(pi k/N),
  and step parity with the oracle;
* cuPentUniformBatch and cuPentBatchRewrite.
"""
import math

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2101_06550_b200 as pb  # noqa: E402


def relerr(x, ref):
    return float(np.max(np.abs(x - ref)) / max(np.max(np.abs(ref)), 1e-300))


def cn_hyper_run(n, m=32, T=1e-4, dt=1e-8, kk=2):
    """eq:1d_hyper_scheme on n points of [0, 1), m identical interleaved systems."""
    dx = 1.0 / n
    s = dt / (2 * dx ** 4)
    h = pb.pent_factor_uniform(s, -4 * s, 1 + 6 * s, -4 * s, s, batch=m, n=n, periodic=True)
    x = dx * np.arange(n)
    c = torch.from_numpy(np.repeat(np.cos(2 * math.pi * kk * x)[:, None], m, axis=1).copy()).cuda()
    f = torch.empty_like(c)
    w = np.array([-s, 4 * s, 1 - 6 * s, 4 * s, -s])   # rows j-2..j+2 (the unknown index is the row)
    steps = synth.ch_nsteps(T, dt)
    for _ in range(steps):
        pb.stencil_apply(c, f, w, left=0, right=0, top=2, bottom=2, periodic=True)
        h.solve(f)
        c, f = f, c
    torch.cuda.synchronize()
    out = c.cpu().numpy()
    assert np.max(np.abs(out - out[:, :1])) == 0.0
    k = 2 * math.pi * kk
    exact = math.exp(-k ** 4 * steps * dt) * np.cos(k * x)
    return oracle.l2_error(out[:, 0], exact)   # eq:myerr


@pytest.mark.timeout(900)
def test_hyperdiffusion_cn_validation():
    """eps_N(T) for N = 16..1024 equals the CPU reference values of
    SURVEY §8(c) (1.62e-2 ... 3.66e-6, 3 digits) and decays as N^-2 (least
    squares slope within 0.003 of the paper's -2.0162)."""
    ns = [16, 32, 64, 128, 256, 512, 1024]
    ref = [1.62e-2, 3.82e-3, 9.41e-4, 2.34e-4, 5.85e-5, 1.46e-5, 3.66e-6]
    eps = [cn_hyper_run(n) for n in ns]
    for n, e, r in zip(ns, eps, ref):
        print(f"eps_{n} = {e:.4e} (CPU {r})")
        assert abs(e - r) <= 0.006 * r + 1e-9, (n, e, r)
    slope = np.polyfit(np.log(ns), np.log(eps), 1)[0]
    print(f"slope {slope:.4f} (paper -2.0162)")
    assert abs(slope - (-2.0162)) <= 0.003


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_tri_cn_diffusion_amplification_and_parity(dtype):
    """P:2283-2315 (eq5:1ddiffscheme): periodic CN diffusion on [0, 1), dt = 1e-4.
    One step multiplies cos(2 pi k x) by exactly (1 - 4 s S^2)/(1 + 4 s S^2),
    S = sin(pi k / N); a random RHS batch matches the oracle step."""
    n, m, dt = 512, 64, 1e-4
    dx = 1.0 / n
    s = dt / (2 * dx * dx)
    h = pb.tri_factor_uniform(-s, 1 + 2 * s, -s, batch=m, n=n, periodic=True, dtype=dtype)
    x = dx * np.arange(n)
    ks = np.arange(m) % 40 + 1
    c0 = np.cos(2 * math.pi * x[:, None] * ks[None, :])
    tdt = torch.float64 if dtype == "f64" else torch.float32
    c = torch.from_numpy(c0).to(tdt).cuda()
    f = torch.empty_like(c)
    pb.stencil_apply(c, f, np.array([s, 1 - 2 * s, s]), left=0, right=0, top=1, bottom=1, periodic=True)
    h.solve(f)
    torch.cuda.synchronize()
    S = np.sin(math.pi * ks / n) ** 2
    amp = (1 - 4 * s * S) / (1 + 4 * s * S)
    tol = 1e-12 if dtype == "f64" else 1e-5
    assert relerr(f.double().cpu().numpy(), c0 * amp[None, :]) <= tol
    # random RHS vs the oracle (stencil + Thomas / Sherman–Morrison)
    r0 = synth.rng(5).uniform(-1, 1, size=(n, m))
    rr = oracle.stencil_apply(r0, np.array([s, 1 - 2 * s, s]), left=0, right=0, top=1, bottom=1, periodic=True)
    a = np.full(n, -s)
    ref = oracle.tri_batch_solve(a, np.full(n, 1 + 2 * s), a, rr.reshape(-1), n=n, m=m, periodic=True).reshape(n, m)
    c = torch.from_numpy(r0).to(tdt).cuda()
    pb.stencil_apply(c, f, np.array([s, 1 - 2 * s, s]), left=0, right=0, top=1, bottom=1, periodic=True)
    h.solve(f)
    torch.cuda.synchronize()
    assert relerr(f.double().cpu().numpy(), ref) <= tol


@pytest.mark.parametrize("periodic", [False, True])
def test_uniform_equals_explicit_diagonals(periodic):
    """pent_factor_uniform builds the same shared LHS as explicit constant
    diagonals (bit-identical solutions)."""
    n, m = 777, 96
    s = synth.SIGMA_STATS
    diags = synth.const_penta(n, s, -4 * s, 1 + 6 * s, -4 * s, s)
    h1 = pb.pent_factor(*[torch.from_numpy(v).cuda() for v in diags], batch=m, n=n, periodic=periodic)
    h2 = pb.pent_factor_uniform(s, -4 * s, 1 + 6 * s, -4 * s, s, batch=m, n=n, periodic=periodic)
    f = torch.from_numpy(synth.rhs_uniform(n, m, seed=9)).cuda()
    x1, x2 = h1.solve(f.clone()), h2.solve(f.clone())
    torch.cuda.synchronize()
    assert torch.equal(x1, x2)


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("periodic", [False, True])
def test_rewrite_refactor_every_step(periodic, dtype):
    """cuPentBatchRewrite: a per-system LHS re-factored in place
    every step (pent_refactor, no sync) then solved; each step matches the
    oracle on that step's matrices."""
    n, m = 300, 64
    h = None
    tdt = torch.float64 if dtype == "f64" else torch.float32
    for step in range(3):
        a, b, c, d, e = synth.dd_penta(n, m, seed=100 + step)
        dev = [torch.from_numpy(v).cuda() for v in (a, b, c, d, e)]
        if h is None:
            h = pb.pent_factor(*dev, batch=m, n=n, lhs_count=m, periodic=periodic, dtype=dtype)
        else:
            h.refactor(*dev)
        f = synth.rhs_uniform(n, m, seed=200 + step)
        ref = oracle.penta_batch_solve(a, b, c, d, e, f, n=n, m=m, periodic=periodic)
        x = torch.from_numpy(f).to(tdt).cuda()
        h.solve(x)
        torch.cuda.synchronize()
        assert relerr(x.double().cpu().numpy(), ref) <= (1e-12 if dtype == "f64" else 1e-5), step
