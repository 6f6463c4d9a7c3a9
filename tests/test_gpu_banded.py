"""GPU parity: pent_solve / tri_solve (CUDA, through the C ABI) vs the CPU oracle.

Bars (BASELINE.json north_star): max-norm relative error <= 1e-12 (fp64) and
<= 1e-5 (fp32, against the fp64 oracle), on identical seeded inputs; the
residual ||Ax - b||/||b|| is computed and reported.
"""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2101_06550_b200 as pb  # noqa: E402

TOL = {"f64": 1e-12, "f32": 1e-5}
TDT = {"f64": torch.float64, "f32": torch.float32}


def relerr(x, ref):
    return float(np.max(np.abs(x - ref)) / max(np.max(np.abs(ref)), 1e-300))


def to_layout(f_inter, n, m, layout):
    return f_inter if layout == "interleaved" else f_inter.reshape(n, m).T.reshape(-1).copy()


def from_layout(x, n, m, layout):
    return x if layout == "interleaved" else x.reshape(m, n).T.reshape(-1).copy()


def residual(a, b, c, d, e, x, f, n, m, periodic):
    """||Ax - f||_inf / ||f||_inf (fp64, wrapped matrix), interleaved x, f, shared LHS."""
    X = x.reshape(n, m)
    F = f.reshape(n, m)
    R = c[:, None] * X - F
    for off, v in ((-2, a), (-1, b), (1, d), (2, e)):
        sh = np.roll(X, -off, axis=0)
        if not periodic:
            if off < 0:
                sh[:(-off)] = 0
            else:
                sh[n - off:] = 0
        R += v[:, None] * sh
    return float(np.max(np.abs(R)) / np.max(np.abs(F)))


def run_penta(n, m, *, periodic, layout, dtype, lhs="shared", sigma=None, seed=0):
    if sigma is not None:
        a, b, c, d, e = synth.const_penta(n, sigma, -4 * sigma, 1 + 6 * sigma, -4 * sigma, sigma)
    else:
        a, b, c, d, e = synth.dd_penta(n, 1 if lhs == "shared" else m, seed=seed + 1)
    f = synth.rhs_uniform(n, m, seed=seed + 2)
    ref = oracle.penta_batch_solve(a, b, c, d, e, f, n=n, m=m, periodic=periodic)
    dev = [torch.from_numpy(v).cuda() for v in (a, b, c, d, e)]
    h = pb.pent_factor(*dev, batch=m, n=n, lhs_count=1 if a.size == n else m, periodic=periodic, dtype=dtype)
    x = torch.from_numpy(to_layout(f, n, m, layout)).to(TDT[dtype]).cuda()
    h.solve(x, layout=layout)
    torch.cuda.synchronize()
    got = from_layout(x.double().cpu().numpy(), n, m, layout)
    return got, ref, (a, b, c, d, e, f)


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("layout", ["interleaved", "contiguous"])
@pytest.mark.parametrize("periodic", [False, True])
@pytest.mark.parametrize("n,m", [(7, 5), (13, 16), (64, 64), (100, 37), (257, 33), (1000, 20), (1024, 48),
                                 (3000, 17), (5000, 16)])
def test_penta_shared_parity(n, m, periodic, layout, dtype):
    got, ref, _ = run_penta(n, m, periodic=periodic, layout=layout, dtype=dtype, seed=n + m)
    assert relerr(got, ref) <= TOL[dtype]


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("n", [64, 256, 1024, 4096, 8192])
def test_penta_hyperdiffusion_kappa722(n, dtype):
    """The thesis CH matrix at dx = 2 pi/256 (sigma = 45.09, kappa = 722), periodic."""
    m = 32
    got, ref, (a, b, c, d, e, f) = run_penta(n, m, periodic=True, layout="interleaved", dtype=dtype,
                                             sigma=synth.SIGMA_STATS, seed=3)
    assert relerr(got, ref) <= TOL[dtype]
    res = residual(a, b, c, d, e, got, f, n, m, True)
    print(f"n={n} {dtype} relerr={relerr(got, ref):.2e} residual={res:.2e}")
    assert res <= (1e-12 if dtype == "f64" else 1e-4)  # fp32: ~ eps32 * ||A|| (||A|| = 1 + 16 sigma)


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("layout", ["interleaved", "contiguous"])
@pytest.mark.parametrize("periodic", [False, True])
def test_penta_per_system_lhs_cfg1(periodic, layout, dtype):
    """cfg1: 64 independent diagonally-dominant systems, N = 64, per-system LHS."""
    got, ref, _ = run_penta(64, 64, periodic=periodic, layout=layout, dtype=dtype, lhs="per", seed=1)
    assert relerr(got, ref) <= TOL[dtype]


def test_penta_full_size_sampled():
    """Bench workload (N = M = 8192, fp64, periodic kappa = 722, interleaved, one
    launch as bench.py times it): sampled systems against the oracle."""
    n = m = 8192
    s_ = synth.SIGMA_STATS
    a, b, c, d, e = synth.const_penta(n, s_, -4 * s_, 1 + 6 * s_, -4 * s_, s_)
    f = synth.rhs_uniform(n, m, seed=2)
    h = pb.pent_factor(*[torch.from_numpy(v).cuda() for v in (a, b, c, d, e)], batch=m, n=n, periodic=True)
    x = torch.from_numpy(f).cuda()
    h.solve(x)
    torch.cuda.synchronize()
    X = x.cpu().numpy().reshape(n, m)
    F = f.reshape(n, m)
    for s in (0, 1, 15, 16, 4097, 8191):
        ref = oracle.penta_batch_solve(a, b, c, d, e, F[:, s].copy(), n=n, m=1, periodic=True)
        assert relerr(X[:, s], ref) <= 1e-12


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("layout", ["interleaved", "contiguous"])
@pytest.mark.parametrize("periodic", [False, True])
@pytest.mark.parametrize("n,m", [(3, 4), (6, 16), (64, 64), (333, 40), (2048, 32), (7000, 33)])
def test_tri_shared_parity(n, m, periodic, layout, dtype):
    a, b, c = synth.dd_tri(n, 1, seed=n)
    f = synth.rhs_uniform(n, m, seed=m)
    ref = oracle.tri_batch_solve(a, b, c, f, n=n, m=m, periodic=periodic)
    h = pb.tri_factor(*[torch.from_numpy(v).cuda() for v in (a, b, c)], batch=m, n=n, periodic=periodic, dtype=dtype)
    x = torch.from_numpy(to_layout(f, n, m, layout)).to(TDT[dtype]).cuda()
    h.solve(x, layout=layout)
    torch.cuda.synchronize()
    assert relerr(from_layout(x.double().cpu().numpy(), n, m, layout), ref) <= TOL[dtype]


@pytest.mark.parametrize("periodic", [False, True])
def test_tri_per_system_and_cn_diffusion(periodic):
    n, m = 128, 50
    a, b, c = synth.dd_tri(n, m, seed=9)
    f = synth.rhs_uniform(n, m, seed=10)
    ref = oracle.tri_batch_solve(a, b, c, f, n=n, m=m, periodic=periodic)
    h = pb.tri_factor(*[torch.from_numpy(v).cuda() for v in (a, b, c)], batch=m, n=n, lhs_count=m, periodic=periodic)
    x = torch.from_numpy(f).cuda()
    h.solve(x)
    torch.cuda.synchronize()
    assert relerr(x.cpu().numpy(), ref) <= 1e-12
    # CN diffusion, sigma_x = 0.25, periodic constant LHS
    a, b, c = synth.const_tri(n, -0.25, 1.5, -0.25)
    ref = oracle.tri_batch_solve(a, b, c, f, n=n, m=m, periodic=True)
    h = pb.tri_factor(*[torch.from_numpy(v).cuda() for v in (a, b, c)], batch=m, n=n, periodic=True)
    x = torch.from_numpy(f).cuda()
    h.solve(x)
    torch.cuda.synchronize()
    assert relerr(x.cpu().numpy(), ref) <= 1e-12


def test_host_buffers_and_solve_many():
    n, m = 300, 24
    a, b, c, d, e = synth.dd_penta(n, 1, seed=4)
    f = synth.rhs_uniform(n, 3 * m, seed=5)  # three batches back to back (each interleaved n x m)
    ref = np.concatenate([oracle.penta_batch_solve(a, b, c, d, e, f[k * n * m:(k + 1) * n * m], n=n, m=m)
                          for k in range(3)])
    h = pb.pent_factor(a, b, c, d, e, batch=m, n=n)  # host (numpy) diagonals
    xh = f.copy()
    h.solve_many(xh, 3, n * m)  # host rhs: staged by the library
    assert relerr(xh, ref) <= 1e-12


def test_zero_pivot_reported():
    n = 16
    a, b, c, d, e = synth.dd_penta(n, 1, seed=3)
    c = c.copy()
    c[5] = 0.0
    a, b, d, e = (np.zeros(n) for _ in range(4))
    with pytest.raises(pb.PentabError) as ei:
        pb.pent_factor(*[torch.from_numpy(v).cuda() for v in (a, b, c, d, e)], batch=4, n=n)
    assert ei.value.code == pb.PB_EZEROPIVOT and ei.value.row == 5


def test_deterministic_and_launch_counted():
    n, m = 512, 64
    a, b, c, d, e = synth.dd_penta(n, 1, seed=7)
    h = pb.pent_factor(*[torch.from_numpy(v).cuda() for v in (a, b, c, d, e)], batch=m, n=n, periodic=True)
    f = torch.from_numpy(synth.rhs_uniform(n, m, seed=8)).cuda()
    pb.reset_launch_count()
    x1 = h.solve(f.clone())
    per_solve = pb.launch_count()
    x2 = h.solve(f.clone())
    torch.cuda.synchronize()
    assert torch.equal(x1, x2)
    # the fused streaming solve is one launch per solve
    assert per_solve == 1 and pb.launch_count() == 2 * per_solve
