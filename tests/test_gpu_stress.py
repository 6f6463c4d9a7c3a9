"""GPU stress tests of the persistent TMA-ring solve in the regimes where the
round-1 ring protocol faulted (many tile groups per chunk, batched launches,
the ADI y-sweep as one batch of sims*n systems).  Long chains of solves are
queued back to back with no host sync and must equal, bit for bit, the same
chain run with a synchronisation after every call; the first solve is checked
against the oracle on sampled systems."""
import math

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2101_06550_b200 as pb  # noqa: E402


def thesis_handle(n, m):
    s = synth.SIGMA_STATS
    diags = synth.const_penta(n, s, -4 * s, 1 + 6 * s, -4 * s, s)
    h = pb.pent_factor(*[torch.from_numpy(v).cuda() for v in diags], batch=m, n=n, periodic=True)
    return h, diags


def chain(h, x, reps, sync, count=1):
    for _ in range(reps):
        if count == 1:
            h.solve(x)
        else:
            h.solve_many(x, count, h.batch * h.n)
        if sync:
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    return x


@pytest.mark.timeout(600)
@pytest.mark.parametrize("n,m,count,reps", [(512, 262144, 1, 2000), (512, 512, 512, 400), (1100, 300, 3, 2000)])
def test_queued_equals_synchronised(n, m, count, reps):
    h, diags = thesis_handle(n, m)
    g = torch.Generator(device="cuda")
    g.manual_seed(n + m + count)
    f = torch.rand(count * n * m, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    # first solve vs the oracle on sampled systems of the first and last batch
    x = chain(h, f.clone(), 1, True, count)
    F = f.view(count, n, m).cpu().numpy()
    X = x.view(count, n, m).cpu().numpy()
    for b in sorted({0, count - 1}):
        for s in (0, 1, m // 2 + 3, m - 1):
            ref = oracle.penta_batch_solve(*diags, np.ascontiguousarray(F[b, :, s]), n=n, m=1, periodic=True)
            err = np.max(np.abs(X[b, :, s] - ref)) / np.max(np.abs(ref))
            assert err <= 1e-12, (b, s, err)
    q = chain(h, f.clone(), reps, False, count)
    r = chain(h, f.clone(), reps, True, count)
    assert torch.isfinite(q).all()
    assert torch.equal(q, r)


@pytest.mark.timeout(600)
def test_adi_cfg4_shape_queued_equals_synchronised():
    """The cfg4 shape (512 sims x 512^2): 30 queued steps == 30 synchronised steps,
    and sampled simulations of the first step match the oracle."""
    n, sims, steps = 512, 512, 30
    L = n * synth.DX_STATS
    dt = synth.ch_dt(n, L)
    g = torch.Generator(device="cuda")
    g.manual_seed(4)
    c0 = (torch.rand((sims, n, n), dtype=torch.float64, device="cuda", generator=g) * 0.2 - 0.1)
    st = pb.CHState(c0)
    pb.ch_adi_step(st, dt, D=1.0, gamma=0.01, L=L, nsteps=1)
    torch.cuda.synchronize()
    got = st.c_cur.cpu().numpy()
    c0h = c0.cpu().numpy()
    for k in (0, 255, 511):
        rn, _ = oracle.ch_adi_steps(c0h[k:k + 1], c0h[k:k + 1], 1, dt=dt, D=1.0, gamma=0.01, L=L)
        err = np.max(np.abs(got[k] - rn[0])) / np.max(np.abs(rn))
        assert err <= 1e-12, (k, err)
    a = pb.CHState(c0)
    b = pb.CHState(c0)
    pb.ch_adi_step(a, dt, D=1.0, gamma=0.01, L=L, nsteps=steps)
    for _ in range(steps):
        pb.ch_adi_step(b, dt, D=1.0, gamma=0.01, L=L, nsteps=1)
        torch.cuda.synchronize()
    torch.cuda.synchronize()
    assert torch.equal(a.c_cur, b.c_cur)
    assert math.isfinite(float(a.c_cur.abs().max()))
