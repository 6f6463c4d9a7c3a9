"""GPU parity of the coarsening-statistics row through the C
ABI: ch_free_energy, ch_coarsening_beta and the Cahn–Hilliard–Cook step
ch_adi_step_cook against the oracle (readings r24-r27)."""
import math

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2101_06550_b200 as pb  # noqa: E402

TDT = {"f64": torch.float64, "f32": torch.float32}


def relerr(x, ref):
    return float(np.max(np.abs(x - ref)) / max(np.max(np.abs(ref)), 1e-300))


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("sims,n", [(3, 100), (2, 512), (1, 9)])
def test_free_energy_parity(sims, n, dtype):
    L, g = n * synth.DX_STATS, 0.01
    c = synth.ch_ic_random(sims, n, seed=21, lo=-1.1, hi=1.1)
    c = c.astype(np.float32).astype(np.float64) if dtype == "f32" else c
    ref = oracle.ch_free_energy(c, L=L, gamma=g)
    st = pb.CHState(torch.from_numpy(c).to(TDT[dtype]).cuda())
    F = torch.empty(sims, dtype=torch.float64, device="cuda")
    pb.ch_free_energy(st, F, gamma=g, L=L)
    torch.cuda.synchronize()
    assert relerr(F.cpu().numpy(), ref) <= 1e-13


def test_beta_parity():
    t = np.linspace(10.0, 100.0, 91)
    F = np.stack([t ** -0.3, 5.0 / (1 + t), 2.0 - 0.01 * t], axis=1)
    ref = oracle.coarsening_beta(t, F)
    td, Fd = torch.from_numpy(t).cuda(), torch.from_numpy(F).cuda()
    beta = torch.empty_like(Fd)
    pb.ch_coarsening_beta(td, Fd, beta)
    torch.cuda.synchronize()
    assert relerr(beta.cpu().numpy(), ref) <= 1e-14


@pytest.mark.parametrize("sims,n", [(2, 64), (1, 100), (3, 256)])
def test_cook_step_parity_fp64(sims, n):
    """IC 0, sigma = 1e-14: the field is all noise; 3 steps as one call
    and as 2 + 1 calls (step0 continues the counter)."""
    L = n * synth.DX_STATS
    dt = synth.ch_dt(n, L)
    z = np.zeros((sims, n, n))
    rn, rm = oracle.ch_adi_steps_cook(z, z, 3, dt=dt, D=1.0, gamma=0.01, L=L, sigma=1e-14, seed=77)
    st = pb.CHState(torch.zeros((sims, n, n), dtype=torch.float64, device="cuda"))
    pb.ch_adi_step_cook(st, dt, sigma=1e-14, seed=77, L=L, nsteps=3)
    torch.cuda.synchronize()
    assert np.max(np.abs(rn)) > 0
    assert relerr(st.c_cur.cpu().numpy(), rn) <= 1e-12
    assert relerr(st.c_prev.cpu().numpy(), rm) <= 1e-12
    s2 = pb.CHState(torch.zeros((sims, n, n), dtype=torch.float64, device="cuda"))
    pb.ch_adi_step_cook(s2, dt, sigma=1e-14, seed=77, step0=0, L=L, nsteps=2)
    pb.ch_adi_step_cook(s2, dt, sigma=1e-14, seed=77, step0=2, L=L, nsteps=1)
    torch.cuda.synchronize()
    assert torch.equal(s2.c_cur, st.c_cur)


def test_cook_with_state_and_zero_sigma():
    """A random quench plus noise matches the oracle; sigma = 0 is ch_adi_step bitwise."""
    sims, n = 2, 128
    L = n * synth.DX_STATS
    dt = synth.ch_dt(n, L)
    c0 = synth.ch_ic_random(sims, n, seed=31)
    rn, _ = oracle.ch_adi_steps_cook(c0, c0, 4, dt=dt, D=1.0, gamma=0.01, L=L, sigma=1e-6, seed=5, step0=10)
    st = pb.CHState(torch.from_numpy(c0).cuda())
    pb.ch_adi_step_cook(st, dt, sigma=1e-6, seed=5, step0=10, L=L, nsteps=4)
    torch.cuda.synchronize()
    assert relerr(st.c_cur.cpu().numpy(), rn) <= 1e-12
    a = pb.CHState(torch.from_numpy(c0).cuda())
    b = pb.CHState(torch.from_numpy(c0).cuda())
    pb.ch_adi_step(a, dt, L=L, nsteps=3)
    pb.ch_adi_step_cook(b, dt, sigma=0.0, seed=5, L=L, nsteps=3)
    torch.cuda.synchronize()
    assert torch.equal(a.c_cur, b.c_cur) and torch.equal(a.c_prev, b.c_prev)


def test_cook_fp32_state():
    sims, n = 2, 128
    L = n * synth.DX_STATS
    dt = synth.ch_dt(n, L)
    c0 = synth.ch_ic_random(sims, n, seed=41).astype(np.float32).astype(np.float64)
    rn, _ = oracle.ch_adi_steps_cook(c0, c0, 3, dt=dt, D=1.0, gamma=0.01, L=L, sigma=1e-6, seed=9)
    st = pb.CHState(torch.from_numpy(c0).to(torch.float32).cuda())
    pb.ch_adi_step_cook(st, dt, sigma=1e-6, seed=9, L=L, nsteps=3)
    torch.cuda.synchronize()
    assert relerr(st.c_cur.double().cpu().numpy(), rn) <= 1e-5


def test_coarsening_pipeline_free_energy_decays():
    """The statistics pipeline of thesis §7.5 on a small batch: CHC from C = 0,
    F sampled on the device every 10 steps, beta on the device; F(t) has the
    oracle's values and decreases once the domains have formed."""
    sims, n = 2, 64
    L = n * synth.DX_STATS
    dt = synth.ch_dt(n, L)
    st = pb.CHState(torch.zeros((sims, n, n), dtype=torch.float64, device="cuda"))
    ts, Fs = [], []
    cn = cm = np.zeros((sims, n, n))
    F = torch.empty(sims, dtype=torch.float64, device="cuda")
    for k in range(6):
        pb.ch_adi_step_cook(st, dt, sigma=1e-8, seed=3, step0=10 * k, L=L, nsteps=10)
        cn, cm = oracle.ch_adi_steps_cook(cn, cm, 10, dt=dt, D=1.0, gamma=0.01, L=L, sigma=1e-8, seed=3, step0=10 * k)
        pb.ch_free_energy(st, F, L=L)
        torch.cuda.synchronize()
        ts.append(10 * (k + 1) * dt)
        Fs.append(F.cpu().numpy().copy())
        assert relerr(Fs[-1], oracle.ch_free_energy(cn, L=L, gamma=0.01)) <= 1e-12
    beta = torch.empty((6, sims), dtype=torch.float64, device="cuda")
    pb.ch_coarsening_beta(torch.tensor(ts, dtype=torch.float64, device="cuda"),
                          torch.tensor(np.array(Fs), device="cuda"), beta)
    torch.cuda.synchronize()
    assert np.allclose(beta.cpu().numpy(), oracle.coarsening_beta(np.array(ts), np.array(Fs)), rtol=1e-12, atol=0)
