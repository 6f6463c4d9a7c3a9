"""GPU parity: stencil_apply and ch_adi_step (CUDA, through the C ABI) vs the
CPU oracle, plus the printed Table 3.1 reproduced by the CUDA path."""
import math
import os

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


# ------------------------------------------------------------------ stencil_apply
@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("periodic", [True, False])
@pytest.mark.parametrize("win", [(2, 2, 0, 0), (0, 0, 3, 1), (1, 1, 1, 1), (2, 2, 2, 2), (0, 3, 2, 0), (7, 7, 7, 7)])
@pytest.mark.parametrize("shape", [(1, 64, 64), (3, 37, 101), (2, 130, 70)])
def test_stencil_parity(shape, win, periodic, dtype):
    left, right, top, bottom = win
    g = synth.rng(sum(shape) + sum(win)).standard_normal(shape)
    w = synth.rng(7).standard_normal((top + bottom + 1) * (left + right + 1))
    init = np.full(shape, 3.0)
    ref = oracle.stencil_apply(g, w, left=left, right=right, top=top, bottom=bottom, periodic=periodic, out=init)
    gi = torch.from_numpy(g).to(TDT[dtype]).cuda()
    go = torch.from_numpy(init).to(TDT[dtype]).cuda()
    pb.stencil_apply(gi, go, w, left=left, right=right, top=top, bottom=bottom, periodic=periodic)
    torch.cuda.synchronize()
    got = go.double().cpu().numpy()
    tol = 1e-13 if dtype == "f64" else 1e-5
    assert np.max(np.abs(got - ref)) <= tol * max(1.0, np.max(np.abs(ref)))
    if not periodic:  # untouched boundary
        assert np.all(got[..., :top, :] == 3.0) and np.all(got[..., :, :left] == 3.0)


def test_stencil_sin_example_and_host_buffers():
    """cuSten 2d_x_np, host (numpy) buffers through the C ABI."""
    nx, ny = 1024, 512
    dx = 2 * math.pi / nx
    g = np.tile(np.sin(dx * np.arange(nx)), (ny, 1))
    w = np.array([-1 / 560, 8 / 315, -1 / 5, 8 / 5, -205 / 72, 8 / 5, -1 / 5, 8 / 315, -1 / 560]) / dx ** 2
    out = np.zeros_like(g)
    pb.stencil_apply(g, out, w, left=4, right=4, top=0, bottom=0, periodic=False)
    assert np.max(np.abs(out[:, 4:-4] + g[:, 4:-4])) < 1e-9
    ref = oracle.stencil_apply(g, w, left=4, right=4, top=0, bottom=0, periodic=False)
    # the 9 terms are ~1e5 and cancel to ~1: bound by the rounding of the terms, 16 eps sum|w| max|g|
    assert np.max(np.abs(out - ref)) <= 16 * 2.2e-16 * np.sum(np.abs(w)) * np.max(np.abs(g))


def test_stencil_rejects_aliasing():
    x = torch.zeros(8, 8, dtype=torch.float64, device="cuda")
    with pytest.raises(pb.PentabError) as ei:
        pb.stencil_apply(x, x, np.ones(3), left=1, right=1, top=0, bottom=0)
    assert ei.value.code == pb.PB_EINVAL


# ------------------------------------------------------------------ ch_adi_step
def gpu_adi(c0, nsteps, *, dt, L, dtype="f64", cprev=None):
    st = pb.CHState(torch.from_numpy(c0).to(TDT[dtype]).cuda())
    if cprev is not None:
        st.c_prev.copy_(torch.from_numpy(cprev).to(TDT[dtype]))
    pb.ch_adi_step(st, dt, D=1.0, gamma=0.01, L=L, nsteps=nsteps)
    torch.cuda.synchronize()
    return st.c_cur.double().cpu().numpy(), st.c_prev.double().cpu().numpy()


@pytest.mark.parametrize("n,sims,L", [(64, 3, None), (100, 2, None), (128, 2, 2 * math.pi), (256, 2, None),
                                      (512, 1, None), (1024, 1, None), (2048, 1, None), (65, 2, None), (99, 1, None)])
def test_adi_parity_fp64(n, sims, L):
    L = L if L is not None else n * synth.DX_STATS  # dx = 2 pi/256 (sigma = 45.09)
    dt = synth.ch_dt(n, L)
    c0 = synth.ch_ic_random(sims, n, seed=3)
    c1, _ = oracle.ch_adi_steps(c0, c0, 1, dt=dt, D=1.0, gamma=0.01, L=L)
    nsteps = 4 if n <= 512 else 1
    rn, rm = oracle.ch_adi_steps(c1, c0, nsteps, dt=dt, D=1.0, gamma=0.01, L=L)
    gn, gm = gpu_adi(c1, nsteps, dt=dt, L=L, cprev=c0)
    assert relerr(gn, rn) <= 1e-12
    assert relerr(gm, rm) <= 1e-12


@pytest.mark.parametrize("n", [64, 256, 512])
def test_adi_parity_fp32(n):
    """fp32 state vs the fp64 oracle at the north-star bar (<= 1e-5), 3 steps.
    The RHS and both sweeps run on an fp64 workspace (reading r22: the explicit
    biharmonic term is ~64 sigma |C| before the sweeps cancel it), so only the
    stored levels round to fp32."""
    L = n * synth.DX_STATS
    dt = synth.ch_dt(n, L)
    c0 = synth.ch_ic_random(2, n, seed=4).astype(np.float32).astype(np.float64)
    rn, _ = oracle.ch_adi_steps(c0, c0, 3, dt=dt, D=1.0, gamma=0.01, L=L)
    gn, _ = gpu_adi(c0, 3, dt=dt, L=L, dtype="f32")
    err = relerr(gn, rn)
    print(f"ADI fp32 n={n} relerr {err:.2e}")
    assert err <= 1e-5


def test_adi_mass_conservation_and_fixed_point():
    n, L = 256, 4 * math.pi
    dt = synth.ch_dt(n, L)
    c0 = synth.ch_ic_random(4, n, seed=5, lo=0.4, hi=0.6)  # asymmetric quench
    gn, _ = gpu_adi(c0, 200, dt=dt, L=L)
    m0, m1 = c0.sum(axis=(1, 2)), gn.sum(axis=(1, 2))
    assert np.max(np.abs(m1 - m0)) <= 1e-11 * n * n
    k = np.full((1, 64, 64), -0.25)
    kn, _ = gpu_adi(k, 10, dt=synth.ch_dt(64, 2 * math.pi), L=2 * math.pi)
    assert np.max(np.abs(kn + 0.25)) <= 1e-15


def run_table31(n):
    L = 2 * math.pi
    dt = synth.ch_dt(n, L)
    c0 = synth.ch_ic_tanh(n, L)[None]
    gn, _ = gpu_adi(c0, synth.ch_nsteps(10.0, dt), dt=dt, L=L)
    return gn[0]


def golden31():
    rows = {}
    for line in open(os.path.join(os.path.dirname(__file__), "golden", "table3_1.txt")):
        if line.strip() and not line.startswith("#"):
            n, e, _ = line.split()
            rows[int(n)] = float(e)
    return rows


def test_table_3_1_on_gpu():
    """Table 3.1: E_128 .. E_1024 by the CUDA path, 4 printed decimals."""
    rows = golden31()
    runs = {n: run_table31(n) for n in (64, 128, 256, 512, 1024)}
    for n in (128, 256, 512, 1024):
        e = oracle.convergence_error_2d(runs[n], runs[n // 2], 2 * math.pi)
        print(f"E_{n} = {e:.6f} (paper {rows[n]})")
        assert abs(e - rows[n]) <= 5e-5


@pytest.mark.timeout(900)
def test_adi_cfg4_shape_sampled_sims():
    """configs[3] launch shape (512 sims x 512^2, L = 4 pi, the bench's sharding
    unit) for 2 steps; sims 0, 1, 255, 511 against the oracle (each simulation
    is independent, so a sampled sim is an exact check of the full launch)."""
    sims, n = 512, 512
    L = n * synth.DX_STATS
    dt = synth.ch_dt(n, L)
    c0 = synth.ch_ic_random(sims, n, seed=4)
    gn, gm = gpu_adi(c0, 2, dt=dt, L=L)
    for k in (0, 1, 255, 511):
        rn, rm = oracle.ch_adi_steps(c0[k:k + 1], c0[k:k + 1], 2, dt=dt, D=1.0, gamma=0.01, L=L)
        assert relerr(gn[k:k + 1], rn) <= 1e-12, k
        assert relerr(gm[k:k + 1], rm) <= 1e-12, k


@pytest.mark.timeout(1200)
def test_adi_16384_single_grid():
    """configs[4] grid size on one GPU: one 16384^2 simulation (L = 128 pi), one
    ADI step through ch_adi_step against the oracle's full step (fp64)."""
    n = 16384
    L = n * synth.DX_STATS
    dt = synth.ch_dt(n, L)
    c0 = synth.ch_ic_random(1, n, seed=5)
    rn, _ = oracle.ch_adi_steps(c0, c0, 1, dt=dt, D=1.0, gamma=0.01, L=L)
    gn, gm = gpu_adi(c0, 1, dt=dt, L=L)
    assert relerr(gn, rn) <= 1e-12
    assert np.array_equal(gm, c0)


def test_stencil_rejects_partial_overlap():
    """Overlapping (not only identical) in/out ranges are rejected."""
    x = torch.zeros(2, 8, 8, dtype=torch.float64, device="cuda")
    with pytest.raises(pb.PentabError) as ei:
        pb.stencil_apply(x[0:1], x.view(-1)[32:96].view(1, 8, 8), np.ones(3), left=1, right=1, top=0, bottom=0)
    assert ei.value.code == pb.PB_EINVAL
