"""GPU parity of the batched 1D Cahn–Hilliard step (ch1d_step, thesis §6.2,
eq6:1Dnumerical) against the oracle's orc_ch1d_steps, and Table
6.1 reproduced by the CUDA path."""
import math
import os

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2101_06550_b200 as pb  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
TDT = {"f64": torch.float64, "f32": torch.float32}


def relerr(x, ref):
    return float(np.max(np.abs(x - ref)) / max(np.max(np.abs(ref)), 1e-300))


def gpu_ch1d(c0, nsteps, *, dt, L, dtype="f64", gamma=0.01):
    n, m = c0.shape
    st = pb.CH1DState(torch.from_numpy(c0).to(TDT[dtype]).cuda())
    pb.ch1d_step(st, dt, gamma=gamma, L=L, nsteps=nsteps)
    torch.cuda.synchronize()
    return st.c.double().cpu().numpy()


@pytest.mark.parametrize("n,m,steps", [(256, 64, 10), (100, 32, 7), (1000, 96, 3), (64, 32, 40)])
def test_ch1d_parity_fp64(n, m, steps):
    """dx = 2 pi / 256 as in the thesis's batch runs (N = 256 on 2 pi):
    kappa(A) = 1 + 16 gamma dt/dx^4 ~ 1.1e3 at every n, where fp64 parity
    <= 1e-12 is attainable (SURVEY §8(c) tolerances; at fixed L = 2 pi and
    n = 1000 kappa = 6.4e4 and the two solves differ by ~1.5e-12)."""
    L = n * 2 * math.pi / 256
    dt = synth.ch_dt(n, L)
    c0 = np.ascontiguousarray(synth.rng(7).uniform(-0.1, 0.1, size=(n, m)))   # U(-0.1, 0.1) quench
    ref = oracle.ch1d_steps(c0.reshape(-1).copy(), steps, n=n, m=m, dt=dt, gamma=0.01, L=L).reshape(n, m)
    got = gpu_ch1d(c0, steps, dt=dt, L=L)
    assert relerr(got, ref) <= 1e-12


def test_ch1d_parity_fp32():
    """fp32 vs the fp64 oracle, one step (kappa(A) = 1 + 16 sigma ~ 1.1e3 at n = 256)."""
    n, m = 256, 64
    L = 2 * math.pi
    dt = synth.ch_dt(n, L)
    c0 = np.ascontiguousarray(synth.rng(8).uniform(-0.1, 0.1, size=(n, m)))
    ref = oracle.ch1d_steps(c0.reshape(-1).copy(), 1, n=n, m=m, dt=dt, gamma=0.01, L=L).reshape(n, m)
    got = gpu_ch1d(c0.astype(np.float32).astype(np.float64), 1, dt=dt, L=L, dtype="f32")
    err = relerr(got, ref)
    print(f"ch1d fp32 relerr {err:.2e}")
    assert err <= 1e-5


def test_ch1d_rejects_ragged_batch():
    c = torch.zeros((64, 33), dtype=torch.float64, device="cuda")
    st = pb.CH1DState(c)
    with pytest.raises(pb.PentabError) as ei:
        pb.ch1d_step(st, 0.01, L=1.0)
    assert ei.value.code == pb.PB_EINVAL


def run_ch1d(n, T=20.0, L=2 * math.pi):
    dt = synth.ch_dt(n, L)
    c0 = np.repeat(synth.ch_ic_cos1d(n, L)[:, None], 32, axis=1)   # 32 identical systems (one tile)
    out = gpu_ch1d(np.ascontiguousarray(c0), synth.ch_nsteps(T, dt), dt=dt, L=L)
    assert np.max(np.abs(out - out[:, :1])) == 0.0   # identical systems stay bitwise identical
    return out[:, 0]


@pytest.mark.timeout(900)
def test_table_6_1_on_gpu():
    """Table 6.1: E_128 .. E_4096 by the CUDA path to the printed
    digits and the order column to 4 decimals for N <= 1024 (reading r11: T =
    20).  The N = 2048 order uses E_4096, which after 130 000 steps is set by
    accumulated rounding (reading r23: the oracle gives 1.9986, this path
    2.0001, the paper 2.0005), so it is reported, not asserted."""
    rows = []
    for line in open(os.path.join(GOLDEN, "table6_1.txt")):
        if line.strip() and not line.startswith("#"):
            n, e, o = line.split()
            rows.append((int(n), float(e), float(o)))
    runs = {n: run_ch1d(n) for n in (64, 128, 256, 512, 1024, 2048, 4096)}
    E = {n: oracle.convergence_error_1d(runs[n], runs[n // 2], 2 * math.pi) for n in (128, 256, 512, 1024, 2048, 4096)}
    for n, e, order in rows:
        if n not in E:
            continue
        print(f"E_{n} = {E[n]:.6e} (paper {e})")
        digits = 3 if e < 1e-3 else 4
        if e < 1e-3:
            assert float(f"{E[n]:.{digits - 1}e}") == pytest.approx(e, rel=1e-9)
        else:
            assert round(E[n], 4) == e
        if n * 2 in E and n <= 1024:
            assert abs(math.log2(E[n] / E[2 * n]) - order) <= 5e-5
    print(f"order at 2048 (E_2048 / E_4096): {math.log2(E[2048] / E[4096]):.4f} (paper 2.0005, reading r23)")


@pytest.mark.parametrize("n,m", [(256, 32768), (200, 32768), (1000, 64)])
def test_ch1d_large_and_long_batches(n, m):
    """The bench's batch shape at reduced size (32 K systems, N = 256 and a
    ragged 200) and a longer system (N = 1000: a cluster of held-tile CTAs);
    sampled systems of a 3-step run against the oracle (dx = 2 pi / 256 as in
    test_ch1d_parity_fp64, where fp64 parity <= 1e-12 is attainable)."""
    L = n * 2 * math.pi / 256
    dt = synth.ch_dt(n, L)
    g = torch.Generator(device="cuda")
    g.manual_seed(n + m)
    c0 = (torch.rand((n, m), dtype=torch.float64, device="cuda", generator=g) * 0.2 - 0.1)
    st = pb.CH1DState(c0)
    pb.ch1d_step(st, dt, gamma=0.01, L=L, nsteps=3)
    torch.cuda.synchronize()
    got = st.c.cpu().numpy()
    C0 = c0.cpu().numpy()
    for s in sorted({0, 1, 31, 32, m // 2, m - 1}):
        ref = oracle.ch1d_steps(np.ascontiguousarray(C0[:, s]), 3, n=n, m=1, dt=dt, gamma=0.01, L=L)
        assert relerr(got[:, s], ref) <= 1e-12, s
