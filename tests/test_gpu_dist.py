"""GPU parity of the row-partitioned ADI step (configs[4] kernels:
ch_dist_pass_a, ch_dist_pack, pent_solve y-sweep, ch_dist_combine), with P
ranks emulated on one device (LocalExchange moves the same blocks the NCCL
all-to-all moves): equal to the oracle's single-grid step (<= 1e-12) and to
the library's own single-grid ch_adi_step."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2101_06550_b200 as pb  # noqa: E402
from paper_2101_06550_b200 import dist  # noqa: E402


def _run(n, parts, steps, dtype=torch.float64, seed=6):
    L = n * synth.DX_STATS
    dt = synth.ch_dt(n, L)
    c0 = synth.ch_ic_random(1, n, seed=seed)[0]
    c1, _ = oracle.ch_adi_steps(c0, c0, 1, dt=dt, D=1.0, gamma=0.01, L=L)
    prm = dist.Params(n=n, parts=parts, dt=dt, L=L)
    r = prm.rows
    dev = torch.device("cuda")
    states = [dist.RankState(prm, k, torch.from_numpy(c1[k * r:(k + 1) * r]).to(dev, dtype),
                             torch.from_numpy(c0[k * r:(k + 1) * r]).to(dev, dtype),
                             dist.LibCompute(prm, dev, dtype)) for k in range(parts)]
    for _ in range(steps):
        dist.step(states, dist.LocalExchange())
    torch.cuda.synchronize()
    got = np.concatenate([s.interior("cn").double().cpu().numpy() for s in states])
    ref, _ = oracle.ch_adi_steps(c1, c0, steps, dt=dt, D=1.0, gamma=0.01, L=L)
    return got, ref, (c0, c1, dt, L)


@pytest.mark.parametrize("n,parts", [(64, 1), (64, 2), (128, 4), (256, 8), (512, 2)])
def test_dist_matches_oracle(n, parts):
    got, ref, _ = _run(n, parts, 3)
    assert np.max(np.abs(got - ref)) / np.max(np.abs(ref)) <= 1e-12


def test_dist_matches_single_grid_library():
    n, parts, steps = 256, 4, 4
    got, _, (c0, c1, dt, L) = _run(n, parts, steps)
    st = pb.CHState(torch.from_numpy(c1[None]).cuda())
    st.c_prev.copy_(torch.from_numpy(c0[None]).cuda())
    pb.ch_adi_step(st, dt, D=1.0, gamma=0.01, L=L, nsteps=steps)
    torch.cuda.synchronize()
    one = st.c_cur[0].cpu().numpy()
    assert np.max(np.abs(got - one)) / np.max(np.abs(one)) <= 1e-13
