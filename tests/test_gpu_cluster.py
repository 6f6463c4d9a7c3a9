"""GPU parity of the TMA cluster solve (cluster_solve.cuh, PB_SOLVER=cluster):
interleaved shared-LHS penta / tri, cyclic and not, fp64 (<= 1e-12) and fp32
(<= 1e-5 against the fp64 oracle), cluster sizes 1..16 (N up to 8192), ragged
row tails and partial system groups."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2101_06550_b200 as pb  # noqa: E402

TOL = {"f64": 1e-12, "f32": 1e-5}
TDT = {"f64": torch.float64, "f32": torch.float32}


@pytest.fixture(autouse=True)
def _cluster_path(monkeypatch):
    monkeypatch.setenv("PB_SOLVER", "cluster")


def relerr(x, ref):
    return float(np.max(np.abs(x - ref)) / max(np.max(np.abs(ref)), 1e-300))


SIZES = [(40, 16), (512, 32), (700, 20), (2100, 48), (5000, 36), (8192, 16)]


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("periodic", [False, True])
@pytest.mark.parametrize("n,m", SIZES)
def test_cluster_penta(n, m, periodic, dtype):
    a, b, c, d, e = synth.dd_penta(n, 1, seed=n + 5)
    f = synth.rhs_uniform(n, m, seed=m + 7)
    ref = oracle.penta_batch_solve(a, b, c, d, e, f, n=n, m=m, periodic=periodic)
    h = pb.pent_factor(*[torch.from_numpy(v).cuda() for v in (a, b, c, d, e)], batch=m, n=n, periodic=periodic,
                       dtype=dtype)
    x = torch.from_numpy(f).to(TDT[dtype]).cuda()
    h.solve(x)
    torch.cuda.synchronize()
    assert relerr(x.double().cpu().numpy(), ref) <= TOL[dtype]


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("periodic", [False, True])
@pytest.mark.parametrize("n,m", SIZES)
def test_cluster_tri(n, m, periodic, dtype):
    a, b, c = synth.dd_tri(n, 1, seed=n + 9)
    f = synth.rhs_uniform(n, m, seed=m + 3)
    ref = oracle.tri_batch_solve(a, b, c, f, n=n, m=m, periodic=periodic)
    h = pb.tri_factor(*[torch.from_numpy(v).cuda() for v in (a, b, c)], batch=m, n=n, periodic=periodic, dtype=dtype)
    x = torch.from_numpy(f).to(TDT[dtype]).cuda()
    h.solve(x)
    torch.cuda.synchronize()
    assert relerr(x.double().cpu().numpy(), ref) <= TOL[dtype]


def test_cluster_thesis_matrix_many():
    """The thesis CH operator (kappa = 722), cyclic, three batches in one launch."""
    n, m, cnt = 4096, 32, 3
    s_ = synth.SIGMA_STATS
    diags = synth.const_penta(n, s_, -4 * s_, 1 + 6 * s_, -4 * s_, s_)
    f = synth.rhs_uniform(n, cnt * m, seed=31)
    ref = np.concatenate([oracle.penta_batch_solve(*diags, f[k * n * m:(k + 1) * n * m], n=n, m=m, periodic=True)
                          for k in range(cnt)])
    h = pb.pent_factor(*[torch.from_numpy(v).cuda() for v in diags], batch=m, n=n, periodic=True)
    x = torch.from_numpy(f).cuda()
    h.solve_many(x, cnt, n * m)
    torch.cuda.synchronize()
    assert relerr(x.cpu().numpy(), ref) <= 1e-12
