"""Test-only compute backend for paper_2101_06550_b200.dist built from the
CPU oracle, so the partitioned orchestration (halo rows, pack, the two
all-to-all transposes, combine, level rotation) can run on CPU ranks over
gloo and be compared with the oracle's single-grid ADI step."""
import numpy as np

import oracle


def _bih_weights(dx):
    # delta_x^4 + delta_y^4 + 2 delta_x^2 delta_y^2 (reading r9), 5x5 window row-major from the top-left
    w = np.zeros((5, 5))
    w[2, 2] = 20.0
    for (a, b) in ((1, 2), (3, 2), (2, 1), (2, 3)):
        w[a, b] = -8.0
    for (a, b) in ((1, 1), (1, 3), (3, 1), (3, 3)):
        w[a, b] = 2.0
    for (a, b) in ((0, 2), (4, 2), (2, 0), (2, 4)):
        w[a, b] = 1.0
    return w / dx ** 4


def _lap_weights(dx):
    return np.array([[0.0, 1.0, 0.0], [1.0, -4.0, 1.0], [0.0, 1.0, 0.0]]) / dx ** 2   # reading r8


class OracleCompute:
    def __init__(self, prm):
        self.prm = prm
        s = (2.0 / 3.0) * prm.D * prm.gamma * prm.dt / (prm.L / prm.n) ** 4   # L_y
        self.diag = [np.full(prm.n, v) for v in (s, -4 * s, 1 + 6 * s, -4 * s, s)]

    def pass_a(self, cn_ext, cm_ext, w):
        p = self.prm
        r, n, dx = p.rows, p.n, p.L / p.n
        cn, cm = cn_ext.numpy(), cm_ext.numpy()
        # window sums on the extended block (wrap in j only touches the halo rows' own values)
        bih = oracle.stencil_apply(2 * cn - cm, _bih_weights(dx), left=2, right=2, top=2, bottom=2, periodic=True)
        lap = oracle.stencil_apply(cn ** 3 - cn, _lap_weights(dx), left=1, right=1, top=1, bottom=1, periodic=True)
        R = (-(2.0 / 3.0) * (cn - cm) - (2.0 / 3.0) * p.dt * p.D * p.gamma * bih + (2.0 / 3.0) * p.D * p.dt * lap)
        Rin = np.ascontiguousarray(R[2:r + 2]).reshape(-1)
        x = oracle.penta_batch_solve(*self.diag, Rin, n=n, m=r, layout="contiguous", periodic=True)
        w.numpy()[:] = x.reshape(r, n)

    def pack(self, w, packed):
        p = self.prm
        nb = p.n // p.parts
        W = w.numpy()
        for q in range(p.parts):
            packed.numpy()[q] = W[:, q * nb:(q + 1) * nb]

    def ysolve(self, cols):
        p = self.prm
        nb = p.n // p.parts
        c = cols.numpy().reshape(-1)
        c[:] = oracle.penta_batch_solve(*self.diag, c.copy(), n=p.n, m=nb, layout="interleaved", periodic=True)

    def combine(self, cn_ext, cm_ext, v_packed):
        p = self.prm
        r, nb = p.rows, p.n // p.parts
        v = np.concatenate([v_packed.numpy()[q] for q in range(p.parts)], axis=1)   # [r][n]
        cm = cm_ext.numpy()
        cm[2:r + 2] = 2 * cn_ext.numpy()[2:r + 2] - cm[2:r + 2] + v
