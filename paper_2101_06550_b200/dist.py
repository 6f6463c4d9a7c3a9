"""Row-partitioned ADI Cahn–Hilliard step over P ranks (configs[4]: one n x n
grid); orchestration only — every arithmetic step runs in
libpentab.so (ch_dist_pass_a, ch_dist_pack, ch_dist_ysweep, ch_dist_combine).

Rank r owns rows [r n/P, (r+1) n/P).  One step of Eq 3.1:
  1. halo exchange: 2 rows above / below of C^n and C^{n-1} (periodic across
     ranks) into the extended buffers (rows + 4) x n;
  2. RHS + x-sweep on the rank's rows (ch_dist_pass_a) -> w;
  3. pack w by column block and all-to-all: rank r receives the n x n/P
     column block r of w (rows in order, columns interleaved = the systems);
  4. y-sweep: ch_dist_ysweep on that block (cyclic L_y, n/P systems, interleaved);
  5. all-to-all back: rank r receives v for its rows, block q = columns of q;
  6. C^{n+1} = 2 C^n - C^{n-1} + v (ch_dist_combine), levels rotate.
The exchange is the only communication (2 all-to-all of one field + halo
rows per step).  ``Exchange`` implementations: ``TorchExchange`` (one process
per rank, torch.distributed — NCCL on GPUs, gloo on CPU) and ``LocalExchange``
(all ranks in one process: single-GPU emulation of the same data movement).
The compute backend is pluggable for host-logic tests; the product backend
is ``LibCompute`` (the CUDA library, no fallback).
"""
from __future__ import annotations

from dataclasses import dataclass

import paper_2101_06550_b200 as pb


@dataclass
class Params:
    n: int
    parts: int
    dt: float
    L: float
    D: float = 1.0
    gamma: float = 0.01

    @property
    def rows(self) -> int:
        return self.n // self.parts



class LibCompute:
    """The product backend: libpentab.so kernels on the rank's device."""

    def __init__(self, prm: Params, device, dtype):
        self.prm, self.device, self.dtype = prm, device, dtype

    def pass_a(self, cn_ext, cm_ext, w):
        p = self.prm
        pb.ch_dist_pass_a(cn_ext, cm_ext, w, rows=p.rows, n=p.n, dt=p.dt, D=p.D, gamma=p.gamma, L=p.L)

    def pack(self, w, packed):
        p = self.prm
        pb.ch_dist_pack(w, packed, rows=p.rows, n=p.n, parts=p.parts)

    def ysolve(self, cols):
        p = self.prm
        pb.ch_dist_ysweep(cols, ncols=p.rows, n=p.n, dt=p.dt, D=p.D, gamma=p.gamma, L=p.L)

    def combine(self, cn_ext, cm_ext, v_packed):
        p = self.prm
        pb.ch_dist_combine(cn_ext, cm_ext, v_packed, rows=p.rows, n=p.n, parts=p.parts)


class RankState:
    """Buffers of one rank: C^n, C^{n-1} with halo rows, w, transpose buffers."""

    def __init__(self, prm: Params, rank: int, cn_rows, cm_rows, compute):
        import torch
        self.prm, self.rank, self.compute = prm, rank, compute
        r, n, P = prm.rows, prm.n, prm.parts
        dev, dt = cn_rows.device, cn_rows.dtype
        self.cn = torch.zeros((r + 4, n), dtype=dt, device=dev)
        self.cm = torch.zeros((r + 4, n), dtype=dt, device=dev)
        self.cn[2:r + 2] = cn_rows
        self.cm[2:r + 2] = cm_rows
        # the sweep intermediates are fp64 for either state dtype (pentab.h ch_dist_pass_a)
        f64 = torch.float64
        self.w = torch.empty((r, n), dtype=f64, device=dev)
        self.packed = torch.empty((P, r, n // P), dtype=f64, device=dev)
        self.cols = torch.empty((P, r, n // P), dtype=f64, device=dev)   # = [n][n/P] column block
        self.back = torch.empty((P, r, n // P), dtype=f64, device=dev)

    def interior(self, which="cn"):
        r = self.prm.rows
        return (self.cn if which == "cn" else self.cm)[2:r + 2]

    def rotate(self):
        self.cn, self.cm = self.cm, self.cn   # C^{n+1} was written over C^{n-1}


class LocalExchange:
    """All P ranks in one process (single device): the same data movement as
    the distributed exchange, used to test the partitioned kernels on 1 GPU."""

    def halo(self, states):
        P, r = len(states), states[0].prm.rows
        for k, st in enumerate(states):
            up, dn = states[(k - 1) % P], states[(k + 1) % P]
            for buf, ub, db in ((st.cn, up.cn, dn.cn), (st.cm, up.cm, dn.cm)):
                buf[0:2] = ub[r:r + 2]
                buf[r + 2:r + 4] = db[2:4]

    def alltoall(self, states, src, dst):
        P = len(states)
        for k, st in enumerate(states):
            out = getattr(st, dst)
            for q in range(P):
                out[q].copy_(getattr(states[q], src)[k])


class TorchExchange:
    """One rank per process over torch.distributed (NCCL / gloo)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group

    def halo(self, states):
        (st,) = states
        dist, r = self.dist, st.prm.rows
        P, k = dist.get_world_size(self.group), dist.get_rank(self.group)
        if P == 1:
            LocalExchange().halo(states)
            return
        up, dn = (k - 1) % P, (k + 1) % P
        ops, recv = [], []
        for f, buf in enumerate((st.cn, st.cm)):
            # NCCL matches the k-th send to a peer with the k-th receive from it
            # and ignores tags, so the posting order itself must pair up when
            # up == dn (P = 2): every rank posts send(bottom rows -> dn) before
            # send(top rows -> up), and recv(<- up) before recv(<- dn); the peer's
            # first message is then its bottom rows = our upper halo.  Tags (gloo)
            # agree with that pairing.
            t_up, t_dn = 1 + 2 * f, 2 + 2 * f
            top, bot = buf[2:4].contiguous(), buf[r:r + 2].contiguous()
            rt, rb = buf.new_empty((2, buf.shape[1])), buf.new_empty((2, buf.shape[1]))
            ops += [dist.P2POp(dist.isend, bot, dn, self.group, t_dn), dist.P2POp(dist.isend, top, up, self.group, t_up),
                    dist.P2POp(dist.irecv, rt, up, self.group, t_dn), dist.P2POp(dist.irecv, rb, dn, self.group, t_up)]
            recv.append((buf, rt, rb))
        for req in dist.batch_isend_irecv(ops):
            req.wait()
        for buf, rt, rb in recv:
            buf[0:2] = rt       # previous rank's last two rows
            buf[r + 2:r + 4] = rb   # next rank's first two rows

    def alltoall(self, states, src, dst):
        (st,) = states
        self.dist.all_to_all_single(getattr(st, dst), getattr(st, src), group=self.group)


def step(states, exchange):
    """One ADI step on every rank in `states` (all ranks for LocalExchange,
    the calling rank for TorchExchange)."""
    exchange.halo(states)
    for st in states:
        st.compute.pass_a(st.cn, st.cm, st.w)
        st.compute.pack(st.w, st.packed)
    exchange.alltoall(states, "packed", "cols")
    for st in states:
        st.compute.ysolve(st.cols)
    exchange.alltoall(states, "cols", "back")
    for st in states:
        st.compute.combine(st.cn, st.cm, st.back)
        st.rotate()
