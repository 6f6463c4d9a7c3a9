"""Host logic of the row-partitioned ADI step (paper_2101_06550_b200.dist,
configs[4]) on CPU: P ranks emulated in one process (LocalExchange) and two
real gloo ranks (TorchExchange), with the oracle as compute backend; the
partitioned result must equal the oracle's single-grid ADI step."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import oracle
import synth
from paper_2101_06550_b200 import dist
from dist_helpers import OracleCompute


def _setup(n, parts, seed=5):
    L = n * synth.DX_STATS
    dt = synth.ch_dt(n, L)
    c0 = synth.ch_ic_random(1, n, seed=seed)[0]
    c1, _ = oracle.ch_adi_steps(c0, c0, 1, dt=dt, D=1.0, gamma=0.01, L=L)
    prm = dist.Params(n=n, parts=parts, dt=dt, L=L)
    return prm, c0, c1


@pytest.mark.parametrize("n,parts", [(32, 1), (32, 2), (48, 4), (64, 8)])
def test_local_exchange_matches_single_grid(n, parts):
    prm, c0, c1 = _setup(n, parts)
    r = prm.rows
    states = [dist.RankState(prm, k, torch.from_numpy(c1[k * r:(k + 1) * r]), torch.from_numpy(c0[k * r:(k + 1) * r]),
                             OracleCompute(prm)) for k in range(parts)]
    for _ in range(3):
        dist.step(states, dist.LocalExchange())
    got = np.concatenate([s.interior("cn").numpy() for s in states])
    ref, _ = oracle.ch_adi_steps(c1, c0, 3, dt=prm.dt, D=1.0, gamma=0.01, L=prm.L)
    assert np.max(np.abs(got - ref)) / np.max(np.abs(ref)) <= 1e-12


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, q):
    import torch.distributed as tdist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        prm, c0, c1 = _setup(n, world)
        r = prm.rows
        st = dist.RankState(prm, rank, torch.from_numpy(c1[rank * r:(rank + 1) * r]),
                            torch.from_numpy(c0[rank * r:(rank + 1) * r]), OracleCompute(prm))
        for _ in range(2):
            dist.step([st], dist.TorchExchange())
        q.put((rank, st.interior("cn").numpy().copy()))
    finally:
        tdist.destroy_process_group()


def test_gloo_two_ranks_match_single_grid():
    n, world = 32, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    got = np.concatenate([out[r] for r in range(world)])
    prm, c0, c1 = _setup(n, world)
    ref, _ = oracle.ch_adi_steps(c1, c0, 2, dt=prm.dt, D=1.0, gamma=0.01, L=prm.L)
    assert np.max(np.abs(got - ref)) / np.max(np.abs(ref)) <= 1e-12


class _FakeNccl:
    """torch.distributed stand-in with NCCL's point-to-point matching: the k-th
    send from a to b pairs with the k-th receive on b from a, tags ignored."""

    import queue as _q
    import threading as _t

    def __init__(self, world):
        self.world = world
        self.chan = {(a, b): self._q.Queue() for a in range(world) for b in range(world)}
        self.local = self._t.local()

    def get_world_size(self, group=None):
        return self.world

    def get_rank(self, group=None):
        return self.local.rank

    def isend(self):  # markers only
        pass

    def irecv(self):
        pass

    class P2POp:
        def __init__(self, op, tensor, peer, group=None, tag=0):
            self.op, self.tensor, self.peer = op, tensor, peer

    def batch_isend_irecv(self, ops):
        me = self.local.rank
        reqs = []
        for o in ops:
            if o.op == self.isend:
                self.chan[(me, o.peer)].put(o.tensor.clone())
        for o in ops:
            if o.op == self.irecv:
                reqs.append((o.tensor, self.chan[(o.peer, me)]))

        class _Req:
            def __init__(self, t, ch):
                self.t, self.ch = t, ch

            def wait(self):
                self.t.copy_(self.ch.get(timeout=30))

        return [_Req(t, ch) for t, ch in reqs]


@pytest.mark.parametrize("world", [2, 3])
def test_halo_posting_order_pairs_under_nccl_matching(world):
    """The halo exchange must be correct when messages pair by posting order
    (NCCL), not by tag: at P = 2 both neighbours are the same peer."""
    import threading

    n = 16
    r = n // world if n % world == 0 else None
    n = r * world if r else 12 * world
    prm = dist.Params(n=n, parts=world, dt=0.01, L=1.0)
    r = prm.rows
    full = torch.arange(n * n, dtype=torch.float64).reshape(n, n)
    fake = _FakeNccl(world)
    ex = dist.TorchExchange()
    ex.dist = fake
    states = [dist.RankState(prm, k, full[k * r:(k + 1) * r], -full[k * r:(k + 1) * r], None) for k in range(world)]

    def run(k):
        fake.local.rank = k
        ex.halo([states[k]])

    th = [threading.Thread(target=run, args=(k,)) for k in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=60)
    for k, st in enumerate(states):
        rows = [(k * r + j) % n for j in range(-2, r + 2)]
        assert torch.equal(st.cn, full[rows]), k
        assert torch.equal(st.cm, -full[rows]), k
