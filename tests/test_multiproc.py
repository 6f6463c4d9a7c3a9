"""World-size-2 gloo tests of bench.py's multi-rank host logic (CPU only):
sharding of independent units and max-over-ranks timing."""
import os
import socket

import pytest
import torch.multiprocessing as mp

import bench


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        t = bench.max_over_ranks(10.0 + rank, device="cpu")
        s = bench.sum_over_ranks(1.5 * (rank + 1), device="cpu")
        lo, hi = bench.shard(512, world, rank)
        q.put((rank, t, s, lo, hi))
    finally:
        dist.destroy_process_group()


def test_shard_partitions_exactly():
    for total in (0, 1, 7, 512, 513):
        for world in (1, 2, 3, 8):
            spans = [bench.shard(total, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def test_gloo_two_ranks_max_and_shard():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = sorted(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, t, s, lo, hi in out:
        assert t == 11.0  # max over ranks
        assert s == pytest.approx(4.5)
    assert [(lo, hi) for _, _, _, lo, hi in out] == [(0, 256), (256, 512)]


def test_reference_arm_runs_on_cpu(capsys):
    """--impl reference times the oracle (the reference arm of this tier) on rank 0."""
    import json
    bench.main(["--impl", "reference", "--steps", "1", "--warmup", "3"])
    line = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "oracle"
