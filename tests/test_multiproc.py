"""Multi-rank host logic on CPU with the gloo backend (world_size 2): sharding,
shard-invariant input generation, and the final statistics reduction."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from cvsr_inputs.awgn import torch_quadratures
from paper_2108_08418_b200 import dist as cdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    F = 5
    first, cnt = cdist.shard(F, rank)
    x, y = torch_quadratures(cnt, 33, 1.0, "cpu", first_frame=first, chunk=4)
    stats = {"bits": 100 * (rank + 1), "frames": cnt, "frames_ok": cnt - rank, "undetected": rank}
    sums, it, ei, tm = cdist.reduce_stats(stats, [1.0 + rank, 2.0], [10.0, 20.0 * rank], [3.0 + rank, 7.0 - rank],
                                          "cpu")
    q.put((rank, first, x.numpy(), y.numpy(), sums, it, ei, tm))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_two_ranks_shard_and_reduce():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # shard-invariant data: the two shards equal one 10-frame generation
    x_all, y_all = torch_quadratures(10, 33, 1.0, "cpu", first_frame=0, chunk=4)
    assert (res[0][2] == x_all[:5].numpy()).all() and (res[1][2] == x_all[5:].numpy()).all()
    assert (res[1][3] == y_all[5:].numpy()).all()
    for r in res:
        sums, it, ei, tm = r[4:]
        assert sums == {"bits": 300.0, "frames": 10.0, "frames_ok": 9.0, "undetected": 1.0}
        assert it == [3.0, 4.0] and ei == [20.0, 20.0]
        assert tm == [4.0, 7.0]  # MAX over ranks


def test_reduce_without_process_group_is_identity():
    s, it, ei, tm = cdist.reduce_stats({"bits": 1, "frames": 2, "frames_ok": 2, "undetected": 0}, [5], [6], [7.5],
                                       "cpu")
    assert s["bits"] == 1 and it == [5] and ei == [6] and tm == [7.5]
