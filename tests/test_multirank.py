"""Multi-rank host logic on CPU (gloo, world size 2): the LPT tensor sharding
every rank computes independently must agree across ranks, partition the
model, stay balanced, and the timing reduction must give max-over-ranks time
and summed bytes (the bench's whole-job throughput)."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2410_20650_b200 import shard


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def llama_sizes(layers, h, f, kv, vocab):
    sizes = []
    for _ in range(layers):
        sizes += [h * h, kv * h, kv * h, h * h, f * h, f * h, h * f, h, h]
    return sizes + [vocab * h, vocab * h, h]


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sizes = llama_sizes(80, 8192, 28672, 1024, 128256)  # Llama-3-70B (config C4)
        owner = shard.lpt_assign(sizes, world)
        plans = [None] * world
        dist.all_gather_object(plans, owner)
        mine = [i for i, r in enumerate(owner) if r == rank]
        local_bytes = sum(sizes[i] for i in mine)
        t_max, total = shard.reduce_timing(dist, 0.5 + rank, local_bytes)
        q.put((rank, plans[0] == plans[1], sorted(mine), local_bytes, t_max, total))
    finally:
        dist.destroy_process_group()


def test_lpt_two_ranks_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    sizes = llama_sizes(80, 8192, 28672, 1024, 128256)
    assert all(r[1] for r in res)  # identical plans on every rank
    a, b = set(res[0][2]), set(res[1][2])
    assert not (a & b) and a | b == set(range(len(sizes)))  # disjoint cover
    assert res[0][3] + res[1][3] == sum(sizes)
    assert all(r[4] == 1.5 for r in res)  # max over ranks
    assert all(r[5] == sum(sizes) for r in res)  # summed bytes
    assert max(res[0][3], res[1][3]) / (sum(sizes) / 2) < 1.01


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_lpt_balance_llama70b(world):
    sizes = llama_sizes(80, 8192, 28672, 1024, 128256)
    assert sum(sizes) == 70553706496
    assert shard.imbalance(sizes, world) < 1.02


def test_lpt_deterministic_and_complete():
    sizes = [5, 5, 3, 3, 3, 1, 0, 7]
    o = shard.lpt_assign(sizes, 3)
    assert o == shard.lpt_assign(sizes, 3)
    assert sorted(set(o)) == [0, 1, 2]
    loads = shard.shard_loads(sizes, o, 3)
    assert sum(loads) == 27 and max(loads) <= 10  # LPT bound: <= 4/3 of optimal (9)
