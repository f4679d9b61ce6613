"""N > 1 host logic on CPU (gloo, world_size 2, 4 and 8): every rank computes its placement with
the library's host-only plan functions; the union over ranks must assign each routed expert to
exactly one GPU of the layer's group (P:104 one-to-one; S:288 sorted pairing; l mod N_G round
robin) and every rank's pool must hold whatever it can be assigned."""
import os
import random

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2512_03927_b200 import odmoe
    E, k, L = 8, 2, 32
    rng = random.Random(1234)  # same routing stream on every rank
    ok = True
    for _ in range(200):
        l = rng.randrange(L)
        ids = rng.sample(range(E), k)
        mine = odmoe.plan_layer(k, world, l, ids, rank)
        for e in mine:
            ok &= odmoe.plan_pool_holds(E, k, world, l, e, rank)
        gathered = [None] * world
        dist.all_gather_object(gathered, (l, ids, mine))
        if rank == 0:
            G = O.plan_group_size(k, world)
            NG = world // G
            groups = O.plan_groups(world, G)
            want = O.assign_experts(ids, groups[O.assign_layer(l, NG)])
            got = {}
            for r, (_, _, m) in enumerate(gathered):
                for e in m:
                    assert e not in got, "expert computed twice"
                    got[e] = r
            ok &= got == want
    # pool coverage: a blob is held by rank r iff some routing can send it there
    for l in range(L):
        for e in range(E):
            holders = [r for r in range(world) if odmoe.plan_pool_holds(E, k, world, l, e, r)]
            ok &= len(holders) >= 1
    # max-over-ranks timing reduction used by bench.py
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ok &= float(t) == float(world)
    dist.barrier()
    dist.destroy_process_group()
    q.put((rank, bool(ok)))


@pytest.mark.parametrize("world", [2, 4, 8])
def test_multirank_placement_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + world * 7 + os.getpid() % 97
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok in res), res


def test_plan_single_gpu_takes_all():
    from paper_2512_03927_b200 import odmoe
    assert odmoe.plan_layer(2, 1, 7, [5, 1], 0) == [1, 5]
    assert all(odmoe.plan_pool_holds(8, 2, 1, l, e, 0) for l in range(4) for e in range(8))
    # at 8 GPUs (4 groups) layer 5 goes to group 1 = GPUs {2, 3}
    assert odmoe.plan_layer(2, 8, 5, [6, 2], 2) == [2]
    assert odmoe.plan_layer(2, 8, 5, [6, 2], 3) == [6]
    assert odmoe.plan_layer(2, 8, 5, [6, 2], 0) == []
    # position 0 of a pair never receives expert 7; position 1 never expert 0
    assert not odmoe.plan_pool_holds(8, 2, 2, 0, 7, 0) and not odmoe.plan_pool_holds(8, 2, 2, 0, 0, 1)
    with pytest.raises(odmoe.OdmoeError):
        odmoe.plan_layer(2, 3, 0, [0, 1], 0)
