"""Multi-process host logic of the DP rollout workers on CPU (gloo, world_size 2).

HistoPipe assignment restated from rhymesim/scheduler.py:22-88 and the
epoch-boundary rollout routing (all-to-all-v) used between GPU workers.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2508_18588_b200 import workers as W


def test_assignment_matches_reference_semantics():
    med = {f"p{i:02d}": float(l) for i, l in enumerate([5, 1, 9, 3, 3, 7, 2, 8, 6])}
    groups = W.build_groups(med, 4)
    assert [len(g.prompt_ids) for g in groups] == [2, 2, 2, 3]          # remainder to the longest
    assert groups[0].prompt_ids == ["p01", "p06"]                          # lengths 1, 2
    assert groups[1].prompt_ids == ["p03", "p04"]                          # ties by id
    assert W.assignment_order(1, 4) == [0, 1, 2, 3] and W.assignment_order(2, 4) == [3, 2, 1, 0]
    a1, a2 = W.assign_prompts(med, 4, 1), W.assign_prompts(med, 4, 2)
    assert a1[0] == a2[3] and a1[3] == a2[0]
    with pytest.raises(ValueError):
        W.assignment_order(0, 4)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(rank)
    med = {i: float(100 + (i * 37) % 11) for i in range(12)}
    mine = W.assign_prompts(med, world, 1)[rank]
    rollouts = [(pid, rng.integers(0, 1000, size=int(rng.integers(1, 50))).astype(np.int32),
                 float(rng.integers(0, 64)) / 64.0) for pid in mine for _ in range(3)]
    owner = W.owner_map(W.assign_prompts(med, world, 2))
    got = W.route_rollouts(rollouts, owner, rank, world)
    out[rank] = ([(p, t.tolist(), r) for p, t, r in rollouts], [(p, t.tolist(), r) for p, t, r in got], owner)
    dist.destroy_process_group()


def test_route_rollouts_all_to_all_world2():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    sent = [r for k in range(world) for r in out[k][0]]
    owner = out[0][2]
    for rank in range(world):
        expect = [r for src in range(world) for r in out[src][0] if owner[r[0]] == rank]
        assert out[rank][1] == expect
    assert sum(len(out[k][1]) for k in range(world)) == len(sent)


def _meta_worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(10 + rank)
    med = {i: float(100 + (i * 37) % 11) for i in range(12)}
    mine = W.assign_prompts(med, world, 1)[rank]
    pids = np.repeat(np.asarray(mine, np.int64), 2)
    lens = rng.integers(1, 50, size=len(pids))
    keys = np.arange(len(pids)) + 100 * rank
    rew = rng.integers(0, 4, size=len(pids)) << 30
    owner = W.owner_map(W.assign_prompts(med, world, 2))
    plan = W.plan_routes(pids, lens, owner, world)
    meta = np.stack([pids, keys, lens, rew], axis=1).astype(np.int64)
    rc, got = W.exchange_route_meta(plan, meta, "cpu")
    out[rank] = (meta.tolist(), got.tolist(), rc.tolist(), owner)
    dist.destroy_process_group()


def test_route_meta_exchange_world2():
    """Device routing's host plan + record-table exchange (workers.plan_routes / exchange_route_meta)."""
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_meta_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    owner = out[0][3]
    for rank in range(world):
        expect = []
        for src in range(world):
            rows = [r for r in out[src][0] if owner[r[0]] == rank]
            rows.sort(key=lambda r: r[0])            # send order: destination, prompt, input order (stable)
            expect += rows
        assert out[rank][1] == expect
        assert [c[1] for c in out[rank][2]] == [sum(r[2] for r in out[src][0] if owner[r[0]] == rank)
                                                for src in range(world)]


def _broker_worker(rank, world, port, out):
    import time

    import torch.distributed as dist
    from torch.distributed import distributed_c10d as c10d
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b = W.MigrationBroker(c10d._get_default_store(), rank, world, tag="t")
    dist.barrier()
    got = []
    if rank == 0:
        for i in range(3):
            b.post(1, {"key": i, "tokens": list(range(i + 1))})
            time.sleep(0.05)
    t0 = time.time()
    while True:
        got += b.poll()
        if not b.keep_alive():
            break
        assert time.time() - t0 < 30, "broker never terminated"
        time.sleep(0.01)
    out[rank] = got
    dist.barrier()
    dist.destroy_process_group()


def test_migration_broker_delivers_and_terminates():
    """MigrationBroker (intra-step migration transport): every posted rollout is taken exactly once by its
    destination and no worker stops while a message is in flight."""
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_broker_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    assert out[0] == []
    assert [m["key"] for m in out[1]] == [0, 1, 2] and out[1][2]["tokens"] == [0, 1, 2]
