"""Multi-GPU batch path, host side (runs on CPU): LPT sharding of independent
atlases and a world_size-2 gloo run of the rank-sharded batch
loop that bench.py uses under torchrun (no collective on the data path; the
only collectives are the barrier and the max-over-ranks timing)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import chartgen


def test_shard_plan_lpt_properties():
    from paper_2602_07782_b200 import shard_plan
    sizes = chartgen.config5_sizes(512)
    for g in (1, 2, 3, 4, 8):
        a = shard_plan(sizes, g)
        assert a.min() >= 0 and a.max() < g
        cost = np.array([n * (1 + np.log2(n + 1)) for n in sizes])
        load = np.bincount(a, weights=cost, minlength=g)
        # LPT: the spread of loads is at most the largest single job
        assert load.max() - load.min() <= cost.max() + 1e-6
        assert np.array_equal(a, shard_plan(sizes, g))  # deterministic


def test_shard_plan_rejects_bad_args():
    from paper_2602_07782_b200 import TabiError, shard_plan
    with pytest.raises(TabiError):
        shard_plan([10, 20], 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, sizes, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    import torch
    from paper_2602_07782_b200 import shard_plan
    a = shard_plan(sizes, ws)
    mine = [i for i in range(len(sizes)) if a[i] == rank]
    t = torch.zeros(len(sizes), dtype=torch.int32)
    t[mine] = rank + 1
    dist.all_reduce(t)  # gather of the assignment only (the "collective" of §8(e))
    load = torch.tensor([float(sum(sizes[i] for i in mine))])
    dist.all_reduce(load, op=dist.ReduceOp.MAX)
    if rank == 0:
        q.put((t.tolist(), float(load.item())))
    dist.destroy_process_group()


def test_gloo_world2_disjoint_cover():
    sizes = chartgen.config5_sizes(64)
    q = mp.get_context("spawn").SimpleQueue()
    port = _free_port()
    ctx = mp.get_context("spawn")
    ps = [ctx.Process(target=_worker, args=(r, 2, port, sizes, q)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(120)
        assert p.exitcode == 0
    owners, maxload = q.get()
    assert sorted(set(owners)) == [1, 2]  # every atlas owned by exactly one rank
    assert maxload <= sum(sizes) * 0.5 + max(sizes)


def _bench_worker(rank, ws, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    import sys
    import torch
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    from paper_2602_07782_b200 import concat_chart_sets
    share = bench.rank_share(ws, rank)  # the exact code path of bench.py's C5 step
    t = torch.zeros(bench.C5_ATLASES, dtype=torch.int32)
    t[share] = 1
    dist.all_reduce(t)
    # the rank's batch layout for tabi_pack_many (first three atlases of its share)
    sets = [chartgen.config5(i) for i in share[:3]]
    xy, cst, abase, res = concat_chart_sets(sets)
    ok = (abase[0] == 0 and abase[-1] == sum(cs.n_charts for cs in sets) and
          cst[-1] * 2 == xy.shape[0] and
          all(np.array_equal(cst[abase[j]:abase[j + 1] + 1] - cst[abase[j]], sets[j].start)
              for j in range(3)))
    okt = torch.tensor([1 if ok else 0], dtype=torch.int32)
    dist.all_reduce(okt, op=dist.ReduceOp.MIN)
    if rank == 0:
        q.put((t.tolist(), int(okt.item())))
    dist.destroy_process_group()


def test_gloo_world2_bench_batch_shares():
    """bench.py's multi-GPU C5 step under a world-size-2 gloo group: the two
    ranks' LPT shares cover the 512 atlases exactly once, and each rank's
    concatenated tabi_pack_many layout (global vertex offsets, atlas offsets)
    reproduces every atlas's own outline offsets."""
    q = mp.get_context("spawn").SimpleQueue()
    port = _free_port()
    ctx = mp.get_context("spawn")
    ps = [ctx.Process(target=_bench_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(300)
        assert p.exitcode == 0
    cover, ok = q.get()
    assert cover == [1] * 512 and ok == 1
