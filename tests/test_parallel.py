"""Multi-process (world size 2, gloo, CPU) tests of the SNP-batch sharding and the result
gather used by the multi-GPU path."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1902_04303_b200.parallel import ShardPlan, batch_owner, shard_batches


def test_shard_batches_cover_exactly_once():
    for nb in (1, 2, 5, 21, 22):
        for world in (1, 2, 3, 8):
            seen = sorted(i for r in range(world) for i in shard_batches(nb, r, world))
            assert seen == list(range(nb))
            counts = ShardPlan(nb, world).per_rank_counts()
            assert max(counts) - min(counts) <= 1
            assert all(batch_owner(i, world) == r for r in range(world) for i in shard_batches(nb, r, world))
    with pytest.raises(ValueError):
        shard_batches(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_1902_04303_b200.parallel import gather_to_root, shard_batches

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    nb = 21
    local = {i: np.full(4, i, dtype=np.uint32) for i in shard_batches(nb, rank, world)}
    merged = gather_to_root(local, world)
    # max-over-ranks timing reduction as in bench.py
    import torch

    t = torch.tensor([1.0 + rank], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        q.put((sorted(merged), [int(v[0]) for _, v in sorted(merged.items())], float(t.item())))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_gather_and_max():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    keys, vals, tmax = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert keys == list(range(21)) and vals == list(range(21))
    assert tmax == 2.0


def _gather_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_1902_04303_b200 import CkksParams
    from paper_1902_04303_b200.ckks import Ciphertext
    from paper_1902_04303_b200.parallel import all_gather_ciphertexts, owned_columns
    from paper_1902_04303_b200.ring import RingElement

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    params = CkksParams(log_n=4, log_l=200, log_p=45, log_p_small=30, h=4)
    n, total, lv = params.n, 7, 100

    def words(i, part):   # a recognisable pattern per (column, poly)
        return torch.full(((lv + 31) // 32, n), 1000 * i + part, dtype=torch.int32)

    local = {i: Ciphertext(c0=RingElement(n, lv, words=words(i, 0)), c1=RingElement(n, lv, words=words(i, 1)),
                           level_bits=lv, scale_bits=45 + i, slots=params.slot_count, params=params, depth_ct=i)
             for i in owned_columns(total, rank, world)}
    got = all_gather_ciphertexts(local, total, world)
    ok = len(got) == total and all(
        int(c.c0.words[0, 0]) == 1000 * i and int(c.c1.words[-1, -1]) == 1000 * i + 1
        and c.scale_bits == 45 + i and c.depth_ct == i for i, c in enumerate(got))
    q.put((rank, ok))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_all_gather_ciphertexts_order_and_metadata():
    """The setup split's exchange (parallel.all_gather_ciphertexts): 7 columns owned round-robin
    by 2 ranks come back on both ranks in column order with their own metadata."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res == {0: True, 1: True}
