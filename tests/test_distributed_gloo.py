"""Multi-rank plumbing on CPU (gloo, world_size 2): sharding + the winner exchange.

Chains are sharded across ranks; each rank reduces its chains to one record,
records are all-gathered and reduced in the same fixed order everywhere, and
the winner equals the single-process winner (sharding invariance).
"""

import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2304_09781_b200.distributed import (gather_records, make_record, reduce_records_host, shard,
                                               order_key)


def _chain_outcomes(total):
    rng = np.random.default_rng(123)
    sla = rng.random(total) < 0.4
    h = np.round(rng.normal(-10, 3, total), 1)     # coarse values force ties broken by index
    return sla, h


def _worker(rank, world, port, total, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sla, h = _chain_outcomes(total)
    b, e = shard(total, rank, world)
    recs = np.concatenate([make_record(bool(sla[i]), float(h[i]), i) for i in range(b, e)])
    local = reduce_records_host(recs)
    t = torch.from_numpy(np.frombuffer(local.tobytes(), dtype=np.uint8).copy())
    g = gather_records(t)
    allrecs = np.frombuffer(g.numpy().tobytes(), dtype=local.dtype)
    win = reduce_records_host(allrecs)
    out[rank] = int(win["index"])
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_balanced():
    for total in (0, 1, 7, 1024):
        for world in (1, 2, 3, 8):
            spans = [shard(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(e - b for b, e in spans) - min(e - b for b, e in spans) <= 1


def test_order_key_monotone():
    xs = np.sort(np.concatenate([np.random.default_rng(0).normal(0, 100, 1000), [-0.0, 0.0, -1e-300, 1e-300]]))
    keys = [order_key(float(x)) for x in xs]
    assert all(a <= b for a, b in zip(keys, keys[1:]))
    assert order_key(-0.0) == order_key(0.0)


def test_two_rank_exchange_matches_single_process():
    total = 37
    sla, h = _chain_outcomes(total)
    single = reduce_records_host(np.concatenate([make_record(bool(sla[i]), float(h[i]), i) for i in range(total)]))
    manager = mp.Manager()
    out = manager.dict()
    mp.start_processes(_worker, args=(2, _free_port(), total, out), nprocs=2, join=True, start_method="spawn")
    assert out[0] == out[1] == int(single["index"])
