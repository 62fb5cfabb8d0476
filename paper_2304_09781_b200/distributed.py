"""Multi-GPU plumbing: chain / index sharding and the per-round winner exchange.

Independent chains and ORACLE / sweep index ranges
partition across ranks with no data-path collective; each round ends with one
all-gather of a 32-byte winner record per rank (NCCL over NVLink on the GPU
path, gloo in the CPU tests) and the same fixed-order reduction on every rank,
so the selected configuration is identical for any world size.
"""

from __future__ import annotations

import numpy as np

RECORD_DTYPE = np.dtype([("k1", "<u8"), ("k2", "<u8"), ("index", "<i8"), ("h", "<f8")])
NO_RECORD = np.array([(np.iinfo(np.uint64).max, np.iinfo(np.uint64).max, np.iinfo(np.int64).max, 0.0)],
                     dtype=RECORD_DTYPE)[0]


def shard(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [begin, end) share of ``total`` units for ``rank`` (balanced to within 1)."""
    base, extra = divmod(int(total), int(world))
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def order_key(h: float) -> int:
    """Order-preserving uint64 of a double (the device's okey; -0 folds onto +0)."""
    u = int(np.array([h + 0.0], dtype=np.float64).view(np.uint64)[0])
    return (~u) & ((1 << 64) - 1) if u >> 63 else u | (1 << 63)


def make_record(sla: bool, h: float, index: int) -> np.ndarray:
    return np.array([(0 if sla else 1, order_key(h), int(index), float(h))], dtype=RECORD_DTYPE)


def reduce_records_host(recs: np.ndarray):
    """Fixed-order winner: (SLA desc, h asc, index asc) -- identical to clv_reduce_records."""
    recs = np.asarray(recs, dtype=RECORD_DTYPE).reshape(-1)
    if len(recs) == 0:
        return NO_RECORD
    i = np.lexsort((recs["index"], recs["k2"], recs["k1"]))[0]
    return recs[i]


def gather_records(record, group=None):
    """All-gather one 32-byte record (uint8 tensor) per rank; returns a [world*32] tensor."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    if record.is_cuda:
        out = record.new_empty(world * 32)
        dist.all_gather_into_tensor(out, record, group=group)
        return out
    parts = [torch.empty_like(record) for _ in range(world)]
    dist.all_gather(parts, record, group=group)
    return torch.cat(parts)
