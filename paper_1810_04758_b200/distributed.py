"""Multi-GPU plumbing for knnj_run_shard: one process per GPU under torchrun.

The join itself needs no collective (queries are sharded by contiguous grid-cell
ranges; points and grid are replicated). The run's only exchange is
the eps-selection histogram: each rank bins its slice of the sampled queries and
the u64 bin counts are summed across ranks. ``torch_allreduce`` adapts
torch.distributed (NCCL on GPUs, gloo in the CPU tests) to the C ABI's
``knnj_allreduce_fn``; ``merge_shards`` reassembles the per-rank outputs into the
single-GPU result (rows in ascending query id).
"""
from __future__ import annotations

from typing import Callable, Optional, Sequence

import numpy as np


def torch_allreduce(group=None, device: Optional[str] = None) -> Callable[[np.ndarray], None]:
    """In-place element-wise SUM of a uint64 numpy array over ``group``.

    Counts stay far below 2**63, so they travel as int64; ``device`` is where the
    staging tensor lives ("cuda:<i>" for NCCL, "cpu" for gloo; default: the
    backend's natural device)."""
    import torch
    import torch.distributed as dist

    if device is None:
        device = "cpu" if dist.get_backend(group) == "gloo" else f"cuda:{torch.cuda.current_device()}"

    def reduce(a: np.ndarray) -> None:
        if a.dtype != np.uint64:
            raise TypeError("allreduce expects uint64 counts")
        if a.size and int(a.max()) >= 2 ** 63:
            raise OverflowError("count exceeds the int64 transport range")
        t = torch.from_numpy(a.view(np.int64).copy()).to(device)
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        a[:] = t.cpu().numpy().view(np.uint64)

    return reduce


def merge_shards(parts: Sequence[tuple], n_queries: int, k: int):
    """Union of per-shard (queries, ids, dist, prov) into full arrays ordered by query id.

    Raises if the shards overlap or leave a query uncovered (the partition must tile
    the query set exactly)."""
    ids = np.zeros((n_queries, k), np.uint32)
    dist = np.zeros((n_queries, k), np.float64)
    prov = np.zeros(n_queries, np.uint8)
    seen = np.zeros(n_queries, np.int32)
    allq = np.concatenate([np.asarray(p[0], np.int64) for p in parts]) if parts else np.zeros(0)
    order = np.unique(allq)
    if order.size != n_queries or allq.size != n_queries:
        raise ValueError(f"shards cover {allq.size} rows / {order.size} queries, expected {n_queries}")
    index = {int(q): i for i, q in enumerate(order)} if order.size else {}
    for q, i_, d_, p_ in parts:
        rows = np.fromiter((index[int(x)] for x in q), np.int64, len(q))
        ids[rows] = np.asarray(i_).reshape(len(q), k)
        dist[rows] = np.asarray(d_).reshape(len(q), k)
        prov[rows] = np.asarray(p_)[:len(q)]
        seen[rows] += 1
    if (seen != 1).any():
        raise ValueError("shards overlap")
    return order.astype(np.uint32), ids, dist, prov
