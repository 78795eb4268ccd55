"""CPU (gloo, world_size 2): the host side of the multi-GPU path.

* torch_allreduce — the knnj_allreduce_fn adapter the bench hands to knnj_run_shard —
  sums uint64 histogram counts across ranks;
* knnj_shard_range (host-only C ABI, no GPU) gives every rank the same partition:
  contiguous runs that tile the items with balanced cost;
* merge_shards rebuilds the single-GPU output order from the per-rank rows.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch.distributed as dist

    from paper_1810_04758_b200.distributed import torch_allreduce
    from paper_1810_04758_b200.engine import shard_range
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        red = torch_allreduce()
        a = np.arange(100, dtype=np.uint64) * np.uint64(rank + 1) + np.uint64(2 ** 40)
        red(a)
        want = np.arange(100, dtype=np.uint64) * np.uint64(sum(range(1, world + 1))) + \
            np.uint64(world * 2 ** 40)
        ok_reduce = bool(np.array_equal(a, want))
        rng = np.random.default_rng(5)
        cost = rng.exponential(1.0, 1000) * 1000 + 1024   # skewed cells (C4-like)
        mine = shard_range(cost, rank, world)
        gathered = [None] * world
        dist.all_gather_object(gathered, mine)
        out[rank] = (ok_reduce, gathered, float(cost[mine[0]:mine[1]].sum() / cost.sum()))
    finally:
        dist.destroy_process_group()


def test_gloo_allreduce_and_partition():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    assert all(out[r][0] for r in range(world))
    ranges = out[0][1]
    assert ranges == out[1][1]                     # same partition on every rank
    assert ranges[0][0] == 0 and ranges[-1][1] == 1000
    for (a, b), (c, d) in zip(ranges, ranges[1:]):
        assert b == c                              # contiguous tiling
    shares = [out[r][2] for r in range(world)]
    assert all(abs(s - 1 / world) < 0.01 for s in shares), shares


@pytest.mark.parametrize("ns", [1, 2, 3, 8])
def test_shard_range_tiles(ns):
    from paper_1810_04758_b200.engine import shard_range
    cost = np.random.default_rng(ns).uniform(1, 10, 377)
    runs = [shard_range(cost, k, ns) for k in range(ns)]
    assert runs[0][0] == 0 and runs[-1][1] == 377
    assert all(runs[i][1] == runs[i + 1][0] for i in range(ns - 1))
    if ns > 1:
        shares = [cost[a:b].sum() / cost.sum() for a, b in runs]
        assert max(shares) - min(shares) < 2 * cost.max() / cost.sum() + 1e-12


def test_merge_shards_roundtrip():
    from paper_1810_04758_b200.distributed import merge_shards
    N, k = 50, 3
    ids = np.arange(N * k, dtype=np.uint32).reshape(N, k)
    dist = ids.astype(np.float64) / 7
    prov = (np.arange(N) % 3).astype(np.uint8)
    perm = np.random.default_rng(1).permutation(N)
    parts = []
    for chunk in np.array_split(perm, 3):
        q = np.sort(chunk)
        parts.append((q.astype(np.uint32), ids[q], dist[q], prov[q]))
    q, i2, d2, p2 = merge_shards(parts, N, k)
    assert np.array_equal(q, np.arange(N)) and np.array_equal(i2, ids)
    assert np.array_equal(d2, dist) and np.array_equal(p2, prov)
    with pytest.raises(ValueError):
        merge_shards(parts[:2], N, k)
