"""Streamed level-0 results (knnj_capi.cu run_pass / run_impl): the join runs in launch
chunks, each chunk's finalize overlaps the next chunk's join on a second stream and, for
pinned host outputs, stores its rows straight into host memory; rows the exact slow path
or the fallback rewrite afterwards are patched at the end. None of it may change an
output bit: compared with one launch and a bulk copy into pageable buffers, and with the
oracle's exact brute force on sampled queries."""
import ctypes as C

import numpy as np
import pytest

from paper_1810_04758_b200 import RunConfig
from paper_1810_04758_b200.synthetic import generate

pytestmark = pytest.mark.gpu


def _lattice(N, n, seed):
    rng = np.random.default_rng(seed)
    X = rng.integers(0, 24, (N, n)).astype(np.float64) / 8.0
    X[: N // 10] += rng.random((N // 10, n)) * 1e-9
    return X


def _pinned(lib, count, dtype):
    nbytes = count * np.dtype(dtype).itemsize
    p = lib.knnj_alloc_pinned(nbytes)
    assert p
    buf = (C.c_char * nbytes).from_address(p)
    return p, np.frombuffer(buf, dtype=dtype, count=count)


@pytest.mark.parametrize("spec,N,n,k", [("clusters:16:0.05", 40000, 18, 32), ("exponential", 40000, 6, 40),
                                        ("uniform", 60000, 2, 10), ("lattice", 30000, 4, 12),
                                        ("uniform", 50000, 4, 32)])
def test_streamed_results_identical(engine, oracle, spec, N, n, k):
    X = _lattice(N, n, 3) if spec == "lattice" else generate(spec, N, n, 61)
    cfg = RunConfig(k=k, mode="hybrid", seed=61)
    lib = engine.lib
    # reference run: one launch, results copied after the run into pageable buffers
    engine.set_option("join_chunks", 1)
    engine.set_points(X)
    a = engine.run(cfg, want_hist=False)
    # streamed: 8 chunks of >= 1 row, pinned outputs written by the finalize
    engine.set_option("join_chunks", 8)
    engine.set_option("chunk_min_rows", 1)
    ptrs = []
    got = []
    try:
        pi, ids = _pinned(lib, N * k, np.uint32)
        pd, dist = _pinned(lib, N * k, np.float64)
        pp, prov = _pinned(lib, N, np.uint8)
        ptrs = [pi, pd, pp]
        for cb in (74, 0):  # the row copy on a bounded grid, then one warp per row
            engine.set_option("copy_blocks", cb)
            ids[:] = 0xFFFFFFFF
            dist[:] = -1.0
            engine.set_points(X)
            b = engine.run(cfg, out=(pi, pd, pp), want_hist=False)
            got.append((ids.reshape(N, k).copy(), dist.reshape(N, k).copy(), prov.copy()))
        # device-resident leg, pageable copy
        engine.set_points(X)
        c = engine.run(cfg, want_hist=False)
    finally:
        engine.set_option("chunk_min_rows", 65536)
        engine.set_option("copy_blocks", 74)
        for p in ptrs:
            lib.knnj_free_pinned(p)
    for bi, bd, bp in got:
        assert np.array_equal(bi, a.ids) and np.array_equal(bd, a.dist)
        assert np.array_equal(bp, a.provenance)
    bi, bd, bp = got[0]
    assert np.array_equal(c.ids, a.ids) and np.array_equal(c.dist, a.dist)
    assert b.info["fallback_queries"] == a.info["fallback_queries"]
    assert b.info["slow_path_queries"] == a.info["slow_path_queries"]
    W = X[:, a.info["perm"]]
    q = np.random.default_rng(5).choice(N, 40, replace=False).astype(np.uint32)
    oi, od = oracle.brute_knn(W, q, k)
    assert np.array_equal(bi[q], oi) and np.array_equal(bd[q], od)


@pytest.mark.parametrize("spec,N,n,k,q,grid", [("clusters:16:0.05", 40000, 18, 32, 990, 0),
                                               ("uniform", 60000, 4, 32, 500, 0),
                                               ("uniform", 60000, 4, 32, 500, 1),
                                               ("exponential", 40000, 6, 40, 990, 1),
                                               ("lattice", 30000, 4, 12, 900, 1),
                                               ("uniform", 50000, 2, 10, 300, 1),
                                               ("mixture:8:0.05", 20000, 90, 16, 990, 0)])
def test_radius_bounded_pass_identical(engine, oracle, spec, N, n, k, q, grid):
    """The radius-bounded level-0 pass (the K-th of a query sample at quantile q bounds
    the box filter and the list cut; rows it misses are re-run without it) gives every
    row exactly the unbounded pass's output. Low quantiles force many misses."""
    X = _lattice(N, n, 4) if spec == "lattice" else generate(spec, N, n, 67)
    cfg = RunConfig(k=k, mode="hybrid", seed=67)
    engine.set_option("kth_bound", 0)
    engine.set_points(X)
    a = engine.run(cfg, want_hist=False)
    engine.set_option("kth_bound", 1)
    engine.set_option("bound_min_rows", 0)
    engine.set_option("bound_sample", 512)
    engine.set_option("kth_bound_q", q)
    engine.set_option("bound_grid", grid)  # 1: the bounded pass on a grid of width ~B, cell runs
    try:
        engine.set_points(X)
        b = engine.run(cfg, want_hist=False)
    finally:
        engine.set_option("bound_min_rows", 200000)
        engine.set_option("bound_sample", 4096)
        engine.set_option("kth_bound_q", 999)
        engine.set_option("bound_grid", 0)
    assert np.array_equal(b.ids, a.ids) and np.array_equal(b.dist, a.dist)
    assert np.array_equal(b.provenance, a.provenance)
    assert b.info["failed_count"] == a.info["failed_count"]
    assert b.info["fallback_queries"] == a.info["fallback_queries"]
    if b.info["kth_bound2"] > 0:
        assert b.info["join_screened_pairs"] <= a.info["join_screened_pairs"] + \
            b.info["bound_retried"] * N
    W = X[:, a.info["perm"]]
    qs = np.random.default_rng(9).choice(N, 32, replace=False).astype(np.uint32)
    oi, od = oracle.brute_knn(W, qs, k)
    assert np.array_equal(b.ids[qs], oi) and np.array_equal(b.dist[qs], od)
