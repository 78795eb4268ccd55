"""GPU: the capped eps-selection histogram and the cell-range sharded run.

* hist_cap: when the profile is not requested, only the low bins select_eps_beta
  reads are counted (pilot slice in full, the rest below the cap edge). eps and
  every output must be identical to the full-histogram run / the oracle.
* knnj_run_shard: S shards (threads, one context each, on cuda:0, summing the
  histogram counts through an in-process allreduce) must reproduce knnj_run's
  output exactly when their rows are merged.
"""
import threading

import numpy as np
import pytest

from paper_1810_04758_b200 import Engine, RunConfig
from paper_1810_04758_b200.distributed import merge_shards
from paper_1810_04758_b200.synthetic import generate

pytestmark = pytest.mark.gpu

CASES = [  # (spec, |D|, n, k, m, beta, seed)
    ("clusters:16:0.05", 6000, 18, 32, 0, 0.0, 1),
    ("uniform", 5000, 3, 7, 0, 0.0, 2),
    ("mixture", 4000, 24, 12, 0, 0.2, 3),
    ("exponential", 5000, 6, 40, 0, 0.0, 4),
    ("clusters:4:0.05", 3000, 12, 9, 2, 1.0, 5),
]


@pytest.mark.parametrize("pilot_cap", [1, 0])
@pytest.mark.parametrize("case", CASES, ids=[f"{c[0]}-{c[2]}d-k{c[3]}" for c in CASES])
def test_capped_histogram_selects_same_eps(engine, oracle, case, pilot_cap):
    """pilot_cap: the pilot slice itself first bins only the lowest third of the bins."""
    spec, N, n, k, m, beta, seed = case
    X = generate(spec, N, n, seed)
    o = oracle.run(X, k=k, m=m, beta=beta, mode="hybrid", seed=seed)
    engine.set_option("hist_cap", 2)
    engine.set_option("pilot_cap", pilot_cap)
    try:
        engine.set_points(X)
        r = engine.run(RunConfig(k=k, m=m, beta=beta, mode="hybrid", seed=seed), want_hist=False)
    finally:
        engine.set_option("hist_cap", 1)
        engine.set_option("pilot_cap", 2)
    assert r.info["eps_used"] == o["eps_used"]
    assert r.info["eps_default"] == o["eps_default"]
    assert np.array_equal(r.ids, o["ids"]) and np.array_equal(r.dist, o["dist"])
    assert np.array_equal(r.provenance, o["prov"])
    nb = int(r.info["hist_bins_counted"])
    assert 1 <= nb <= 100
    # the counted bins are exact: the capped kernels over the run's own sampled queries
    # (sample_without_replacement, seed derive_seed(seed, 2)) count bins [0, nb) exactly as
    # the oracle's full histogram does, and nothing above
    want = min(max(int(0.01 * N), 100), N)
    q = oracle.sample(N, want, oracle.derive_seed(seed, 2))
    for ncount in sorted({1, max(1, nb // 2), nb}):
        raw = engine.histogram_queries_capped(q, r.info["eps_mean"], 100, ncount)
        assert np.array_equal(raw[:ncount], o["raw_hist"][:ncount]), ncount
        assert not raw[ncount:].any()


class ThreadAllreduce:
    """Element-wise sum across `parts` threads (a stand-in for NCCL on one GPU)."""

    def __init__(self, parts):
        self.parts = parts
        self.slots = [None] * parts
        self.barrier = threading.Barrier(parts)

    def fn(self, rank):
        def reduce(a):
            self.slots[rank] = a.copy()
            self.barrier.wait()
            total = np.sum(np.stack(self.slots), axis=0, dtype=np.uint64)
            self.barrier.wait()
            a[:] = total
        return reduce


GRID_HIST = {"hist_cap": 2, "hist_grid": 2}  # capped rounds on the grid histogram


@pytest.mark.parametrize("shards", [2, 3])
@pytest.mark.parametrize("spec,N,n,k,opts", [("clusters:16:0.05", 8000, 18, 32, {}),
                                             ("exponential", 6000, 6, 20, {}),
                                             ("uniform", 5000, 2, 5, {}),
                                             ("uniform", 30000, 4, 16, GRID_HIST),
                                             ("exponential", 20000, 6, 12, GRID_HIST)])
def test_sharded_run_equals_single(engine, spec, N, n, k, opts, shards):
    """Shards (threads on one GPU, counts summed through a thread all-reduce) merge to the
    single run; with GRID_HIST every shard bins all sampled queries against its own
    slice of the candidates (the candidate-split grid histogram)."""
    X = generate(spec, N, n, 7)
    cfg = RunConfig(k=k, mode="hybrid", seed=7)
    for o, v in opts.items():
        engine.set_option(o, v)
    try:
        engine.set_points(X)
        ref = engine.run(cfg, want_hist=False)
    finally:
        engine.set_option("hist_cap", 1)
        engine.set_option("hist_grid", 1)
    ar = ThreadAllreduce(shards)
    parts, errs, infos = [None] * shards, [], [None] * shards

    def work(rank):
        try:
            e = Engine(0)
            for o, v in opts.items():
                e.set_option(o, v)
            e.set_points(X)
            r = e.run(cfg, want_hist=False, shard=(rank, shards, ar.fn(rank)))
            parts[rank] = (r.queries.copy(), r.ids.copy(), r.dist.copy(), r.provenance.copy())
            infos[rank] = r.info
            e.close()
        except Exception as ex:  # noqa: BLE001
            errs.append(ex)
            ar.barrier.abort()

    th = [threading.Thread(target=work, args=(i,)) for i in range(shards)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    q, ids, dist, prov = merge_shards(parts, N, k)
    assert np.array_equal(q, np.arange(N))
    assert np.array_equal(ids, ref.ids) and np.array_equal(dist, ref.dist)
    assert np.array_equal(prov, ref.provenance)
    assert all(i["eps_used"] == ref.info["eps_used"] for i in infos)
    assert all(i["hist_bins_counted"] == ref.info["hist_bins_counted"] for i in infos)
    assert sum(i["n_owned"] for i in infos) == N
    assert sum(i["failed_count"] for i in infos) == ref.info["failed_count"]
    # every shard owns a share of the work
    assert all(i["n_owned"] > 0 for i in infos)


@pytest.mark.parametrize("spec,N,n,k,m", [("mixture", 60000, 5, 8, 0), ("uniform", 80000, 2, 20, 0),
                                          ("mixture:4:0.02", 40000, 18, 32, 6)])
def test_split_items_identical(engine, oracle, spec, N, n, k, m):
    """Oversized work items are split into candidate-range parts and merged; the
    output must not depend on it, and must equal brute force on sampled queries."""
    X = generate(spec, N, n, 17)
    cfg = RunConfig(k=k, m=m, mode="hybrid", seed=17)
    out = []
    for split in (0, 1):
        engine.set_option("split_items", split)
        engine.set_points(X)
        out.append(engine.run(cfg, want_hist=False))
    engine.set_option("split_items", 1)
    a, b = out
    assert np.array_equal(a.ids, b.ids) and np.array_equal(a.dist, b.dist)
    assert np.array_equal(a.provenance, b.provenance)
    W = X[:, b.info["perm"]]
    q = np.random.default_rng(3).choice(N, 64, replace=False).astype(np.uint32)
    oi, od = oracle.brute_knn(W, q, k)
    assert np.array_equal(b.ids[q], oi) and np.array_equal(b.dist[q], od)


@pytest.mark.parametrize("spec,N,n,k", [("clusters:16:0.05", 30000, 18, 32), ("mixture", 40000, 5, 8),
                                        ("exponential", 30000, 6, 40), ("mixture:8:0.05", 6000, 90, 16)])
def test_box_filter_identical(engine, oracle, spec, N, n, k):
    """Dropping candidate blocks outside the pass radius (eps at level 0, the cell
    width in the fallback) leaves every output bit unchanged."""
    X = generate(spec, N, n, 29)
    cfg = RunConfig(k=k, mode="hybrid", seed=29)
    out = []
    for f in (0, 1):
        engine.set_option("box_filter", f)
        engine.set_points(X)
        out.append(engine.run(cfg, want_hist=False))
    engine.set_option("box_filter", 1)
    a, b = out
    assert np.array_equal(a.ids, b.ids) and np.array_equal(a.dist, b.dist)
    assert np.array_equal(a.provenance, b.provenance)
    assert a.info["failed_count"] == b.info["failed_count"]
    # the filter only drops pairs (with cell runs the screened union can exceed the
    # reference walk's count, so compare filtered against unfiltered)
    assert b.info["join_screened_pairs"] <= a.info["join_screened_pairs"]
    W = X[:, b.info["perm"]]
    q = np.random.default_rng(9).choice(N, 48, replace=False).astype(np.uint32)
    oi, od = oracle.brute_knn(W, q, k)
    assert np.array_equal(b.ids[q], oi) and np.array_equal(b.dist[q], od)


@pytest.mark.parametrize("spec,N,n,k", [("clusters:16:0.05", 30000, 18, 32), ("exponential", 40000, 6, 40),
                                        ("uniform", 50000, 2, 10), ("mixture:8:0.05", 6000, 90, 16)])
def test_fine_cascade_identical(engine, oracle, spec, N, n, k):
    """Rows certified on the fine grids (width f*eps) skip level 0; every output bit,
    the provenance and the failure count equal the plain level-0 run."""
    X = generate(spec, N, n, 37)
    cfg = RunConfig(k=k, mode="hybrid", seed=37)
    out = []
    for f1, f2 in ((0, 0), (700, 0), (500, 700)):
        engine.set_option("fine", f1)
        engine.set_option("fine2", f2)
        engine.set_points(X)
        out.append(engine.run(cfg, want_hist=False))
    engine.set_option("fine", 0)
    engine.set_option("fine2", 0)
    a = out[0]
    for b in out[1:]:
        assert np.array_equal(a.ids, b.ids) and np.array_equal(a.dist, b.dist)
        assert np.array_equal(a.provenance, b.provenance)
        assert a.info["failed_count"] == b.info["failed_count"]
        assert a.info["candidates_examined"] == b.info["candidates_examined"]
    W = X[:, a.info["perm"]]
    q = np.random.default_rng(4).choice(N, 48, replace=False).astype(np.uint32)
    oi, od = oracle.brute_knn(W, q, k)
    assert np.array_equal(out[2].ids[q], oi) and np.array_equal(out[2].dist[q], od)


@pytest.mark.parametrize("spec,N,n,k", [("clusters:16:0.05", 30000, 18, 32), ("exponential", 40000, 6, 40),
                                        ("mixture", 40000, 5, 8), ("mixture:8:0.05", 6000, 90, 16)])
def test_sweep_order_identical(engine, oracle, spec, N, n, k):
    """Sweeping each item's kept blocks nearest-first (per-block ranges, segmented
    sort) changes only the order candidates are screened in, never the output."""
    X = generate(spec, N, n, 41)
    cfg = RunConfig(k=k, mode="hybrid", seed=41)
    out = []
    for o in (0, 1):
        engine.set_option("sweep_order", o)
        engine.set_points(X)
        out.append(engine.run(cfg, want_hist=False))
    engine.set_option("sweep_order", 0)
    a, b = out
    assert np.array_equal(a.ids, b.ids) and np.array_equal(a.dist, b.dist)
    assert np.array_equal(a.provenance, b.provenance)
    assert a.info["failed_count"] == b.info["failed_count"]
    assert a.info["join_screened_pairs"] == b.info["join_screened_pairs"]
    W = X[:, b.info["perm"]]
    q = np.random.default_rng(6).choice(N, 48, replace=False).astype(np.uint32)
    oi, od = oracle.brute_knn(W, q, k)
    assert np.array_equal(b.ids[q], oi) and np.array_equal(b.dist[q], od)


@pytest.mark.parametrize("spec,N,n,k", [("clusters:16:0.05", 30000, 18, 32), ("exponential", 40000, 6, 40),
                                        ("uniform", 50000, 2, 10)])
def test_early_d2h_identical(engine, spec, N, n, k):
    """Host results copied during classification + fallback (rows the fallback rewrites
    patched afterwards) equal the copy taken after the whole run."""
    X = generate(spec, N, n, 47)
    cfg = RunConfig(k=k, mode="hybrid", seed=47)
    out = []
    for o in (0, 1):
        engine.set_option("early_d2h", o)
        engine.set_points(X)
        out.append(engine.run(cfg, want_hist=False))
    engine.set_option("early_d2h", 1)
    a, b = out
    assert b.info["fallback_queries"] > 0 or spec == "clusters:16:0.05"
    assert np.array_equal(a.ids, b.ids) and np.array_equal(a.dist, b.dist)
    assert np.array_equal(a.provenance, b.provenance)


@pytest.mark.parametrize("opt,val,default", [("morton_dims", 6, 10), ("morton_bits", 5, 3),
                                             ("finalize_xj", 0, 1), ("tc_slack", 12, 24),
                                             ("sweep_order", 0, 1), ("tc_small_cta", 0, 2),
                                             ("item_radius", 0, 1)])
def test_engine_knobs_identical(engine, oracle, opt, val, default):
    """The remaining engine knobs change only work order and layout, never an output bit
    (70k points so the finalize's join-ordered copy is in play)."""
    N, n, k = 70000, 18, 32
    X = generate("clusters:16:0.05", N, n, 53)
    cfg = RunConfig(k=k, mode="hybrid", seed=53)
    out = []
    for v in (default, val):
        engine.set_option(opt, v)
        engine.set_points(X)
        out.append(engine.run(cfg, want_hist=False))
    engine.set_option(opt, default)
    a, b = out
    assert np.array_equal(a.ids, b.ids) and np.array_equal(a.dist, b.dist)
    assert np.array_equal(a.provenance, b.provenance)
    W = X[:, b.info["perm"]]
    q = np.random.default_rng(11).choice(N, 32, replace=False).astype(np.uint32)
    oi, od = oracle.brute_knn(W, q, k)
    assert np.array_equal(b.ids[q], oi) and np.array_equal(b.dist[q], od)


@pytest.mark.parametrize("opt", ["filter_skip_all_dims", "adj_norm_order"])
@pytest.mark.parametrize("spec,N,n,k", [("uniform", 200000, 4, 32), ("exponential", 60000, 6, 20),
                                        ("mixture", 50000, 3, 8)])
def test_all_dims_knobs_identical(engine, oracle, opt, spec, N, n, k):
    """On grids over every dim: skipping the box filter at level 0 and the nearer-rows-first
    adjacency order change only which pairs are screened and in what order."""
    X = generate(spec, N, n, 61)
    cfg = RunConfig(k=k, mode="hybrid", seed=61)
    out = []
    for v in (1, 0):
        engine.set_option(opt, v)
        engine.set_points(X)
        out.append(engine.run(cfg, want_hist=False))
    engine.set_option(opt, 1)
    a, b = out
    assert np.array_equal(a.ids, b.ids) and np.array_equal(a.dist, b.dist)
    assert np.array_equal(a.provenance, b.provenance)
    assert a.info["failed_count"] == b.info["failed_count"]
    W = X[:, a.info["perm"]]
    q = np.random.default_rng(8).choice(N, 32, replace=False).astype(np.uint32)
    oi, od = oracle.brute_knn(W, q, k)
    assert np.array_equal(a.ids[q], oi) and np.array_equal(a.dist[q], od)


@pytest.mark.parametrize("small,halves", [(0, 1), (1, 0), (1, 1)])
def test_item_halves_identical(engine, oracle, small, halves):
    """128-query CTAs launched over 256-query items (tc_halves: 4-D, the grid indexes every
    dim) and 128-query items give the same bits as the 256-query CTA shape."""
    N, n, k = 300000, 4, 32
    X = generate("uniform", N, n, 59)
    cfg = RunConfig(k=k, mode="hybrid", seed=59)
    out = []
    for sm, hv in ((0, 1), (small, halves)):
        engine.set_option("tc_small_cta", sm)
        engine.set_option("tc_item_halves", hv)
        engine.set_points(X)
        out.append(engine.run(cfg, want_hist=False))
    engine.set_option("tc_small_cta", 2)
    engine.set_option("tc_item_halves", 1)
    a, b = out
    assert b.info["join_tensor_cores"] == 1
    assert np.array_equal(a.ids, b.ids) and np.array_equal(a.dist, b.dist)
    assert np.array_equal(a.provenance, b.provenance)
    W = X[:, b.info["perm"]]
    q = np.random.default_rng(5).choice(N, 32, replace=False).astype(np.uint32)
    oi, od = oracle.brute_knn(W, q, k)
    assert np.array_equal(b.ids[q], oi) and np.array_equal(b.dist[q], od)


@pytest.mark.parametrize("spec,N,n,k", [("uniform", 40000, 4, 32), ("exponential", 30000, 6, 20),
                                        ("uniform", 50000, 2, 5), ("mixture", 30000, 3, 8),
                                        ("clusters:4:0.05", 20000, 8, 16)])
def test_grid_histogram_counts_exact(engine, oracle, spec, N, n, k):
    """The capped histogram on a grid of the cap radius (k_hist_grid, n <= 8) counts
    bins [0, n_count) exactly like the reference's binning (epsilon.cpp:76-104), and a
    run through it is bit-identical to one through the tensor-core histogram."""
    X = generate(spec, N, n, 13)
    o = oracle.run(X, k=k, mode="hybrid", seed=13)
    engine.set_option("hist_cap", 2)
    engine.set_option("hist_grid", 2)
    try:
        engine.set_points(X)
        r = engine.run(RunConfig(k=k, mode="hybrid", seed=13), want_hist=False)
        want = min(max(int(0.01 * N), 100), N)
        q = oracle.sample(N, want, oracle.derive_seed(13, 2))
        for ncount in (1, 3, 7, 20):
            raw = engine.histogram_queries_capped(q, r.info["eps_mean"], 100, ncount)
            assert np.array_equal(raw[:ncount], o["raw_hist"][:ncount]), ncount
            assert not raw[ncount:].any()
        engine.set_option("hist_grid", 0)
        engine.set_points(X)
        t = engine.run(RunConfig(k=k, mode="hybrid", seed=13), want_hist=False)
    finally:
        engine.set_option("hist_cap", 1)
        engine.set_option("hist_grid", 1)
    assert r.info["eps_used"] == o["eps_used"] == t.info["eps_used"]
    assert np.array_equal(r.ids, o["ids"]) and np.array_equal(r.dist, o["dist"])
    assert np.array_equal(t.ids, r.ids) and np.array_equal(t.provenance, r.provenance)
