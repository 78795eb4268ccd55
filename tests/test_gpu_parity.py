"""GPU parity: the CUDA path (through the C ABI) against the reference.

Bar: neighbour ids and FP64 distances BIT-IDENTICAL to the
reference run with its scalar kernel, identical provenance / eps / failed
counts / histogram counts / grid tables. Checked against (a) the golden
fixtures made by the unmodified reference and (b) the pinned C oracle on
seeded random instances, plus the edge cases the reference tests cover.
"""
import math

import numpy as np
import pytest

from conftest import golden_cases, load_golden
from paper_1810_04758_b200 import KnnjError, RunConfig
from paper_1810_04758_b200.synthetic import generate

pytestmark = pytest.mark.gpu


def _cfg(cfg, mode):
    cfg = dict(cfg)
    hf = cfg.pop("hist_frac", 0.01)
    return RunConfig(mode=mode, hist_query_fraction=hf, **cfg)


@pytest.mark.parametrize("name", golden_cases())
def test_run_hybrid_matches_reference_golden(engine, name):
    g, cfg = load_golden(name)
    for mode in ("hybrid", "dense", "sparse", "oracle"):
        engine.set_points(g["X"])
        r = engine.run(_cfg(cfg, mode))
        assert np.array_equal(r.ids, g["ids"]), mode
        assert np.array_equal(r.dist, g["dist"]), mode          # bit-identical FP64
        assert np.array_equal(r.provenance, g[f"{mode}_prov"]), mode
        assert np.array_equal(r.info["perm"], g["perm"])
        if mode in ("hybrid", "dense"):
            i = r.info
            assert i["eps_mean"] == g[f"{mode}_eps_mean"]
            assert i["eps_used"] == g[f"{mode}_eps_used"]
            assert i["eps_default"] == g[f"{mode}_eps_default"]
            assert i["failed_count"] == g[f"{mode}_failed_count"]
            assert i["q_gpu"] == g[f"{mode}_q_gpu"] and i["q_cpu"] == g[f"{mode}_q_cpu"]
            assert i["demoted"] == g[f"{mode}_demoted"]
            assert i["n_thresh"] == g[f"{mode}_n_thresh"]
            assert i["candidates_examined"] == g[f"{mode}_candidates_examined"]
            qc = int(g[f"{mode}_hist_query_count"])
            assert i["hist_query_count"] == qc
            assert np.array_equal(r.raw_hist / qc, g[f"{mode}_hist_counts"])


@pytest.mark.parametrize("name", golden_cases())
def test_phases_match_reference_golden(engine, name):
    g, cfg = load_golden(name)
    X = g["X"]
    engine.set_points(X)
    perm, var = engine.reorder_by_variance(1)
    assert np.array_equal(perm, g["perm"])
    W = engine.working_points()
    assert np.array_equal(W, X[:, g["perm"]])
    m = cfg.get("m", 0) or min(6, X.shape[1])
    eps = float(g["dense_eps_used"])
    info = engine.grid_build(m, eps)
    assert np.array_equal(info["cells_per_dim"], g["grid_cpd"])
    t = engine.grid_export(info["n_cells"])
    assert np.array_equal(t["B"], g["grid_B"])
    assert np.array_equal(t["G"], g["grid_G"])
    assert np.array_equal(t["A"], g["grid_A"])
    q = np.arange(X.shape[0], dtype=np.uint32)
    ine, cand = engine.range_count(q)
    assert np.array_equal(ine, g["range_in_eps"])
    assert np.array_equal(cand, g["range_candidates"])


def test_pair_sq_bit_exact(engine, oracle):
    rng = np.random.default_rng(3)
    for n in (1, 2, 3, 7, 8, 9, 18, 33, 90, 128):
        X = rng.uniform(-5, 5, (200, n))
        engine.set_points(X)
        ij = rng.integers(0, 200, (500, 2)).astype(np.uint64)
        got = engine.pair_sq(ij)
        want = np.array([oracle.sq_dist_limited(X[i], X[j]) for i, j in ij])
        assert np.array_equal(got, want), n
        lim = float(np.median(want))
        got = engine.pair_sq(ij, lim)
        assert np.array_equal(got, np.where(want > lim, np.inf, want))


RANDOM = [  # (spec, |D|, n, k, m, beta, gamma, rho, seed) — acceptance C1-style instances
    ("uniform", 1500, 3, 7, 0, 0.0, 0.0, 0.0, 1),
    ("clusters:4:0.05", 1200, 12, 25, 2, 0.1, 0.4, 0.25, 2),
    ("mixture", 1800, 32, 11, 6, 0.3, 0.8, 0.5, 3),
    ("uniform", 900, 1, 3, 1, 0.5, 1.0, 0.0, 4),
    ("exponential", 2500, 6, 40, 0, 0.0, 0.0, 0.0, 5),
    ("clusters:16:0.05", 3000, 18, 32, 0, 0.0, 0.0, 0.0, 6),
    ("mixture:8:0.05", 1000, 90, 16, 0, 0.0, 0.0, 0.0, 7),
    ("uniform", 4000, 2, 5, 0, 1.0, 0.0, 0.0, 8),
    ("clusters:3:0.2", 700, 5, 100, 3, 0.0, 0.0, 0.0, 9),
    ("mixture", 2000, 48, 8, 4, 0.1, 0.0, 0.0, 10),
]


RANDOM += [
    ("clusters:16:0.05", 6000, 18, 32, 0, 0.0, 0.0, 0.0, 11),
    ("clusters:8:0.02", 4000, 12, 9, 0, 0.2, 0.3, 0.1, 12),
    ("mixture:4:0.05", 3000, 24, 20, 5, 0.0, 0.0, 0.0, 13),
    ("clusters:6:0.1", 2500, 40, 3, 0, 0.0, 0.0, 0.0, 14),
    ("uniform", 2000, 16, 64, 0, 0.0, 0.0, 0.0, 15),
]


@pytest.mark.parametrize("tc", [1, 0], ids=["tcgen05", "simt"])
@pytest.mark.parametrize("case", RANDOM, ids=[f"{c[0]}-{c[2]}d-k{c[3]}" for c in RANDOM])
def test_random_instances_vs_oracle(engine, oracle, case, tc):
    spec, N, n, k, m, beta, gamma, rho, seed = case
    engine.set_option("tensor_cores", tc)
    X = generate(spec, N, n, seed)
    for mode in ("hybrid", "dense"):
        o = oracle.run(X, k=k, m=m, beta=beta, gamma=gamma, rho=rho, mode=mode, seed=seed)
        engine.set_points(X)
        r = engine.run(RunConfig(k=k, m=m, beta=beta, gamma=gamma, rho=rho, mode=mode, seed=seed))
        assert np.array_equal(r.ids, o["ids"]), mode
        assert np.array_equal(r.dist, o["dist"]), mode
        assert np.array_equal(r.provenance, o["prov"]), mode
        assert r.info["failed_count"] == o["failed_count"]
        assert r.info["eps_used"] == o["eps_used"]
        assert np.array_equal(r.raw_hist, o["raw_hist"])
        # the screen list holds the exact top-K without the slow path (no exact ties here)
        assert r.info["slow_path_queries"] == 0, r.info["slow_path_queries"]
    engine.set_option("tensor_cores", 1)


def test_exact_knn_matches_brute(engine, oracle):
    rng = np.random.default_rng(12)
    for spec, n, k in (("uniform", 3, 10), ("clusters:5:0.02", 8, 17), ("exponential", 6, 64)):
        X = generate(spec, 3000, n, int(rng.integers(1 << 30)))
        engine.set_points(X)
        q = rng.choice(3000, 300, replace=False).astype(np.uint32)
        ids, dist = engine.exact_knn(q, k)
        oi, od = oracle.brute_knn(X, q, k)
        assert np.array_equal(ids, oi) and np.array_equal(dist, od)


def test_query_subset(engine, oracle):
    X = generate("mixture", 2000, 4, 21)
    sub = np.array([5, 3, 3, 1999, 0, 700, 5], np.uint32)
    engine.set_points(X)
    r = engine.run(RunConfig(k=6, query_subset=sub, seed=4))
    assert list(r.queries) == [0, 3, 5, 700, 1999]
    Wi = X[:, r.info["perm"]]
    oi, od = oracle.brute_knn(Wi, r.queries, 6)
    assert np.array_equal(r.ids, oi) and np.array_equal(r.dist, od)


def test_duplicates_and_ties(engine, oracle):
    # duplicate at distance 0 is a neighbour (test_sparse_engine.cpp:89-96); ties by id
    X = np.concatenate([np.zeros((40, 2)), np.ones((40, 2)), np.eye(2)])
    for mode in ("oracle", "sparse", "dense", "hybrid"):
        engine.set_points(X)
        r = engine.run(RunConfig(k=50, mode=mode, seed=2))
        o = oracle.run(X, k=50, mode=mode, seed=2)
        assert np.array_equal(r.ids, o["ids"]) and np.array_equal(r.dist, o["dist"]), mode


def test_k_clamp_and_tiny(engine, oracle):
    X = np.array([[0.0, 0.0], [3.0, 4.0], [1.0, 1.0]])
    engine.set_points(X)
    r = engine.run(RunConfig(k=10, mode="oracle"))
    assert r.k_effective == 2 and r.warnings
    o = oracle.run(X, k=10, mode="oracle")
    assert np.array_equal(r.ids, o["ids"]) and np.array_equal(r.dist, o["dist"])
    assert r.dist[0, 1] == 5.0
    engine.set_points(np.array([[1.0, 2.0]]))
    r = engine.run(RunConfig(k=3))
    assert r.k_effective == 0 and r.ids.size == 0


def test_errors_mirror_reference(engine):
    with pytest.raises(KnnjError) as e:
        engine.set_points(np.array([[0.0, np.nan]]))
    assert e.value.kind == "UsageError" and "non-finite coordinate at point 0, dimension 1" in str(e.value)
    engine.set_points(np.full((30, 2), 1.5))
    with pytest.raises(KnnjError) as e:
        engine.run(RunConfig(k=3))          # all points identical: eps_mean == 0
    assert e.value.kind == "DegenerateProfileError"
    engine.set_points(generate("uniform", 100, 3, 1))
    with pytest.raises(KnnjError) as e:
        engine.run(RunConfig(k=3, beta=1.5))
    assert e.value.kind == "UsageError"
    # 64-bit linear id overflow (test_grid_index.cpp:52-60)
    X = np.zeros((4, 8))
    X[1] = 1e6
    engine.set_points(X)
    engine.reorder_by_variance(8)
    with pytest.raises(KnnjError) as e:
        engine.grid_build(8, 1e-3)
    assert e.value.kind == "IndexingError" and "required extent" in str(e.value)


def test_split_matches_reference_semantics(engine, oracle):
    X = generate("mixture", 3000, 3, 9)
    engine.set_points(X)
    perm, _ = engine.reorder_by_variance(3)
    W = X[:, perm]
    eps = 0.15
    info = engine.grid_build(3, eps)
    q = np.arange(3000, dtype=np.uint32)
    for gamma, rho in ((0.0, 0.0), (0.4, 0.0), (0.2, 0.5), (1.0, 0.9)):
        s = engine.split_work(q, 5, 0.2, gamma, rho)
        g = oracle.grid(W, 3, eps)
        pop = (g["G"][:, 1] - g["G"][:, 0])[g["slot"]]
        assert np.array_equal(s["cell_population"], pop)
        n_thresh = oracle.n_thresh(oracle.n_min(5, 3), gamma)
        assert s["n_thresh"] == n_thresh
        dense = pop.astype(np.float64) >= n_thresh
        floor_cpu = math.ceil(rho * 3000)
        ncpu = int((~dense).sum())
        if ncpu < floor_cpu:
            order = sorted((int(pop[i]), int(g["B"][g["slot"][i]]), i) for i in range(3000) if dense[i])
            for _, _, i in order[:floor_cpu - ncpu]:
                dense[i] = False
        assert np.array_equal(s["is_dense"].astype(bool), dense)
        assert s["q_cpu"] >= floor_cpu


@pytest.mark.parametrize("name", golden_cases())
def test_phase_entries_match_reference_golden(engine, oracle, name):
    """The phase-level C-ABI entries called directly, each against the unmodified
    reference's own values for the same data (tests/golden): estimate_eps_mean
    (epsilon.cpp:14-44), build_distance_histogram (epsilon.cpp:46-120) and
    run_dense_join + filter_keys in DenseOnly mode (dense_engine.cpp:165-303)."""
    g, cfg = load_golden(name)
    X = g["X"]
    N = X.shape[0]
    k = min(int(cfg["k"]), N - 1)
    seed = int(cfg.get("seed", 0))
    engine.set_points(X)
    engine.reorder_by_variance(1)
    em = engine.estimate_eps_mean(min(10 * N, 1_000_000), oracle.derive_seed(seed, 1))
    assert em == g["hybrid_eps_mean"]
    raw, qc = engine.build_distance_histogram(em, 100, cfg.get("hist_frac", 0.01),
                                              oracle.derive_seed(seed, 2))
    assert qc == int(g["hybrid_hist_query_count"])
    assert np.array_equal(raw / qc, g["hybrid_hist_counts"])
    m = cfg.get("m", 0) or min(6, X.shape[1])
    engine.grid_build(m, float(g["dense_eps_used"]))
    q = np.arange(N, dtype=np.uint32)
    ids, dist, solved, st = engine.dense_join(q, k)
    ok = g["dense_prov"] == 0
    assert np.array_equal(solved, ok)
    assert np.array_equal(ids[ok], g["ids"][ok]) and np.array_equal(dist[ok], g["dist"][ok])
    assert (ids[~ok] == 0xFFFFFFFF).all() and np.isinf(dist[~ok]).all()
    assert st["candidates_examined"] == g["dense_candidates_examined"]
    assert st["solved"] == int(ok.sum()) and st["failed"] == int((~ok).sum())
