"""CPU: pin the C restatement (oracle/) to the reference.

1. The reference's own known-answer tests for this path (cited per case).
2. The golden fixtures produced by the UNMODIFIED reference (tests/golden).
3. When oracle/_ref is built here, random cross-checks against it.
"""
import math

import numpy as np
import pytest

from conftest import golden_cases, load_golden
from oracle.oracle import Ref, ref_available


# ---- 1. known-answer tests -------------------------------------------------
def test_345_triangle(oracle):
    # proj/tests/test_core.cpp:14-17
    assert math.sqrt(oracle.sq_dist_limited([0, 0], [3, 4])) == 5.0


def test_direct_formula(oracle):
    # proj/tests/test_core.cpp:24-27
    assert abs(math.sqrt(oracle.sq_dist_limited([1, 1, 1], [2, 3, 4])) - 3.7416573867739413) < 1e-15


def test_short_circuit_boundary(oracle):
    # proj/tests/test_core.cpp:34-47: inclusive at 5.0, exceeded at 4.9
    assert oracle.sq_dist_limited([0, 0], [3, 4], 25.0) == 25.0
    assert math.isinf(oracle.sq_dist_limited([0, 0], [3, 4], 4.9 * 4.9))


def test_limited_bit_exact_and_inf(oracle):
    # proj/tests/test_kernels.cpp:46-66
    rng = np.random.default_rng(11)
    for _ in range(300):
        n = int(rng.integers(1, 300))
        a, b = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
        full = oracle.sq_dist_limited(a, b)
        assert oracle.sq_dist_limited(a, b, full) == full
        assert oracle.sq_dist_limited(a, b, np.nextafter(full, np.inf)) == full
        if full > 0:
            assert math.isinf(oracle.sq_dist_limited(a, b, np.nextafter(full, -np.inf)))


def test_eps_mean_known_answers(oracle):
    # proj/tests/test_epsilon.cpp:13-30
    assert oracle.eps_mean(np.array([[0, 0], [3, 4]], float), 50, 1) == 5.0
    assert oracle.eps_mean(np.array([[0, 0], [3, 4]], float), 1, 1) == 5.0
    assert abs(oracle.eps_mean(np.array([[0], [1], [2], [3]], float), 12, 7) - 10 / 6) < 1e-15


def test_histogram_known_answer(oracle):
    # proj/tests/test_epsilon.cpp:37-48: {0,1,2,3}, 2 bins -> counts (0, 1.5)
    raw, qc = oracle.histogram(np.array([[0], [1], [2], [3]], float), 10 / 6, 2, 1.0, 0)
    assert qc == 4
    assert list(raw / qc) == [0.0, 1.5]


def test_histogram_identical_points(oracle):
    # proj/tests/test_epsilon.cpp:50-56
    raw, qc = oracle.histogram(np.full((20, 1), 4.25), 1.0, 5, 1.0, 0)
    assert raw[0] / qc == 19.0 and all(raw[1:] == 0)


def test_n_min_spots(oracle):
    # proj/tests/test_partitioner.cpp:51-56 / acceptance.cpp:116-118
    assert abs(oracle.n_min(5, 2) - 4 * 5 / math.pi) <= 1e-10 * oracle.n_min(5, 2)
    assert abs(oracle.n_min(10, 3) - 19.0986) <= 1e-4


def test_select_eps_unreachable(oracle):
    # proj/tests/test_epsilon.cpp:91-103: beta=1, K=5 -> target 500 unreachable
    cum = np.linspace(0, 10, 100)
    with pytest.raises(ValueError):
        oracle.select_eps(cum, 0.01, 5, 1.0, allow_fallback=False)


def test_variance_order_example(oracle):
    # proj/tests/test_core.cpp:85-98 shape: ranges [0,1] x [0,0.01] x [0.2,0.6] -> {0,2,1}
    rng = np.random.default_rng(5)
    X = np.stack([rng.uniform(0, 1, 400), rng.uniform(0, 0.01, 400), rng.uniform(0.2, 0.6, 400)], 1)
    order, _ = oracle.variance_order(X)
    assert list(order) == [0, 2, 1]


def test_grid_two_close_one_far(oracle):
    # proj/tests/test_grid_index.cpp:13-25
    g = oracle.grid(np.array([[0.0, 0.0], [0.1, 0.1], [5.0, 5.0]]), 2, 1.0)
    assert len(g["B"]) == 2
    assert list(g["A"]) == [0, 1, 2]


def test_grid_boundary_goes_up(oracle):
    # proj/tests/test_grid_index.cpp:69-91: a coordinate on a face goes to the higher cell
    g = oracle.grid(np.array([[0.0], [1.0], [2.0], [2.5]]), 1, 1.0)
    assert list(g["B"]) == [0, 1, 2]


def test_mt19937_64_reference_value(oracle):
    # [rand.predef]: the 10000th output of default-seeded mt19937_64
    assert int(oracle.mt_stream(5489, 10000)[-1]) == 9981545732273789042


# ---- 2. golden fixtures from the unmodified reference -----------------------
@pytest.mark.parametrize("name", golden_cases())
def test_oracle_matches_reference_golden(oracle, name):
    g, cfg = load_golden(name)
    X = g["X"]
    hist_frac = cfg.pop("hist_frac", 0.01)
    for mode in ("hybrid", "dense", "sparse", "oracle"):
        r = oracle.run(X, mode=mode, hist_frac=hist_frac, threads=4, **cfg)
        assert (r["ids"] == g["ids"]).all(), mode
        assert (r["dist"] == g["dist"]).all(), mode  # bit-identical FP64
        assert (r["prov"] == g[f"{mode}_prov"]).all(), mode
        if mode in ("hybrid", "dense"):
            assert r["eps_mean"] == g[f"{mode}_eps_mean"]
            assert r["eps_used"] == g[f"{mode}_eps_used"]
            assert r["failed_count"] == g[f"{mode}_failed_count"]
            assert r["q_gpu"] == g[f"{mode}_q_gpu"]
            assert r["candidates_examined"] == g[f"{mode}_candidates_examined"]
            qc = int(g[f"{mode}_hist_query_count"])
            assert r["hist_query_count"] == qc
            assert np.array_equal(r["raw_hist"] / qc, g[f"{mode}_hist_counts"])
            assert (r["perm"] == g[f"{mode}_perm"]).all()
    W = np.ascontiguousarray(X[:, g["perm"]])
    m = cfg.get("m", 0) or min(6, X.shape[1])
    grid = oracle.grid(W, m, float(g["dense_eps_used"]))
    assert (grid["B"] == g["grid_B"]).all()
    assert (grid["G"] == g["grid_G"]).all()
    assert (grid["A"] == g["grid_A"]).all()


# ---- 3. random cross-checks against the compiled reference (here only) -----
@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built (no /root/reference)")
def test_oracle_vs_ref_random(oracle):
    ref = Ref()
    ref.set_kernel("scalar")
    rng = np.random.default_rng(20260810)
    for i in range(12):
        size = int(rng.integers(100, 900))
        dims = int(rng.integers(1, 20))
        k = int(rng.integers(1, 20))
        m = int(rng.integers(0, min(6, dims) + 1))
        spec = ["uniform", "clusters:4:0.05", "mixture"][i % 3]
        X = ref.generate(spec, size, dims, int(rng.integers(1 << 30)))
        kw = dict(k=k, m=m, beta=[0, 0.1, 0.5][i % 3], gamma=[0, 0.4, 1.0][i % 3],
                  rho=[0, 0.25, 0.5][i % 3], seed=int(rng.integers(1 << 30)))
        r = ref.run(X, mode="hybrid", workers=2, buffer_size=10**12, **kw)
        o = oracle.run(X, mode="hybrid", **kw)
        assert (r["ids"] == o["ids"]).all() and (r["dist"] == o["dist"]).all()
        assert (r["prov"] == o["prov"]).all()


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built (no /root/reference)")
def test_sampler_matches_reference(oracle):
    ref = Ref()
    for n, k, s in [(1000, 100, 3), (10**8, 3000, 5), (50, 60, 1), (7, 7, 2)]:
        assert (oracle.sample(n, k, s) == ref.sample(n, k, s)).all()
