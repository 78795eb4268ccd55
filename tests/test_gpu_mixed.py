"""Mixed level passes (knnj_capi.cu pass_mixed / run_pass): when the tensor-core screen's
global precision rule fails (data far from the centre somewhere, e.g. skewed Exp(1)
coordinates), work items whose own data lie close to the centre run on the tcgen05 screen
with a per-item error bound (tc_delta_poly at the item's radius, measured by the box
filter), the rest on the SIMT screen. Neither screen may change an output bit: compared
with an all-SIMT run and with the oracle."""
import numpy as np
import pytest

from paper_1810_04758_b200 import RunConfig
from paper_1810_04758_b200.synthetic import generate

pytestmark = pytest.mark.gpu


def _far_cluster(N, n, seed):
    """A blob at the origin plus a sparse far shell: the global radius is large, the
    blob's items are small. (A blob much smaller than the global scale would fail the
    per-item rule too: the FP16 split's absolute floor, tc_delta_poly's C term.)"""
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((N, n))
    far = rng.standard_normal((N // 50, n))
    far *= 40.0 / np.linalg.norm(far, axis=1)[:, None]
    X[: far.shape[0]] = far
    return X


# mixed passes need 128-query items (G = 1): K > 40 for n <= 20, or n >= 21
@pytest.mark.parametrize("spec,N,n,k,minq", [("exponential", 60000, 6, 64, 8), ("exponential", 50000, 5, 48, 16),
                                             ("far", 40000, 4, 44, 1), ("far", 40000, 6, 64, 8),
                                             ("exponential", 40000, 24, 16, 32), ("far", 30000, 22, 12, 1),
                                             ("exponential", 80000, 6, 64, 64)])
def test_mixed_pass_identical(engine, oracle, spec, N, n, k, minq):
    X = _far_cluster(N, n, 5) if spec == "far" else generate(spec, N, n, 71)
    cfg = RunConfig(k=k, mode="hybrid", seed=71)
    engine.set_option("item_tc", 0)
    engine.set_points(X)
    a = engine.run(cfg, want_hist=False)
    engine.set_option("item_tc", 1)
    engine.set_option("item_tc_min_q", minq)
    try:
        engine.set_points(X)
        b = engine.run(cfg, want_hist=False)
    finally:
        engine.set_option("item_tc_min_q", 32)
    assert np.array_equal(b.ids, a.ids) and np.array_equal(b.dist, a.dist)
    assert np.array_equal(b.provenance, a.provenance)
    assert b.info["failed_count"] == a.info["failed_count"]
    if minq == 1:
        assert b.info["join_tensor_cores"] == 1, "no item ran on the tensor cores"
    W = X[:, a.info["perm"]]
    q = np.random.default_rng(3).choice(N, 40, replace=False).astype(np.uint32)
    oi, od = oracle.brute_knn(W, q, k)
    assert np.array_equal(b.ids[q], oi) and np.array_equal(b.dist[q], od)


@pytest.mark.parametrize("spec,N,n,k", [("exponential", 80000, 6, 64), ("uniform", 60000, 2, 10),
                                        ("exponential", 50000, 5, 16), ("far", 40000, 4, 44),
                                        ("clusters:16:0.05", 40000, 18, 32)])
def test_cell_runs_identical(engine, oracle, spec, N, n, k):
    """Cell runs (level0_group_span, fallback_group_span): consecutive sparse cells of a
    grid row share a work item whose candidates are the union of their neighbourhoods.
    Outputs, provenance and the reference's per-cell walk counters (candidates_examined)
    are unchanged."""
    X = _far_cluster(N, n, 9) if spec == "far" else generate(spec, N, n, 73)
    cfg = RunConfig(k=k, mode="hybrid", seed=73)
    out = []
    try:
        for span in (0, 8):
            engine.set_option("level0_group_span", span)
            engine.set_option("fallback_group_span", span)
            engine.set_points(X)
            out.append(engine.run(cfg, want_hist=False))
    finally:
        engine.set_option("level0_group_span", 8)
        engine.set_option("fallback_group_span", 8)
    a, b = out
    assert np.array_equal(b.ids, a.ids) and np.array_equal(b.dist, a.dist)
    assert np.array_equal(b.provenance, a.provenance)
    assert b.info["candidates_examined"] == a.info["candidates_examined"]
    assert b.info["join_candidate_pairs"] == a.info["join_candidate_pairs"]
    W = X[:, a.info["perm"]]
    q = np.random.default_rng(4).choice(N, 32, replace=False).astype(np.uint32)
    oi, od = oracle.brute_knn(W, q, k)
    assert np.array_equal(b.ids[q], oi) and np.array_equal(b.dist[q], od)
