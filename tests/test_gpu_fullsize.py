"""GPU parity at BASELINE.json's full sizes, through size-independent properties
(the CPU oracle cannot replay a 5M-point run):

* sampled queries: neighbour ids and FP64 distances bit-identical to brute force
  (the oracle's exact scalar-order search over ALL points);
* every row: distances non-decreasing, ids distinct, self never listed;
* provenance consistent with eps: dense-solved rows have their K-th neighbour
  within eps, dense-failed rows do not (dense_engine.cpp:182-192);
* the capped eps histogram selects the same eps, and so the same output, as the
  full one (epsilon.cpp:46-141);
* determinism: a second run is bit-identical.
"""
import os

import numpy as np
import pytest

from paper_1810_04758_b200 import RunConfig
from paper_1810_04758_b200.synthetic import CONFIGS, generate

pytestmark = pytest.mark.gpu

CASES = [("C2", None), ("C3", None), ("C4", 5_000_000), ("NS", None), ("C1", None)]
# C5 (100M points) takes ~220 s, most of it the full (uncapped) histogram of 1e14 pairs
# the capped-vs-full check needs; opt in with KNNJ_FULLSIZE_C5=1 (passed on B200, round 1)
if os.environ.get("KNNJ_FULLSIZE_C5"):
    CASES.append(("C5", None))


@pytest.mark.parametrize("name,size", CASES, ids=[c[0] for c in CASES])
def test_full_size_properties(engine, oracle, name, size):
    c = CONFIGS[name]
    N = size or c["size"]
    X = generate(c["spec"], N, c["dims"], seed=1)
    k = c["k"]
    engine.set_points(X)
    r = engine.run(RunConfig(k=k, mode="hybrid", seed=1), want_hist=False)
    i = r.info
    assert r.ids.shape == (N, k)
    eps = i["eps_used"]
    W = X[:, i["perm"]]

    rng = np.random.default_rng(7)
    q = np.sort(rng.choice(N, 96, replace=False)).astype(np.uint32)
    oi, od = oracle.brute_knn(W, q, k, threads=os.cpu_count() or 8)
    assert np.array_equal(r.ids[q], oi), "sampled neighbour ids differ from brute force"
    assert np.array_equal(r.dist[q], od), "sampled distances differ from brute force"

    assert (np.diff(r.dist, axis=1) >= 0).all()
    assert not (r.ids == np.arange(N, dtype=np.uint32)[:, None]).any(), "self listed"
    s = np.sort(r.ids, axis=1)
    assert (s[:, 1:] != s[:, :-1]).all(), "duplicate neighbour id"

    kth = r.dist[:, -1]
    dense_ok, failed = r.provenance == 0, r.provenance == 2
    assert (kth[dense_ok] <= eps * (1 + 1e-15)).all()
    assert (kth[failed] >= eps * (1 - 1e-15)).all()
    assert int(failed.sum()) == i["failed_count"]

    # capped (the run above) vs full histogram: same eps, identical output
    engine.set_option("hist_cap", 0)
    try:
        engine.set_points(X)
        full = engine.run(RunConfig(k=k, mode="hybrid", seed=1), want_hist=True)
    finally:
        engine.set_option("hist_cap", 1)
    assert full.info["eps_used"] == eps
    assert np.array_equal(full.ids, r.ids) and np.array_equal(full.dist, r.dist)
    assert np.array_equal(full.provenance, r.provenance)
