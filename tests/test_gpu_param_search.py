"""GPU: parameter_search (proj/src/orchestrator.cpp:252-303) through knnj_parameter_search.

The seeded f-fraction subset (derive_seed(seed, kSeedQuerySubset = 4),
sample_without_replacement) and every candidate run (hybrid, rho = 0.5) follow the
reference; the winner is the fastest candidate by device time, so only its membership
is checked. Invalid inputs raise the reference's error kinds and messages.
"""
import math

import numpy as np
import pytest

from paper_1810_04758_b200 import KnnjError, RunConfig, parameter_search
from paper_1810_04758_b200.synthetic import generate

pytestmark = pytest.mark.gpu


def test_parameter_search_candidates_and_subset(engine, oracle):
    N, n, k, seed, f = 6000, 8, 10, 7, 0.05
    X = generate("clusters:4:0.05", N, n, seed)
    engine.set_points(X)
    cands = [(0.0, 0.0), (0.5, 0.2), (1.5, 0.0), (0.2, 1.0)]  # (1.5, .) is invalid
    res = parameter_search(engine, k, f, cands, RunConfig(k=k, seed=seed))
    assert [(c.beta, c.gamma) for c in res.candidates] == cands
    bad = res.candidates[2]
    assert bad.error == "beta, gamma, rho must all be in [0, 1]"
    ok = [c for c in res.candidates if not c.error]
    assert len(ok) == 3 and all(c.wall_seconds > 0 for c in ok)
    best = min(ok, key=lambda c: c.wall_seconds)
    assert (res.best_beta, res.best_gamma) == (best.beta, best.gamma)
    assert res.t1 is None and res.rho_model is None
    # the candidate runs are plain hybrid runs over the reference's subset
    subset = oracle.sample(N, math.floor(f * N), oracle.derive_seed(seed, 4)).astype(np.uint32)
    assert subset.size == math.floor(f * N)
    o = oracle.run(X, k=k, beta=0.5, gamma=0.2, rho=0.5, seed=seed)
    engine.set_points(X)
    r = engine.run(RunConfig(k=k, beta=0.5, gamma=0.2, rho=0.5, seed=seed, query_subset=subset),
                   want_hist=False)
    q = np.unique(subset)
    assert np.array_equal(r.queries, q)
    assert np.array_equal(r.ids, o["ids"][q]) and np.array_equal(r.dist, o["dist"][q])


@pytest.mark.parametrize("f,cands,code,msg", [
    (0.0, [(0.0, 0.0)], 1, "query fraction f must be in (0, 1]"),
    (1.5, [(0.0, 0.0)], 1, "query fraction f must be in (0, 1]"),
    (0.5, [], 1, "parameter search needs at least one candidate"),
    (0.01, [(0.0, 0.0)], 7, "parameter search sample of 40 queries is below the floor of 50"),
    (0.5, [(2.0, 0.0), (0.0, -1.0)], 1, "every parameter-search candidate failed"),
])
def test_parameter_search_errors(engine, f, cands, code, msg):
    X = generate("uniform", 4000, 3, 3)
    engine.set_points(X)
    with pytest.raises(KnnjError) as ei:
        parameter_search(engine, 5, f, cands, RunConfig(k=5, seed=3))
    assert ei.value.code == code and msg in str(ei.value)
