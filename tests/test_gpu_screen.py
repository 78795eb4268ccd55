"""GPU: the tcgen05 distance screen and its error bound.

* Raw tiles: one 128x128 TMEM accumulator tile per case is compared with the same
  GEMM-form value computed from the FP16 operands in float64 (the accumulation error,
  which tc_delta bounds for any internal order / rounding of the UMMA chain), and the
  key with the FP64 scalar distance (the whole bound delta).
* Adversarial runs: data built to sit on the screen's decision boundaries - points on
  cell faces and lattice ties, near-ties a few ulps apart at the K-th distance, a large
  common offset - must give the oracle's output bit for bit through the tcgen05 path.
"""
import ctypes as C

import numpy as np
import pytest

from paper_1810_04758_b200 import RunConfig
from paper_1810_04758_b200.synthetic import generate

pytestmark = pytest.mark.gpu


def _tile(engine, q0, c0, n):
    L = engine.lib
    rh = 64 * ((3 * n + 2 + 63) // 64)
    D = np.zeros((128, 128), np.float32)
    Bq = np.zeros((128, rh), np.uint16)
    Bc = np.zeros((128, rh), np.uint16)
    S, dl = C.c_double(), C.c_double()
    pq = np.zeros(128, np.uint32)
    pc = np.zeros(128, np.uint32)
    engine._check(L.knnj_debug_tc_tile(engine.h, q0, c0, D.ctypes.data, Bq.ctypes.data,
                                       Bc.ctypes.data, C.byref(S), C.byref(dl), pq.ctypes.data,
                                       pc.ctypes.data))
    return (D, Bq.view(np.float16).astype(np.float64), Bc.view(np.float16).astype(np.float64),
            S.value, dl.value, pq, pc)


def _acc_bound(n, bq, bc):
    """The accumulation term of tc_delta evaluated with this tile's actual magnitudes:
    18 * 2^-23 * sum over the UMMA steps of (sum |p| of the step + |D_in|)."""
    a = np.zeros_like(bq)
    a[:, :n] = -2 * bq[:, n:2 * n]
    a[:, n:2 * n] = -2 * bq[:, :n]
    a[:, 2 * n:3 * n] = -2 * bq[:, 2 * n:3 * n]
    a[:, 3 * n:3 * n + 2] = 1
    steps = (3 * n + 2 + 15) // 16
    total = np.zeros((a.shape[0], bc.shape[0]))
    prefix = np.zeros_like(total)
    for s in range(steps):
        sl = slice(16 * s, 16 * s + 16)
        S_s = np.abs(a[:, sl]) @ np.abs(bc[:, sl]).T
        total += S_s + prefix
        prefix += S_s
    return a, 18 * 2.0 ** -23 * total


@pytest.mark.parametrize("spec,n,shift", [("clusters:16:0.05", 18, 0.0), ("uniform", 12, 0.0),
                                          ("clusters:4:0.01", 24, 1e3), ("mixture", 40, -7.5),
                                          ("clusters:16:0.05", 18, 1e5), ("uniform", 2, 0.0),
                                          ("uniform", 4, 0.0), ("exponential", 6, 0.0)])
def test_tc_accumulator_within_bound(engine, spec, n, shift):
    X = generate(spec, 6000, n, 3) + shift
    engine.set_points(X)
    m = min(6, n)
    engine.reorder_by_variance(m)
    engine.grid_build(m, 0.5)
    W = engine.working_points()
    for q0, c0 in ((0, 0), (1000, 3000), (5800, 17), (2500, 2500)):
        D, bq, bc, S, delta, pq, pc = _tile(engine, q0, c0, n)
        a, acc = _acc_bound(n, bq, bc)
        gemm = a @ bc.T                       # exact in float64 (22-bit products, short sums)
        err = np.abs(D.astype(np.float64) - gemm)
        assert (err <= acc).all(), float((err / acc).max())
        # key vs the exact FP64 distance, in scaled units: within the whole bound
        na = bq[:, 3 * n] + bq[:, 3 * n + 1]
        key = D.astype(np.float64) + na.astype(np.float32).astype(np.float64)[:, None]
        P, Q = W[pq], W[pc]
        sq = ((P[:, None, :] - Q[None, :, :]) ** 2).sum(-1) / (S * S)
        assert np.abs(key - sq).max() <= delta, (np.abs(key - sq).max(), delta)


def _faces(N, n, seed):
    """Lattice points (spacing 1/8) with duplicates and exact ties, sitting on cell faces
    of every grid whose width divides the spacing, plus a few off-lattice points."""
    rng = np.random.default_rng(seed)
    X = rng.integers(0, 24, (N, n)).astype(np.float64) / 8.0
    X[: N // 10] += rng.random((N // 10, n)) * 1e-9
    return X


def _shells(N, n, k, seed):
    """Groups of k + 12 points at distances r (1 + j 2^-40) from a centre: near-ties a few
    ulps apart at each centre's K-th distance, far inside the screen band."""
    rng = np.random.default_rng(seed)
    g = k + 13
    centres = rng.random((N // g, n))
    out = []
    for c in centres:
        d = rng.standard_normal((g - 1, n))
        d /= np.linalg.norm(d, axis=1)[:, None]
        r = 0.01 * (1.0 + np.arange(g - 1) * 2.0 ** -40)
        out.append(np.vstack([c, c + d * r[:, None]]))
    return np.vstack(out)


@pytest.mark.parametrize("name,k", [("faces4", 12), ("faces6", 20), ("shells18", 16), ("shells4", 8),
                                    ("offset18", 32), ("offset4", 16)])
def test_screen_adversarial_matches_oracle(engine, oracle, name, k):
    if name.startswith("faces"):
        n = int(name[5:])
        X = _faces(12000, n, 5)
    elif name.startswith("shells"):
        n = int(name[6:])
        X = _shells(12000, n, k, 6)
    else:
        n = int(name[6:])
        X = generate("clusters:8:0.05" if n > 4 else "uniform", 15000, n, 7) + 1e5
    engine.set_points(X)
    r = engine.run(RunConfig(k=k, mode="hybrid", seed=11), want_hist=False)
    o = oracle.run(X, k=k, mode="hybrid", seed=11)
    assert r.info["eps_used"] == o["eps_used"]
    assert np.array_equal(r.ids, o["ids"]), "neighbour ids differ from the oracle"
    assert np.array_equal(r.dist, o["dist"]), "distances differ from the oracle"
    assert np.array_equal(r.provenance, o["prov"])
    # the same run on the SIMT screen agrees too (two independent screens)
    engine.set_option("tensor_cores", 0)
    try:
        engine.set_points(X)
        s = engine.run(RunConfig(k=k, mode="hybrid", seed=11), want_hist=False)
    finally:
        engine.set_option("tensor_cores", 1)
    assert np.array_equal(s.ids, r.ids) and np.array_equal(s.dist, r.dist)
