"""GPU: the tcgen05 distance screen's error stays far inside the bound the exact
re-decision relies on. One raw 128x128 TMEM accumulator tile per
case is compared with the same GEMM-form value computed from the FP16 operands
in float64, and the key with the FP64 scalar distance."""
import ctypes as C

import numpy as np
import pytest

from paper_1810_04758_b200.synthetic import generate

pytestmark = pytest.mark.gpu


def _tile(engine, q0, c0, n):
    L = engine.lib
    L.knnj_debug_tc_tile.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p,
                                     C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                     C.c_void_p, C.c_void_p]
    split = 3 if 3 * n + 2 <= 128 else 1
    rh = 64 if split * n + 2 <= 64 else 128
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


@pytest.mark.parametrize("spec,n,shift", [("clusters:16:0.05", 18, 0.0), ("uniform", 12, 0.0),
                                          ("clusters:4:0.01", 24, 1e3), ("mixture", 40, -7.5),
                                          ("clusters:16:0.05", 18, 1e5), ("uniform", 2, 0.0),
                                          ("exponential", 6, 0.0)])
def test_tc_accumulator_error_far_below_delta(engine, spec, n, shift):
    X = generate(spec, 6000, n, 3) + shift
    engine.set_points(X)
    m = min(6, n)
    engine.reorder_by_variance(m)
    engine.grid_build(m, 0.5)
    W = engine.working_points()
    worst = 0.0
    for q0, c0 in ((0, 0), (1000, 3000), (5800, 17)):
        D, bq, bc, S, delta, pq, pc = _tile(engine, q0, c0, n)
        split = 3 if 3 * n + 2 <= 128 else 1   # hi|lo|hi operand, or hi only (n > 42)
        a = np.zeros_like(bq)
        a[:, :n] = -2 * bq[:, :n]
        if split == 3:
            a[:, n:2 * n] = -2 * bq[:, :n]
            a[:, 2 * n:3 * n] = -2 * bq[:, n:2 * n]
        a[:, split * n:split * n + 2] = 1
        gemm = a @ bc.T
        worst = max(worst, float(np.abs(D - gemm).max()) / delta)
        # key vs the exact FP64 distance, in scaled units
        na = bq[:, split * n] + bq[:, split * n + 1]
        key = D.astype(np.float64) + na.astype(np.float32).astype(np.float64)[:, None]
        P, Q = W[pq], W[pc]
        sq = ((P[:, None, :] - Q[None, :, :]) ** 2).sum(-1) / (S * S)
        assert np.abs(key - sq).max() <= delta, (np.abs(key - sq).max(), delta)
    assert worst < 0.2, worst   # accumulation error uses < 1/5 of the budget
