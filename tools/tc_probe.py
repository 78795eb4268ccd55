"""Probe one tcgen05 tile: raw TMEM accumulators vs the same GEMM-form value from
the FP16 operands (numpy, float64) and vs the exact distance (dev tool)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1810_04758_b200 import Engine
from paper_1810_04758_b200.synthetic import generate
eng = Engine(0)
L = eng.lib
L.knnj_debug_tc_tile.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p,
                                 C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_void_p, C.c_void_p]
X = generate("clusters:16:0.05", 20000, 18, 1)
eng.set_points(X)
eng.reorder_by_variance(6)
eng.grid_build(6, 0.35)
n = 18
D = np.zeros((128, 128), np.float32)
rh = 64
Bq = np.zeros((128, rh), np.uint16); Bc = np.zeros((128, rh), np.uint16)
S, dl = C.c_double(), C.c_double()
eng._check(L.knnj_debug_tc_tile(eng.h, 1000, 5000, D.ctypes.data, Bq.ctypes.data, Bc.ctypes.data,
                                C.byref(S), C.byref(dl), np.zeros(128,np.uint32).ctypes.data, np.zeros(128,np.uint32).ctypes.data))
bq = Bq.view(np.float16).astype(np.float64); bc = Bc.view(np.float16).astype(np.float64)
A = np.zeros_like(bq)
A[:, :n] = -2 * bq[:, :n]; A[:, n:2*n] = -2 * bq[:, :n]; A[:, 2*n:3*n] = -2 * bq[:, n:2*n]; A[:, 3*n:3*n+2] = 1
want = A @ bc.T
print("S", S.value, "delta", dl.value)
print("D[0,:6]   ", D[0, :6])
print("want[0,:6]", want[0, :6])
err = np.abs(D - want)
print("max |D-want|", err.max(), "rel to delta", err.max() / dl.value)
i, j = np.unravel_index(np.argmax(err), err.shape); print("argmax", i, j, D[i, j], want[i, j])
# which transposition/layout would match?
for name, cand in [("want.T", want.T)]:
    print(name, np.abs(D - cand).max())
