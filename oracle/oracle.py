"""TEST INFRASTRUCTURE ONLY — ctypes bindings for the CPU checkers.

* ``Oracle``: the C restatement in oracle/knnj_oracle.c (liboracle.so).
* ``Ref``:    the unmodified reference compiled by oracle/Makefile
              (oracle/_ref/libknnjoin_ref.so), when it has been built.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline leg may
import this module, and only as the checker / the timed CPU baseline — the
product path (paper_1810_04758_b200) never routes through it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libknnjoin_ref.so")

MODES = {"hybrid": 0, "sparse": 1, "dense": 2, "oracle": 3}

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")


def build_oracle() -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)


class _OrcCfg(C.Structure):
    _fields_ = [("k", C.c_uint32), ("m", C.c_uint32), ("mode", C.c_uint32),
                ("threads", C.c_uint32), ("n_bins", C.c_uint32), ("beta", C.c_double),
                ("gamma", C.c_double), ("rho", C.c_double), ("hist_frac", C.c_double),
                ("seed", C.c_uint64), ("eps_mean_cap", C.c_uint64)]


class _OrcInfo(C.Structure):
    _fields_ = [("k_eff", C.c_uint32), ("m_used", C.c_uint32), ("eps_fallback", C.c_uint32),
                ("eps_mean", C.c_double), ("bin_width", C.c_double),
                ("eps_default", C.c_double), ("eps_beta", C.c_double),
                ("eps_used", C.c_double), ("n_min", C.c_double), ("n_thresh", C.c_double),
                ("hist_query_count", C.c_uint64), ("q_gpu", C.c_uint64),
                ("q_cpu", C.c_uint64), ("demoted", C.c_uint64),
                ("failed_count", C.c_uint64), ("candidates_examined", C.c_uint64),
                ("perm", C.c_uint32 * 1024)]


class _OrcGrid(C.Structure):
    _fields_ = [("m", C.c_uint32), ("eps", C.c_double), ("mins", C.c_double * 64),
                ("maxs", C.c_double * 64), ("cpd", C.c_uint64 * 64),
                ("strides", C.c_uint64 * 64), ("ncells", C.c_uint64),
                ("B", C.POINTER(C.c_uint64)), ("G", C.POINTER(C.c_uint64)),
                ("A", C.POINTER(C.c_uint32)), ("slot", C.POINTER(C.c_uint32))]


class _MT(C.Structure):
    _fields_ = [("mt", C.c_uint64 * 312), ("mti", C.c_int)]


class Oracle:
    """The C restatement (see oracle/knnj_oracle.h)."""

    def __init__(self) -> None:
        if not os.path.exists(ORACLE_SO):
            build_oracle()
        L = C.CDLL(ORACLE_SO)
        L.orc_sq_dist_limited.restype = C.c_double
        L.orc_sq_dist_limited.argtypes = [_dp, _dp, C.c_size_t, C.c_double]
        L.orc_mt_seed.argtypes = [C.POINTER(_MT), C.c_uint64]
        L.orc_mt_next.restype = C.c_uint64
        L.orc_mt_next.argtypes = [C.POINTER(_MT)]
        L.orc_uniform_u64.restype = C.c_uint64
        L.orc_uniform_u64.argtypes = [C.POINTER(_MT), C.c_uint64, C.c_uint64]
        L.orc_derive_seed.restype = C.c_uint64
        L.orc_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_sample_without_replacement.restype = C.c_uint64
        L.orc_sample_without_replacement.argtypes = [C.c_uint64, C.c_uint64, C.POINTER(_MT),
                                                     _u64p]
        L.orc_variance_order.argtypes = [_dp, C.c_uint64, C.c_uint32, _u32p, _dp]
        L.orc_eps_mean.argtypes = [_dp, C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64,
                                   C.POINTER(C.c_double)]
        L.orc_histogram.argtypes = [_dp, C.c_uint64, C.c_uint32, C.c_double, C.c_uint32,
                                    C.c_double, C.c_uint64, C.c_uint32, _u64p,
                                    C.POINTER(C.c_uint64)]
        L.orc_histogram_queries.argtypes = [_dp, C.c_uint64, C.c_uint32, C.c_double,
                                            C.c_uint32, _u64p, C.c_uint64, C.c_uint32, _u64p]
        L.orc_select_eps.argtypes = [_dp, C.c_uint32, C.c_double, C.c_uint32, C.c_double,
                                     C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                     C.POINTER(C.c_uint64), C.POINTER(C.c_int)]
        L.orc_grid_build.argtypes = [_dp, C.c_uint64, C.c_uint32, C.c_uint32, C.c_double,
                                     C.POINTER(_OrcGrid), C.c_char_p, C.c_size_t]
        L.orc_grid_free.argtypes = [C.POINTER(_OrcGrid)]
        L.orc_n_min.restype = C.c_double
        L.orc_n_min.argtypes = [C.c_uint32, C.c_uint32]
        L.orc_n_thresh.restype = C.c_double
        L.orc_n_thresh.argtypes = [C.c_double, C.c_double]
        L.orc_run.argtypes = [_dp, C.c_uint64, C.c_uint32, C.POINTER(_OrcCfg), _u32p, _dp,
                              _u8p, _u64p, C.POINTER(_OrcInfo), C.c_char_p, C.c_size_t]
        L.orc_brute_knn.argtypes = [_dp, C.c_uint64, C.c_uint32, _u32p, C.c_uint64,
                                    C.c_uint32, C.c_uint32, _u32p, _dp]
        self.L = L

    # -- primitives ---------------------------------------------------------
    def sq_dist_limited(self, a, b, limit=np.inf) -> float:
        a = np.ascontiguousarray(a, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        return self.L.orc_sq_dist_limited(a, b, a.size, limit)

    def mt_stream(self, seed: int, count: int) -> np.ndarray:
        st = _MT()
        self.L.orc_mt_seed(C.byref(st), seed)
        return np.array([self.L.orc_mt_next(C.byref(st)) for _ in range(count)], np.uint64)

    def derive_seed(self, master: int, tag: int) -> int:
        return self.L.orc_derive_seed(master, tag)

    def sample(self, n: int, k: int, seed: int) -> np.ndarray:
        st = _MT()
        self.L.orc_mt_seed(C.byref(st), seed)
        out = np.zeros(max(min(n, k), 1), np.uint64)
        c = self.L.orc_sample_without_replacement(n, k, C.byref(st), out)
        return out[:c]

    def variance_order(self, X):
        X = np.ascontiguousarray(X, np.float64)
        N, n = X.shape
        order = np.zeros(n, np.uint32)
        var = np.zeros(n, np.float64)
        self.L.orc_variance_order(X, N, n, order, var)
        return order, var

    def eps_mean(self, X, pairs: int, seed: int) -> float:
        X = np.ascontiguousarray(X, np.float64)
        out = C.c_double()
        rc = self.L.orc_eps_mean(X, X.shape[0], X.shape[1], pairs, seed, C.byref(out))
        if rc:
            raise ValueError("eps_mean usage error")
        return out.value

    def histogram(self, X, eps_mean, n_bins, frac, seed, threads=8):
        X = np.ascontiguousarray(X, np.float64)
        raw = np.zeros(n_bins, np.uint64)
        qc = C.c_uint64()
        rc = self.L.orc_histogram(X, X.shape[0], X.shape[1], eps_mean, n_bins, frac, seed,
                                  threads, raw, C.byref(qc))
        if rc:
            raise ValueError(f"histogram error {rc}")
        return raw, qc.value

    def histogram_queries(self, X, eps_mean, n_bins, queries, threads=8):
        X = np.ascontiguousarray(X, np.float64)
        q = np.ascontiguousarray(queries, np.uint64)
        raw = np.zeros(n_bins, np.uint64)
        rc = self.L.orc_histogram_queries(X, X.shape[0], X.shape[1], eps_mean, n_bins, q,
                                          q.size, threads, raw)
        if rc:
            raise ValueError(f"histogram error {rc}")
        return raw

    def select_eps(self, cum, bin_width, k, beta, allow_fallback=True):
        cum = np.ascontiguousarray(cum, np.float64)
        eb, ef, b, fb = C.c_double(), C.c_double(), C.c_uint64(), C.c_int()
        rc = self.L.orc_select_eps(cum, cum.size, bin_width, k, beta, int(allow_fallback),
                                   C.byref(eb), C.byref(ef), C.byref(b), C.byref(fb))
        if rc:
            raise ValueError("target unreachable")
        return eb.value, ef.value, b.value, bool(fb.value)

    def grid(self, X, m, eps):
        X = np.ascontiguousarray(X, np.float64)
        N = X.shape[0]
        g = _OrcGrid()
        err = C.create_string_buffer(256)
        rc = self.L.orc_grid_build(X, N, X.shape[1], m, eps, C.byref(g), err, 256)
        if rc:
            raise ValueError(f"grid error {rc}: {err.value.decode()}")
        nc = g.ncells
        out = dict(
            B=np.ctypeslib.as_array(g.B, (nc,)).copy(),
            G=np.ctypeslib.as_array(g.G, (2 * nc,)).copy().reshape(nc, 2),
            A=np.ctypeslib.as_array(g.A, (N,)).copy(),
            slot=np.ctypeslib.as_array(g.slot, (N,)).copy(),
            cpd=np.array(g.cpd[:m], np.uint64), mins=np.array(g.mins[:m]),
            maxs=np.array(g.maxs[:m]))
        self.L.orc_grid_free(C.byref(g))
        return out

    def n_min(self, k, m):
        return self.L.orc_n_min(k, m)

    def n_thresh(self, n_min, gamma):
        return self.L.orc_n_thresh(n_min, gamma)

    def brute_knn(self, Xw, queries, k, threads=8):
        Xw = np.ascontiguousarray(Xw, np.float64)
        q = np.ascontiguousarray(queries, np.uint32)
        ids = np.zeros(q.size * k, np.uint32)
        dist = np.zeros(q.size * k, np.float64)
        self.L.orc_brute_knn(Xw, Xw.shape[0], Xw.shape[1], q, q.size, k, threads, ids, dist)
        return ids.reshape(q.size, k), dist.reshape(q.size, k)

    def run(self, X, k=5, m=0, beta=0.0, gamma=0.0, rho=0.0, mode="hybrid", seed=0,
            n_bins=100, hist_frac=0.01, eps_mean_cap=1_000_000, threads=8):
        X = np.ascontiguousarray(X, np.float64)
        N, n = X.shape
        cfg = _OrcCfg(k, m, MODES[mode], threads, n_bins, beta, gamma, rho, hist_frac, seed,
                      eps_mean_cap)
        k_eff = min(k, N - 1)
        ids = np.zeros(max(N * k_eff, 1), np.uint32)
        dist = np.zeros(max(N * k_eff, 1), np.float64)
        prov = np.zeros(N, np.uint8)
        raw = np.zeros(n_bins, np.uint64)
        info = _OrcInfo()
        err = C.create_string_buffer(256)
        rc = self.L.orc_run(X, N, n, C.byref(cfg), ids, dist, prov, raw, C.byref(info), err, 256)
        if rc:
            raise RuntimeError(f"oracle run failed ({rc}): {err.value.decode()}")
        out = {f: getattr(info, f) for f, _ in _OrcInfo._fields_ if f != "perm"}
        out.update(ids=ids[:N * k_eff].reshape(N, k_eff), dist=dist[:N * k_eff].reshape(N, k_eff),
                   prov=prov, raw_hist=raw, perm=np.array(info.perm[:n], np.uint32))
        return out


# ---------------------------------------------------------------------------
class _RefCfg(C.Structure):
    _fields_ = [("k", C.c_uint32), ("m", C.c_uint32), ("beta", C.c_double),
                ("gamma", C.c_double), ("rho", C.c_double), ("mode", C.c_uint32),
                ("workers", C.c_uint32), ("seed", C.c_uint64), ("n_bins", C.c_uint32),
                ("hist_frac", C.c_double), ("batch_frac", C.c_double),
                ("buffer_size", C.c_uint64), ("eps_mean_cap", C.c_uint64),
                ("policy_dynamic", C.c_uint32), ("policy_count", C.c_uint64),
                ("subset", C.POINTER(C.c_uint32)), ("n_subset", C.c_uint64),
                ("force_n_batches", C.c_uint64)]


class _RefInfo(C.Structure):
    _fields_ = [("n_queries", C.c_uint64), ("k_eff", C.c_uint32), ("m_used", C.c_uint32),
                ("eps_used", C.c_double), ("eps_mean", C.c_double),
                ("eps_default", C.c_double), ("eps_beta", C.c_double),
                ("bin_width", C.c_double), ("hist_query_count", C.c_uint64),
                ("q_gpu", C.c_uint64), ("q_cpu", C.c_uint64), ("demoted", C.c_uint64),
                ("failed_count", C.c_uint64), ("n_min", C.c_double), ("n_thresh", C.c_double),
                ("eps_fallback", C.c_uint32), ("has_profile", C.c_uint32),
                ("candidates_examined", C.c_uint64), ("estimate_e", C.c_uint64),
                ("n_batches", C.c_uint64)] + [
                   (f, C.c_double) for f in ("t_reorder", "t_eps", "t_grid", "t_kd", "t_split",
                                             "t_dense", "t_sparse", "t_reassign", "t_merge",
                                             "measured_total")] + [
                   ("perm", C.c_uint32 * 1024)]


def ref_available() -> bool:
    return os.path.exists(REF_SO)


class Ref:
    """The unmodified reference library (oracle/_ref), through oracle/ref_capi.cpp."""

    def __init__(self) -> None:
        if not ref_available():
            raise FileNotFoundError(REF_SO)
        L = C.CDLL(REF_SO)
        L.ref_last_error.restype = C.c_char_p
        L.ref_set_kernel.argtypes = [C.c_char_p]
        L.ref_sq_dist_limited.restype = C.c_double
        L.ref_sq_dist_limited.argtypes = [_dp, _dp, C.c_uint64, C.c_double]
        L.ref_generate.argtypes = [C.c_char_p, C.c_uint64, C.c_uint32, C.c_uint64, _dp]
        L.ref_run.argtypes = [_dp, C.c_uint64, C.c_uint32, C.POINTER(_RefCfg), _u32p, _u32p,
                              _dp, _u32p, _u8p, _dp, _dp, C.POINTER(_RefInfo)]
        L.ref_variance_order.argtypes = [_dp, C.c_uint64, C.c_uint32, C.c_uint32, _u32p, _dp]
        L.ref_eps_mean.argtypes = [_dp, C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64,
                                   C.POINTER(C.c_double)]
        L.ref_histogram.argtypes = [_dp, C.c_uint64, C.c_uint32, C.c_double, C.c_uint32,
                                    C.c_double, C.c_uint64, C.c_uint32, _dp, _dp,
                                    C.POINTER(C.c_uint64)]
        L.ref_sample.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, _u64p]
        L.ref_derive_seed.restype = C.c_uint64
        L.ref_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.ref_grid.argtypes = [_dp, C.c_uint64, C.c_uint32, C.c_uint32, C.c_double,
                               C.POINTER(C.c_uint64), C.c_void_p, C.c_void_p, C.c_void_p,
                               C.c_void_p, C.c_void_p, C.c_void_p]
        L.ref_range_counts.argtypes = [_dp, C.c_uint64, C.c_uint32, C.c_uint32, C.c_double,
                                       _u32p, C.c_uint64, _u64p, _u64p]
        L.ref_split.argtypes = [_dp, C.c_uint64, C.c_uint32, C.c_uint32, C.c_double,
                                C.c_uint32, C.c_double, C.c_double, C.c_double, _u32p,
                                C.c_uint64, _u8p, _u64p, C.POINTER(C.c_double),
                                C.POINTER(C.c_double), C.POINTER(C.c_uint64)]
        L.ref_brute_knn.argtypes = [_dp, C.c_uint64, C.c_uint32, _u32p, C.c_uint64, C.c_uint32,
                                    C.c_uint32, _u32p, _dp]
        L.ref_sparse_knn.argtypes = [_dp, C.c_uint64, C.c_uint32, _u32p, C.c_uint64,
                                     C.c_uint32, C.c_uint32, _u32p, _dp,
                                     C.POINTER(C.c_double)]
        L.ref_hardware_concurrency.restype = C.c_uint
        L.ref_kd_create.restype = C.c_void_p
        L.ref_kd_create.argtypes = [_dp, C.c_uint64, C.c_uint32, C.c_uint32,
                                    C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.ref_kd_query.argtypes = [C.c_void_p, _u32p, C.c_uint64, C.c_uint32, C.c_uint32,
                                   _u32p, _dp, C.POINTER(C.c_double)]
        L.ref_kd_destroy.argtypes = [C.c_void_p]
        self.L = L

    def _check(self, rc):
        if rc:
            raise RuntimeError(f"reference error {rc}: {self.L.ref_last_error().decode()}")

    def set_kernel(self, name: str) -> None:
        if self.L.ref_set_kernel(name.encode()):
            raise ValueError(name)

    def sq_dist_limited(self, a, b, limit=np.inf) -> float:
        a = np.ascontiguousarray(a, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        return self.L.ref_sq_dist_limited(a, b, a.size, limit)

    def generate(self, spec: str, size: int, dims: int, seed: int) -> np.ndarray:
        out = np.zeros(size * dims, np.float64)
        self._check(self.L.ref_generate(spec.encode(), size, dims, seed, out))
        return out.reshape(size, dims)

    def variance_order(self, X, m=1):
        X = np.ascontiguousarray(X, np.float64)
        perm = np.zeros(X.shape[1], np.uint32)
        var = np.zeros(X.shape[1], np.float64)
        self._check(self.L.ref_variance_order(X, X.shape[0], X.shape[1], m, perm, var))
        return perm, var

    def eps_mean(self, X, pairs, seed):
        X = np.ascontiguousarray(X, np.float64)
        out = C.c_double()
        self._check(self.L.ref_eps_mean(X, X.shape[0], X.shape[1], pairs, seed, C.byref(out)))
        return out.value

    def histogram(self, X, eps_mean, n_bins, frac, seed, threads=8):
        X = np.ascontiguousarray(X, np.float64)
        counts = np.zeros(n_bins)
        cum = np.zeros(n_bins)
        qc = C.c_uint64()
        self._check(self.L.ref_histogram(X, X.shape[0], X.shape[1], eps_mean, n_bins, frac,
                                         seed, threads, counts, cum, C.byref(qc)))
        return counts, cum, qc.value

    def sample(self, n, k, seed):
        out = np.zeros(max(min(n, k), 1), np.uint64)
        self._check(self.L.ref_sample(n, k, seed, out))
        return out[:min(n, k)]

    def derive_seed(self, master, tag):
        return self.L.ref_derive_seed(master, tag)

    def grid(self, X, m, eps):
        X = np.ascontiguousarray(X, np.float64)
        N, n = X.shape
        nc = C.c_uint64()
        self._check(self.L.ref_grid(X, N, n, m, eps, C.byref(nc), None, None, None, None,
                                    None, None))
        c = nc.value
        B = np.zeros(c, np.uint64)
        G = np.zeros(2 * c, np.uint64)
        A = np.zeros(N, np.uint32)
        cpd = np.zeros(m, np.uint64)
        mins = np.zeros(m)
        maxs = np.zeros(m)
        p = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
        self._check(self.L.ref_grid(X, N, n, m, eps, C.byref(nc), p(B), p(G), p(A), p(cpd),
                                    p(mins), p(maxs)))
        return dict(B=B, G=G.reshape(c, 2), A=A, cpd=cpd, mins=mins, maxs=maxs)

    def range_counts(self, X, m, eps, queries):
        X = np.ascontiguousarray(X, np.float64)
        q = np.ascontiguousarray(queries, np.uint32)
        cand = np.zeros(q.size, np.uint64)
        ine = np.zeros(q.size, np.uint64)
        self._check(self.L.ref_range_counts(X, X.shape[0], X.shape[1], m, eps, q, q.size,
                                            cand, ine))
        return cand, ine

    def split(self, X, m, eps, k, beta, gamma, rho, queries):
        X = np.ascontiguousarray(X, np.float64)
        q = np.ascontiguousarray(queries, np.uint32)
        dense = np.zeros(q.size, np.uint8)
        pop = np.zeros(q.size, np.uint64)
        nmin, nth, dem = C.c_double(), C.c_double(), C.c_uint64()
        self._check(self.L.ref_split(X, X.shape[0], X.shape[1], m, eps, k, beta, gamma, rho,
                                     q, q.size, dense, pop, C.byref(nmin), C.byref(nth),
                                     C.byref(dem)))
        return dict(is_dense=dense, pop=pop, n_min=nmin.value, n_thresh=nth.value,
                    demoted=dem.value)

    def brute_knn(self, Xw, queries, k, threads=8):
        Xw = np.ascontiguousarray(Xw, np.float64)
        q = np.ascontiguousarray(queries, np.uint32)
        ids = np.zeros(q.size * k, np.uint32)
        dist = np.zeros(q.size * k, np.float64)
        self._check(self.L.ref_brute_knn(Xw, Xw.shape[0], Xw.shape[1], q, q.size, k, threads,
                                         ids, dist))
        return ids.reshape(q.size, k), dist.reshape(q.size, k)

    def sparse_knn(self, Xw, queries, k, threads=0):
        Xw = np.ascontiguousarray(Xw, np.float64)
        q = np.ascontiguousarray(queries, np.uint32)
        ids = np.zeros(q.size * k, np.uint32)
        dist = np.zeros(q.size * k, np.float64)
        secs = C.c_double()
        threads = threads or self.hardware_concurrency()
        self._check(self.L.ref_sparse_knn(Xw, Xw.shape[0], Xw.shape[1], q, q.size, k, threads,
                                          ids, dist, C.byref(secs)))
        return ids.reshape(q.size, k), dist.reshape(q.size, k), secs.value

    def kd_create(self, X, m):
        """reorder_by_variance + KdTree::build once; returns (handle, t_reorder, t_build)."""
        X = np.ascontiguousarray(X, np.float64)
        a, b = C.c_double(), C.c_double()
        h = self.L.ref_kd_create(X, X.shape[0], X.shape[1], m, C.byref(a), C.byref(b))
        if not h:
            raise RuntimeError(self.L.ref_last_error().decode())
        return h, a.value, b.value

    def kd_query(self, h, queries, k, threads=0):
        q = np.ascontiguousarray(queries, np.uint32)
        ids = np.zeros(q.size * k, np.uint32)
        dist = np.zeros(q.size * k, np.float64)
        secs = C.c_double()
        threads = threads or self.hardware_concurrency()
        self._check(self.L.ref_kd_query(h, q, q.size, k, threads, ids, dist, C.byref(secs)))
        return ids.reshape(q.size, k), dist.reshape(q.size, k), secs.value

    def kd_destroy(self, h):
        self.L.ref_kd_destroy(h)

    def hardware_concurrency(self) -> int:
        return int(self.L.ref_hardware_concurrency())

    def run(self, X, k=5, m=0, beta=0.0, gamma=0.0, rho=0.0, mode="hybrid", seed=0,
            n_bins=100, hist_frac=0.01, batch_frac=0.01, buffer_size=1_000_000,
            eps_mean_cap=1_000_000, workers=0, policy=("static", 8), subset=None,
            force_n_batches=0):
        X = np.ascontiguousarray(X, np.float64)
        N, n = X.shape
        sub = None
        nsub = 0
        if subset is not None:
            sub_arr = np.ascontiguousarray(subset, np.uint32)
            sub = sub_arr.ctypes.data_as(C.POINTER(C.c_uint32))
            nsub = sub_arr.size
        cfg = _RefCfg(k, m, beta, gamma, rho, MODES[mode], workers, seed, n_bins, hist_frac,
                      batch_frac, buffer_size, eps_mean_cap, int(policy[0] == "dynamic"),
                      policy[1], sub, nsub, force_n_batches)
        nq = N if subset is None else len(np.unique(subset))
        qids = np.zeros(max(nq, 1), np.uint32)
        ids = np.zeros(max(nq * k, 1), np.uint32)
        dist = np.zeros(max(nq * k, 1), np.float64)
        counts = np.zeros(max(nq, 1), np.uint32)
        prov = np.zeros(max(nq, 1), np.uint8)
        hc = np.zeros(n_bins)
        hcum = np.zeros(n_bins)
        info = _RefInfo()
        self._check(self.L.ref_run(X, N, n, C.byref(cfg), qids, ids, dist, counts, prov, hc,
                                   hcum, C.byref(info)))
        out = {f: getattr(info, f) for f, _ in _RefInfo._fields_ if f != "perm"}
        ke = info.k_eff
        out.update(queries=qids[:nq], ids=ids[:nq * k].reshape(nq, k)[:, :ke],
                   dist=dist[:nq * k].reshape(nq, k)[:, :ke], counts=counts[:nq],
                   prov=prov[:nq], hist_counts=hc, hist_cum=hcum,
                   perm=np.array(info.perm[:n], np.uint32))
        return out
