"""Python mirror of the reference ``knnjoin`` API over the C ABI.

Names, defaults, argument meaning and error behaviour follow the reference
C++ library (/root/reference/proj/include/knnjoin/*.hpp); every call runs on
the GPU through libknnj_b200.so. This is the interface the parity tests and
bench.py use; C++ callers link the same library through include/knnj_c.h.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
from typing import Optional, Sequence

import numpy as np

from . import _capi
from ._capi import KnnjError

HYBRID, SPARSE_ONLY, DENSE_ONLY, BRUTE_ORACLE = 0, 1, 2, 3
MODE_NAMES = {"hybrid": HYBRID, "sparse": SPARSE_ONLY, "dense": DENSE_ONLY,
              "oracle": BRUTE_ORACLE}
PROVENANCE_NAMES = {0: "dense", 1: "sparse", 2: "dense_failed_then_sparse"}

# seed sub-stream tags, proj/include/knnjoin/util.hpp:26-29
SEED_EPS_MEAN, SEED_HISTOGRAM, SEED_BATCH_ESTIMATE, SEED_QUERY_SUBSET = 1, 2, 3, 4


def splitmix64(x: int) -> int:
    m = (1 << 64) - 1
    x = (x + 0x9E3779B97F4A7C15) & m
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & m
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & m
    return x ^ (x >> 31)


def derive_seed(master: int, tag: int) -> int:
    """proj/include/knnjoin/util.hpp:22-24"""
    return splitmix64(master ^ splitmix64(tag))


@dataclasses.dataclass
class RunConfig:
    """RunConfig, proj/include/knnjoin/orchestrator.hpp:17-41 (device-relevant fields)."""
    k: int = 5
    m: int = 0                      # 0 -> min(6, n)
    beta: float = 0.0
    gamma: float = 0.0
    rho: float = 0.0
    mode: str = "hybrid"            # hybrid | sparse | dense | oracle
    n_bins: int = 100
    hist_query_fraction: float = 0.01
    eps_mean_pair_cap: int = 1_000_000
    seed: int = 0
    query_subset: Optional[Sequence[int]] = None


@dataclasses.dataclass
class KnnRunResult:
    """KnnRunResult, proj/include/knnjoin/orchestrator.hpp:67-89."""
    queries: np.ndarray              # ascending point ids
    ids: np.ndarray                  # [n_queries, k_effective] neighbour ids, (dist, id) order
    dist: np.ndarray                 # [n_queries, k_effective] FP64 distances
    provenance: np.ndarray           # uint8 per query (0 dense, 1 sparse, 2 dense-failed)
    k_effective: int
    info: dict
    raw_hist: Optional[np.ndarray] = None
    warnings: list = dataclasses.field(default_factory=list)

    @property
    def failed_count(self) -> int:
        return int(self.info["failed_count"])

    @property
    def eps_used(self) -> float:
        return float(self.info["eps_used"])

    def profile_counts(self) -> np.ndarray:
        return self.raw_hist / float(self.info["hist_query_count"])

    def profile_cumulative(self) -> np.ndarray:
        return np.cumsum(self.raw_hist).astype(np.float64) / float(self.info["hist_query_count"])


def tsv_string(r: KnnRunResult) -> str:
    """proj/src/io.cpp:141-154: '%u\\t%u\\t%.17g' per (query, rank)."""
    out = []
    for qi, q in enumerate(r.queries):
        for j in range(r.ids.shape[1]):
            out.append(f"{int(q)}\t{int(r.ids[qi, j])}\t{float(r.dist[qi, j]):.17g}\n")
    # %.17g in Python matches C's printf %.17g
    return "".join(out)


class Engine:
    """One knnj_ctx on one GPU (the C ABI's unit of ownership)."""

    def __init__(self, device: int = 0):
        self.lib = _capi.load_library()
        h = C.c_void_p()
        rc = self.lib.knnj_create(device, C.byref(h))
        if rc:
            raise KnnjError(rc, f"cannot create context on device {device}")
        self.h = h
        self.device = device
        self.N = 0
        self.n = 0
        self._all_queries = None

    def close(self) -> None:
        if getattr(self, "h", None):
            self.lib.knnj_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc: int) -> None:
        if rc:
            raise KnnjError(rc, self.lib.knnj_last_error(self.h).decode())

    def set_option(self, name: str, value: int) -> None:
        self._check(self.lib.knnj_set_option(self.h, name.encode(), int(value)))

    # ------------------------------------------------------------- dataset
    def set_points(self, X) -> None:
        """Dataset(coords, dims) upload (validates finiteness like dataset.cpp:22-33).
        Accepts a C-contiguous float64 numpy array or a raw (pointer, N, n) tuple."""
        if isinstance(X, tuple):
            ptr, N, n = X
        else:
            X = np.ascontiguousarray(X, np.float64)
            if X.ndim != 2:
                raise KnnjError(1, "points must be a 2-D array")
            ptr, (N, n) = X.ctypes.data, X.shape
            self._keep = X
        self._check(self.lib.knnj_set_points(self.h, C.c_void_p(ptr), N, n))
        self.N, self.n = int(N), int(n)

    def reorder_by_variance(self, m: int):
        perm = np.zeros(self.n, np.uint32)
        var = np.zeros(self.n, np.float64)
        self._check(self.lib.knnj_reorder_by_variance(self.h, m, perm, var))
        return perm, var

    def working_points(self) -> np.ndarray:
        out = np.zeros((self.N, self.n), np.float64)
        self._check(self.lib.knnj_get_points(self.h, out))
        return out

    # ------------------------------------------------------------- phases
    def pair_sq(self, pairs, limit: float = np.inf) -> np.ndarray:
        ij = np.ascontiguousarray(pairs, np.uint64).reshape(-1)
        out = np.zeros(ij.size // 2, np.float64)
        self._check(self.lib.knnj_pair_sq(self.h, ij, ij.size // 2, limit, out))
        return out

    def estimate_eps_mean(self, sample_pairs: int, seed: int) -> float:
        out = C.c_double()
        self._check(self.lib.knnj_eps_mean(self.h, sample_pairs, seed, C.byref(out)))
        return out.value

    def build_distance_histogram(self, eps_mean: float, n_bins: int, query_fraction: float,
                                 seed: int):
        raw = np.zeros(n_bins, np.uint64)
        qc = C.c_uint64()
        self._check(self.lib.knnj_histogram(self.h, eps_mean, n_bins, query_fraction, seed, raw,
                                            C.byref(qc)))
        return raw, qc.value

    def histogram_queries(self, qids, eps_mean: float, n_bins: int, raw=None):
        q = np.ascontiguousarray(qids, np.uint64)
        raw = np.zeros(n_bins, np.uint64) if raw is None else raw
        self._check(self.lib.knnj_histogram_queries(self.h, q, q.size, eps_mean, n_bins, raw))
        return raw

    def histogram_queries_capped(self, qids, eps_mean: float, n_bins: int, n_count: int):
        """Test hook: the capped histogram's kernels, counting bins [0, n_count) only."""
        q = np.ascontiguousarray(qids, np.uint64)
        raw = np.zeros(n_bins, np.uint64)
        self._check(self.lib.knnj_histogram_queries_capped(self.h, q, q.size, eps_mean, n_bins,
                                                           n_count, raw))
        return raw

    def grid_build(self, m: int, eps: float) -> dict:
        gi = _capi.GridInfo()
        self._check(self.lib.knnj_grid_build(self.h, m, eps, C.byref(gi)))
        return dict(m=gi.m, eps=gi.eps, n_cells=gi.n_cells, mins=np.array(gi.mins[:m]),
                    maxs=np.array(gi.maxs[:m]),
                    cells_per_dim=np.array(gi.cells_per_dim[:m], np.uint64))

    def grid_export(self, n_cells: int) -> dict:
        B = np.zeros(n_cells, np.uint64)
        G = np.zeros(2 * n_cells, np.uint64)
        A = np.zeros(self.N, np.uint32)
        slot = np.zeros(self.N, np.uint32)
        p = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
        self._check(self.lib.knnj_grid_export(self.h, p(B), p(G), p(A), p(slot)))
        return dict(B=B, G=G.reshape(n_cells, 2), A=A, slot=slot)

    def range_count(self, queries):
        q = np.ascontiguousarray(queries, np.uint32)
        ine = np.zeros(q.size, np.uint64)
        cand = np.zeros(q.size, np.uint64)
        self._check(self.lib.knnj_range_count(self.h, q, q.size, ine, cand))
        return ine, cand

    def split_work(self, queries, k: int, beta: float, gamma: float, rho: float) -> dict:
        q = np.ascontiguousarray(queries, np.uint32)
        dense = np.zeros(q.size, np.uint8)
        pop = np.zeros(q.size, np.uint64)
        si = _capi.SplitInfo()
        self._check(self.lib.knnj_split(self.h, q, q.size, k, beta, gamma, rho, dense, pop,
                                        C.byref(si)))
        return dict(is_dense=dense, cell_population=pop, n_min=si.n_min, n_thresh=si.n_thresh,
                    q_gpu=si.q_gpu, q_cpu=si.q_cpu, demoted=si.demoted)

    def dense_join(self, queries, k: int):
        q = np.ascontiguousarray(queries, np.uint32)
        ids = np.zeros(q.size * k, np.uint32)
        dist = np.zeros(q.size * k, np.float64)
        solved = np.zeros(q.size, np.uint8)
        st = _capi.JoinStats()
        self._check(self.lib.knnj_dense_join(self.h, q, q.size, k, ids, dist, solved,
                                             C.byref(st)))
        return (ids.reshape(q.size, k), dist.reshape(q.size, k), solved.astype(bool),
                dict(candidates_examined=st.candidates_examined, solved=st.solved,
                     failed=st.failed, kernel_ms=st.kernel_ms))

    def exact_knn(self, queries, k: int):
        q = np.ascontiguousarray(queries, np.uint32)
        ids = np.zeros(q.size * k, np.uint32)
        dist = np.zeros(q.size * k, np.float64)
        self._check(self.lib.knnj_exact_knn(self.h, q, q.size, k, ids, dist))
        return ids.reshape(q.size, k), dist.reshape(q.size, k)

    # ------------------------------------------------------------- pipeline
    def run(self, cfg: RunConfig, out=None, want_hist: bool = True,
            shard: Optional[tuple] = None) -> KnnRunResult:
        """run_hybrid (orchestrator.cpp:67-250) over the points set by set_points.

        ``out`` may supply preallocated (ids, dist, prov) host buffers (e.g. pinned).
        ``shard = (index, count, allreduce)`` runs this GPU's share of a multi-GPU job
        (knnj_run_shard): ``allreduce(a)`` must sum the uint64 array ``a`` in place over
        all shards (see distributed.py); the result then holds this shard's queries only.
        """
        N = self.N
        sub = None
        nsub = 0
        if cfg.query_subset is not None:
            sub_arr = np.ascontiguousarray(cfg.query_subset, np.uint32)
            sub = sub_arr.ctypes.data_as(C.POINTER(C.c_uint32))
            nsub = sub_arr.size
            queries = np.unique(sub_arr)
        else:
            queries = None
        mode = MODE_NAMES[cfg.mode] if isinstance(cfg.mode, str) else int(cfg.mode)
        c = _capi.Config(cfg.k, cfg.m, cfg.beta, cfg.gamma, cfg.rho, mode, cfg.n_bins,
                         cfg.hist_query_fraction, cfg.eps_mean_pair_cap, cfg.seed, sub, nsub)
        nq = N if queries is None else queries.size
        k_eff = min(cfg.k, N - 1)
        if out is None:
            ids = np.zeros(max(nq * k_eff, 1), np.uint32)
            dist = np.zeros(max(nq * k_eff, 1), np.float64)
            prov = np.zeros(max(nq, 1), np.uint8)
            ptrs = (ids.ctypes.data, dist.ctypes.data, prov.ctypes.data)
        else:
            ids, dist, prov = out
            ptrs = tuple(x.ctypes.data if hasattr(x, "ctypes") else x for x in out)
        raw = np.zeros(cfg.n_bins, np.uint64) if want_hist else None
        rawp = raw.ctypes.data_as(C.c_void_p) if raw is not None else None
        info = _capi.RunInfo()
        owned = None
        if shard is None:
            self._check(self.lib.knnj_run(self.h, C.byref(c), C.c_void_p(ptrs[0]),
                                          C.c_void_p(ptrs[1]), C.c_void_p(ptrs[2]), rawp,
                                          C.byref(info)))
        else:
            index, count, reduce = shard
            owned = np.zeros(max(nq, 1), np.uint32)

            def _cb(ptr, n, _user):
                try:
                    reduce(np.ctypeslib.as_array(ptr, shape=(int(n),)))
                    return 0
                except Exception:  # noqa: BLE001 - reported as a CUDA-class failure
                    return 1
            cb = _capi.ALLREDUCE_FN(_cb)
            self._check(self.lib.knnj_run_shard(self.h, C.byref(c), index, count, cb, None,
                                                C.c_void_p(ptrs[0]), C.c_void_p(ptrs[1]),
                                                C.c_void_p(ptrs[2]), C.c_void_p(owned.ctypes.data),
                                                rawp, C.byref(info)))
        d = {f: getattr(info, f) for f, _ in _capi.RUN_INFO_FIELDS if f != "perm"}
        d["perm"] = np.array(info.perm[:self.n], np.uint32)
        warnings = []
        if info.k_clamped:
            warnings.append(f"k clamped to |D|-1 = {k_eff}")
        if info.eps_fallback:
            warnings.append("beta target unreachable within eps_mean; clamped to the histogram maximum")
        if queries is None:
            # every point is a query: one read-only 0..N-1 array per point set (a fresh
            # 4N-byte array per run costs the host ~50 ms at 100M points)
            if self._all_queries is None or self._all_queries.size != N:
                self._all_queries = np.arange(N, dtype=np.uint32)
                self._all_queries.flags.writeable = False
            queries = self._all_queries
        rows = nq
        if owned is not None:
            rows = int(info.n_owned)
            queries = owned[:rows]
        if out is None:
            ids = ids[:rows * k_eff].reshape(rows, k_eff)
            dist = dist[:rows * k_eff].reshape(rows, k_eff)
            prov = prov[:rows]
        return KnnRunResult(queries=queries, ids=ids, dist=dist, provenance=prov,
                            k_effective=k_eff, info=d, raw_hist=raw, warnings=warnings)


@dataclasses.dataclass
class CandidateOutcome:
    """CandidateOutcome, proj/include/knnjoin/orchestrator.hpp:96-102."""
    beta: float
    gamma: float
    wall_seconds: float
    error: str = ""
    t1: Optional[float] = None       # the reference's CPU load-balance model: no analogue
    t2: Optional[float] = None


@dataclasses.dataclass
class ParameterSearchResult:
    """ParameterSearchResult, proj/include/knnjoin/orchestrator.hpp:104-110."""
    best_beta: float
    best_gamma: float
    candidates: list
    t1: Optional[float] = None
    t2: Optional[float] = None
    rho_model: Optional[float] = None


def parameter_search(engine, k: int, f: float, candidates, base: Optional[RunConfig] = None
                     ) -> ParameterSearchResult:
    """parameter_search (proj/src/orchestrator.cpp:252-303) through knnj_parameter_search:
    each (beta, gamma) candidate runs hybrid at rho = 0.5 over the same seeded f-fraction
    query subset; the fastest (device time) wins. Raises KnnjError like the reference's
    UsageError / SampleTooSmallError; a failing candidate keeps its message."""
    base = base or RunConfig(k=k)
    cand = list(candidates)
    betas = np.ascontiguousarray([b for b, _ in cand], np.float64)
    gammas = np.ascontiguousarray([g for _, g in cand], np.float64)
    mode = MODE_NAMES[base.mode] if isinstance(base.mode, str) else int(base.mode)
    c = _capi.Config(k, base.m, base.beta, base.gamma, base.rho, mode, base.n_bins,
                     base.hist_query_fraction, base.eps_mean_pair_cap, base.seed, None, 0)
    rows = (_capi.SearchRow * max(len(cand), 1))()
    bb, bg = C.c_double(), C.c_double()
    engine._check(engine.lib.knnj_parameter_search(engine.h, C.byref(c), float(f), betas, gammas,
                                                   len(cand), rows, C.byref(bb), C.byref(bg)))
    out = [CandidateOutcome(r.beta, r.gamma, r.wall_seconds, r.error.decode())
           for r in rows[:len(cand)]]
    return ParameterSearchResult(bb.value, bg.value, out)


def shard_range(cost, shard_index: int, shard_count: int) -> tuple:
    """knnj_shard_range: the contiguous item run [first, last) a shard owns (host-only)."""
    lib = _capi.load_library()
    a = np.ascontiguousarray(cost, np.float64)
    f, l = C.c_uint64(), C.c_uint64()
    rc = lib.knnj_shard_range(a, a.size, shard_index, shard_count, C.byref(f), C.byref(l))
    if rc:
        raise KnnjError(rc, "invalid shard_range arguments")
    return int(f.value), int(l.value)


def run_hybrid(X, cfg: RunConfig, device: int = 0) -> KnnRunResult:
    """One-shot run_hybrid(Dataset, RunConfig) on a fresh context."""
    eng = Engine(device)
    try:
        eng.set_points(X)
        return eng.run(cfg)
    finally:
        eng.close()


def tsv_bytes(r: KnnRunResult, threads: int = 0) -> bytes:
    """io::tsv_string (proj/src/io.cpp:141-154) through the native multi-threaded
    formatter (knnj_tsv_format): byte-identical to ``tsv_string``."""
    lib = _capi.load_library()
    q = np.ascontiguousarray(r.queries, np.uint32)
    ids = np.ascontiguousarray(r.ids, np.uint32)
    dist = np.ascontiguousarray(r.dist, np.float64)
    n = C.c_uint64()
    k = ids.shape[1] if ids.ndim == 2 else 0
    args = (q.ctypes.data, ids.ctypes.data, dist.ctypes.data, q.size, k)
    if lib.knnj_tsv_format(*args, None, 0, C.byref(n), threads):
        raise KnnjError(1, lib.knnj_io_last_error().decode())
    buf = C.create_string_buffer(max(1, n.value))
    if lib.knnj_tsv_format(*args, buf, n.value, C.byref(n), threads):
        raise KnnjError(1, lib.knnj_io_last_error().decode())
    return buf.raw[:n.value]


def write_tsv(path: str, r: KnnRunResult, threads: int = 0) -> int:
    """write_tsv (proj/src/io.cpp:137-139), formatted and written in parallel."""
    lib = _capi.load_library()
    q = np.ascontiguousarray(r.queries, np.uint32)
    ids = np.ascontiguousarray(r.ids, np.uint32)
    dist = np.ascontiguousarray(r.dist, np.float64)
    k = ids.shape[1] if ids.ndim == 2 else 0
    n = C.c_uint64()
    rc = lib.knnj_tsv_write(path.encode(), q.ctypes.data, ids.ctypes.data, dist.ctypes.data,
                            q.size, k, threads, C.byref(n))
    if rc:
        raise KnnjError(rc, lib.knnj_io_last_error().decode())
    return n.value


def read_binary_f64(path: str, out=None) -> np.ndarray:
    """ingest_binary (proj/src/io.cpp:69-91): |D| x n float64 (into ``out`` if given,
    e.g. a pinned buffer); IngestError-kind failures carry the reference messages."""
    lib = _capi.load_library()
    N, n = C.c_uint64(), C.c_uint64()
    rc = lib.knnj_binary_header(path.encode(), C.byref(N), C.byref(n))
    if rc:
        raise KnnjError(rc, lib.knnj_io_last_error().decode())
    X = np.empty((N.value, n.value), np.float64) if out is None else out
    rc = lib.knnj_binary_read(path.encode(), X.ctypes.data, X.size)
    if rc:
        raise KnnjError(rc, lib.knnj_io_last_error().decode())
    return X


def read_text(path: str, sep: str = ",", threads: int = 0, out=None) -> np.ndarray:
    """ingest_text (proj/src/io.cpp:24-67): CSV (sep ',') or TSV (sep '\\t') into a
    |D| x n float64 array (``out`` if given, e.g. a pinned buffer), parsed by ``threads``
    host threads; IngestError-kind failures carry the reference messages."""
    lib = _capi.load_library()
    h, N, n = C.c_void_p(), C.c_uint64(), C.c_uint64()
    rc = lib.knnj_text_parse(path.encode(), sep.encode(), threads, C.byref(h), C.byref(N),
                             C.byref(n))
    if rc:
        raise KnnjError(rc, lib.knnj_io_last_error().decode())
    try:
        X = np.empty((N.value, n.value), np.float64) if out is None else out
        rc = lib.knnj_text_copy(h, X.ctypes.data, X.size)
        if rc:
            raise KnnjError(rc, lib.knnj_io_last_error().decode())
    finally:
        lib.knnj_text_free(h)
    return X


def format_from_string(s: str) -> str:
    """format_from_string (proj/src/io.cpp:15-20)."""
    if s in ("csv", "tsv"):
        return s
    if s in ("bin", "binary-f64"):
        return "bin"
    raise KnnjError(1, f"unknown dataset format '{s}' (expected csv, tsv, or bin)")


def ingest_dataset(path: str, fmt: str = "bin", threads: int = 0, out=None) -> np.ndarray:
    """ingest_dataset (proj/src/io.cpp:99-106): csv, tsv or binary-f64."""
    f = format_from_string(fmt)
    if f == "bin":
        return read_binary_f64(path, out)
    return read_text(path, "," if f == "csv" else "\t", threads, out)
