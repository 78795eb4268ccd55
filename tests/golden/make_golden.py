"""Generate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref).

Run here (where /root/reference exists): ``make -C oracle ref && python
tests/golden/make_golden.py``. The fixtures are committed; the GPU box never
needs /root/reference. The reference runs with kernel "scalar" so its
distances are in the summation order the contract pins.
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import Ref  # noqa: E402
from paper_1810_04758_b200.synthetic import generate  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

# name, generator spec, |D|, n, run kwargs
CASES = [
    ("uniform2d", "uniform", 3000, 2, dict(k=5)),
    ("clusters18d", "clusters:16:0.05", 2500, 18, dict(k=32)),
    ("mixture90d", "mixture:8:0.05", 1200, 90, dict(k=16)),
    ("exp6d", "exponential", 4000, 6, dict(k=64)),
    ("uniform4d", "uniform", 5000, 4, dict(k=32)),
    ("mixture5d_rho", "mixture", 1500, 5, dict(k=6, beta=0.3, gamma=0.4, rho=0.25, seed=99)),
    ("clusters7d_m3", "clusters:4:0.1", 1800, 7, dict(k=10, m=3, beta=0.1, gamma=0.8)),
    ("uniform1d", "uniform", 700, 1, dict(k=9)),
]


def sheet() -> np.ndarray:
    """Acceptance C8's adversarial sheet (proj/tests/acceptance.cpp:263-303), drawn with numpy."""
    rng = np.random.default_rng(7)
    a = np.stack([rng.uniform(0, 100, 1300), 0.0001 * (np.arange(1300) % 7)], 1)
    b = np.stack([rng.uniform(0, 100, 700), rng.uniform(5, 63, 700)], 1)
    return np.concatenate([a, b])


def dups() -> np.ndarray:
    """Exact duplicates and equal-distance ties (test_sparse_engine.cpp:89-96 style)."""
    rng = np.random.default_rng(3)
    base = np.round(rng.random((300, 3)) * 4) / 4.0   # lattice: many equal distances
    return np.concatenate([base, base[:100]])           # plus exact duplicates


def main() -> None:
    ref = Ref()
    ref.set_kernel("scalar")
    cases = [(name, generate(spec, size, dims, seed=11 + i), kw)
             for i, (name, spec, size, dims, kw) in enumerate(CASES)]
    cases.append(("sheet_c8", sheet(), dict(k=5, m=1, seed=11, hist_frac=1.0)))
    cases.append(("lattice_dups", dups(), dict(k=7, seed=5)))
    for name, X, kw in cases:
        rec = {"X": X}
        kw = dict(kw)
        kw.setdefault("seed", 1)
        for key, val in kw.items():
            rec["cfg_" + key] = np.array(val)
        for mode in ("hybrid", "dense", "sparse", "oracle"):
            r = ref.run(X, mode=mode, workers=4, buffer_size=10**12, **kw)
            if mode == "hybrid":
                rec["ids"] = r["ids"]
                rec["dist"] = r["dist"]
            else:  # the reference's own cross-mode contract (test_orchestrator.cpp:42-63)
                assert (r["ids"] == rec["ids"]).all() and (r["dist"] == rec["dist"]).all(), mode
            rec[f"{mode}_prov"] = r["prov"]
            if mode in ("hybrid", "dense"):
                for f in ("eps_mean", "eps_used", "eps_default", "eps_beta", "bin_width",
                          "hist_query_count", "q_gpu", "q_cpu", "demoted", "failed_count",
                          "n_min", "n_thresh", "candidates_examined"):
                    rec[f"{mode}_{f}"] = np.array(r[f])
                rec[f"{mode}_hist_counts"] = r["hist_counts"]
                rec[f"{mode}_perm"] = r["perm"]
        # phase-level vectors on the reordered dataset
        perm, var = ref.variance_order(X)
        W = np.ascontiguousarray(X[:, perm])
        rec["perm"] = perm
        rec["var"] = var
        m = kw.get("m", 0) or min(6, X.shape[1])
        eps = float(rec["dense_eps_used"])
        g = ref.grid(W, m, eps)
        for f in ("B", "G", "A", "cpd", "mins", "maxs"):
            rec[f"grid_{f}"] = g[f]
        q = np.arange(X.shape[0], dtype=np.uint32)
        cand, ine = ref.range_counts(W, m, eps, q)
        rec["range_candidates"] = cand
        rec["range_in_eps"] = ine
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **rec)
        print(name, X.shape, "eps", eps, "failed", int(rec["hybrid_failed_count"]))


if __name__ == "__main__":
    main()
