"""Per-step phase timings of knnj_run on a BASELINE config (dev tool).

  python tools/probe_steps.py [--config C2] [--size N] [--steps 6] [--hist]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_04758_b200 import Engine, RunConfig  # noqa: E402
from paper_1810_04758_b200.synthetic import CONFIGS, generate  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--size", type=int, default=0)
ap.add_argument("--steps", type=int, default=6)
ap.add_argument("--hist", action="store_true")
ap.add_argument("--opt", action="append", default=[], help="name=value engine option")
ap.add_argument("--pinned", action="store_true", help="results into pinned host buffers (e2e path)")
a = ap.parse_args()
c = dict(CONFIGS[a.config])
N = a.size or c["size"]
X = generate(c["spec"], N, c["dims"], seed=1)
eng = Engine(0)
for o in a.opt:
    k, v = o.split("=")
    eng.set_option(k, int(v))
eng.set_points(X)
keys = ["ms_total", "ms_download", "ms_eps_mean", "ms_histogram", "ms_hist_kernel", "ms_grid", "ms_join_build",
        "ms_join", "ms_join_kernel", "ms_fallback", "fallback_queries", "fallback_passes",
        "slow_path_queries", "failed_count", "q_cpu", "hist_bins_counted", "join_candidate_pairs", "join_screened_pairs",
        "kth_bound2", "bound_retried", "eps_used"]
out = (0, 0, 0)
if a.pinned:
    out = (eng.lib.knnj_alloc_pinned(N * c["k"] * 4), eng.lib.knnj_alloc_pinned(N * c["k"] * 8),
           eng.lib.knnj_alloc_pinned(N))
for st in range(a.steps):
    t = time.time()
    r = eng.run(RunConfig(k=c["k"], mode="hybrid", seed=1), out=out, want_hist=a.hist)
    w = time.time() - t
    i = r.info
    print(f"[{a.config} N={N} step {st}] wall={w*1e3:.1f}ms " +
          " ".join(f"{k}={i[k]:.4g}" if isinstance(i[k], float) else f"{k}={i[k]}" for k in keys),
          flush=True)
