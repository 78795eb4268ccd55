"""Small runs of every device kernel family for compute-sanitizer (memcheck, racecheck,
synccheck): the tcgen05 join + histogram (18-D clustered, 90-D wide operands), the SIMT
join (forced, and 2-D / 6-D skewed data where the precision rule picks it), the grid
histogram (n <= 8), the exact fallback levels and the split-item merge. Each run is
checked against the CPU oracle so a sanitizer-clean run is also a correct one.

  compute-sanitizer --tool racecheck python tools/sanitize_run.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.oracle import Oracle  # noqa: E402  (the checker)
from paper_1810_04758_b200 import Engine, RunConfig  # noqa: E402
from paper_1810_04758_b200.synthetic import generate  # noqa: E402

CASES = [  # (spec, N, n, K, options)
    ("clusters:16:0.05", 6000, 18, 32, {}),
    ("clusters:16:0.05", 4000, 18, 32, {"tensor_cores": 0}),
    ("mixture", 3000, 90, 16, {}),
    ("exponential", 8000, 6, 64, {"hist_grid": 2, "hist_cap": 2}),
    ("uniform", 12000, 4, 32, {"hist_grid": 2, "hist_cap": 2}),
    ("uniform", 5000, 2, 5, {}),
]
ora = Oracle()
bad = 0
for spec, N, n, k, opts in CASES:
    X = generate(spec, N, n, seed=3)
    eng = Engine(0)
    for o, v in opts.items():
        eng.set_option(o, v)
    eng.set_points(X)
    r = eng.run(RunConfig(k=k, mode="hybrid", seed=1))
    o = ora.run(X, k=k, mode="hybrid", seed=1)
    ok = np.array_equal(r.ids, o["ids"]) and np.array_equal(r.dist, o["dist"])
    bad += not ok
    print(f"{spec} N={N} n={n} K={k} {opts}: {'ok' if ok else 'MISMATCH'} "
          f"tc={r.info['join_tensor_cores']} fallback={r.info['fallback_queries']}", flush=True)
    eng.close()
sys.exit(1 if bad else 0)
