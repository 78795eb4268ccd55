"""Quick timing probe of knnj_run on BASELINE-shaped synthetic data (dev tool)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1810_04758_b200 import Engine, RunConfig
from paper_1810_04758_b200.synthetic import generate

cases = [a.split(",") for a in sys.argv[1:]] or [["clusters:16:0.05", "200000", "18", "32"]]
eng = Engine(0)
for spec, N, n, k in cases:
    N, n, k = int(N), int(n), int(k)
    t = time.time(); X = generate(spec, N, n, 1); tg = time.time() - t
    for rep in range(2):
        t = time.time()
        eng.set_points(X)
        r = eng.run(RunConfig(k=k, mode="hybrid", seed=1), want_hist=True)
        wall = time.time() - t
    i = r.info
    keys = ["eps_used", "grid_cells", "q_gpu", "failed_count", "candidates_examined", "fallback_queries",
            "fallback_passes", "slow_path_queries", "ms_reorder", "ms_eps_mean", "ms_histogram", "ms_hist_kernel",
            "ms_grid", "ms_split", "ms_join", "ms_join_kernel", "ms_fallback", "ms_download", "ms_total"]
    print(f"{spec} N={N} n={n} k={k} gen={tg:.1f}s wall={wall:.3f}s pts/s={N/wall:.3e}")
    print("   " + " ".join(f"{k}={i[k]:.4g}" if isinstance(i[k], float) else f"{k}={i[k]}" for k in keys))
    cand = i["candidates_examined"]
    if i["ms_join_kernel"] > 0:
        print(f"   join: {cand/i['ms_join_kernel']/1e6:.3f} Gpairs/s  ({cand/N:.0f} cand/q) "
              f"eff FP32 {3*n*cand/i['ms_join_kernel']/1e9:.2f} TFLOP/s(3n def)")
