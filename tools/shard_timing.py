"""Per-shard phase times of an S-way sharded run, all shards on one GPU in turn (dev tool).

Approximates the per-GPU critical path of `bench.py --gpus S`: the histogram all-reduce
is replaced by scaling this shard's counts by S (timing only; outputs are not checked).

  python tools/shard_timing.py [--config C2] [--shards 8] [--steps 2]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_04758_b200 import Engine, RunConfig  # noqa: E402
from paper_1810_04758_b200.synthetic import CONFIGS, generate  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--shards", type=int, default=8)
ap.add_argument("--steps", type=int, default=2)
a = ap.parse_args()
c = CONFIGS[a.config]
X = generate(c["spec"], c["size"], c["dims"], seed=1)
eng = Engine(0)
eng.set_points(X)
keys = ["ms_total", "ms_reorder", "ms_eps_mean", "ms_histogram", "ms_grid", "ms_join_build", "ms_join",
        "ms_join_kernel", "ms_fallback", "n_owned"]


def scaled(arr):
    arr *= a.shards


for st in range(a.steps):
    worst = 0.0
    for sh in range(a.shards):
        r = eng.run(RunConfig(k=c["k"], mode="hybrid", seed=1), out=(0, 0, 0), want_hist=False,
                    shard=(sh, a.shards, scaled))
        i = r.info
        worst = max(worst, i["ms_total"])
        if st == a.steps - 1:
            print(f"shard {sh}/{a.shards} " + " ".join(
                f"{k}={i[k]:.1f}" if isinstance(i[k], float) else f"{k}={i[k]}" for k in keys), flush=True)
    print(f"step {st}: max ms_total over shards {worst:.1f}", flush=True)
