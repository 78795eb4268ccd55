"""One small knnj_run (dev aid for debugger runs)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_04758_b200 import Engine, RunConfig  # noqa: E402
from paper_1810_04758_b200.synthetic import generate  # noqa: E402

spec, N, n, k = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
X = generate(spec, N, n, 61)
eng = Engine(0)
for o in sys.argv[5:]:
    a, b = o.split("=")
    eng.set_option(a, int(b))
eng.set_points(X)
r = eng.run(RunConfig(k=k, mode="hybrid", seed=61), want_hist=False)
print("ok", r.info["eps_used"], r.info["join_tensor_cores"])
