import sys, os, numpy as np
sys.path.insert(0, os.getcwd())
from paper_1810_04758_b200 import Engine, RunConfig
from paper_1810_04758_b200.synthetic import CONFIGS, generate
for cname in sys.argv[1:]:
    c = CONFIGS[cname]; N = c["size"]
    X = generate(c["spec"], N, c["dims"], seed=1)
    eng = Engine(0); eng.set_points(X)
    r = eng.run(RunConfig(k=c["k"], mode="hybrid", seed=1))
    eps = r.eps_used
    kth = np.sqrt(np.asarray(r.dist)[:, c["k"]-1]) if False else np.asarray(r.dist)[:, c["k"]-1]
    ratio = kth / eps
    qs = np.quantile(ratio, [0.01, 0.1, 0.25, 0.5, 0.75, 0.9, 0.99])
    print(cname, "eps", eps, "m", r.info.get("m_used"), "kth/eps quantiles", np.round(qs, 3))
    for f in (0.25, 0.35, 0.5, 0.7, 1.0):
        print("  frac kth < %.2f eps: %.3f" % (f, (ratio < f).mean()))
