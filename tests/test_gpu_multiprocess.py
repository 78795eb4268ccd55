"""GPU: the sharded engine in separate processes, launched like bench.py's N-GPU path
(torchrun, one process per rank, knnj_run_shard, the eps histogram counts summed through
torch.distributed). On a 1-GPU box the ranks share cuda:0 over gloo. The ranks' rows,
merged by query id, must equal the single-process knnj_run output bit for bit
(shared-nothing ranks over contiguous cell ranges,
proj/src/sparse_engine.cpp:22-27's independent queries)."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from paper_1810_04758_b200 import Engine, RunConfig
from paper_1810_04758_b200.distributed import merge_shards
from paper_1810_04758_b200.synthetic import generate

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,spec,size,dims,k", [(2, "clusters:16:0.05", 20000, 18, 16),
                                                    (3, "uniform", 60000, 4, 32),
                                                    (2, "exponential", 40000, 6, 20)])
def test_torchrun_shards_merge_to_single_run(tmp_path, world, spec, size, dims, k):
    env = dict(os.environ, KNNJ_DIST_BACKEND="gloo", PYTHONPATH=ROOT)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr=127.0.0.1", f"--master-port={_port()}",
           os.path.join(ROOT, "tools", "shard_worker.py"), "--spec", spec, "--size", str(size),
           "--dims", str(dims), "--k", str(k), "--seed", "3", "--out", str(tmp_path)]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    parts, eps = [], set()
    for r in range(world):
        z = np.load(tmp_path / f"rank{r}.npz")
        parts.append((z["q"], z["ids"], z["dist"], z["prov"]))
        eps.add(float(z["eps"]))
    assert len(eps) == 1, "ranks selected different eps"
    q, ids, dist, prov = merge_shards(parts, size, k)
    X = generate(spec, size, dims, seed=3)
    eng = Engine(0)
    eng.set_points(X)
    ref = eng.run(RunConfig(k=k, mode="hybrid", seed=3), want_hist=False)
    eng.close()
    assert ref.info["eps_used"] in eps
    assert np.array_equal(q, np.arange(size, dtype=np.uint32))
    assert np.array_equal(ids, ref.ids) and np.array_equal(dist, ref.dist)
    assert np.array_equal(prov, ref.provenance)
