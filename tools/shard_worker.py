"""One rank of a multi-process sharded run (launched by torchrun; used by
tests/test_gpu_multiprocess.py): knnj_run_shard over this rank's contiguous cell range,
the histogram counts summed through torch.distributed, the rank's rows saved to
<out>/rank<r>.npz. KNNJ_DIST_BACKEND=gloo puts every rank on the visible GPUs
round-robin (a multi-rank check on a 1-GPU box)."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--spec", default="clusters:16:0.05")
    ap.add_argument("--size", type=int, default=20000)
    ap.add_argument("--dims", type=int, default=18)
    ap.add_argument("--k", type=int, default=16)
    ap.add_argument("--seed", type=int, default=3)
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    import torch
    import torch.distributed as dist

    from paper_1810_04758_b200 import Engine, RunConfig
    from paper_1810_04758_b200.distributed import torch_allreduce
    from paper_1810_04758_b200.synthetic import generate
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    backend = os.environ.get("KNNJ_DIST_BACKEND", "nccl")
    local = int(os.environ.get("LOCAL_RANK", rank)) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group(backend)
    X = generate(a.spec, a.size, a.dims, seed=a.seed)
    eng = Engine(local)
    eng.set_points(X)
    r = eng.run(RunConfig(k=a.k, mode="hybrid", seed=a.seed), want_hist=False,
                shard=(rank, world, torch_allreduce()))
    np.savez(os.path.join(a.out, f"rank{rank}.npz"), q=r.queries, ids=r.ids, dist=r.dist,
             prov=r.provenance, eps=r.info["eps_used"], failed=r.info["failed_count"])
    eng.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
