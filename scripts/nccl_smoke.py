"""NCCL world > 1 smoke for a multi-GPU node (one rank per GPU; not runnable on the one-GPU
gpurun boxes): every rank holds its mode-0 slab of a C4-shaped problem, runs sweeps through the
library's NCCL exchange, and the ranks compare their cores bit for bit and against a world-1
context holding the whole tensor (same oracle tolerance as the tests: 1e-4).

  torchrun --standalone --nproc-per-node 2 scripts/nccl_smoke.py [--config C4] [--sweeps 3]
"""
import argparse
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--sweeps", type=int, default=3)
    args = ap.parse_args()
    import bench
    from paper_2305_09044_b200 import TRD, nccl_unique_id
    from synth.generate import CONFIGS, make_problem, scaled_spec

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    spec = scaled_spec(CONFIGS[args.config], [32, 24, 20, 16], sketch=[16, 12, 10, 8])
    prob = make_problem(spec, device="cuda", keep_mask_bool=True)
    (b, e), vals, words, _ = bench.local_shard(prob, rank, world)
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    kw = dict(sigma_mode=spec.sigma_mode, sketch=spec.sketch, seed=spec.sampler_seed, packed=True)
    ctx = TRD(spec.dims, spec.ranks, vals, words, prob.init, shard_mode=0, shard_range=(b, e),
              world=world, rank=rank, nccl_id=obj[0], **kw)
    recs = ctx.sweep(args.sweeps)
    cores = ctx.get_cores()
    ctx.close()
    assert all(r["replica_mismatch"] == 0 for r in recs)
    flat = torch.from_numpy(np.concatenate([c.ravel() for c in cores])).cuda()
    gathered = [torch.empty_like(flat) for _ in range(world)]
    dist.all_gather(gathered, flat)
    same = all(torch.equal(gathered[0], g) for g in gathered)
    if rank == 0:
        one = TRD(spec.dims, spec.ranks, prob.X[prob.mask_bool].contiguous(), prob.mask, prob.init, **kw)
        one.sweep(args.sweeps, stats=False)
        ref = one.get_cores()
        one.close()
        err = max(float(np.linalg.norm(a - r) / np.linalg.norm(r)) for a, r in zip(cores, ref))
        print(f"nccl smoke: world {world}, replicas bitwise equal: {same}, cores vs world 1: {err:.2e}, "
              f"sigma per sweep {[round(r['sigma'], 6) for r in recs]}", flush=True)
        assert same and err <= 1e-4
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
