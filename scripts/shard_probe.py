"""Per-rank sweep time of the data-parallel plans, measured on one GPU: a world-1 context that
holds only rank r's slab i_0 in [b, e) of the C5b workload (no NCCL), for world = 1, 2, 4, 8."""
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import bench  # noqa: E402
from synth.generate import CONFIGS  # noqa: E402
from paper_2305_09044_b200.trd import TRD  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5b"
spec = CONFIGS[cfg]
prob = bench.make_workload(spec, "cuda")
for world in (1, 2, 4, 8):
    (b, e), vals, words, _ = bench.local_shard(prob, 0, world)
    ctx = TRD(spec.dims, spec.ranks, vals, words, prob.init, sigma_mode=spec.sigma_mode, sketch=spec.sketch,
              seed=spec.sampler_seed, shard_mode=0, shard_range=(b, e), world=1, rank=0, packed=True)
    ctx.sweep(2, stats=False)
    torch.cuda.synchronize()
    r = ctx.sweep(3, stats=True)
    ms = sum(x["ms"] for x in r) / 3
    print(f"world {world}: rank-0 slab i_0 in [{b}, {e}): {ms:.2f} ms/sweep, {r[0]['n_obs']} entries/sweep")
    ctx.close()
    del vals, words
    torch.cuda.empty_cache()
