"""Break the end-to-end step (bench.py e2e) into H2D upload, staging + sweep, and the sum."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import bench  # noqa: E402
from paper_2305_09044_b200.trd import TRD  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5b"
from synth.generate import CONFIGS  # noqa: E402
spec = CONFIGS[cfg]
prob = bench.make_workload(spec, "cuda")
(b, e), vals, words, Ml = bench.local_shard(prob, 0, 1)
kw = dict(sigma_mode=spec.sigma_mode, sketch=spec.sketch, seed=spec.sampler_seed, shard_mode=0,
          shard_range=(b, e), world=1, rank=0, nccl_id=None, packed=True)
vals_h = vals.cpu().pin_memory()
words_h = words.cpu().pin_memory()
print("pinned:", vals_h.is_pinned(), words_h.is_pinned(), "bytes", vals_h.numel() * 4 + words_h.numel() * 4)
ctx = TRD(spec.dims, spec.ranks, vals_h, words_h, prob.init, host=True, **kw)
ctx.sweep(1, stats=False)
torch.cuda.synchronize()
s = torch.cuda.current_stream()


def timed(fn, n=3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(n):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


def host_ms(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    return (t1 - t0) * 1e3, (t2 - t0) * 1e3


for st in (False, True, False, True):
    print("sweep stats=%d host enqueue %.2f ms, host total %.2f ms" % ((st,) + host_ms(lambda: ctx.sweep(1, stats=st))))
for i in range(4):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(s)
    ctx.sweep(1, stats=True)
    t1 = time.perf_counter()
    e1.record(s)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print("call %d: wall %.2f ms, wall+sync %.2f ms, events %.2f ms" % (i, (t1 - t0) * 1e3, (t2 - t0) * 1e3,
                                                                     e0.elapsed_time(e1)))
print("sweep (cached)   %.2f ms" % timed(lambda: ctx.sweep(1, stats=True)))
print("sweep x3 / 3     %.2f ms" % timed(lambda: ctx.sweep(3, stats=True), n=1) + " (per 3)")
print("sweep no stats   %.2f ms" % timed(lambda: ctx.sweep(1, stats=False)))
print("upload + sweep   %.2f ms (copy in line)" % timed(lambda: (ctx.upload(vals_h, words_h), ctx.sweep(1, stats=True))))
x = torch.empty(vals_h.numel() + words_h.numel(), dtype=torch.float32, device="cuda")
h = torch.empty(x.numel(), dtype=torch.float32).pin_memory()
print("torch H2D copy   %.2f ms" % timed(lambda: x.copy_(h, non_blocking=True)))
ctx.set_profiling(True)
ctx.upload(vals_h, words_h)
ctx.sweep(1, stats=True)
torch.cuda.synchronize()
print(ctx.get_profile())
ctx.close()
