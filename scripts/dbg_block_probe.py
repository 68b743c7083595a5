import sys, os, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from tests.helpers import small_spec, gpu_context
from synth.generate import make_problem
name, dims, sk = sys.argv[1], eval(sys.argv[2]), eval(sys.argv[3])
spec = small_spec(name, dims, sk)
prob = make_problem(spec)
ctx = gpu_context(prob, packed=True)
for k in range(len(dims)):
    t0=time.time(); g = ctx.block_probe(0, k); torch.cuda.synchronize()
    print("block", k, "ok", time.time()-t0, flush=True)
print("sweep", ctx.sweep(1)[0]["n_obs"], flush=True)
