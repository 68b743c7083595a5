"""debug: sigma per sweep of the MAD rule, GPU vs oracle (C1 small)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import trd_oracle as O
from synth.generate import make_problem
from tests.helpers import small_spec, oracle_source, oracle_config, gpu_context
for name, dims, sk in [("C1", [32, 32, 32], None), ("C4", [16, 16, 16, 16], [8, 8, 8, 8])]:
    spec = small_spec(name, dims, sk)
    prob = make_problem(spec)
    src, _ = oracle_source(prob)
    st, recs = O.run(oracle_config(spec, sigma_mode=O.SIGMA_MAD), prob.init, src, 3)
    ctx = gpu_context(prob, packed=True, sigma_mode=O.SIGMA_MAD)
    g = ctx.sweep(3)
    print(name, os.environ.get("TRD_NO_PERM"), [(round(x["sigma"], 6), round(r.sigma, 6), x["n_obs"], r.n_obs) for x, r in zip(g, recs)])
    ctx.close()
