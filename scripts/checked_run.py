"""Driver of tests/test_gpu_checked.py (one process per library / jitter setting): runs the
cases below through the library TRD_LIB_PATH points at and saves cores and sweep records to an
npz.  usage: checked_run.py OUT.npz [case ...]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("TRD_GRAPH", "0")

from paper_2305_09044_b200 import TRD                             # noqa: E402
from paper_2305_09044_b200.trd import TRD_SAMPLING_ROWS           # noqa: E402
from synth.generate import CONFIGS, make_problem, scaled_spec     # noqa: E402

# name -> (config, dims, sketch, spec overrides, context overrides)
CASES = {
    "rsts4": ("C4", [16, 12, 10, 8], [8, 6, 5, 4], {}, {}),
    "mad3": ("C1", [24, 20, 16], None, {}, {"sigma_mode": 3}),
    "full5": ("C5b", [10, 9, 8, 7, 6], None, {}, {}),
    "dense": ("C2", [140, 70, 3], None, {"observed": 1.0}, {}),        # rho = 1: full tiles, odd row tiles
    "sparse": ("C4", [40, 30, 20, 10], [0, 0, 0, 0], {"observed": 0.002}, {}),  # mostly empty tiles
    "rows": ("C4", [16, 12, 10, 8], [8, 6, 5, 4], {}, {"sampling": TRD_SAMPLING_ROWS}),
}


def run(case):
    cfg, dims, sk, spec_over, ctx_over = CASES[case]
    spec = scaled_spec(CONFIGS[cfg], dims, sketch=sk)
    for k, v in spec_over.items():
        setattr(spec, k, v)
    prob = make_problem(spec)
    kw = dict(sigma_mode=spec.sigma_mode, sketch=spec.sketch, seed=spec.sampler_seed)
    kw.update(ctx_over)
    ctx = TRD(spec.dims, spec.ranks, prob.packed_values().cuda(), prob.mask.cuda(), prob.init, packed=True, **kw)
    recs = ctx.sweep(2)
    probe = ctx.block_probe(2, 1)
    cores = ctx.get_cores()
    ctx.close()
    out = {f"{case}_core{k}": c for k, c in enumerate(cores)}
    out[f"{case}_sigma"] = np.array([r["sigma"] for r in recs])
    out[f"{case}_eta"] = np.array([r["eta"] for r in recs])
    out[f"{case}_d"] = probe["d"]
    out[f"{case}_den"] = np.array([probe["den"]])
    return out


if __name__ == "__main__":
    dst = sys.argv[1]
    cases = sys.argv[2:] or list(CASES)
    res = {}
    for c in cases:
        res.update(run(c))
    np.savez(dst, **res)
    print(f"checked_run: {len(cases)} cases ok ({os.environ.get('TRD_LIB_PATH', 'libtrd.so')}, "
          f"jitter {os.environ.get('TRD_JITTER_NS', '0')} ns)", flush=True)
