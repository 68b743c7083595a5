"""Tiny sweeps of the whole path (pass kernels, staging, sampler, solve, MAD select) for
profiler checks, e.g. the NVTX ranges (scripts/gpu_nvtx.sh).  usage (GPU box):
  python scripts/tiny_sweep.py [C4|C1|C5]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("TRD_GRAPH", "0")

from paper_2305_09044_b200 import TRD            # noqa: E402
from synth.generate import make_problem, scaled_spec, CONFIGS   # noqa: E402

CASES = {
    "C4": ([16, 12, 10, 8], [8, 6, 5, 4], {}),                 # RStS, order 4
    "C1": ([24, 20, 16], None, {"sigma_mode": 3}),             # full sets, exact-median sigma
    "C5": ([10, 9, 8, 7, 6], None, {}),                        # order 5, full working set
}


def main(name):
    dims, sk, over = CASES[name]
    spec = scaled_spec(CONFIGS[name if name != "C5" else "C5b"], dims, sketch=sk)
    prob = make_problem(spec)
    kw = dict(sigma_mode=spec.sigma_mode, sketch=spec.sketch, seed=spec.sampler_seed)
    kw.update(over)
    ctx = TRD(spec.dims, spec.ranks, prob.packed_values().cuda(), prob.mask.cuda(), prob.init, packed=True, **kw)
    recs = ctx.sweep(2)
    ctx.get_cores()
    ctx.close()
    print(f"tiny_sweep {name}: sigma {[round(r['sigma'], 6) for r in recs]} n_obs {recs[-1]['n_obs']}", flush=True)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "C4")
