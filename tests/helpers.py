"""Shared helpers of the parity tests: one seeded Problem feeds both the oracle and libtrd."""
import numpy as np
import torch

from oracle import trd_oracle as O
from synth.generate import CONFIGS, ProblemSpec, make_problem, scaled_spec, to_numpy_views


def small_spec(name, dims, sketch=None, **over):
    s = scaled_spec(CONFIGS[name], dims, sketch=sketch)
    for k, v in over.items():
        setattr(s, k, v)
    return s


def oracle_config(spec: ProblemSpec, **over):
    kw = dict(sigma_mode=spec.sigma_mode, sketch=spec.sketch, seed=spec.sampler_seed)
    kw.update(over)
    return O.Config(spec.dims, spec.ranks, **kw)


def gpu_context(prob, packed=False, host=False, **over):
    from paper_2305_09044_b200 import TRD
    spec = prob.spec
    if packed:
        vals = prob.packed_values()
    else:
        vals = prob.X
    mask = prob.mask
    if host:
        vals = vals.cpu().pin_memory()
        mask = mask.cpu().pin_memory()
    else:
        vals = vals.cuda()
        mask = mask.cuda()
    kw = dict(sigma_mode=spec.sigma_mode, sketch=spec.sketch, seed=spec.sampler_seed)
    kw.update(over)
    return TRD(spec.dims, spec.ranks, vals, mask, prob.init, packed=packed, host=host, **kw)


def rel_fro(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def cores_rel_err(gpu_cores, oracle_cores):
    return max(rel_fro(g, o) for g, o in zip(gpu_cores, oracle_cores))


def oracle_source(prob):
    X, P, Xc = to_numpy_views(prob)
    return O.DenseSource(X, P), Xc
