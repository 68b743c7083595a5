"""Full-size parity on every BASELINE config (-m gpu): the bench's storage and launch
configuration (packed values + bitmask, persistent CTA pairs) against the float64 oracle with
the entry-wise data source (oracle/entries.py: the per-entry sums of Eq. 7 / 9 / 12 in C, the
rest of Alg. 1 in numpy).  North-star bars: cores after one sweep within 1e-4 relative
Frobenius, final relative error within 1e-3 (absolute difference, reading R19), sampled
indices and observed counts exact.  Citations are PAPER.md lines (P:L)."""
import math

import numpy as np
import pytest
import torch

from oracle import trd_oracle as O
from oracle.entries import EntrySource
from synth.generate import CONFIGS, make_problem
from tests.helpers import cores_rel_err, rel_fro

pytestmark = pytest.mark.gpu


def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _setup(name):
    spec = CONFIGS[name]
    prob = make_problem(spec, device="cuda", keep_mask_bool=True)
    vals = prob.X[prob.mask_bool].contiguous()
    words = prob.mask
    src = EntrySource(spec.dims, words.cpu().numpy().view(np.uint32), vals.cpu().numpy(), True)
    assert src.n_obs == prob.n_obs
    return spec, prob, vals, words, src


def _ctx(spec, prob, vals, words, **over):
    from paper_2305_09044_b200 import TRD
    kw = dict(sigma_mode=spec.sigma_mode, sketch=spec.sketch, seed=spec.sampler_seed, packed=True)
    kw.update(over)
    return TRD(spec.dims, spec.ranks, vals, words, prob.init, **kw)


def _eval_subset(spec, n_eval, seed):
    """Evaluation entries for the relative error at full size (both sides use the same ones):
    n_eval distinct linear indices (or all entries when the tensor is smaller)."""
    n = spec.numel
    if n <= n_eval:
        return np.arange(n, dtype=np.int64)
    rng = np.random.default_rng(seed)
    return np.unique(rng.integers(0, n, size=n_eval, dtype=np.int64))


def _bits(lin, n):
    words = np.zeros((n + 31) // 32, dtype=np.uint32)
    np.bitwise_or.at(words, lin >> 5, (np.uint32(1) << (lin & 31).astype(np.uint32)))
    return torch.from_numpy(words.view(np.int32)).cuda()


@pytest.mark.parametrize("name", ["C2", "C3", "C4", "C5a"])
def test_full_size_cores_after_one_sweep(name):
    """Cores after one sweep (sigma_0 from all observed residuals, the RMS schedule, RStS
    sketches of the config), observed counts per block exact."""
    _cuda()
    spec, prob, vals, words, src = _setup(name)
    cfg = O.Config(spec.dims, spec.ranks, sigma_mode=spec.sigma_mode, sketch=spec.sketch, seed=spec.sampler_seed)
    st, recs = O.run(cfg, prob.init, src, 1)
    ctx = _ctx(spec, prob, vals, words)
    g = ctx.sweep(1)[0]
    assert abs(g["sigma"] - recs[0].sigma) <= 1e-6 * recs[0].sigma
    for k in range(spec.order):
        assert g["nnz"][k] == recs[0].nnz[k], k
    err = cores_rel_err(ctx.get_cores(), st.cores)
    ctx.close()
    assert err <= 1e-4, err


@pytest.mark.parametrize("name", ["C2", "C3", "C4"])
def test_full_size_final_error(name):
    """Final relative reconstruction error after the config's 20 sweeps, over a shared
    evaluation subset (all entries for C2), within 1e-3 of the oracle's."""
    _cuda()
    spec, prob, vals, words, src = _setup(name)
    cfg = O.Config(spec.dims, spec.ranks, sigma_mode=spec.sigma_mode, sketch=spec.sketch, seed=spec.sampler_seed)
    st, _ = O.run(cfg, prob.init, src, spec.sweeps)
    lin = _eval_subset(spec, 1 << 21, 7)
    xc = prob.X_clean[torch.from_numpy(lin).cuda()].double().cpu().numpy()
    xo = src.reconstruct(st.cores, spec.ranks, lin)
    e_or = float(np.linalg.norm(xo - xc) / np.linalg.norm(xc))
    ctx = _ctx(spec, prob, vals, words)
    ctx.sweep(spec.sweeps, stats=False)
    g = ctx.error(prob.X_clean, _bits(lin, spec.numel))
    xg = src.reconstruct([c.astype(np.float64) for c in ctx.get_cores()], spec.ranks, lin)
    ctx.close()
    e_gpu = float(np.linalg.norm(xg - xc) / np.linalg.norm(xc))
    assert g["n_eval"] == len(lin)
    assert abs(g["rel_err_all"] - e_gpu) <= 1e-5                 # trd_error vs Def. 1 at the GPU cores
    assert abs(e_gpu - e_or) <= 1e-3, (e_gpu, e_or)


def test_full_size_c5b_block_and_sweep():
    """C5b (80^5, ranks 8, 5 % observed, full working set): every row of d (Eq. 9), n_obs and
    den (Eq. 12) of one whole block at the initial cores (fixed sigma, element-wise rows), then
    the cores after one sweep in the bench's sigma rule."""
    _cuda()
    spec, prob, vals, words, src = _setup("C5b")
    cores = [c.astype(np.float64) for c in prob.init]
    N = spec.order
    k = 2
    ctx = _ctx(spec, prob, vals, words, sigma_mode=O.SIGMA_FIXED, sigma=1.0)
    g = ctx.block_probe(0, k)
    ctx.close()
    sets = [np.arange(d, dtype=np.int64) for d in spec.dims]
    d, e2, _, n, _ = src.pass1(cores, k, sets, spec.ranks, 1.0, False)
    assert g["n_obs"] == n == prob.n_obs
    rn = np.linalg.norm(d, axis=1)
    row_err = np.linalg.norm(g["d"] - d, axis=1) / np.maximum(rn, 1e-6 * rn.max())
    assert float(row_err.max()) <= 1e-4, float(row_err.max())
    assert abs(g["sum_e2"] - e2) <= 1e-5 * e2
    G = O.gram_fgmc([O.q_matrix(Z) for Z in cores], k, spec.ranks)
    h, _ = O.scaled_gradient(d, G, 1e-6)
    den = src.pass2(cores, k, sets, spec.ranks, 1.0, False, h)
    assert abs(g["den"] - den) <= 1e-4 * den
    # one sweep of Alg. 1 in the bench configuration
    cfg = O.Config(spec.dims, spec.ranks, sigma_mode=spec.sigma_mode, sketch=spec.sketch, seed=spec.sampler_seed)
    st, recs = O.run(cfg, prob.init, src, 1)
    ctx = _ctx(spec, prob, vals, words)
    gs = ctx.sweep(1)[0]
    assert abs(gs["sigma"] - recs[0].sigma) <= 1e-6 * recs[0].sigma
    assert gs["n_obs"] == recs[0].n_obs
    err = cores_rel_err(ctx.get_cores(), st.cores)
    ctx.close()
    assert err <= 1e-4, err
