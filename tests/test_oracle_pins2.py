"""More pins of the float64 oracle (-m "not gpu"): the Philox generator against CUDA's curand
host implementation, the sigma schedules (R9 / R21) against residuals computed by brute force,
the lambda retry rule (R23), and the entry-wise data source (oracle/entries.py) against the
dense form.  Citations are PAPER.md lines (P:L)."""
import ctypes
import math
import os

import numpy as np
import pytest

from oracle import trd_oracle as O
from oracle.entries import EntrySource
from oracle.philox import philox4x32_10, sample_indices

from tests.test_oracle_pins import _problem, brute_entry, rand_cores

CURAND = "/usr/local/cuda/lib64/libcurand.so"


# ---------------------------------------------------------------- Philox4x32-10 (R11)
@pytest.mark.skipif(not os.path.exists(CURAND), reason="CUDA toolkit curand library absent")
def test_philox_matches_curand_host_generator():
    """The oracle's Philox4x32-10 equals an independent implementation of the same published
    generator: curand's host Philox4_32_10 generator (CPU, no GPU needed).  With seed s, block
    j of its output stream (4 words, curandSetGeneratorOffset(4 j)) is the Philox output at
    key (s lo32, s hi32) and counter (lo32(j >> 16), hi32(j >> 16), j mod 2^16, 0) -- the
    layout of curand's 65536 host subsequences -- so every counter word but the last, both
    key words, the round function and the key schedule are exercised."""
    lib = ctypes.CDLL(CURAND)
    philox = 161                                   # CURAND_RNG_PSEUDO_PHILOX4_32_10

    def block(seed, j):
        g = ctypes.c_void_p()
        assert lib.curandCreateGeneratorHost(ctypes.byref(g), philox) == 0
        try:
            assert lib.curandSetPseudoRandomGeneratorSeed(g, ctypes.c_ulonglong(seed)) == 0
            assert lib.curandSetGeneratorOffset(g, ctypes.c_ulonglong(4 * j)) == 0
            out = np.zeros(4, dtype=np.uint32)
            assert lib.curandGenerate(g, out.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(4)) == 0
        finally:
            lib.curandDestroyGenerator(g)
        return [int(x) for x in out]

    for seed in (0, 3000, 0xFEDCBA9876543210, (1 << 64) - 1):
        for j in (0, 1, 4464, 65535, 70000, 1 << 20, (5 << 48) + (7 << 16) + 3, (0x3FFF << 48) + 0xFFFF):
            q = j >> 16
            o = philox4x32_10(q & 0xFFFFFFFF, q >> 32, j & 0xFFFF, 0, seed & 0xFFFFFFFF, seed >> 32)
            assert block(seed, j) == [int(x) for x in o], (seed, j)


# ---------------------------------------------------------------- sigma schedules (R9, R21)
def _observed_residuals(cores, X, P, sets=None):
    """e = x - Tr(prod Z_m(i_m)) of every observed entry (of the product set), by brute force
    over the ring indices (Def. 1)."""
    dims = X.shape
    sets = sets or [range(d) for d in dims]
    out = []
    for idx in np.ndindex(*[len(s) for s in sets]):
        ix = tuple(int(sets[m][idx[m]]) for m in range(len(dims)))
        if P[ix]:
            out.append(float(X[ix]) - brute_entry(cores, ix))
    return np.asarray(out)


@pytest.mark.parametrize("mode", [O.SIGMA_RMS, O.SIGMA_MAD])
def test_initial_sigma_from_brute_force_residuals(mode):
    """sigma_0 (R9 / R21) = max(sigma_min, theta * RMS (or 1.4826 median |e|)) over all
    observed entries at the initial cores."""
    dims, ranks = [5, 4, 3], [2, 3, 2]
    _, _, X, P = _problem(dims, ranks, 0.6, 300, outliers=0.1, noise=0.05)
    cores = O.init_cores(dims, ranks, 301)
    cfg = O.Config(dims, ranks, sigma_mode=mode, sigma_theta=1.3, sigma_min=1e-3)
    e = _observed_residuals([c.astype(np.float64) for c in cores], X, P)
    want = 1.3 * (math.sqrt(float(np.mean(e * e))) if mode == O.SIGMA_RMS
                  else 1.4826 * float(np.median(np.abs(e))))
    got = O.State(cfg, cores, O.DenseSource(X, P)).sigma
    assert got == pytest.approx(want, rel=1e-12)


@pytest.mark.parametrize("mode", [O.SIGMA_RMS, O.SIGMA_MAD])
def test_sigma_schedule_uses_each_blocks_pass1_residuals(mode):
    """sigma_{t+1} (R9 / R21) is computed from the pass-1 residuals of sweep t: block k's
    residuals over its own sketch, at the cores *before* block k's update (Alg. 1 order,
    P:267-274), pooled over the N blocks -- divided by the number of observed residuals, not
    by |WS|.  Residuals recomputed here by brute force from snapshots of the cores."""
    dims, ranks = [6, 5, 4, 3], [2, 2, 3, 2]
    _, _, X, P = _problem(dims, ranks, 0.5, 310, outliers=0.1, noise=0.05)
    cores = O.init_cores(dims, ranks, 311)
    cfg = O.Config(dims, ranks, sigma_mode=mode, sketch=[4, 3, 3, 2], seed=5)
    src = O.DenseSource(X, P)
    st = O.State(cfg, cores, src)
    for t in range(2):
        pooled = []
        rec = O.SweepRecord(4)
        rec.sigma = st.sigma
        for k in range(4):
            sets = O.index_sets_for_block(cfg, st.t, k)
            pooled.append(_observed_residuals([c.copy() for c in st.cores], X, P, sets))
            O.block_update(cfg, st, src, k, rec)
        e = np.concatenate(pooled)
        assert rec.n_obs == e.size
        want = math.sqrt(float(np.mean(e * e))) if mode == O.SIGMA_RMS else 1.4826 * float(np.median(np.abs(e)))
        # the sweep driver's update of sigma from this record
        if mode == O.SIGMA_RMS:
            got = max(cfg.sigma_min, cfg.sigma_theta * math.sqrt(rec.sum_e2 / rec.n_obs))
        else:
            got = O.mad_sigma(cfg, np.concatenate(rec.abs_e))
        assert got == pytest.approx(want, rel=1e-12)
        # ... and O.sweep applies exactly this update
        st2 = O.State(cfg, cores, src)
        for _ in range(t + 1):
            O.sweep(cfg, st2, src)
        assert st2.sigma == pytest.approx(got, rel=1e-12)
        st.t += 1
        st.sigma = got


# ---------------------------------------------------------------- lambda retry (R23)
def test_lambda_retry_rule():
    """R23: a failed Cholesky of G + lambda I retries with lambda x 10 (from
    2^-40 tr(G)/R^2 when lambda_rel = 0); a Gram with exactly zero rows fails at lambda = 0
    and succeeds on the first retry, after which h solves the regularised system on the
    nonzero block and vanishes on the zero rows; G = 0 stays singular -> NotSPD."""
    rng = np.random.default_rng(7)
    n, z = 9, 3
    B = rng.standard_normal((n, n))
    G = B @ B.T
    G[:z, :] = 0.0
    G[:, :z] = 0.0
    d = rng.standard_normal((4, n))
    d[:, :z] = 0.0
    h, lam = O.scaled_gradient(d, G, 0.0)
    assert lam == pytest.approx(2.0 ** -40 * np.trace(G) / n, rel=1e-15)
    A = G + lam * np.eye(n)
    want = d @ np.linalg.inv(A) @ G @ np.linalg.inv(A)
    assert np.linalg.norm(h - want) <= 1e-9 * np.linalg.norm(want)
    assert np.all(h[:, :z] == 0.0)
    with pytest.raises(O.NotSPD):
        O.scaled_gradient(d, np.zeros((n, n)), 1e-6)
    # a positive definite G never retries
    h2, lam2 = O.scaled_gradient(d, B @ B.T, 1e-6)
    assert lam2 == pytest.approx(1e-6 * np.trace(B @ B.T) / n, rel=1e-15)


# ---------------------------------------------------------------- entry-wise source
def _words(P):
    flat = P.transpose().reshape(-1)            # mode 0 fastest (Def. 2)
    n = flat.size
    pad = np.zeros((n + 31) // 32 * 32, dtype=bool)
    pad[:n] = flat
    bits = pad.reshape(-1, 32).astype(np.uint64) << np.arange(32, dtype=np.uint64)
    return bits.sum(axis=1).astype(np.uint32)


def _entry_source(X, P, packed):
    flatX = X.transpose().reshape(-1).astype(np.float32)
    flatP = P.transpose().reshape(-1)
    vals = flatX[flatP] if packed else flatX
    return EntrySource(X.shape, _words(P), vals, packed)


@pytest.mark.parametrize("packed", [False, True])
@pytest.mark.parametrize("mode", [O.SIGMA_RMS, O.SIGMA_INF, O.SIGMA_MAD])
def test_entry_source_equals_dense_form(packed, mode):
    """The entry-wise passes (oracle/trd_entries.c) give the dense form's d, statistics, den
    and sweeps (Eq. 9/15, 12/18 on the same sketch), to rounding order."""
    dims, ranks = [7, 5, 6, 4], [3, 2, 3, 2]
    _, _, X, P = _problem(dims, ranks, 0.4, 320, outliers=0.1, noise=0.05)
    cores = O.init_cores(dims, ranks, 321)
    cfg = O.Config(dims, ranks, sigma_mode=mode, sketch=[5, 3, 4, 0], seed=11)
    dense, ent = O.DenseSource(X, P), _entry_source(X, P, packed)
    s1, s2 = O.State(cfg, cores, dense), O.State(cfg, cores, ent)
    assert s2.sigma == pytest.approx(s1.sigma, rel=1e-12)
    for t in range(2):
        r1, r2 = O.sweep(cfg, s1, dense), O.sweep(cfg, s2, ent)
        for k in range(4):
            assert r2.nnz[k] == r1.nnz[k]
            assert r2.num[k] == pytest.approx(r1.num[k], rel=1e-10)
            assert r2.den[k] == pytest.approx(r1.den[k], rel=1e-10)
        assert r2.sum_e2 == pytest.approx(r1.sum_e2, rel=1e-12)
        assert r2.welsch == pytest.approx(r1.welsch, rel=1e-12, abs=1e-300)
        assert s2.sigma == pytest.approx(s1.sigma, rel=1e-12)
        for a, b in zip(s2.cores, s1.cores):
            assert np.linalg.norm(a - b) <= 1e-11 * np.linalg.norm(b)


def test_entry_source_block_pass_and_reconstruct():
    """Block quantities entry by entry vs gradient_block / line_search_den on the unfolded
    sketch, and reconstruct() vs Def. 1 by brute force."""
    dims, ranks = [6, 4, 5], [2, 3, 2]
    _, _, X, P = _problem(dims, ranks, 0.5, 330)
    cores = [c.astype(np.float64) for c in O.init_cores(dims, ranks, 331)]
    ent = _entry_source(X, P, True)
    for k in range(3):
        sets = [sample_indices(4, 0, k, m, dims[m], 3 if m != k else 0) for m in range(3)]
        Xk, Pk = O.working_set(O.DenseSource(X, P), k, sets)
        S = O.subchain(cores, k, sets)
        d, E, W = O.gradient_block(Xk, Pk, O.core_unfold2(cores[k]), S, 0.7)
        d2, e2, _, n, ae = ent.pass1(cores, k, sets, ranks, 0.7, False, want_abs=True)
        assert n == int(Pk.sum())
        assert np.linalg.norm(d2 - d) <= 1e-12 * np.linalg.norm(d)
        assert e2 == pytest.approx(float(np.sum(E[Pk] ** 2)), rel=1e-12)
        assert np.allclose(np.sort(ae), np.sort(np.abs(E[Pk])), rtol=1e-12, atol=0)
        h = np.random.default_rng(k).standard_normal(d.shape)
        assert ent.pass2(cores, k, sets, ranks, 0.7, False, h) == pytest.approx(
            O.line_search_den(h, Pk, W, S), rel=1e-12)
    lin = np.array([0, 5, 17, 119, 6 * 4 * 5 - 1])
    got = ent.reconstruct(cores, ranks, lin)
    for t, l in enumerate(lin):
        ix = (l % 6, (l // 6) % 4, l // 24)
        assert got[t] == pytest.approx(brute_entry(cores, ix), rel=1e-12, abs=1e-14)
