"""Float64 CPU oracle of AWRTRD / SAWRTRD (arXiv 2305.09044), written from PAPER.md.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this module.  The product path
(``paper_2305_09044_b200``) never imports it and shares no code with it.

Every function follows the paper's equations in the paper's order and notation, in float64,
using plain numpy primitives (einsum / matmul / Cholesky) as single steps.  Indices are
0-based; the paper's are 1-based.  Readings of silent or garbled passages are labelled Rn
and listed in DESIGN.md section 3.

Conventions (pinned by tests/test_oracle_pins.py):
  * A tensor X of shape (I_0..I_{N-1}) is indexed X[i_0, .., i_{N-1}]; its flat storage is
    the paper's multi-index order (Def. 2): mode 0 fastest.
  * Core Z_k is an array of shape (r_k, I_k, r_{k+1}) (Def. 1); its lateral
    slice Z_k(i) = Z_k[:, i, :].
  * Classical mode-2 unfolding Zk2 (Thm 1): Zk2[i, a + r_k*b] = Z_k[a, i, b].
  * Subchain (Thm 1): S(j) = Z_{k+1}(i_{k+1}) .. Z_{N-1}(i_{N-1}) Z_0(i_0) ..
    Z_{k-1}(i_{k-1}) in R^{r_{k+1} x r_k}; j enumerates (i_{k+1}, .., i_{k-1}) with i_{k+1}
    fastest; its [2]-unfolding row is S_[2][j, c + r_k*b] = S(j)[b, c].
  * Shifted unfolding X_[k] (Thm 1): rows i_k, columns j as above.

Parity status: every function below is pinned by an independent test (brute force, closed
form, finite differences, optimality or an invariant); see DESIGN.md section 4.  The exact
iterates of the non-convex iteration are not printed by the paper, so the whole-run
trajectory is pinned only through those invariants.
"""
import math
import numpy as np

from .philox import philox4x32_10, sample_indices

SIGMA_FIXED, SIGMA_INF, SIGMA_RMS, SIGMA_MAD = 0, 1, 2, 3
# robust sigma (reading R21): sigma = max(sigma_min, theta * MAD_C * median |e|), the exact
# median of the sweep's pass-1 residual magnitudes
MAD_C = 1.4826                     # 1 / Phi^-1(3/4): MAD -> standard deviation for Gaussians
# operator of the update direction: the paper's scaled gradient (Eq. 16) and the two
# ablation arms of Sec. 6.1 built on the same sketch
SCALING_GLOBAL, SCALING_NONE, SCALING_LOCAL = 0, 1, 2
# working set of a block: the RStS subtensor (Eq. 14) or the 'uniform row sampling' arm
SAMPLING_RSTS, SAMPLING_ROWS = 0, 1
ROW_TAG = 0x524F5753                 # Philox counter word of the row sampler ('ROWS')


# ----------------------------------------------------------------------------------------
# TR algebra: Def. 1, Def. 2, Theorem 1
# ----------------------------------------------------------------------------------------
def tr_entry(cores, index):
    """Def. 1: X_{i_1..i_N} = Tr(prod_k Z_k(i_k))."""
    M = np.eye(cores[0].shape[0])
    for Z, i in zip(cores, index):
        M = M @ Z[:, i, :]
    return float(np.trace(M))


def merge_cores(A, B):
    """Def. 2: Z^{(k,k+1)}(i_k + I_k*i_{k+1}) = Z_k(i_k) Z_{k+1}(i_{k+1})."""
    ra, Ia, _ = A.shape
    _, Ib, rc = B.shape
    M = np.einsum('aib,bjc->ajic', A, B)          # [a, j, i, c]; flat (j, i) = i + Ia*j
    return M.reshape(ra, Ib * Ia, rc)


def tr_reconstruct(cores):
    """Def. 1 via Def. 2: merge all cores, then take the trace of every merged slice.

    Returns X indexed X[i_0, .., i_{N-1}] (a Fortran-ordered view of the flat, mode-0-fastest
    buffer)."""
    M = cores[0]
    for Z in cores[1:]:
        M = merge_cores(M, Z)
    flat = np.einsum('aja->j', M)                 # flat index is the paper's multi-index
    dims = [Z.shape[1] for Z in cores]
    return flat.reshape(dims[::-1]).transpose()


def core_unfold2(Z):
    """Classical mode-2 unfolding Z_{k(2)} (Thm 1): [i, a + r_k*b] = Z[a,i,b]."""
    r0, I, r1 = Z.shape
    return Z.transpose(1, 2, 0).reshape(I, r1 * r0)   # column = b*r0 + a


def core_fold2(Zk2, r0, r1):
    """Inverse of core_unfold2: the fold(.) of Eq. (11)."""
    I = Zk2.shape[0]
    return Zk2.reshape(I, r1, r0).transpose(2, 0, 1)


def subchain(cores, k, index_sets=None):
    """Subchain Z^{!=k} (Thm 1), optionally on sampled lateral slices
    (Eq. (14) and the sampled subchain of Eq. (15)).

    Merges Z_{k+1}, .., Z_{N-1}, Z_0, .., Z_{k-1} left to right (Def. 2).  Returns the
    [2]-unfolding S_[2] of shape (J, r_k*r_{k+1}) with S_[2][j, c + r_k*b] = S(j)[b, c].
    """
    N = len(cores)
    order = [(k + 1 + q) % N for q in range(N - 1)]
    def sl(m):
        Z = cores[m]
        return Z if index_sets is None else Z[:, index_sets[m], :]
    M = sl(order[0])
    for m in order[1:]:
        M = merge_cores(M, sl(m))
    rk1, J, rk = M.shape                           # S(j)[b, c] = M[b, j, c]
    return M.transpose(1, 0, 2).reshape(J, rk1 * rk)  # column = b*r_k + c


def unfold_shifted(X, k):
    """Mode-k unfolding X_[k] (Thm 1): columns (i_{k+1}..i_N i_1..i_{k-1}),
    i_{k+1} fastest."""
    N = X.ndim
    cols_slow_to_fast = [(k - 1 - q) % N for q in range(N - 1)]   # k-1, .., 0, N-1, .., k+1
    Y = np.transpose(X, [k] + cols_slow_to_fast)
    return Y.reshape(X.shape[k], -1)


def unfold_classical(X, n):
    """Classical mode-n unfolding X_(n) (Thm 1): i_1 fastest among the rest."""
    N = X.ndim
    rest = [m for m in range(N) if m != n]
    Y = np.transpose(X, [n] + rest[::-1])
    return Y.reshape(X.shape[n], -1)


# ----------------------------------------------------------------------------------------
# FGMC: Proposition 2 / Eq. (13)
# ----------------------------------------------------------------------------------------
def q_matrix(Z):
    """Per-core FGMC matrix Q_k (Eq. (13); reading R6):
    Q[(a*r_k + a'), (b*r_{k+1} + b')] = sum_i Z[a,i,b] Z[a',i,b'] = sum_i Z(i) (x) Z(i)."""
    r0, _, r1 = Z.shape
    Q = np.einsum('aib,cid->acbd', Z, Z)
    return Q.reshape(r0 * r0, r1 * r1)


def gram_fgmc(Qs, k, ranks):
    """G_{Z^{!=k}} = Phi(prod Q) (Eq. (13); reading R6).

    Chain C = Q_{k+1} .. Q_{N-1} Q_0 .. Q_{k-1} (same cyclic order as the subchain),
    shape (r_{k+1}^2, r_k^2); Phi: G[c + r_k*b, c' + r_k*b'] = C[b*r_{k+1} + b', c*r_k + c']
    so that G matches the column map of subchain()."""
    N = len(Qs)
    rk, rk1 = ranks[k], ranks[(k + 1) % N]
    C = np.eye(rk1 * rk1)
    for q in range(N - 1):
        C = C @ Qs[(k + 1 + q) % N]
    C4 = C.reshape(rk1, rk1, rk, rk)               # [b, b', c, c']
    # G index (row = b*r_k + c, col = b'*r_k + c') -> C4[b, b', c, c']
    return C4.transpose(0, 2, 1, 3).reshape(rk1 * rk, rk1 * rk)


def gram_explicit(S):
    """Explicit Gram S_[2]^T S_[2] (the O(I^N r^4) computation FGMC replaces)."""
    return S.T @ S


# ----------------------------------------------------------------------------------------
# Correntropy / half-quadratic weights: Eq. (4)-(7)
# ----------------------------------------------------------------------------------------
def g_sigma(x, sigma):
    """Eq. (4) kernel g_sigma(x) = sigma^2 exp(-x^2 / (2 sigma^2))."""
    return sigma * sigma * np.exp(-np.square(x) / (2.0 * sigma * sigma))


def hq_weight(e, sigma, sigma_inf=False):
    """Eq. (7) weight, sign reading R1: w = exp(-e^2/(2 sigma^2)) = -g'_sigma(e)/e
    (PAPER.md:136); sigma -> inf gives w = 1."""
    e = np.asarray(e, dtype=np.float64)
    if sigma_inf:
        return np.ones_like(e)
    return np.exp(-np.square(e) / (2.0 * sigma * sigma))


def welsch_loss(E, P, sigma):
    """sum_Omega sigma^2 - g_sigma(e): minimising it maximises Eq. (4) (reading R3)."""
    e = E[P]
    return float(np.sum(sigma * sigma - g_sigma(e, sigma)))


def hq_surrogate(E, P, W):
    """First term of Eq. (6): 1/2 || sqrt(W) o P o E ||_F^2."""
    return 0.5 * float(np.sum(W * P * E * E))


# ----------------------------------------------------------------------------------------
# Block step: Eq. (9)/(15), Eq. (10)/(16), Eq. (12)/(18), Eq. (11)/(17)
# ----------------------------------------------------------------------------------------
def gradient_block(Xk, Pk, Zk2, S, sigma, sigma_inf=False):
    """Eq. (7) + Eq. (9), or Eq. (15) on a sketch.

    Xk, Pk: X_[k] and P_[k] restricted to the working set (I_k x J); S: S_[2] (J x R^2).
    Returns d = (W o P o (X_[k] - Zk2 S^T)) S, and E, W for the same entries."""
    E = Xk - Zk2 @ S.T
    W = hq_weight(E, sigma, sigma_inf)
    Y = W * Pk * E
    return Y @ S, E, W


def gradient_entries(cores, k, index, x, sigma, sigma_inf=False):
    """Eq. (7) + Eq. (9) summed entry by entry, for a list of observed
    entries: index (n x N int, the multi-indices), x (n,) their values.  For each entry j,
    S(j) = Z_{k+1}(i_{k+1}) .. Z_{k-1}(i_{k-1}) (Thm 1), e = x - Tr(Z_k(i_k) S(j)),
    w = exp(-e^2 / 2 sigma^2) (reading R1), and d[i_k, c + r_k b] += w e S(j)[b, c].
    Same quantity as gradient_block restricted to the given entries (pinned against it);
    used to check single rows of d at sizes where the dense unfolding does not fit.
    Returns (d, sum_e2) with d of shape (I_k, r_k * r_{k+1})."""
    N = len(cores)
    index = np.asarray(index, dtype=np.int64)
    x = np.asarray(x, dtype=np.float64)
    rk, Ik, rk1 = cores[k].shape
    order = [(k + 1 + q) % N for q in range(N - 1)]
    S = cores[order[0]][:, index[:, order[0]], :].transpose(1, 0, 2)        # (n, r, r')
    for m in order[1:]:
        S = np.einsum('nab,nbc->nac', S, cores[m][:, index[:, m], :].transpose(1, 0, 2))
    # S[n] = S(j) in R^{r_{k+1} x r_k};  Tr(Z_k(i_k) S(j)) = sum_{a,b} Z_k[a, i_k, b] S(j)[b, a]
    Zs = cores[k][:, index[:, k], :].transpose(1, 0, 2)                    # (n, r_k, r_{k+1})
    xhat = np.einsum('nab,nba->n', Zs, S)
    e = x - xhat
    w = hq_weight(e, sigma, sigma_inf)
    y = w * e
    d = np.zeros((Ik, rk * rk1))
    contrib = (y[:, None, None] * S).reshape(len(x), rk1 * rk)             # column b*r_k + c
    np.add.at(d, index[:, k], contrib)
    return d, float(np.sum(e * e))


class NotSPD(ArithmeticError):
    """G + lambda I stayed not positive definite through the retries (reading R23)."""


LAMBDA_RETRIES = 3
LAMBDA_FLOOR = 2.0 ** -40          # R23: first retry when lambda_rel = 0, relative to tr(G)/R^2


def scaled_gradient(d, G, lambda_rel):
    """Eq. (10)/(16) with reading R5:
    lambda = lambda_rel * tr(G) / R^2, A = G + lambda I = L L^T and the filtered solve
    h = d A^{-1} G A^{-1} (= d (G + lambda I)^{-1} up to O(lambda/mu) on range(G)).
    Reading R23: if the Cholesky factorisation of A fails, lambda <- 10 lambda
    (from 2^-40 tr(G)/R^2 when lambda = 0), at most 3 retries, then NotSPD.
    Returns (h, lambda)."""
    R2 = G.shape[0]
    scale = float(np.trace(G)) / R2
    lam = lambda_rel * scale
    for attempt in range(LAMBDA_RETRIES + 1):
        if attempt > 0:
            lam = 10.0 * lam if lam > 0.0 else LAMBDA_FLOOR * scale
        try:
            L = np.linalg.cholesky(G + lam * np.eye(R2))
            break
        except np.linalg.LinAlgError:
            L = None
    if L is None:
        raise NotSPD(f"G + lambda I not positive definite (lambda = {lam:g})")
    # row-wise h = d A^{-1} G A^{-1}: solve A u^T = d^T, then A h^T = G u^T (A, G symmetric)
    U = _chol_solve(L, d.T)
    H = _chol_solve(L, G @ U)
    return H.T, lam


def _chol_solve(L, B):
    """Solve (L L^T) X = B by two triangular solves (plain numpy)."""
    Y = np.linalg.solve(L, B)
    return np.linalg.solve(L.T, Y)


def line_search_den(h, Pk, Wk, S):
    """Denominator of Eq. (12)/(18): || sqrt(W) o P o (h S^T) ||_F^2."""
    T = h @ S.T
    return float(np.sum(Wk * Pk * T * T))


# ----------------------------------------------------------------------------------------
# Working-set access (Eq. (14) sketch) -- a data source returns the sub-tensor of X and P
# ----------------------------------------------------------------------------------------
class DenseSource:
    """X (float64 view of the fp32 bytes) and P (bool) held in host memory."""

    def __init__(self, X, P):
        self.X = np.asarray(X, dtype=np.float64)
        self.P = np.asarray(P, dtype=bool)
        self.dims = self.X.shape

    def subtensor(self, index_sets):
        ix = np.ix_(*index_sets)
        return self.X[ix], self.P[ix]

    def all_observed_values(self):
        return self.X[self.P]


def working_set(source, k, index_sets):
    """Obtain X_I and P_I (Alg. 1 line 5) unfolded along mode k (Thm 1)."""
    Xs, Ps = source.subtensor(index_sets)
    return unfold_shifted(Xs, k), unfold_shifted(Ps, k)


# ----------------------------------------------------------------------------------------
# Sweep driver: Algorithm 1; full-data AWRTRD is the s_m = I_m case
# ----------------------------------------------------------------------------------------
def init_cores(dims, ranks, seed):
    """Alg. 1 line 1 'Initialize Z_k', reading R16: i.i.d. N(0, std^2) with
    std = (r_k r_{k+1})^(-1/4), rounded to fp32 (the bytes both sides consume)."""
    rng = np.random.default_rng(seed)
    N = len(dims)
    cores = []
    for k in range(N):
        r0, r1 = ranks[k], ranks[(k + 1) % N]
        std = (r0 * r1) ** -0.25
        cores.append((rng.standard_normal((r0, dims[k], r1)) * std).astype(np.float32))
    return cores


class Config:
    """Algorithm 1 inputs plus the readings' parameters."""

    def __init__(self, dims, ranks, sigma_mode=SIGMA_RMS, sigma=1.0, sigma_theta=1.0,
                 sigma_min=1e-3, lambda_rel=1e-6, step=0.0, sketch=None, seed=0, eps=0.0,
                 scaling=SCALING_GLOBAL, sampling=SAMPLING_RSTS):
        self.dims = list(dims)
        self.ranks = list(ranks)
        self.sigma_mode = sigma_mode
        self.sigma = sigma
        self.sigma_theta = sigma_theta
        self.sigma_min = sigma_min
        self.lambda_rel = lambda_rel
        self.step = step
        self.sketch = list(sketch) if sketch is not None else [0] * len(dims)
        self.seed = seed
        self.eps = eps
        self.scaling = scaling
        self.sampling = sampling
        if sampling == SAMPLING_ROWS and scaling == SCALING_LOCAL:
            raise ValueError("the local scaled term needs RStS index sets")


def gram_local(cores, k, sets, ranks):
    """'Local scaled term' ablation arm: the Gram G_{Z_I^{!=k}} of the
    subchain of the sampled cores {(Z_m)_{I_m}}, computed as Eq. (13) with
    each Q_m summed over the sampled slices only."""
    N = len(cores)
    Qs = [q_matrix(cores[m][:, sets[m], :]) if m != k else None for m in range(N)]
    return gram_fgmc(Qs, k, ranks)


def update_direction(cfg, d, G_global, cores, k, sets):
    """Update direction of block k: h = d (G + lambda I)^-1-filtered (Eq. 16) with the FGMC
    Gram, or an ablation arm of Sec. 6.1: 'gradient descent' h = d (Eq. 15's
    d_I instead of h_I), 'local scaled term' the same filtered solve with gram_local."""
    if cfg.scaling == SCALING_NONE:
        return d.copy()
    if cfg.scaling == SCALING_LOCAL:
        h, _ = scaled_gradient(d, gram_local(cores, k, sets, cfg.ranks), cfg.lambda_rel)
        return h
    h, _ = scaled_gradient(d, G_global, cfg.lambda_rel)
    return h


def row_samples(cfg, t, k):
    """'Uniform row sampling' ablation arm (reading R22): J = prod_{m != k} s_m
    rows of the shifted unfolding X_[k] drawn uniformly with replacement.  Draw q:
    kappa_q = (out0 << 32) | out1 of Philox(key = seed, ctr = (q, ROW_TAG, k, t)), row
    rho_q = floor(kappa_q R / 2^64) with R = prod_{m != k} I_m, decoded with i_{k+1} fastest
    (Thm 1's column order of X_[k]).  Returns per-mode index lists: mode k all of I_k, the
    others J entries each (entry q of every list belongs to draw q)."""
    N = len(cfg.dims)
    order = [(k + 1 + q) % N for q in range(N - 1)]
    J, R = 1, 1
    for m in order:
        s_m = cfg.sketch[m]
        J *= cfg.dims[m] if (s_m <= 0 or s_m >= cfg.dims[m]) else s_m
        R *= cfg.dims[m]
    q = np.arange(J, dtype=np.uint64)
    seed = int(cfg.seed)
    o0, o1, _, _ = philox4x32_10(q, ROW_TAG, k, t, seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF)
    kappa = (o0 << np.uint64(32)) | o1
    rho = [(int(x) * R) >> 64 for x in kappa]
    lists = [None] * N
    lists[k] = np.arange(cfg.dims[k], dtype=np.int64)
    for m in order:
        lists[m] = np.array([r % cfg.dims[m] for r in rho], dtype=np.int64)
        rho = [r // cfg.dims[m] for r in rho]
    return lists


def working_set_rows(source, k, lists):
    """X_I and P_I for explicit rows (draw q = column q): X_k[i_k, q] = X[.., i_k, .., lists[m][q], ..]."""
    N = len(lists)
    idx = [lists[m][None, :] if m != k else lists[k][:, None] for m in range(N)]
    return source.X[tuple(idx)], source.P[tuple(idx)]


def subchain_rows(cores, k, lists):
    """Subchain rows S(j_q) = Z_{k+1}(i_{k+1}^q) .. Z_{k-1}(i_{k-1}^q) for explicit multi-indices
    (Thm 1, one row per draw); S_[2][q, c + r_k b] = S(j_q)[b, c]."""
    N = len(cores)
    order = [(k + 1 + q) % N for q in range(N - 1)]
    M = cores[order[0]][:, lists[order[0]], :]
    for m in order[1:]:
        M = np.einsum('ajb,bjc->ajc', M, cores[m][:, lists[m], :])
    rk1, J, rk = M.shape
    return M.transpose(1, 0, 2).reshape(J, rk1 * rk)


def index_sets_for_block(cfg, t, k):
    """Alg. 1 line 4: I_k = all of mode k, I_m sampled for m != k."""
    N = len(cfg.dims)
    sets = []
    for m in range(N):
        if m == k:
            sets.append(np.arange(cfg.dims[m], dtype=np.int64))
        else:
            sets.append(sample_indices(cfg.seed, t, k, m, cfg.dims[m], cfg.sketch[m]))
    return sets


def mad_sigma(cfg, abs_e):
    """R21: sigma = max(sigma_min, theta * 1.4826 * median |e|) -- the exact median (numpy's:
    the middle value, or the mean of the two middle values of an even count)."""
    return max(cfg.sigma_min, cfg.sigma_theta * MAD_C * float(np.median(np.asarray(abs_e, dtype=np.float64))))


def initial_sigma(cfg, cores, source):
    """sigma_0 for the RMS reading R9 (or the MAD reading R21): max(sigma_min, theta * RMS
    (or 1.4826 median |e|)) of the observed residuals at the initial cores, over all
    observed entries."""
    if cfg.sigma_mode not in (SIGMA_RMS, SIGMA_MAD):
        return cfg.sigma
    if hasattr(source, "pass1"):                  # entry-wise source: all observed entries
        N = len(cfg.dims)
        sets = [np.arange(cfg.dims[m], dtype=np.int64) for m in range(N)]
        _, sum_e2, _, n, abs_e = source.pass1([np.asarray(c, dtype=np.float64) for c in cores], 0, sets,
                                              cfg.ranks, 1.0, True, want_abs=cfg.sigma_mode == SIGMA_MAD)
        if cfg.sigma_mode == SIGMA_MAD:
            return mad_sigma(cfg, abs_e)
        return max(cfg.sigma_min, cfg.sigma_theta * math.sqrt(sum_e2 / n))
    Xhat = tr_reconstruct([c.astype(np.float64) for c in cores])
    E = (source.X - Xhat)[source.P]
    if cfg.sigma_mode == SIGMA_MAD:
        return mad_sigma(cfg, np.abs(E))
    return max(cfg.sigma_min, cfg.sigma_theta * math.sqrt(float(np.mean(E * E))))


class SweepRecord:
    def __init__(self, N):
        self.sigma = 0.0
        self.sum_e2 = 0.0
        self.n_obs = 0
        self.welsch = 0.0
        self.stop_e = float('nan')
        self.eta = [0.0] * N
        self.num = [0.0] * N
        self.den = [0.0] * N
        self.nnz = [0] * N
        self.skipped = [False] * N
        self.abs_e = []                      # |e| of every pass-1 residual (MAD rule, R21)


class State:
    """Solver state carried across sweeps (cores, Q cache, sigma, D^{t-1}, t)."""

    def __init__(self, cfg, cores, source):
        self.cores = [np.asarray(c, dtype=np.float64).copy() for c in cores]
        self.Qs = [q_matrix(Z) for Z in self.cores]     # Alg. 1 line 1: Q_k
        self.sigma = initial_sigma(cfg, cores, source)
        self.D_prev = None
        self.t = 0


def block_update(cfg, st, source, k, rec, check_gram=False):
    """One block k of Alg. 1 (lines 4-10)."""
    N = len(cfg.dims)
    ranks = cfg.ranks
    rk, rk1 = ranks[k], ranks[(k + 1) % N]
    sigma_inf = cfg.sigma_mode == SIGMA_INF
    if hasattr(source, "pass1"):
        return block_update_entries(cfg, st, source, k, rec)
    # line 4-5: index sets and sketch (or the uniform-row-sampling arm)
    if cfg.sampling == SAMPLING_ROWS:
        sets = row_samples(cfg, st.t, k)
        Xk, Pk = working_set_rows(source, k, sets)
        S = subchain_rows(st.cores, k, sets)
    else:
        sets = index_sets_for_block(cfg, st.t, k)
        Xk, Pk = working_set(source, k, sets)
        S = subchain(st.cores, k, sets)
    Zk2 = core_unfold2(st.cores[k])
    # lines 6-7: weights (Eq. 7) and gradient (Eq. 9/15)
    d, E, W = gradient_block(Xk, Pk, Zk2, S, st.sigma, sigma_inf)
    e_obs = E[Pk]
    rec.sum_e2 += float(np.sum(e_obs * e_obs))
    if cfg.sigma_mode == SIGMA_MAD:
        rec.abs_e.append(np.abs(e_obs))
    rec.n_obs += int(e_obs.size)
    rec.nnz[k] = int(e_obs.size)
    s2 = st.sigma * st.sigma if abs(st.sigma) < 1e150 else float('inf')
    if not sigma_inf and math.isfinite(s2):
        rec.welsch += float(np.sum(s2 * (1.0 - W[Pk])))
    # line 8: FGMC Gram of the full cores (Eq. 13/16)
    G = gram_fgmc(st.Qs, k, ranks)
    if check_gram:
        Sf = subchain(st.cores, k)
        Gx = gram_explicit(Sf)
        assert np.linalg.norm(G - Gx) <= 1e-10 * max(np.linalg.norm(Gx), 1e-300)
    # line 9: scaled gradient (Eq. 10/16; or an ablation arm), step (Eq. 12/18), update
    # (Eq. 11/17, reading R2)
    h = update_direction(cfg, d, G, st.cores, k, sets)
    num = float(np.sum(d * h))
    den = line_search_den(h, Pk, W, S)
    rec.num[k], rec.den[k] = num, den
    if cfg.step > 0.0:
        eta = cfg.step
    elif num > 0.0 and den > 0.0:
        eta = num / den
    else:
        eta = 0.0
    rec.eta[k] = eta
    if eta == 0.0:
        rec.skipped[k] = True
    else:
        st.cores[k] = st.cores[k] + eta * core_fold2(h, rk, rk1)
    # line 10: refresh Q_k
    st.Qs[k] = q_matrix(st.cores[k])
    return G


def block_update_entries(cfg, st, source, k, rec):
    """block_update with the two per-entry sums taken entry by entry (oracle/entries.py):
    same lines 4-10 of Alg. 1 in the same order, for problems whose sketch does not fit the
    dense unfolding (RStS subtensors only)."""
    if cfg.sampling != SAMPLING_RSTS:
        raise ValueError("entry-wise source: RStS index sets only")
    N = len(cfg.dims)
    rk, rk1 = cfg.ranks[k], cfg.ranks[(k + 1) % N]
    sigma_inf = cfg.sigma_mode == SIGMA_INF
    sets = index_sets_for_block(cfg, st.t, k)                       # line 4
    s2 = st.sigma * st.sigma if abs(st.sigma) < 1e150 else float('inf')
    sig = 1.0 if sigma_inf else st.sigma
    d, sum_e2, welsch, n, abs_e = source.pass1(st.cores, k, sets, cfg.ranks, sig, sigma_inf,
                                               want_abs=cfg.sigma_mode == SIGMA_MAD)   # lines 5-7
    rec.sum_e2 += sum_e2
    rec.n_obs += n
    rec.nnz[k] = n
    if cfg.sigma_mode == SIGMA_MAD:
        rec.abs_e.append(abs_e)
    if not sigma_inf and math.isfinite(s2):
        rec.welsch += welsch
    G = gram_fgmc(st.Qs, k, cfg.ranks)                              # line 8
    h = update_direction(cfg, d, G, st.cores, k, sets)              # line 9
    num = float(np.sum(d * h))
    den = source.pass2(st.cores, k, sets, cfg.ranks, sig, sigma_inf, h)
    rec.num[k], rec.den[k] = num, den
    if cfg.step > 0.0:
        eta = cfg.step
    elif num > 0.0 and den > 0.0:
        eta = num / den
    else:
        eta = 0.0
    rec.eta[k] = eta
    if eta == 0.0:
        rec.skipped[k] = True
    else:
        st.cores[k] = st.cores[k] + eta * core_fold2(h, rk, rk1)
    st.Qs[k] = q_matrix(st.cores[k])                                # line 10
    return G


def sweep(cfg, st, source, check_gram=False):
    """One iteration of Alg. 1's repeat loop; returns a SweepRecord."""
    N = len(cfg.dims)
    rec = SweepRecord(N)
    rec.sigma = st.sigma
    G_last = None
    for k in range(N):                       # line 3: cyclic k = 1..N
        G_last = block_update(cfg, st, source, k, rec, check_gram)
    # lines 12-13: D^t = Z_N(2) G_{!=N} Z_N(2)^T (reading R15: G of block N, updated Z_N)
    ZN2 = core_unfold2(st.cores[N - 1])
    D = ZN2 @ G_last @ ZN2.T
    if st.D_prev is not None:
        rec.stop_e = float(np.linalg.norm(D - st.D_prev) / np.linalg.norm(D))
    st.D_prev = D
    # sigma for the next sweep (reading R9)
    if cfg.sigma_mode == SIGMA_RMS and rec.n_obs > 0:
        st.sigma = max(cfg.sigma_min, cfg.sigma_theta * math.sqrt(rec.sum_e2 / rec.n_obs))
    elif cfg.sigma_mode == SIGMA_MAD and rec.n_obs > 0:
        st.sigma = mad_sigma(cfg, np.concatenate(rec.abs_e))
        rec.abs_e = []
    st.t += 1
    return rec


def run(cfg, cores, source, n_sweeps, check_gram=False):
    """Algorithm 1 for n_sweeps iterations (stops early only if cfg.eps > 0, line 14)."""
    st = State(cfg, cores, source)
    recs = []
    for _ in range(n_sweeps):
        rec = sweep(cfg, st, source, check_gram)
        recs.append(rec)
        if cfg.eps > 0.0 and not math.isnan(rec.stop_e) and rec.stop_e < cfg.eps:
            break
    return st, recs


# ----------------------------------------------------------------------------------------
# Evaluation
# ----------------------------------------------------------------------------------------
def relative_error(cores, X_true):
    """||X_hat - X*||_F / ||X*||_F over all entries."""
    Xhat = tr_reconstruct([np.asarray(c, dtype=np.float64) for c in cores])
    return float(np.linalg.norm(Xhat - X_true) / np.linalg.norm(X_true))


def psnr(X_true, X_hat, peak=1.0):
    """PSNR = 10 log10(peak^2 / MSE) (the paper's evaluation metric)."""
    mse = float(np.mean(np.square(np.asarray(X_true) - np.asarray(X_hat))))
    return float('inf') if mse == 0.0 else 10.0 * math.log10(peak * peak / mse)
