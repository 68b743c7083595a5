"""Pins of the float64 oracle against what the paper and mathematics fix (-m "not gpu").

Each test checks an oracle function against something other than itself: brute force,
an index enumeration, a closed form, finite differences, optimality, or an invariant.
Citations are PAPER.md lines (P:L).
"""
import itertools
import math

import numpy as np
import pytest

from oracle import trd_oracle as O
from oracle.philox import sample_indices, philox4x32_10, sample_keys


def rand_cores(dims, ranks, seed, scale=None):
    rng = np.random.default_rng(seed)
    N = len(dims)
    out = []
    for k in range(N):
        r0, r1 = ranks[k], ranks[(k + 1) % N]
        s = (r0 * r1) ** -0.25 if scale is None else scale
        out.append(rng.standard_normal((r0, dims[k], r1)) * s)
    return out


def brute_entry(cores, idx):
    """Def. 1 as a full contraction: sum over ring indices a_0..a_{N-1} of
    prod_k Z_k[a_k, i_k, a_{k+1}] (pure Python loops)."""
    N = len(cores)
    ranks = [c.shape[0] for c in cores]
    tot = 0.0
    for a in itertools.product(*[range(r) for r in ranks]):
        p = 1.0
        for k in range(N):
            p *= float(cores[k][a[k], idx[k], a[(k + 1) % N]])
        tot += p
    return tot


def py_matmul(A, B):
    n, m = len(A), len(B[0])
    return [[sum(A[i][t] * B[t][j] for t in range(len(B))) for j in range(m)] for i in range(n)]


CASES = [([3, 4, 2], [2, 3, 2]), ([4, 3, 5, 2], [2, 3, 2, 3]), ([2, 3, 2, 3, 2], [2, 1, 3, 2, 2])]


@pytest.mark.parametrize("dims,ranks", CASES)
def test_reconstruct_matches_bruteforce_trace(dims, ranks):
    """Def. 1: merged reconstruction equals the explicit ring contraction."""
    cores = rand_cores(dims, ranks, 1)
    X = O.tr_reconstruct(cores)
    for idx in itertools.product(*[range(I) for I in dims]):
        assert abs(X[idx] - brute_entry(cores, idx)) <= 1e-12
        assert abs(O.tr_entry(cores, idx) - X[idx]) <= 1e-12


def test_reconstruct_flat_order_is_mode0_fastest():
    """Def. 2 multi-index: flat position i_0 + I_0 i_1 + I_0 I_1 i_2."""
    dims, ranks = [3, 4, 2], [2, 2, 2]
    cores = rand_cores(dims, ranks, 2)
    X = O.tr_reconstruct(cores)
    flat = np.asfortranarray(X).ravel(order="F")
    for idx in itertools.product(*[range(I) for I in dims]):
        lin = idx[0] + dims[0] * (idx[1] + dims[1] * idx[2])
        assert flat[lin] == X[idx]


@pytest.mark.parametrize("dims,ranks", CASES)
def test_unfold_shifted_enumeration(dims, ranks):
    """Thm 1 X_[k] column order by explicit index enumeration."""
    rng = np.random.default_rng(3)
    X = rng.standard_normal(dims)
    N = len(dims)
    for k in range(N):
        Xk = O.unfold_shifted(X, k)
        for idx in itertools.product(*[range(I) for I in dims]):
            j, stride = 0, 1
            for q in range(N - 1):
                m = (k + 1 + q) % N
                j += idx[m] * stride
                stride *= dims[m]
            assert Xk[idx[k], j] == X[idx]
    # classical unfolding X_(n): i_1 fastest among the remaining modes
    Xc = O.unfold_classical(X, 1)
    for idx in itertools.product(*[range(I) for I in dims]):
        j, stride = 0, 1
        for m in range(N):
            if m == 1:
                continue
            j += idx[m] * stride
            stride *= dims[m]
        assert Xc[idx[1], j] == X[idx]


@pytest.mark.parametrize("dims,ranks", CASES)
def test_subchain_rows_are_slice_products(dims, ranks):
    """Thm 1 subchain slices: S(j) = Z_{k+1}(i_{k+1}) .. Z_{k-1}(i_{k-1})."""
    cores = rand_cores(dims, ranks, 4)
    N = len(dims)
    for k in range(N):
        S = O.subchain(cores, k)
        rk, rk1 = ranks[k], ranks[(k + 1) % N]
        modes = [(k + 1 + q) % N for q in range(N - 1)]
        for tup in itertools.product(*[range(dims[m]) for m in modes]):
            j, stride = 0, 1
            for m, i in zip(modes, tup):
                j += i * stride
                stride *= dims[m]
            M = [[1.0 if a == b else 0.0 for b in range(rk1)] for a in range(rk1)]
            for m, i in zip(modes, tup):
                M = py_matmul(M, cores[m][:, i, :].tolist())
            for b in range(rk1):
                for c in range(rk):
                    assert abs(S[j, c + rk * b] - M[b][c]) <= 1e-12


@pytest.mark.parametrize("dims,ranks", CASES)
def test_theorem1_identity(dims, ranks):
    """Thm 1: X_[k] = Z_k(2) (Z^{!=k}_[2])^T for every k (<= 1e-12)."""
    cores = rand_cores(dims, ranks, 5)
    X = np.zeros(dims)
    for idx in itertools.product(*[range(I) for I in dims]):
        X[idx] = brute_entry(cores, idx)
    for k in range(len(dims)):
        lhs = O.unfold_shifted(X, k)
        rhs = O.core_unfold2(cores[k]) @ O.subchain(cores, k).T
        assert np.max(np.abs(lhs - rhs)) <= 1e-12


def test_core_unfold2_enumeration_and_fold():
    """Classical mode-2 unfolding of a core: [i, a + r_k b] = Z[a, i, b]."""
    Z = np.random.default_rng(6).standard_normal((3, 5, 2))
    U = O.core_unfold2(Z)
    for a, i, b in itertools.product(range(3), range(5), range(2)):
        assert U[i, a + 3 * b] == Z[a, i, b]
    assert np.array_equal(O.core_fold2(U, 3, 2), Z)


def test_merge_cores_associative_and_ordered():
    """Def. 2: merged slice at i_a + I_a i_b is Z_a(i_a) Z_b(i_b)."""
    A, B, C = rand_cores([3, 4, 2], [2, 3, 2], 7)
    AB = O.merge_cores(A, B)
    for ia in range(3):
        for ib in range(4):
            assert np.allclose(AB[:, ia + 3 * ib, :], A[:, ia, :] @ B[:, ib, :], atol=1e-14)
    lhs = O.merge_cores(O.merge_cores(A, B), C)
    rhs = O.merge_cores(A, O.merge_cores(B, C))
    assert np.max(np.abs(lhs - rhs)) <= 1e-13


# ---------------------------------------------------------------- FGMC (Eq. 13)
FGMC_CASES = [([4, 3, 5, 2], [2, 3, 2, 3]), ([3, 4, 2], [2, 2, 3]), ([2, 3, 2, 3, 2], [2, 3, 1, 2, 3]),
              ([5, 4, 3], [3, 1, 2])]


@pytest.mark.parametrize("dims,ranks", FGMC_CASES)
def test_fgmc_equals_explicit_gram(dims, ranks):
    """Eq. (13): Phi(prod Q) equals the explicit S^T S, all k (<= 1e-10 rel)."""
    cores = rand_cores(dims, ranks, 8)
    Qs = [O.q_matrix(Z) for Z in cores]
    for k in range(len(dims)):
        S = O.subchain(cores, k)
        Gx = S.T @ S
        G = O.gram_fgmc(Qs, k, ranks)
        assert np.linalg.norm(G - Gx) <= 1e-10 * np.linalg.norm(Gx)
        assert np.max(np.abs(G - G.T)) <= 1e-12 * np.abs(G).max()
        assert np.linalg.eigvalsh(G).min() >= -1e-10 * np.trace(G)


def test_q_matrix_kron_sum():
    """Q_k = sum_i Z(i) (x) Z(i) (reading R6/R7) against np.kron."""
    Z = np.random.default_rng(9).standard_normal((2, 4, 3))
    Q = O.q_matrix(Z)
    ref = sum(np.kron(Z[:, i, :], Z[:, i, :]) for i in range(4))
    assert np.max(np.abs(Q - ref)) <= 1e-13


def test_fgmc_rank_one_all_ones_closed_form():
    """All-ones rank-1 cores: G = prod_{j != k} I_j (SPEC S:224 example)."""
    dims = [3, 4, 5, 2]
    cores = [np.ones((1, I, 1)) for I in dims]
    Qs = [O.q_matrix(Z) for Z in cores]
    for k in range(4):
        G = O.gram_fgmc(Qs, k, [1, 1, 1, 1])
        assert G.shape == (1, 1)
        assert G[0, 0] == np.prod([I for m, I in enumerate(dims) if m != k])


# ---------------------------------------------------------------- weights (Eq. 4-7)
def test_weights_special_values():
    """Eq. (7) with sign reading R1: w(0)=1, w(1; sigma=1)=e^-1/2, sigma=inf -> 1 exactly."""
    assert O.hq_weight(0.0, 1.0) == 1.0
    assert abs(O.hq_weight(1.0, 1.0) - math.exp(-0.5)) <= 1e-16
    e = np.array([0.0, 1e-3, 5.0, 1e6])
    assert np.all(O.hq_weight(e, 1.0, sigma_inf=True) == 1.0)
    # sigma so large that sigma^2 overflows: the FIXED formula gives exactly 1 too
    assert np.all(O.hq_weight(e[:3], 1e200) == 1.0)
    # w = -g'_sigma(e)/e for the Eq. (4) kernel (derivative by central differences)
    s, x, h = 0.7, 0.9, 1e-6
    gp = (O.g_sigma(x + h, s) - O.g_sigma(x - h, s)) / (2 * h)
    assert abs(-gp / x - O.hq_weight(x, s)) <= 1e-8
    # Eq. (4) kernel: g(0)=sigma^2 and g(sigma) = sigma^2 e^-1/2
    assert O.g_sigma(0.0, 2.0) == 4.0
    assert abs(O.g_sigma(2.0, 2.0) - 4.0 * math.exp(-0.5)) <= 1e-15


def test_hq_weight_minimises_half_quadratic():
    """Reading R3: w* = exp(-e^2/2s^2) minimises 1/2 w e^2 + psi(w) with
    psi(w) = s^2 (w log w - w + 1)  (so that min_w = s^2 - g_s(e))."""
    s = 1.3
    for e in [0.0, 0.4, 1.7, 4.0]:
        ws = np.linspace(1e-6, 1.0, 200001)
        f = 0.5 * ws * e * e + s * s * (ws * np.log(ws) - ws + 1.0)
        w_star = ws[np.argmin(f)]
        assert abs(w_star - O.hq_weight(e, s)) <= 1e-4
        assert abs(f.min() - (s * s - O.g_sigma(e, s))) <= 1e-6


# ---------------------------------------------------------------- gradient (Eq. 9)
def _instance(seed, dims=(4, 3, 5), ranks=(2, 3, 2), obs=0.6):
    rng = np.random.default_rng(seed)
    cores = rand_cores(list(dims), list(ranks), seed + 100)
    X = rng.standard_normal(dims)
    P = rng.random(dims) < obs
    return cores, X, P


@pytest.mark.parametrize("seed", range(5))
def test_gradient_is_negative_gradient_by_finite_differences(seed):
    """Eq. (9), reading R2: d = -grad of 1/2||sqrt(W) o P o E||^2 at fixed W."""
    cores, X, P = _instance(seed)
    N = len(cores)
    rng = np.random.default_rng(seed)
    for k in range(N):
        Xk, Pk = O.unfold_shifted(X, k), O.unfold_shifted(P, k)
        S = O.subchain(cores, k)
        Zk2 = O.core_unfold2(cores[k])
        W = rng.random(Xk.shape)                    # any fixed weights
        def f(Z2):
            E = Xk - Z2 @ S.T
            return 0.5 * np.sum(W * Pk * E * E)
        d = (W * Pk * (Xk - Zk2 @ S.T)) @ S
        d_or, _, _ = O.gradient_block(Xk, Pk, Zk2, S, 1.0, sigma_inf=True)
        # the oracle's d with W = 1 matches the formula; check FD against general W
        E1 = Xk - Zk2 @ S.T
        assert np.allclose(d_or, (Pk * E1) @ S, rtol=0, atol=1e-13)
        g = np.zeros_like(Zk2)
        h = 1e-6
        for idx in np.ndindex(*Zk2.shape):
            Zp, Zm = Zk2.copy(), Zk2.copy()
            Zp[idx] += h
            Zm[idx] -= h
            g[idx] = (f(Zp) - f(Zm)) / (2 * h)
        assert np.linalg.norm(d + g) <= 1e-7 * max(np.linalg.norm(d), 1e-12)


def test_gradient_single_observed_entry():
    """One observed entry: d = w e (row of S_[2]) at row i_k."""
    dims, ranks = [3, 4, 2], [2, 2, 3]
    cores = rand_cores(dims, ranks, 11)
    X = np.random.default_rng(11).standard_normal(dims)
    P = np.zeros(dims, dtype=bool)
    P[1, 2, 1] = True
    k = 1
    Xk, Pk = O.unfold_shifted(X, k), O.unfold_shifted(P, k)
    S = O.subchain(cores, k)
    d, E, W = O.gradient_block(Xk, Pk, O.core_unfold2(cores[k]), S, 0.8)
    j = 1 + dims[2] * 1                                # (i_2, i_0) = (1, 1), i_2 fastest
    e = X[1, 2, 1] - brute_entry(cores, (1, 2, 1))
    w = math.exp(-e * e / (2 * 0.64))
    expect = np.zeros_like(d)
    expect[2] = w * e * S[j]
    assert np.max(np.abs(d - expect)) <= 1e-12


# ---------------------------------------------------------------- scaled gradient (Eq. 10)
def test_scaled_gradient_identity_gram():
    """G = I: h = d A^-1 G A^-1 = d / (1 + lambda_rel)^2 (reading R5; S:378 at lambda=0)."""
    d = np.random.default_rng(12).standard_normal((5, 6))
    h, lam = O.scaled_gradient(d, np.eye(6), 1e-3)
    assert lam == 1e-3
    assert np.max(np.abs(h - d / (1.001 ** 2))) <= 1e-15
    h0, _ = O.scaled_gradient(d, np.eye(6), 0.0)
    assert np.array_equal(h0, d)


def test_scaled_gradient_spd_residual_and_nullspace():
    """h A G^-1 A = d for SPD G; for singular G, h has no null(G) component."""
    rng = np.random.default_rng(13)
    B = rng.standard_normal((9, 9))
    G = B @ B.T + 0.5 * np.eye(9)
    d = rng.standard_normal((4, 9))
    h, lam = O.scaled_gradient(d, G, 1e-6)
    A = G + lam * np.eye(9)
    assert np.max(np.abs(h @ A @ np.linalg.inv(G) @ A - d)) <= 1e-10 * np.abs(d).max()
    # exact reading R5 vs the paper's literal d (G + lambda I)^-1: O(lambda/mu) apart
    lit = d @ np.linalg.inv(A)
    assert np.linalg.norm(h - lit) <= 1e-4 * np.linalg.norm(lit)
    # singular Gram (rank 5 of 9): d in the row space -> h in the row space
    B5 = rng.standard_normal((9, 5))
    Gs = B5 @ B5.T
    ds = rng.standard_normal((4, 5)) @ B5.T
    hs, _ = O.scaled_gradient(ds, Gs, 1e-6)
    U, s, Vt = np.linalg.svd(Gs)
    null = U[:, 5:]
    assert np.abs(hs @ null).max() <= 1e-6 * np.abs(hs).max()
    # on range(G) it is the pseudo-inverse solution up to O(lambda_rel)
    pinv = ds @ np.linalg.pinv(Gs)
    assert np.linalg.norm(hs - pinv) <= 1e-3 * np.linalg.norm(pinv)


# ---------------------------------------------------------------- line search (Eq. 12)
@pytest.mark.parametrize("seed", range(5))
def test_exact_line_search_is_optimal(seed):
    """Eq. (12): with the sign reading R2 the step eta = <d,h>/den minimises the
    weighted residual along +h: cost(eta) <= cost(0.99 eta), cost(1.01 eta)."""
    cores, X, P = _instance(seed + 20)
    for k in range(3):
        Xk, Pk = O.unfold_shifted(X, k), O.unfold_shifted(P, k)
        S = O.subchain(cores, k)
        Zk2 = O.core_unfold2(cores[k])
        Qs = [O.q_matrix(Z) for Z in cores]
        d, E, W = O.gradient_block(Xk, Pk, Zk2, S, 1.5)
        h, _ = O.scaled_gradient(d, O.gram_fgmc(Qs, k, [2, 3, 2]), 1e-6)
        num, den = float(np.sum(d * h)), O.line_search_den(h, Pk, W, S)
        assert num > 0 and den > 0
        eta = num / den
        def cost(t):
            Et = Xk - (Zk2 + t * h) @ S.T
            return 0.5 * np.sum(W * Pk * Et * Et)
        c0 = cost(eta)
        assert c0 <= cost(0.99 * eta) + 1e-12 and c0 <= cost(1.01 * eta) + 1e-12
        assert c0 < cost(0.0)
        # the opposite sign (Eq. 11 as printed) increases the cost
        assert cost(-eta) > cost(0.0)


# ---------------------------------------------------------------- whole-method invariants
def _problem(dims, ranks, obs, seed, outliers=0.0, noise=0.0):
    gt = rand_cores(dims, ranks, seed)
    Xc = O.tr_reconstruct(gt)
    rng = np.random.default_rng(seed + 1)
    X = Xc + noise * rng.standard_normal(dims)
    P = rng.random(dims) < obs
    hit = (rng.random(dims) < outliers) & P
    X = np.where(hit, rng.uniform(-10, 10, dims), X)
    X = X.astype(np.float32).astype(np.float64)
    return gt, Xc, X, P


def test_hq_mm_monotone_fixed_sigma():
    """Eq. (5)-(6) MM argument: with fixed sigma, full mode, the Welsch loss (reading R3)
    is non-increasing after every block update (SPEC AC-6)."""
    dims, ranks = [10, 9, 8], [3, 3, 3]
    gt, Xc, X, P = _problem(dims, ranks, 1.0, 30, outliers=0.2, noise=0.05)
    cfg = O.Config(dims, ranks, sigma_mode=O.SIGMA_FIXED, sigma=1.0)
    cores = O.init_cores(dims, ranks, 31)
    src = O.DenseSource(X, P)
    st = O.State(cfg, cores, src)
    def loss():
        E = X - O.tr_reconstruct(st.cores)
        return O.welsch_loss(E, P, 1.0)
    prev = loss()
    for t in range(8):
        rec = O.SweepRecord(3)
        for k in range(3):
            O.block_update(cfg, st, src, k, rec)
            cur = loss()
            assert cur <= prev + 1e-9 * max(1.0, abs(prev))
            prev = cur
        st.t += 1


def test_sigma_inf_equals_huge_fixed_sigma_bitwise():
    """sigma -> inf makes W == 1; FIXED sigma=1e200 (sigma^2 = inf) is bitwise the
    same trajectory as the INF mode (SPEC AC-12)."""
    dims, ranks = [7, 6, 5], [2, 3, 2]
    gt, Xc, X, P = _problem(dims, ranks, 0.7, 40)
    cores = O.init_cores(dims, ranks, 41)
    src = O.DenseSource(X, P)
    a, _ = O.run(O.Config(dims, ranks, sigma_mode=O.SIGMA_INF), cores, src, 3)
    b, _ = O.run(O.Config(dims, ranks, sigma_mode=O.SIGMA_FIXED, sigma=1e200), cores, src, 3)
    for za, zb in zip(a.cores, b.cores):
        assert np.array_equal(za, zb)


def test_rsts_full_sets_reproduce_awrtrd_bitwise():
    """P:246 / SPEC AC-10: sketch sizes >= I_m give the full-data AWRTRD trajectory."""
    dims, ranks = [6, 5, 7, 4], [2, 2, 2, 2]
    gt, Xc, X, P = _problem(dims, ranks, 0.5, 50, outliers=0.1)
    cores = O.init_cores(dims, ranks, 51)
    src = O.DenseSource(X, P)
    a, ra = O.run(O.Config(dims, ranks, sketch=[0, 0, 0, 0], seed=5), cores, src, 2)
    b, rb = O.run(O.Config(dims, ranks, sketch=[6, 99, 7, 4], seed=5), cores, src, 2)
    for za, zb in zip(a.cores, b.cores):
        assert np.array_equal(za, zb)


def test_eq14_sketch_identity():
    """Eq. (14): the subtensor of the TR tensor is the TR tensor of the sampled
    cores (<= 1e-12)."""
    dims, ranks = [6, 5, 7, 4], [2, 3, 2, 2]
    cores = rand_cores(dims, ranks, 60)
    X = O.tr_reconstruct(cores)
    for t in range(5):
        sets = [sample_indices(7, t, 0, m, dims[m], [3, 2, 4, 2][m]) for m in range(4)]
        Xs = X[np.ix_(*sets)]
        Ys = O.tr_reconstruct([c[:, s, :] for c, s in zip(cores, sets)])
        assert np.max(np.abs(Xs - Ys)) <= 1e-12


def test_stationary_at_generator():
    """Cores equal to the generator of a noiseless tensor: d = 0, num = 0 -> skipped (R14)."""
    dims, ranks = [6, 5, 4], [2, 2, 2]
    gt, Xc, X, P = _problem(dims, ranks, 0.6, 70)
    X = Xc                                       # exact, float64
    src = O.DenseSource(X, P)
    cfg = O.Config(dims, ranks, sigma_mode=O.SIGMA_FIXED, sigma=1.0)
    st = O.State(cfg, gt, src)
    rec = O.SweepRecord(3)
    for k in range(3):
        O.block_update(cfg, st, src, k, rec)
    assert all(abs(n) <= 1e-20 for n in rec.num)
    for za, zb in zip(st.cores, gt):
        assert np.max(np.abs(za - zb)) <= 1e-9


def test_stop_metric_equals_gram_of_unfolding():
    """Alg. 1 line 12: D^t = Z_N(2) G_{!=N} Z_N(2)^T equals X_hat_[N] X_hat_[N]^T of
    the model after the sweep (Thm 1 + Eq. 13), so e_t is the change of that Gram."""
    dims, ranks = [6, 5, 4], [2, 3, 2]
    gt, Xc, X, P = _problem(dims, ranks, 0.8, 80, outliers=0.1)
    cfg = O.Config(dims, ranks)
    src = O.DenseSource(X, P)
    st = O.State(cfg, O.init_cores(dims, ranks, 81), src)
    D_list = []
    for t in range(3):
        rec = O.sweep(cfg, st, src)
        Xh = O.tr_reconstruct(st.cores)
        U = O.unfold_shifted(Xh, 2)
        D = U @ U.T
        assert np.max(np.abs(st.D_prev - D)) <= 1e-10 * np.abs(D).max()
        D_list.append(D)
        if t == 0:
            assert math.isnan(rec.stop_e)
        else:
            ref = np.linalg.norm(D_list[-1] - D_list[-2]) / np.linalg.norm(D_list[-1])
            assert abs(rec.stop_e - ref) <= 1e-9 * ref


def test_noiseless_exact_recovery():
    """Noiseless, fully observed TR tensor recovered to <= 1e-4 (SPEC AC-8), sigma = inf."""
    dims, ranks = [8, 7, 6], [2, 2, 2]
    gt, Xc, X, P = _problem(dims, ranks, 1.0, 90)
    X = Xc
    cfg = O.Config(dims, ranks, sigma_mode=O.SIGMA_INF, lambda_rel=1e-9)
    src = O.DenseSource(X, P)
    st, recs = O.run(cfg, O.init_cores(dims, ranks, 91), src, 200)
    assert O.relative_error(st.cores, Xc) <= 1e-4


def test_robust_beats_unweighted_with_outliers():
    """P:129 / SPEC AC-7: correntropy weighting beats sigma = inf under outliers."""
    dims, ranks = [12, 11, 10], [3, 3, 3]
    gt, Xc, X, P = _problem(dims, ranks, 0.8, 100, outliers=0.1, noise=0.05)
    src = O.DenseSource(X, P)
    init = O.init_cores(dims, ranks, 101)
    rob, _ = O.run(O.Config(dims, ranks, sigma_mode=O.SIGMA_RMS), init, src, 20)
    ls, _ = O.run(O.Config(dims, ranks, sigma_mode=O.SIGMA_INF), init, src, 20)
    e_rob, e_ls = O.relative_error(rob.cores, Xc), O.relative_error(ls.cores, Xc)
    assert e_rob <= 0.5 * e_ls


def test_check_gram_inside_sweep():
    """FGMC cache stays coherent with the updated cores through a whole run (Alg. 1 l.10)."""
    dims, ranks = [5, 4, 3, 4], [2, 3, 2, 2]
    gt, Xc, X, P = _problem(dims, ranks, 0.7, 110, outliers=0.1)
    src = O.DenseSource(X, P)
    O.run(O.Config(dims, ranks, sketch=[3, 2, 2, 3], seed=9), O.init_cores(dims, ranks, 111),
          src, 3, check_gram=True)


# ---------------------------------------------------------------- sampler (Alg. 1 line 4)
def test_sampler_basic_properties():
    for (t, k, m, I, s) in [(0, 0, 1, 128, 32), (3, 2, 0, 80, 32), (1, 1, 2, 3, 1), (5, 0, 3, 100, 20)]:
        idx = sample_indices(123, t, k, m, I, s)
        assert len(idx) == s and np.all(np.diff(idx) > 0) and idx[0] >= 0 and idx[-1] < I
        assert np.array_equal(idx, sample_indices(123, t, k, m, I, s))    # deterministic
    assert np.array_equal(sample_indices(1, 0, 0, 1, 10, 10), np.arange(10))
    assert np.array_equal(sample_indices(1, 0, 0, 1, 10, 0), np.arange(10))
    assert np.array_equal(sample_indices(1, 0, 0, 1, 10, 50), np.arange(10))
    a = sample_indices(5, 0, 0, 1, 128, 32)
    assert not np.array_equal(a, sample_indices(5, 1, 0, 1, 128, 32))   # fresh per t
    assert not np.array_equal(a, sample_indices(5, 0, 2, 1, 128, 32))   # per k
    assert not np.array_equal(a, sample_indices(6, 0, 0, 1, 128, 32))   # per seed


def test_sampler_inclusion_frequency_uniform():
    """'randomly and uniformly select': each index is included w.p. s/I."""
    I, s, T = 40, 10, 4000
    counts = np.zeros(I)
    for t in range(T):
        counts[sample_indices(77, t, 1, 0, I, s)] += 1
    p = s / I
    expect = T * p
    # per-index binomial sd * 5
    assert np.max(np.abs(counts - expect)) <= 5 * math.sqrt(T * p * (1 - p))
    chi2 = float(np.sum((counts - expect) ** 2 / (expect * (1 - p))))
    assert chi2 < I + 6 * math.sqrt(2 * I)


def test_philox_output_statistics():
    """Philox4x32-10 words look uniform; one counter-bit flip changes ~half of the bits."""
    n = 1 << 16
    i = np.arange(n, dtype=np.uint64)
    outs = philox4x32_10(i, 3, 5, 7, 0xDEADBEEF, 0x12345678)
    for o in outs:
        u = o.astype(np.float64) / 2 ** 32
        assert abs(u.mean() - 0.5) < 5 * math.sqrt(1 / 12 / n)
        bits = ((o[:, None] >> np.arange(32, dtype=np.uint64)) & np.uint64(1)).mean(axis=0)
        assert np.all(np.abs(bits - 0.5) < 0.02)
    a = np.stack(philox4x32_10(i[:4096], 0, 0, 0, 1, 2))
    b = np.stack(philox4x32_10(i[:4096] ^ np.uint64(1 << 20), 0, 0, 0, 1, 2))
    flips = np.unpackbits((a ^ b).astype(np.uint32).view(np.uint8)).mean()
    assert abs(flips - 0.5) < 0.01
    # keys are 64-bit combinations of words 0 and 1
    kap = sample_keys(9, 1, 2, 3, 16)
    o0, o1, _, _ = philox4x32_10(np.arange(16, dtype=np.uint64), 3, 2, 1, 9, 0)
    assert np.array_equal(kap, (o0 << np.uint64(32)) | o1)


def test_psnr_and_relative_error():
    """PSNR of a constant offset 0.1 at peak 1 is 20 dB."""
    X = np.zeros((4, 4))
    assert abs(O.psnr(X, X + 0.1) - 20.0) <= 1e-12
    assert O.psnr(X, X) == float('inf')


def test_gradient_entries_equals_dense_gradient_block():
    """The entry-wise form of Eq. (9) (used for full-size row checks) equals the dense
    unfolding form on a small random instance, for every block, including sigma = inf."""
    rng = np.random.default_rng(7)
    dims, ranks = [5, 4, 6, 3], [2, 3, 2, 3]
    cores = [rng.standard_normal((ranks[m], dims[m], ranks[(m + 1) % 4])) for m in range(4)]
    X = rng.standard_normal(dims)
    P = rng.random(dims) < 0.4
    idx = np.argwhere(P)
    for k in range(4):
        for sigma, sinf in ((0.7, False), (1.0, True)):
            Xk, Pk = O.unfold_shifted(X, k), O.unfold_shifted(P, k)
            S = O.subchain(cores, k)
            d_dense, E, W = O.gradient_block(Xk, Pk, O.core_unfold2(cores[k]), S, sigma, sinf)
            d_ent, se2 = O.gradient_entries(cores, k, idx, X[P], sigma, sinf)
            assert np.allclose(d_ent, d_dense, rtol=1e-12, atol=1e-12)
            assert abs(se2 - float(np.sum(E[Pk] ** 2))) <= 1e-10 * float(np.sum(E[Pk] ** 2))


# ---------------------------------------------------------------- ablation arms (Sec. 6.1)
@pytest.mark.parametrize("seed", range(3))
def test_local_gram_equals_explicit_gram_of_sampled_subchain(seed):
    """'Local scaled term' arm: the Gram of the subchain of the sampled cores
    (P:239), built as Eq. (13) over the sampled slices, equals S_I^T S_I formed explicitly
    from the sampled subchain rows."""
    dims, ranks = [5, 4, 6, 3], [2, 3, 2, 2]
    cores = rand_cores(dims, ranks, seed + 300)
    rng = np.random.default_rng(seed)
    for k in range(4):
        sets = [np.arange(dims[m]) if m == k else np.sort(rng.choice(dims[m], 2, replace=False))
                for m in range(4)]
        G = O.gram_local(cores, k, sets, ranks)
        Gx = O.gram_explicit(O.subchain(cores, k, sets))
        assert np.linalg.norm(G - Gx) <= 1e-12 * np.linalg.norm(Gx)


def test_local_gram_with_full_sets_is_the_fgmc_gram():
    dims, ranks = [4, 3, 5], [2, 3, 2]
    cores = rand_cores(dims, ranks, 7)
    sets = [np.arange(I) for I in dims]
    Qs = [O.q_matrix(Z) for Z in cores]
    for k in range(3):
        assert np.allclose(O.gram_local(cores, k, sets, ranks), O.gram_fgmc(Qs, k, ranks),
                           rtol=1e-13, atol=0.0)


@pytest.mark.parametrize("scaling", [O.SCALING_NONE, O.SCALING_LOCAL])
def test_ablation_arm_steps_are_exact_line_searches(scaling):
    """Both arms keep Eq. (12)'s exact line search along their own direction: the block step
    minimises the weighted residual along +h (cost(eta) <= cost(0.99 eta), cost(1.01 eta));
    'gradient descent' moves along d itself (d_I instead of h_I)."""
    dims, ranks = [6, 5, 4], [2, 3, 2]
    gt = rand_cores(dims, ranks, 11)
    rng = np.random.default_rng(12)
    X = O.tr_reconstruct(gt) + 0.05 * rng.standard_normal(dims)
    P = rng.random(dims) < 0.7
    cfg = O.Config(dims, ranks, sigma_mode=O.SIGMA_FIXED, sigma=0.8, sketch=[4, 3, 3], seed=5,
                   scaling=scaling)
    src = O.DenseSource(X, P)
    st = O.State(cfg, rand_cores(dims, ranks, 13), src)
    for k in range(3):
        sets = O.index_sets_for_block(cfg, st.t, k)
        Xk, Pk = O.working_set(src, k, sets)
        S = O.subchain(st.cores, k, sets)
        Zk2 = O.core_unfold2(st.cores[k])
        d, E, W = O.gradient_block(Xk, Pk, Zk2, S, st.sigma, False)
        h = O.update_direction(cfg, d, O.gram_fgmc(st.Qs, k, ranks), st.cores, k, sets)
        if scaling == O.SCALING_NONE:
            assert np.array_equal(h, d)
        num, den = float(np.sum(d * h)), O.line_search_den(h, Pk, W, S)
        assert num > 0 and den > 0
        eta = num / den

        def cost(t):
            Et = Xk - (Zk2 + t * h) @ S.T
            return 0.5 * np.sum(W * Pk * Et * Et)
        c0 = cost(eta)
        assert c0 <= cost(0.99 * eta) + 1e-12 and c0 <= cost(1.01 * eta) + 1e-12
        assert c0 < cost(0.0)
        rec = O.SweepRecord(3)
        O.block_update(cfg, st, src, k, rec)
        assert abs(rec.eta[k] - eta) <= 1e-12 * eta


# ---------------------------------------------------------------- robust sigma (R21)
def _py_median(values):
    """Median by sorting in pure Python: the middle element, or the mean of the two middle
    elements of an even count."""
    v = sorted(float(x) for x in values)
    n = len(v)
    return v[n // 2] if n % 2 else 0.5 * (v[n // 2 - 1] + v[n // 2])


def test_mad_sigma_is_the_exact_median():
    """R21: sigma = theta * 1.4826 * median|e| (exact), floored at sigma_min."""
    rng = np.random.default_rng(2)
    cfg = O.Config([2, 2, 2], [1, 1, 1], sigma_mode=O.SIGMA_MAD, sigma_theta=1.5, sigma_min=1e-3)
    for n in (1, 2, 7, 8, 1001, 1000):
        v = np.abs(rng.standard_normal(n)) * 0.3
        assert O.mad_sigma(cfg, v) == pytest.approx(1.5 * 1.4826 * _py_median(v), rel=1e-15)
    assert O.mad_sigma(cfg, [0.1, 0.3]) == pytest.approx(1.5 * 1.4826 * 0.2, rel=1e-15)
    assert O.mad_sigma(cfg, [0.1, 0.2, 0.9]) == pytest.approx(1.5 * 1.4826 * 0.2, rel=1e-15)
    assert O.mad_sigma(cfg, np.zeros(5)) == 1e-3


def test_mad_sigma_is_consistent_for_gaussian_residuals_and_robust_to_outliers():
    """1.4826 median|e| estimates the standard deviation of Gaussian residuals (within the
    sampling error) and, unlike the RMS rule, ignores 20 % gross outliers (P:362's mixture)."""
    rng = np.random.default_rng(4)
    cfg = O.Config([2, 2, 2], [1, 1, 1], sigma_mode=O.SIGMA_MAD)
    e = 0.05 * rng.standard_normal(200000)
    assert abs(O.mad_sigma(cfg, np.abs(e)) - 0.05) <= 0.05 * 0.01
    out = np.where(rng.random(e.size) < 0.2, rng.uniform(-10, 10, e.size), e)
    mad = O.mad_sigma(cfg, np.abs(out))
    rms = float(np.sqrt(np.mean(out * out)))
    assert mad < 0.2 and rms > 2.0


# ---------------------------------------------------------------- uniform row sampling (R22)
def test_rows_of_a_full_enumeration_equal_the_subtensor_forms():
    """Explicit-row working set and subchain: listing every multi-index of a product set in
    Thm 1's order (i_{k+1} fastest) reproduces working_set / subchain of that set."""
    dims, ranks = [4, 3, 5, 2], [2, 3, 2, 2]
    cores = rand_cores(dims, ranks, 21)
    rng = np.random.default_rng(22)
    X = rng.standard_normal(dims)
    P = rng.random(dims) < 0.6
    src = O.DenseSource(X, P)
    for k in range(4):
        sets = [np.arange(I) for I in dims]
        order = [(k + 1 + q) % 4 for q in range(3)]
        grids = np.meshgrid(*[sets[m] for m in order[::-1]], indexing="ij")   # slowest first
        lists = [None] * 4
        lists[k] = sets[k]
        for g, m in zip(grids, order[::-1]):
            lists[m] = g.reshape(-1)
        Xr, Pr = O.working_set_rows(src, k, lists)
        Xs, Ps = O.working_set(src, k, sets)
        assert np.array_equal(Xr, Xs) and np.array_equal(Pr, Ps)
        assert np.allclose(O.subchain_rows(cores, k, lists), O.subchain(cores, k, sets), rtol=1e-13, atol=1e-14)


def test_row_samples_are_uniform_with_replacement_and_decode_in_thm1_order():
    cfg = O.Config([3, 4, 5], [1, 1, 1], sketch=[0, 4, 5], seed=9, sampling=O.SAMPLING_ROWS)
    counts = np.zeros((4, 5))
    for t in range(300):
        L = O.row_samples(cfg, t, 0)
        assert len(L[1]) == len(L[2]) == 20 and np.array_equal(L[0], np.arange(3))
        np.add.at(counts, (L[1], L[2]), 1)
    expected = 300 * 20 / 20.0
    chi2 = float(np.sum((counts - expected) ** 2 / expected))
    assert chi2 < 60.0                                   # 19 dof, p ~ 1e-5
    # decode: the same Philox word, i_{k+1} fastest
    L = O.row_samples(cfg, 7, 1)                        # k = 1: modes 2 (fastest), then 0
    o0, o1, _, _ = O.philox4x32_10(np.arange(len(L[2]), dtype=np.uint64), O.ROW_TAG, 1, 7, 9, 0)
    rho = [(int((a << np.uint64(32)) | b) * 15) >> 64 for a, b in zip(o0, o1)]
    assert [r % 5 for r in rho] == list(L[2]) and [r // 5 for r in rho] == list(L[0])


def test_row_sampling_block_step_is_an_exact_line_search():
    dims, ranks = [6, 5, 4], [2, 3, 2]
    gt = rand_cores(dims, ranks, 31)
    rng = np.random.default_rng(32)
    X = O.tr_reconstruct(gt) + 0.05 * rng.standard_normal(dims)
    P = rng.random(dims) < 0.7
    src = O.DenseSource(X, P)
    cfg = O.Config(dims, ranks, sigma_mode=O.SIGMA_FIXED, sigma=0.8, sketch=[4, 3, 3], seed=5,
                   sampling=O.SAMPLING_ROWS)
    st = O.State(cfg, rand_cores(dims, ranks, 33), src)
    for k in range(3):
        L = O.row_samples(cfg, st.t, k)
        Xk, Pk = O.working_set_rows(src, k, L)
        S = O.subchain_rows(st.cores, k, L)
        Zk2 = O.core_unfold2(st.cores[k])
        d, E, W = O.gradient_block(Xk, Pk, Zk2, S, st.sigma, False)
        h = O.update_direction(cfg, d, O.gram_fgmc(st.Qs, k, ranks), st.cores, k, L)
        eta = float(np.sum(d * h)) / O.line_search_den(h, Pk, W, S)

        def cost(t):
            Et = Xk - (Zk2 + t * h) @ S.T
            return 0.5 * np.sum(W * Pk * Et * Et)
        assert cost(eta) <= min(cost(0.99 * eta), cost(1.01 * eta)) + 1e-12
        rec = O.SweepRecord(3)
        O.block_update(cfg, st, src, k, rec)
        assert abs(rec.eta[k] - eta) <= 1e-12 * eta
