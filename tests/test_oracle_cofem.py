"""Pins for oracle/cofem.py and oracle/exact.py: direct solves, closed forms,
exact EM, estimator statistics."""
import numpy as np
import pytest

import synth
from oracle import closed_forms as cf
from oracle.cofem import cofem_em, estep, mstep, pcg, support, tau_of
from oracle.exact import dense_phi, exact_em, exact_posterior, log_evidence
from oracle.operators import CircConvOp, DCT2MaskedOp, DenseOp
from oracle.philox import rademacher_probes


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


# ---------------------------------------------------------------- PCG
@pytest.mark.parametrize("precond", [False, True])
def test_pcg_identity_one_iteration(precond):
    B = np.random.default_rng(0).standard_normal((7, 3))
    X, rep = pcg(lambda V: V, B, np.ones(7), U=1, precond=precond)
    assert np.allclose(X, B, rtol=1e-15)


def test_pcg_diagonal():
    d = np.array([1.0, 2.0, 4.0])
    X, _ = pcg(lambda V: d[:, None] * V, d[:, None].copy(), d, U=1, precond=True)
    assert np.allclose(X[:, 0], 1.0)
    X, _ = pcg(lambda V: d[:, None] * V, d[:, None].copy(), d, U=3, precond=False)
    assert np.allclose(X[:, 0], 1.0, rtol=1e-12)


@pytest.mark.parametrize("precond", [False, True])
@pytest.mark.parametrize("trial", range(10))
def test_pcg_vs_direct_solve(trial, precond):
    rng = np.random.default_rng(trial)
    D = int(rng.integers(2, 64))
    M = rng.standard_normal((D, D))
    A = M.T @ M + np.eye(D) * rng.uniform(0.1, 2)
    B = rng.standard_normal((D, int(rng.integers(1, 8))))
    X, _ = pcg(lambda V: A @ V, B, np.diag(A).copy(), U=4 * D, precond=precond)
    assert rel(X, np.linalg.solve(A, B)) < 1e-8


def test_pcg_column_permutation_and_anorm_monotone():
    rng = np.random.default_rng(3)
    M = rng.standard_normal((30, 30))
    A = M.T @ M + np.eye(30)
    B = rng.standard_normal((30, 4))
    X, _ = pcg(lambda V: A @ V, B, np.diag(A).copy(), U=10)
    perm = [2, 0, 3, 1]
    Xp, _ = pcg(lambda V: A @ V, B[:, perm], np.diag(A).copy(), U=10)
    assert np.allclose(Xp, X[:, perm], rtol=1e-14, atol=1e-14)
    Xs = np.linalg.solve(A, B)
    errs = []
    for u in range(1, 25):
        Xu, _ = pcg(lambda V: A @ V, B, np.diag(A).copy(), U=u)
        E = Xu - Xs
        errs.append(np.sum(E * (A @ E), axis=0))
    errs = np.array(errs)
    assert np.all(np.diff(errs, axis=0) <= 1e-12 * errs[0])


def test_pcg_freeze_rules():
    # zero rhs -> rho0 = 0 -> frozen at iteration 0, x = 0 (R5)
    B = np.zeros((5, 1))
    X, rep = pcg(lambda V: V, B, np.ones(5), U=5)
    assert rep.frozen_at[0] == 0 and not rep.nonfinite[0] and np.all(X == 0)
    # converged column freezes once rho <= 1e-30 rho0 (diagonal A converges in 1 step)
    d = np.linspace(1, 3, 6)
    X, rep = pcg(lambda V: d[:, None] * V, np.ones((6, 1)), d, U=50)
    assert 0 < rep.frozen_at[0] < 50 and np.allclose(X[:, 0], 1 / d)
    # non-finite operator output flags the column
    X, rep = pcg(lambda V: V * np.nan, np.ones((3, 2)), np.ones(3), U=3)
    assert rep.nonfinite.all()


# ---------------------------------------------------------------- eps stopping (NEXT-1, reading R19)
def test_eps_stopping_identity_one_step():
    """SPEC S:109 with a tolerance: A = I converges in one step; every column freezes at i = 1."""
    B = np.random.default_rng(1).standard_normal((9, 3))
    X, rep = pcg(lambda V: V, B, np.ones(9), U=10, precond=False, tau=tau_of(1e-8))
    assert np.array_equal(X, B) and np.all(rep.frozen_at == 1) and rep.iters_run == 2


@pytest.mark.parametrize("precond", [False, True])
def test_eps_stopping_first_iteration_meeting_the_criterion(precond):
    """Each column stops at the first iteration where rho <= eps^2 rho0 (plain CG: the recursive
    ||r_j|| <= eps ||b_j||); its iterate equals the fixed-U iterate with U = that iteration count,
    one iteration earlier the criterion did not hold, and at the end the paper's Frobenius
    criterion ||AX - B||_F / ||B||_F < eps holds (checked with the true residual)."""
    rng = np.random.default_rng(7)
    D, eps = 40, 1e-6
    M = rng.standard_normal((D, D))
    A = M.T @ M + np.eye(D)
    B = rng.standard_normal((D, 4)) * np.array([1e-3, 1.0, 1e3, 5.0])      # very different column scales
    diag = np.diag(A).copy()
    X, rep = pcg(lambda V: A @ V, B, diag, U=4 * D, precond=precond, tau=tau_of(eps))
    assert np.all(rep.frozen_at > 0) and np.all(rep.frozen_at < 4 * D) and not rep.nonfinite.any()
    minv = 1.0 / diag if precond else np.ones(D)
    for j in range(4):
        u = int(rep.frozen_at[j])
        Xu, _ = pcg(lambda V: A @ V, B[:, [j]], diag, U=u, precond=precond)
        assert rel(Xu[:, 0], X[:, j]) < 1e-7        # same recurrence; BLAS order differs with the block width, amplified by kappa
        Xp, _ = pcg(lambda V: A @ V, B[:, [j]], diag, U=u - 1, precond=precond)
        r_now, r_prev = B[:, j] - A @ X[:, j], B[:, j] - A @ Xp[:, 0]
        rho0 = B[:, j] @ (minv * B[:, j])
        assert r_now @ (minv * r_now) <= eps ** 2 * rho0 * 1.01
        assert r_prev @ (minv * r_prev) > eps ** 2 * rho0 * 0.99
    if not precond:
        assert np.linalg.norm(A @ X - B) / np.linalg.norm(B) < eps


def test_eps_zero_is_the_fixed_u_run():
    rng = np.random.default_rng(2)
    M = rng.standard_normal((20, 20))
    A = M.T @ M + np.eye(20)
    B = rng.standard_normal((20, 3))
    X0, _ = pcg(lambda V: A @ V, B, np.diag(A).copy(), U=15)
    X1, _ = pcg(lambda V: A @ V, B, np.diag(A).copy(), U=15, tau=tau_of(0.0))
    assert np.array_equal(X0, X1) and tau_of(0.0) == 1e-30 and tau_of(1e-3) == 1e-6


# ---------------------------------------------------------------- E/M-step
def test_estep_jacobi_diag_uses_alpha_one_iteration_exact():
    """Pins jacobi_diag's alpha term (R6, diag(A) = beta colsq + alpha, A of Eq. 7 / P:133 depends
    on alpha) through estep.  Phi with orthogonal columns of different norms makes
    A = beta Phi^T Phi + diag(alpha) diagonal; Jacobi-PCG with the TRUE diagonal then solves
    every column in one iteration (z = A^-1 r is already the solution direction, a = 1), so at
    U = 1 and a non-uniform alpha: mu = b0_d / (beta c_d + alpha_d) and, since each x_k is
    exact, s_d = Sigma_dd = 1 / (beta c_d + alpha_d) (Eq. 4/6) for any probes.  A diagonal
    without alpha (or with alpha = 1) leaves z off the solution direction and misses both."""
    rng = np.random.default_rng(7)
    D = 12
    Q, _ = np.linalg.qr(rng.standard_normal((16, D)))       # orthonormal columns (16 x 12)
    c = rng.uniform(0.5, 3.0, D)
    phi = Q * np.sqrt(c)[None, :]                           # Phi^T Phi = diag(c) exactly (up to u)
    y = rng.standard_normal(16)
    beta = 2.0
    alpha = rng.uniform(0.2, 5.0, D)                        # non-uniform prior precisions
    mu, s, rep = estep(DenseOp(phi), y, beta, alpha, K=3, seed=4, t=0, U=1)
    lam = beta * c + alpha                                  # the exact eigenvalues of A
    b0 = beta * (Q.T @ y) * np.sqrt(c)                      # beta Phi^T y, computed from Q, c
    assert np.allclose(mu, b0 / lam, rtol=1e-10, atol=0), np.max(np.abs(mu * lam / b0 - 1))
    assert np.allclose(s, 1.0 / lam, rtol=1e-10, atol=0), np.max(np.abs(s * lam - 1))


def test_estep_phi_zero_gives_identity_system():
    op = DenseOp(np.zeros((3, 10)))
    mu, s, _ = estep(op, np.ones(3), 5.0, np.ones(10), K=4, seed=1, t=0, U=5)
    assert np.all(mu == 0) and np.allclose(s, 1.0, rtol=0, atol=0)


def test_estep_scalar_closed_form():
    op = DenseOp(np.ones((1, 1)))
    mu, s, _ = estep(op, np.array([2.0]), 1.0, np.ones(1), K=3, seed=9, t=0, U=3)
    assert np.allclose(mu, 1.0, rtol=1e-15) and np.allclose(s, 0.5, rtol=1e-15)


def test_estep_mu_vs_exact_d32():
    rng = np.random.default_rng(1)
    phi = rng.standard_normal((16, 32))
    y = rng.standard_normal(16)
    alpha = rng.uniform(0.5, 2.0, 32)
    mu, s, _ = estep(DenseOp(phi), y, 3.0, alpha, K=4, seed=0, t=0, U=200)
    mu_ex, _ = exact_posterior(phi, 3.0, alpha, y)
    assert rel(mu, mu_ex) < 1e-10


def test_mstep_examples():
    assert np.allclose(mstep(np.zeros(3), np.ones(3)), 1.0)
    assert np.allclose(mstep(np.array([1.0, 0.0]), np.array([0.0, 0.5])), [1.0, 2.0])
    assert mstep(np.array([0.0]), np.array([-0.1]))[0] == 1e12                         # S:226 floor + clamp
    assert mstep(np.array([0.0]), np.array([1e-20]))[0] == 1e12


def test_em_phi_zero_fixed_point_and_scalar_trajectory():
    op = DenseOp(np.zeros((2, 4)))
    a, _, _ = cofem_em(op, np.ones(2), 1.0, T=1, K=2, seed=0, U=3)
    assert np.allclose(a, 1.0)
    # scalar D = N = 1, Phi = 1, beta = 1, y = 2: alpha = 1 -> 1/(1 + .5) -> 1/(1.2^2 + .6)
    op = DenseOp(np.ones((1, 1)))
    trace = []
    cofem_em(op, np.array([2.0]), 1.0, T=2, K=2, seed=0, U=3, trace=trace)
    assert np.isclose(trace[0][0][0], 1 / 1.5, rtol=1e-14)
    assert np.isclose(trace[1][0][0], 1 / (1.2 ** 2 + 0.6), rtol=1e-14)


def test_em_resume_equals_continuous_run():
    w = synth.dense(20, 50, 3, K=4, U=40, T=4, seed=2)
    op = DenseOp(w.phi)
    a4, mu4, s4 = cofem_em(op, w.y, w.beta, T=4, K=4, seed=3, U=40)
    a2, _, _ = cofem_em(op, w.y, w.beta, T=2, K=4, seed=3, U=40)
    b4, nu4, r4 = cofem_em(op, w.y, w.beta, T=2, K=4, seed=3, U=40, alpha_init=a2, t0=2)
    assert np.array_equal(a4, b4) and np.array_equal(mu4, nu4) and np.array_equal(s4, r4)


# ---------------------------------------------------------------- closed forms
@pytest.mark.parametrize("beta", [1.0, 1e4])
def test_full_mask_dct_em_trajectory(beta):
    rows, cols = 16, 8
    D = rows * cols
    rng = np.random.default_rng(4)
    y = rng.standard_normal(D) * 0.5
    op = DCT2MaskedOp(rows, cols, np.arange(D))
    aT, muT, sT = cofem_em(op, y, beta, T=6, K=3, seed=1, U=20)
    u = cf.dct_phiT(rows, cols, np.arange(D), y)
    eT, emu, es = cf.full_mask_dct_em(u, beta, 6)
    assert rel(aT, eT) < 1e-12 and rel(muT, emu) < 1e-12 and rel(sT, es) < 1e-12


def test_full_mask_scalar_recursion_values():
    # beta = 1, u = 2: alpha = 1 -> 0.666667 -> 0.490196 -> 0.404482 -> ... -> 1/3
    vals = [cf.full_mask_dct_em(np.array([2.0]), 1.0, T)[0][0] for T in (1, 2, 3)]
    assert np.allclose(vals, [2 / 3, 1 / 2.04, 0.404482], atol=1e-6)
    assert np.isclose(cf.full_mask_dct_em(np.array([2.0]), 1.0, 200)[0][0], 1 / 3, rtol=1e-6)


@pytest.mark.parametrize("conv", [0, 1])
def test_masked_dct_estep1_closed_form(conv):
    w = synth.dct(32, 32, 256, 10, K=6, U=200, T=1, seed=0, convention=conv)
    op = DCT2MaskedOp(w.rows, w.cols, w.obs_idx, conv)
    mu, s, rep, X = estep(op, w.y, w.beta, np.ones(w.D), w.K, seed=11, t=0, U=200, return_x=True)
    P = rademacher_probes(w.D, w.K, 11, 0)
    emu, es, eX = cf.masked_dct_estep1(w.rows, w.cols, w.obs_idx, w.y, w.beta, P, conv)
    assert rel(mu, emu) < 1e-10 and rel(s, es) < 1e-10 and rel(X[:, 1:], eX) < 1e-10


def test_circconv_estep1_closed_form():
    w = synth.circconv(4099, 64, 4, K=4, U=150, T=1, seed=0)
    op = CircConvOp(w.taps, w.D)
    mu, s, rep = estep(op, w.y, w.beta, np.ones(w.D), w.K, seed=2, t=0, U=1500)
    P = rademacher_probes(w.D, w.K, 2, 0)
    emu, es, _ = cf.circconv_estep(w.taps, w.D, w.y, w.beta, 1.0, P)
    assert rel(mu, emu) < 1e-8 and rel(s, es) < 1e-8


def test_dense_estep1_closed_form():
    w = synth.dense(60, 200, 5, K=5, U=200, T=1, seed=0)
    op = DenseOp(w.phi)
    mu, s, _ = estep(op, w.y, w.beta, np.ones(w.D), w.K, seed=0, t=0, U=400)
    P = rademacher_probes(w.D, w.K, 0, 0)
    emu, es, _ = cf.dense_estep(w.phi, w.y, w.beta, 1.0, P)
    assert rel(mu, emu) < 1e-8 and rel(s, es) < 1e-8


# ---------------------------------------------------------------- estimator (Eq. 6, Proposition)
def test_diagonal_estimator_unbiased_and_variance():
    rng = np.random.default_rng(0)
    M = rng.standard_normal((16, 16))
    Sig = M @ M.T / 16 + np.eye(16)
    def est(K, t):
        P = rademacher_probes(16, K, seed=77, t=t)
        return np.mean(P * (Sig @ P), axis=1)
    R = 2000
    S20 = np.array([est(20, t) for t in range(R)])
    m, se = S20.mean(0), S20.std(0) / np.sqrt(R)
    assert np.all(np.abs(m - np.diag(Sig)) < 3.5 * se)
    S80 = np.array([est(80, R + t) for t in range(R)])
    ratio = S20.var(0).mean() / S80.var(0).mean()
    assert 2.5 < ratio < 6.5
    D = np.diag(np.diag(Sig))                                                # exact on diagonal
    P = rademacher_probes(16, 3, 1, 0)
    assert np.allclose(np.mean(P * (D @ P), axis=1), np.diag(Sig))


def test_estep_s_large_K_matches_exact_diag():
    rng = np.random.default_rng(5)
    phi = rng.standard_normal((16, 32))
    y = rng.standard_normal(16)
    mu, s, _ = estep(DenseOp(phi), y, 2.0, np.ones(32), K=2000, seed=3, t=0, U=100)
    _, Sig = exact_posterior(phi, 2.0, np.ones(32), y)
    assert np.max(np.abs(s - np.diag(Sig)) / np.diag(Sig)) < 0.15


# ---------------------------------------------------------------- exact EM + parity of CoFEM vs EM
def test_exact_posterior_scalar_and_prior_only():
    mu, S = exact_posterior(np.ones((1, 1)), 1.0, np.ones(1), np.array([2.0]))
    assert np.isclose(mu[0], 1.0) and np.isclose(S[0, 0], 0.5)
    mu, S = exact_posterior(np.zeros((2, 3)), 1.0, np.array([1.0, 2.0, 4.0]), np.ones(2))
    assert np.allclose(mu, 0) and np.allclose(np.diag(S), [1, 0.5, 0.25])


def test_log_evidence_values_and_monotone():
    assert np.isclose(log_evidence(np.zeros((1, 1)), 1.0, np.ones(1), np.zeros(1)), -0.5 * np.log(2 * np.pi))
    assert np.isclose(log_evidence(np.ones((1, 1)), 1.0, np.ones(1), np.zeros(1)),
                      -0.5 * (np.log(2 * np.pi) + np.log(2)))
    for seed in range(5):
        w = synth.dense(32, 64, 4, K=1, U=1, T=1, seed=seed)
        phi = w.phi.astype(np.float64)
        trace = []
        exact_em(phi, 100.0, w.y, T=15, trace=trace)
        ev = [log_evidence(phi, 100.0, np.ones(64), w.y)] + [log_evidence(phi, 100.0, a, w.y) for a, _ in trace]
        assert np.all(np.diff(ev) > -1e-8)


def test_cofem_first_iteration_mu_equals_exact_em():
    # SPEC acceptance 1: D=128, N=32, mu of E-step 1 within 1e-6 of exact EM
    w = synth.dense(32, 128, 5, K=20, U=256, T=1, seed=0)
    w_beta = 1 / 0.005 ** 2
    op = DenseOp(w.phi)
    mu, _, _ = estep(op, w.y, w_beta, np.ones(128), K=20, seed=0, t=0, U=256)
    mu_ex, _ = exact_posterior(w.phi.astype(np.float64), w_beta, np.ones(128), w.y)
    assert rel(mu, mu_ex) < 1e-6


def test_cofem_nrmse_tracks_exact_em():
    # P:166 "CoFEM converges at the same rate as EM" (acceptance 3-4): D=256,
    # f=4, K=20, U=400, the paper's §4.1 data.  The stochastic s shifts the steep
    # descent by an iteration or so, so "same rate" is checked as: the iteration at
    # which NRMSE first drops below 20% differs by <= 2, and after 30 iterations
    # both reach the same NRMSE (< 1 pp apart, < 5%).
    final = []
    for seed in range(3):
        w = synth.paper_dense(256, 4, seed=seed)
        t_c, t_e = [], []
        cofem_em(DenseOp(w.phi), w.y, w.beta, T=30, K=20, seed=seed, U=400, trace=t_c)
        exact_em(w.phi.astype(np.float64), w.beta, w.y, T=30, trace=t_e)
        nr = lambda mu: 100 * np.linalg.norm(mu - w.z_true) / np.linalg.norm(w.z_true)
        first = lambda tr: next(i for i, x in enumerate(tr) if nr(x[1]) < 20.0)
        assert abs(first(t_c) - first(t_e)) <= 2
        final.append((nr(t_c[-1][1]), nr(t_e[-1][1])))
    for c, e in final:
        assert abs(c - e) < 1.0 and c < 5.0


def test_support_threshold():
    assert list(support(np.array([1.0, -0.002, 0.0005, 0.0]))) == [True, True, False, False]


# ---------------------------------------------------------------- R20: warm start (NEXT-1)
def test_warm_start_from_zero_is_the_cold_start():
    w = synth.dense(30, 80, 4, K=3, U=20, T=1, seed=3)
    op = DenseOp(w.phi)
    a = np.random.default_rng(1).uniform(0.5, 2.0, w.D)
    m1, s1, _ = estep(op, w.y, w.beta, a, 3, 2, 0, 20)
    m2, s2, _ = estep(op, w.y, w.beta, a, 3, 2, 0, 20, mu0=np.zeros(w.D))
    assert np.array_equal(m1, m2) and np.array_equal(s1, s2)


def test_warm_start_at_the_solution_stops_at_once():
    """x0 = A^-1 b: the residual is ~0, so the mean column freezes in its first iteration (R5 with
    rho0 = b^T M^-1 b) and mu stays the exact solution (direct solve)."""
    w = synth.dense(30, 80, 4, K=2, U=20, T=1, seed=4)
    op = DenseOp(w.phi)
    a = np.random.default_rng(2).uniform(0.5, 2.0, w.D)
    A = w.beta * op.phi.T @ op.phi + np.diag(a)
    b0 = w.beta * op.phi.T @ w.y.astype(np.float64)
    xs = np.linalg.solve(A, b0)
    mu, _, rep = estep(op, w.y, w.beta, a, 2, 1, 0, 20, mu0=xs)
    assert rel(mu, xs) < 1e-12
    assert rep.frozen_at[0] <= 1


def test_warm_start_converges_to_the_same_solution():
    """Warm-started CG converges to A^-1 b like the cold start (direct solve), and a good warm
    start reaches a given accuracy in fewer iterations."""
    w = synth.dense(40, 120, 6, K=2, U=60, T=1, seed=5)
    op = DenseOp(w.phi)
    a = np.random.default_rng(3).uniform(0.2, 5.0, w.D)
    A = w.beta * op.phi.T @ op.phi + np.diag(a)                 # condition number ~1e5
    xs = np.linalg.solve(A, w.beta * op.phi.T @ w.y.astype(np.float64))
    near = xs * (1.0 + 1e-3 * np.random.default_rng(4).standard_normal(w.D))
    mu_w, _, _ = estep(op, w.y, w.beta, a, 2, 1, 0, 300, mu0=near)
    assert rel(mu_w, xs) < 1e-10
    for U in (5, 20, 60, 120):          # measured: cold 0.69 / 0.61 / 1.0e-2 / 2.4e-5, warm 1e-3 .. 7e-8
        e_cold = rel(estep(op, w.y, w.beta, a, 2, 1, 0, U)[0], xs)
        e_warm = rel(estep(op, w.y, w.beta, a, 2, 1, 0, U, mu0=near)[0], xs)
        assert e_warm < 1e-2 * e_cold, (U, e_cold, e_warm)


def test_warm_start_em_first_estep_is_cold():
    w = synth.dense(30, 80, 4, K=3, U=15, T=1, seed=6)
    op = DenseOp(w.phi)
    a1, m1, s1 = cofem_em(op, w.y, w.beta, 1, 3, 5, 15)
    a2, m2, s2 = cofem_em(op, w.y, w.beta, 1, 3, 5, 15, warm_start=True)
    assert np.array_equal(a1, a2) and np.array_equal(m1, m2)


# ---------------------------------------------------------------- R22: multi-task SBL (NEXT-4)
def test_multitask_one_task_is_algorithm1():
    from oracle.cofem import cofem_em_multi, estep_multi
    w = synth.dense(30, 80, 4, K=3, U=20, T=1, seed=7)
    op = DenseOp(w.phi)
    mu, s, _ = estep(op, w.y, w.beta, np.ones(w.D), 3, 5, 0, 20)
    MU, s2, _ = estep_multi(op, w.y[:, None], w.beta, np.ones(w.D), 3, 5, 0, 20)
    assert np.array_equal(MU[:, 0], mu) and np.array_equal(s2, s)
    a1, m1, _ = cofem_em(op, w.y, w.beta, 3, 3, 5, 20)
    a2, M2, _ = cofem_em_multi(op, w.y[:, None], w.beta, 3, 3, 5, 20)
    assert np.array_equal(a1, a2) and np.array_equal(M2[:, 0], m1)


def test_multitask_diagonal_closed_form():
    """Phi with orthogonal columns (A diagonal, Jacobi PCG exact in one iteration): every task's
    mu_l,d = beta (Phi^T y_l)_d / lam_d, s_d = 1/lam_d, and the multi-task M-step is
    alpha_d = 1 / (mean_l mu_l,d^2 + 1/lam_d), lam = beta c + alpha (R22)."""
    from oracle.cofem import cofem_em_multi
    rng = np.random.default_rng(11)
    D, N, L = 10, 14, 3
    Q, _ = np.linalg.qr(rng.standard_normal((N, D)))
    c = rng.uniform(0.5, 2.0, D)
    phi = Q * np.sqrt(c)[None, :]
    Y = rng.standard_normal((N, L))
    beta = 3.0
    a, MU, s = cofem_em_multi(DenseOp(phi), Y, beta, 1, 2, 0, 1, alpha_init=np.full(D, 0.7))
    lam = beta * c + 0.7
    u = beta * (Q.T @ Y) * np.sqrt(c)[:, None]              # beta Phi^T Y
    assert np.allclose(MU, u / lam[:, None], rtol=1e-10, atol=0)
    assert np.allclose(s, 1.0 / lam, rtol=1e-10, atol=0)
    assert np.allclose(a, 1.0 / (np.mean((u / lam[:, None]) ** 2, axis=1) + 1.0 / lam), rtol=1e-10, atol=0)


def test_multitask_matches_exact_multitask_em():
    """Converged CG at D = 40 and many probes: the multi-task CoFEM EM tracks the exact multi-task
    EM (Cholesky: Sigma shared, alpha = L / sum_l (mu_l^2 + Sigma_dd))."""
    from oracle.cofem import cofem_em_multi
    from oracle.exact import exact_posterior
    rng = np.random.default_rng(12)
    D, N, L = 40, 20, 4
    phi = rng.standard_normal((N, D)) / np.sqrt(N)
    Y = rng.standard_normal((N, L))
    beta = 50.0
    alpha = np.ones(D)
    for _ in range(3):
        MUe = []
        for l in range(L):
            mu, Sig = exact_posterior(phi, beta, alpha, Y[:, l])
            MUe.append(mu)
        MUe = np.array(MUe).T
        alpha = L / np.sum(MUe ** 2 + np.diag(Sig)[:, None], axis=1)
    from oracle.cofem import estep_multi
    MU1, _, _ = estep_multi(DenseOp(phi), Y, beta, np.ones(D), 8, 1, 0, 200)
    MU1e = np.array([exact_posterior(phi, beta, np.ones(D), Y[:, l])[0] for l in range(L)]).T
    assert rel(MU1, MU1e) < 1e-8                # E-step 1: the task means do not depend on the probes
    a, MU, s = cofem_em_multi(DenseOp(phi), Y, beta, 3, 4000, 1, 200)
    assert rel(1 / a, 1 / alpha) < 0.05         # s is the K-probe estimate of diag(Sigma)
    assert rel(MU, MUe) < 0.05
