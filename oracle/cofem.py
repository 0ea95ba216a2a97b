"""Algorithm 1 (CovarianceFreeEM) in fp64, step by step (oracle; test infrastructure only).

Paper passages followed:
  Eq. 5   Sigma^-1 mu = beta Phi^T y: mu solves A x = b, b = beta Phi^T y
  Eq. 6   s = (1/K) sum_k p_k o Sigma p_k, with Sigma p_k = x_k solving A x = p_k
  Eq. 7   A X = B, A = beta Phi^T Phi + diag(alpha), B = [probes | mean]
  Eq. 8   alpha_new = 1 / (mu o mu + s)
  §3.2   conjugate gradient, matrix-matrix applies, at most U iterations
  Alg. 1 the EM loop; returns alpha, mu, s

Readings of silent/ambiguous passages:
  R2  column 0 of B is the mean system b0 = beta Phi^T y, columns 1..K the probes
  R3  "block" CG = K+1 column-independent CG recurrences batched into one
      matrix-matrix apply per iteration (per-column step scalars), not O'Leary
      block-CG
  R4  X0 = 0 every E-step (no warm start)
  R5  fixed U iterations; a column freezes (stops updating) when
      !(gamma > 0) or !(rho > 1e-30 rho0) or gamma/rho non-finite
  R6  Jacobi preconditioner z = r / (beta colsq + alpha) (BASELINE.json); the
      paper's plain CG is precond=False
  R7  M-step floor 1e-12 and clamp 1e12
  R19 (NEXT-1) the paper's stopping rule ||A X - B||_F / ||B||_F < eps applied per
      column ("columns that individually converge are frozen"): rtol = eps > 0
      raises the R5 threshold to tau = eps^2, i.e. freeze column j once
      rho_j <= eps^2 rho_j(0) with rho = r^T M^-1 r (plain CG: ||r_j|| <= eps ||b_j||); once
      every column is frozen the Frobenius criterion holds.  rtol = 0: fixed U (R5).
  R9  Algorithm 1 returns alpha after the last M-step and mu, s of the last E-step
  R20 (NEXT-1, optional) warm start: the paper's initial guess is unstated (SPEC S:254-256
      lists warm starts as unvalidated); with warm_start the mean system's CG starts from the
      previous E-step's mu (x = mu_prev, r = b0 - A mu_prev), the probes from 0 (they are fresh),
      and rho0 stays b^T M^-1 b so the freeze threshold is relative to b.  Off by default (R4).
  R22 (NEXT-4) multi-task SBL (P:179 names it, no procedure): L tasks y_l = Phi z_l + noise share
      Phi, beta and alpha (z_l ~ N(0, diag(alpha)^-1)); Sigma is shared, so one batched solve of
      A X = [beta Phi^T y_1 .. beta Phi^T y_L | p_1 .. p_K] gives mu_l and the same estimator s,
      and maximising sum_l E[log p(z_l | alpha)] gives alpha = L / sum_l (mu_l^2 + s)
      = 1 / (mean_l mu_l^2 + s).  L = 1 is Algorithm 1.
"""
import numpy as np

from .operators import gram_apply
from .philox import rademacher_probes

FREEZE_TAU = 1e-30
DEN_FLOOR = 1e-12
ALPHA_MAX = 1e12


class PCGReport:
    def __init__(self, m):
        self.frozen_at = np.full(m, -1, dtype=np.int64)   # iteration index at which a column froze
        self.nonfinite = np.zeros(m, dtype=bool)
        self.iters_run = 0
        self.rho_hist = []                                # per-iteration rho (recursive residual^2, M-norm)


def pcg(apply_A, B, diag, U, precond=True, tau=FREEZE_TAU, X0=None):
    """Jacobi-preconditioned CG on every column of B, column-independently (R3-R6).

    Per column j, the textbook PCG recurrence:
        x = 0, r = b, z = M^-1 r, p = z, rho = r^T z, rho0 = rho
    (X0 given -- reading R20, NEXT-1 warm start: x = x0, r = b - A x0, and rho0 = b^T M^-1 b, the
    cold-start value, so the freeze threshold stays relative to b as in the paper's criterion
    ||A X - B||_F / ||B||_F < eps)
        repeat U times (skipping frozen columns):
            q = A p,  gamma = p^T q
            freeze if !(gamma > 0) or !(rho > tau rho0) or non-finite
            a = rho / gamma;  x += a p;  r -= a q
            z = M^-1 r;  rho' = r^T z;  p = z + (rho'/rho) p;  rho = rho'
    Every x_j is materialised (no fused estimator).  Returns (X, PCGReport).
    """
    B = np.asarray(B, dtype=np.float64)
    D, m = B.shape
    minv = 1.0 / diag if precond else np.ones(D)
    rho0 = np.sum(B * (B * minv[:, None]), axis=0)
    if X0 is None:
        X = np.zeros((D, m))
        R = B.copy()
    else:
        X = np.asarray(X0, dtype=np.float64).copy()
        R = B - apply_A(X)
    Z = R * minv[:, None]
    P = Z.copy()
    rho = np.sum(R * Z, axis=0)
    active = np.ones(m, dtype=bool)
    rep = PCGReport(m)
    for i in range(U):
        if not active.any():
            break
        rep.iters_run = i + 1
        idx = np.nonzero(active)[0]
        Q = apply_A(P[:, idx])
        gamma = np.sum(P[:, idx] * Q, axis=0)
        r_i = rho[idx]
        finite = np.isfinite(gamma) & np.isfinite(r_i)
        ok = finite & (gamma > 0) & (r_i > tau * rho0[idx])
        for jj, j in enumerate(idx):
            if not ok[jj]:
                active[j] = False
                rep.frozen_at[j] = i
                rep.nonfinite[j] = not finite[jj]
        keep = ok
        idx, Q, gamma = idx[keep], Q[:, keep], gamma[keep]
        if idx.size == 0:
            continue
        a = rho[idx] / gamma
        X[:, idx] += a * P[:, idx]
        R[:, idx] -= a * Q
        Z[:, idx] = R[:, idx] * minv[:, None]
        rho_new = np.sum(R[:, idx] * Z[:, idx], axis=0)
        b = rho_new / rho[idx]
        P[:, idx] = Z[:, idx] + b * P[:, idx]
        rho[idx] = rho_new
        rep.rho_hist.append(rho.copy())
    return X, rep


def mean_rhs(op, y, beta):
    """b0 = beta Phi^T y (Eq. 5)."""
    return beta * op.apply_T(np.asarray(y, dtype=np.float64)[:, None])[:, 0]


def jacobi_diag(op, beta, alpha):
    """diag(A) = beta diag(Phi^T Phi) + alpha (R6)."""
    return beta * op.colsq() + alpha


def tau_of(rtol):
    """Freeze threshold of R5 / R19: max(1e-30, rtol^2)."""
    return max(FREEZE_TAU, float(rtol) ** 2)


def estep(op, y, beta, alpha, K, seed, t, U, precond=True, k_offset=0, return_x=False, rtol=0.0, mu0=None):
    """Simplified E-step (Alg. 1 lines 3-7; Eq. 6-7).

    B = [b0 | p_1 .. p_K]  (R2),  X = LinearSolver(A, B),
    mu = x_0,  s = (1/K) sum_k p_k o x_k (Eq. 6; Alg. 1 line 7).
    Raises FloatingPointError if a column met a non-finite value.
    """
    alpha = np.asarray(alpha, dtype=np.float64)
    b0 = mean_rhs(op, y, beta)
    diag = jacobi_diag(op, beta, alpha)
    Pk = rademacher_probes(op.D, K, seed, t, k_offset)
    B = np.concatenate([b0[:, None], Pk], axis=1)
    X0 = None
    if mu0 is not None:              # R20 (NEXT-1): warm start of the mean system only (fresh probes)
        X0 = np.zeros_like(B)
        X0[:, 0] = mu0
    X, rep = pcg(lambda V: gram_apply(op, beta, alpha, V), B, diag, U, precond, tau=tau_of(rtol), X0=X0)
    if rep.nonfinite.any():
        raise FloatingPointError("numerical breakdown in column %d" % int(np.argmax(rep.nonfinite)))
    mu = X[:, 0]
    s = np.mean(Pk * X[:, 1:], axis=1)
    if return_x:
        return mu, s, rep, X
    return mu, s, rep


def mstep(mu, s, den_floor=DEN_FLOOR, alpha_max=ALPHA_MAX):
    """alpha = 1 / (mu o mu + s)  (Eq. 8), floored/clamped (R7)."""
    den = np.maximum(mu * mu + s, den_floor)
    return np.minimum(1.0 / den, alpha_max)


def cofem_em(op, y, beta, T, K, seed, U, alpha_init=None, t0=0, precond=True, trace=None, rtol=0.0,
             warm_start=False):
    """Algorithm 1: alpha <- 1; for t in 1..T: E-step with fresh probes
    (probe counter t0 + t), M-step.  Returns (alpha_T, mu, s) where mu, s are
    from the last E-step (R9).  warm_start (R20, NEXT-1): every E-step after the first
    starts the mean system's CG from the previous E-step's mu."""
    alpha = np.ones(op.D) if alpha_init is None else np.asarray(alpha_init, dtype=np.float64).copy()
    mu = s = None
    for t in range(t0, t0 + T):
        mu, s, _ = estep(op, y, beta, alpha, K, seed, t, U, precond, rtol=rtol,
                         mu0=mu if (warm_start and mu is not None) else None)
        alpha = mstep(mu, s)
        if trace is not None:
            trace.append((alpha.copy(), mu.copy(), s.copy()))
    return alpha, mu, s


def support(mu, rel=1e-3):
    """Recovered support |mu_d| > rel * max|mu| (BASELINE.json north_star; reading R16)."""
    mu = np.asarray(mu)
    return np.abs(mu) > rel * np.max(np.abs(mu))


def estep_multi(op, Y, beta, alpha, K, seed, t, U, precond=True):
    """Multi-task E-step (R22): B = [beta Phi^T y_1 .. beta Phi^T y_L | p_1 .. p_K] (the task means
    first, then the probes, R2), one column-independent PCG (R3), mu_l = x_l,
    s = (1/K) sum_k p_k o x_{L+k} (Eq. 6).  Y: N x L.  Returns (MU (D x L), s, report)."""
    Y = np.asarray(Y, dtype=np.float64)
    if Y.ndim == 1:
        Y = Y[:, None]
    L = Y.shape[1]
    alpha = np.asarray(alpha, dtype=np.float64)
    B0 = beta * op.apply_T(Y)
    diag = jacobi_diag(op, beta, alpha)
    Pk = rademacher_probes(op.D, K, seed, t)
    X, rep = pcg(lambda V: gram_apply(op, beta, alpha, V), np.concatenate([B0, Pk], axis=1), diag, U, precond)
    if rep.nonfinite.any():
        raise FloatingPointError("numerical breakdown in column %d" % int(np.argmax(rep.nonfinite)))
    return X[:, :L], np.mean(Pk * X[:, L:], axis=1), rep


def mstep_multi(MU, s, den_floor=DEN_FLOOR, alpha_max=ALPHA_MAX):
    """alpha = 1 / (mean_l mu_l o mu_l + s) (R22), floored / clamped as Eq. 8 (R7)."""
    MU = np.asarray(MU, dtype=np.float64)
    den = np.maximum(np.mean(MU * MU, axis=1) + s, den_floor)
    return np.minimum(1.0 / den, alpha_max)


def cofem_em_multi(op, Y, beta, T, K, seed, U, alpha_init=None, t0=0, precond=True):
    """Multi-task Algorithm 1 (R22): returns (alpha_T, MU (D x L) and s of the last E-step)."""
    alpha = np.ones(op.D) if alpha_init is None else np.asarray(alpha_init, dtype=np.float64).copy()
    MU = s = None
    for t in range(t0, t0 + T):
        MU, s, _ = estep_multi(op, Y, beta, alpha, K, seed, t, U, precond)
        alpha = mstep_multi(MU, s)
    return alpha, MU, s
