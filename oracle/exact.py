"""Exact EM with an explicit covariance (Eq. 3-4) — the oracle's own oracle (test infrastructure only).

Eq. 3:  Sigma = (beta Phi^T Phi + diag alpha)^-1,  mu = beta Sigma Phi^T y
Eq. 4:  alpha_new = 1 / (mu o mu + Sigma[diag])
Eq. 2:  log p(y | alpha), evaluated with the standard Gaussian marginal
                  y ~ N(0, C), C = beta^-1 I + Phi diag(alpha)^-1 Phi^T.
Dense, O(D^3); guarded to D <= 4096.  Uses Cholesky (LAPACK via NumPy/SciPy)
as the library primitive.
"""
import numpy as np
import scipy.linalg as sla

from .cofem import mstep

MAX_D = 4096


def dense_phi(op):
    """Materialise Phi (N x D) of any operator by applying it to the identity."""
    return op.apply(np.eye(op.D))


def exact_posterior(phi, beta, alpha, y):
    """(mu, Sigma) of Eq. 3 by Cholesky factorisation of A = beta Phi^T Phi + diag alpha."""
    phi = np.asarray(phi, dtype=np.float64)
    D = phi.shape[1]
    if D > MAX_D:
        raise ValueError("exact_posterior guarded to D <= %d" % MAX_D)
    A = beta * (phi.T @ phi) + np.diag(np.asarray(alpha, dtype=np.float64))
    cf = sla.cho_factor(A, lower=True)
    Sigma = sla.cho_solve(cf, np.eye(D))
    mu = sla.cho_solve(cf, beta * (phi.T @ np.asarray(y, dtype=np.float64)))
    return mu, Sigma


def exact_em(phi, beta, y, T, alpha_init=None, trace=None):
    """Exact EM: Eq. 3 then Eq. 4 (same floor/clamp as CoFEM)."""
    D = np.asarray(phi).shape[1]
    alpha = np.ones(D) if alpha_init is None else np.asarray(alpha_init, dtype=np.float64).copy()
    mu = Sigma = None
    for _ in range(T):
        mu, Sigma = exact_posterior(phi, beta, alpha, y)
        alpha = mstep(mu, np.diag(Sigma))
        if trace is not None:
            trace.append((alpha.copy(), mu.copy()))
    return alpha, mu, Sigma


def log_evidence(phi, beta, alpha, y):
    """log p(y | alpha) = -1/2 [N log 2pi + log det C + y^T C^-1 y] (Eq. 2)."""
    phi = np.asarray(phi, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    N = phi.shape[0]
    C = np.eye(N) / beta + (phi / np.asarray(alpha)[None, :]) @ phi.T
    cf = sla.cho_factor(C, lower=True)
    logdet = 2.0 * np.sum(np.log(np.diag(cf[0])))
    return -0.5 * (N * np.log(2 * np.pi) + logdet + y @ sla.cho_solve(cf, y))
