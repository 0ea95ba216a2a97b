"""Closed-form E-step / EM results that pin the oracle (and the GPU) at any size.

Test infrastructure only.  Each function states the mathematics that makes the
linear system of Eq. 7 solvable without CG.  They use library
transforms (scipy.fft, numpy.fft, LAPACK), NOT oracle/operators.py, so that a
mistake in the oracle's operator or its PCG shows up as a disagreement.

1. full-mask DCT (N = D): Phi is square orthonormal, Phi^T Phi = I, so
   A = diag(beta + alpha) and, for u = Phi^T y, every coordinate follows
       mu = beta u / (beta + alpha),  Sigma_dd = s = 1 / (beta + alpha)
   (s is exact for ANY probes since p o p = 1, Eq. 6), and the M-step (Eq. 8)
   gives the scalar recursion alpha+ = 1 / (mu^2 + s).  Whole-EM trajectory.
2. masked DCT at alpha = 1: Phi Phi^T = I_N, so P = Phi^T Phi is a projection,
   A = beta P + I, A^-1 = I - beta/(beta+1) P, and since b0 = beta Phi^T y lies in
   range(P): mu = b0 / (beta + 1);  x_k = p_k - beta/(beta+1) P p_k.
3. circular convolution at constant alpha: A = beta Phi^T Phi + alpha I is
   circulant with eigenvalues beta |H(w)|^2 + alpha (H = DFT of zero-padded h),
   so A^-1 v = IFFT(FFT(v) / (beta |H|^2 + alpha)).
4. dense Phi at constant alpha (Woodbury):
   A^-1 = (1/alpha) [I - beta Phi^T (alpha I_N + beta Phi Phi^T)^-1 Phi].
"""
import numpy as np
import scipy.fft as sfft
import scipy.linalg as sla


def _idct2(img, convention):
    return sfft.idctn(img, norm="ortho") if convention == 0 else sfft.dctn(img, norm="ortho")


def _dct2(img, convention):
    return sfft.dctn(img, norm="ortho") if convention == 0 else sfft.idctn(img, norm="ortho")


def dct_phiT(rows, cols, obs_idx, w, convention=0):
    """Phi^T w for the masked 2D DCT via scipy.fft (independent of the oracle)."""
    img = np.zeros(rows * cols)
    img[obs_idx] = w
    return _dct2(img.reshape(rows, cols), convention).ravel()


def dct_phi(rows, cols, obs_idx, v, convention=0):
    return _idct2(np.asarray(v, dtype=np.float64).reshape(rows, cols), convention).ravel()[obs_idx]


def full_mask_dct_em(u, beta, T, alpha0=1.0):
    """Item 1: per-coordinate EM trajectory for Phi^T Phi = I.  Returns
    (alpha_T, mu_{T-1}, s_{T-1}) matching Algorithm 1's return (R9)."""
    u = np.asarray(u, dtype=np.float64)
    alpha = np.full_like(u, alpha0)
    mu = s = None
    for _ in range(T):
        mu = beta * u / (beta + alpha)
        s = 1.0 / (beta + alpha)
        alpha = np.minimum(1.0 / np.maximum(mu * mu + s, 1e-12), 1e12)
    return alpha, mu, s


def masked_dct_estep1(rows, cols, obs_idx, y, beta, probes, convention=0):
    """Item 2: exact (mu, x_k, s) of E-step 1 (alpha = 1) for the masked DCT."""
    b0 = beta * dct_phiT(rows, cols, obs_idx, np.asarray(y, dtype=np.float64), convention)
    mu = b0 / (beta + 1.0)
    c = beta / (beta + 1.0)
    X = np.empty_like(probes)
    for k in range(probes.shape[1]):
        pk = probes[:, k]
        Ppk = dct_phiT(rows, cols, obs_idx, dct_phi(rows, cols, obs_idx, pk, convention), convention)
        X[:, k] = pk - c * Ppk
    s = np.mean(probes * X, axis=1)
    return mu, s, X


def circconv_solve(h, D, beta, alpha, V):
    """Item 3: A^-1 V for circular convolution, constant alpha."""
    H = np.fft.fft(np.concatenate([np.asarray(h, dtype=np.float64), np.zeros(D - len(h))]))
    lam = beta * np.abs(H) ** 2 + alpha
    return np.real(np.fft.ifft(np.fft.fft(V, axis=0) / lam[:, None], axis=0))


def circconv_estep(h, D, y, beta, alpha, probes):
    """Exact (mu, s) at constant alpha: b0 = beta Phi^T y, Phi^T = correlation with h."""
    H = np.fft.fft(np.concatenate([np.asarray(h, dtype=np.float64), np.zeros(D - len(h))]))
    b0 = beta * np.real(np.fft.ifft(np.conj(H) * np.fft.fft(np.asarray(y, dtype=np.float64))))
    mu = circconv_solve(h, D, beta, alpha, b0[:, None])[:, 0]
    X = circconv_solve(h, D, beta, alpha, probes)
    return mu, np.mean(probes * X, axis=1), X


def dense_estep(phi, y, beta, alpha, probes):
    """Item 4: exact (mu, s) at constant alpha via an N x N Cholesky (Woodbury)."""
    phi = np.asarray(phi, dtype=np.float64)
    N = phi.shape[0]
    cf = sla.cho_factor(alpha * np.eye(N) + beta * (phi @ phi.T), lower=True)

    def solve(V):
        return (V - beta * phi.T @ sla.cho_solve(cf, phi @ V)) / alpha

    b0 = beta * (phi.T @ np.asarray(y, dtype=np.float64))
    mu = solve(b0[:, None])[:, 0]
    X = solve(probes)
    return mu, np.mean(probes * X, axis=1), X
