"""Dictionaries Phi for the oracle (fp64, plain definitions; test infrastructure only).

Paper: y ~ N(Phi z, beta^-1 I) with a known dictionary Phi in R^{N x D} (Eq. 1,
P:24-28).  CG needs only a way to apply Phi and Phi^T (§3.2).  The three
dictionaries of the workloads (BASELINE.json configs):

* DenseOp        Phi given as an N x D matrix (§4.1).
* DCT2MaskedOp   "an inverse discrete cosine transform (DCT) followed by an
                 undersampling mask" (§4.2).  Reading R11: orthonormal
                 2D DCT-II C2 on a rows x cols grid, Phi = S * C2^T (paper
                 reading, convention 0) or Phi = S * C2 (convention 1, the
                 literal "rows of DCT-II" of BASELINE.json config 4).
* CircConvOp     circular convolution with a short filter h (named in P:17,
                 P:98; defined by BASELINE.json config 5).  Reading R12:
                 (Phi x)_i = sum_{j<T} h_j x_{(i-j) mod D}, N = D.

Every operator takes and returns 2D blocks (one column per right-hand side), as
in Eq. 7 where the matrix-vector products become matrix-matrix products.
"""
import numpy as np


class DenseOp:
    """Phi as an explicit N x D matrix (fp32 input promoted to fp64)."""

    kind = "dense"

    def __init__(self, phi):
        self.phi = np.asarray(phi, dtype=np.float64)
        self.N, self.D = self.phi.shape

    def apply(self, V):
        """Phi V  (D x m -> N x m)."""
        return self.phi @ V

    def apply_T(self, W):
        """Phi^T W  (N x m -> D x m)."""
        return self.phi.T @ W

    def colsq(self):
        """diag(Phi^T Phi)_d = sum_n Phi_nd^2 (definition)."""
        return np.sum(self.phi * self.phi, axis=0)


def dct2_matrix(L):
    """Orthonormal DCT-II matrix, C[k, n] = s_k cos(pi (2n+1) k / (2L)),
    s_0 = sqrt(1/L), s_k = sqrt(2/L) (the textbook definition; reading R11)."""
    k = np.arange(L, dtype=np.float64)[:, None]
    n = np.arange(L, dtype=np.float64)[None, :]
    C = np.cos(np.pi * (2.0 * n + 1.0) * k / (2.0 * L)) * np.sqrt(2.0 / L)
    C[0, :] = np.sqrt(1.0 / L)
    return C


class DCT2MaskedOp:
    """Phi = S * C2^T (convention 0) or S * C2 (convention 1) on a rows x cols grid.

    The coefficient vector z (length D = rows*cols) and the pixel image are both
    stored row-major: index d = r*cols + c.  C2 = C_r (x) C_c acts on an image X
    as C_r X C_c^T; its transpose (the inverse, since C2 is orthonormal) as
    C_r^T X C_c.  S selects the N sorted, distinct pixel indices obs_idx
    (reading R11).
    """

    kind = "dct2_masked"

    def __init__(self, rows, cols, obs_idx, convention=0):
        self.rows, self.cols = int(rows), int(cols)
        self.D = self.rows * self.cols
        self.obs_idx = np.asarray(obs_idx, dtype=np.int64)
        if np.any(np.diff(self.obs_idx) <= 0) or self.obs_idx[0] < 0 or self.obs_idx[-1] >= self.D:
            raise ValueError("obs_idx must be sorted, distinct, in [0, D)")
        self.N = self.obs_idx.size
        self.convention = int(convention)
        self.Cr = dct2_matrix(self.rows)
        self.Cc = dct2_matrix(self.cols)

    def _img(self, V):
        return V.T.reshape(V.shape[1], self.rows, self.cols)

    def _vec(self, X):
        return X.reshape(X.shape[0], self.D).T

    def _c2(self, X):      # forward 2D DCT-II: C_r X C_c^T
        return self.Cr @ X @ self.Cc.T

    def _c2t(self, X):     # transpose = inverse 2D DCT (DCT-III): C_r^T X C_c
        return self.Cr.T @ X @ self.Cc

    def apply(self, V):
        """Phi V: inverse DCT of each column (conv. 0), then select the masked pixels."""
        X = self._img(V)
        pix = self._c2t(X) if self.convention == 0 else self._c2(X)
        return self._vec(pix)[self.obs_idx, :]

    def apply_T(self, W):
        """Phi^T W: scatter into a zero image, then the forward DCT (conv. 0)."""
        img = np.zeros((self.D, W.shape[1]))
        img[self.obs_idx, :] = W
        X = self._img(img)
        out = self._c2(X) if self.convention == 0 else self._c2t(X)
        return self._vec(out)

    def colsq(self):
        """diag(Phi^T Phi).  Conv. 0: Phi[n, d] = C2[d, obs_n], so
        colsq_d = sum_{pix in mask} C2[d, pix]^2 = (Q_r M Q_c^T)[d] with Q = C o C
        (elementwise square; C2 = C_r (x) C_c).  Conv. 1: (Q_r^T M Q_c)[d].
        Pinned against sum_n Phi_nd^2 with Phi materialised (tests)."""
        M = np.zeros(self.D)
        M[self.obs_idx] = 1.0
        M = M.reshape(self.rows, self.cols)
        Qr, Qc = self.Cr * self.Cr, self.Cc * self.Cc
        if self.convention == 0:
            out = Qr @ M @ Qc.T
        else:
            out = Qr.T @ M @ Qc
        return out.reshape(self.D)


class CircConvOp:
    """(Phi x)_i = sum_{j=0}^{T-1} h_j x_{(i-j) mod D}; N = D (reading R12)."""

    kind = "circconv"

    def __init__(self, h, D):
        self.h = np.asarray(h, dtype=np.float64)
        self.D = self.N = int(D)
        if self.D < self.h.size:
            raise ValueError("D must be >= number of taps")

    def apply(self, V):
        """(Phi V)_i = sum_j h_j V_{(i-j) mod D}, summed in tap order j = 0..T-1.
        The wrapped rows are read from a copy of V with its last T-1 rows in front,
        Vw[i + T-1] = V[(i) mod D] for i >= -(T-1), so Vw[T-1-j : T-1-j+D][i] = V[(i-j) mod D]
        (the same products and sums as np.roll(V, j), without the per-tap copy)."""
        V = np.asarray(V, dtype=np.float64)
        T, D = self.h.size, self.D
        Vw = np.concatenate([V[D - (T - 1):], V]) if T > 1 else V
        out = np.zeros_like(V)
        for j, hj in enumerate(self.h):
            out += hj * Vw[T - 1 - j:T - 1 - j + D]
        return out

    def apply_T(self, W):
        """(Phi^T W)_i = sum_j h_j W_{(i+j) mod D}, tap order j = 0..T-1; Ww[i] = W[i mod D]
        for i < D + T-1, so Ww[j : j+D][i] = W[(i+j) mod D]."""
        W = np.asarray(W, dtype=np.float64)
        T, D = self.h.size, self.D
        Ww = np.concatenate([W, W[:T - 1]]) if T > 1 else W
        out = np.zeros_like(W)
        for j, hj in enumerate(self.h):
            out += hj * Ww[j:j + D]
        return out

    def colsq(self):
        """Column d of Phi holds each tap once (D >= T), so diag(Phi^T Phi) = sum_j h_j^2."""
        return np.full(self.D, np.sum(self.h * self.h))


def gram_apply(op, beta, alpha, V):
    """A V = beta Phi^T (Phi V) + diag(alpha) V  (Eq. 7; reading R1:
    beta is kept in A even though P:98 drops it), one apply and one apply_T."""
    return beta * op.apply_T(op.apply(V)) + alpha[:, None] * V
