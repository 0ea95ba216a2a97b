"""Pins for oracle/operators.py against definitions, library routines and invariants."""
import numpy as np
import pytest
import scipy.fft as sfft

from oracle import closed_forms as cf
from oracle.exact import dense_phi
from oracle.operators import CircConvOp, DCT2MaskedOp, DenseOp, dct2_matrix, gram_apply


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def test_dense_examples():
    op = DenseOp(np.eye(3))
    assert np.array_equal(op.apply(np.array([[0.0], [1.0], [0.0]]))[:, 0], [0, 1, 0])
    op = DenseOp(np.array([[1.0, 2, 3], [4, 5, 6]]))
    assert np.array_equal(op.apply(np.ones((3, 1)))[:, 0], [6, 15])
    assert np.array_equal(DenseOp(np.eye(3)).apply_T(np.array([[1.0], [0], [0]]))[:, 0], [1, 0, 0])


@pytest.mark.parametrize("L", [1, 2, 8, 32, 64])
def test_dct_matrix_vs_scipy(L):
    x = np.random.default_rng(L).standard_normal((L, 3))
    C = dct2_matrix(L)
    assert rel(C @ x, sfft.dct(x, type=2, norm="ortho", axis=0)) < 1e-13
    assert rel(C.T @ x, sfft.dct(x, type=3, norm="ortho", axis=0)) < 1e-13
    assert np.allclose(C @ C.T, np.eye(L), atol=1e-13)


def test_dct8_spike_is_basis_column():
    # full mask, delta spike -> the corresponding inverse-DCT basis column
    op = DCT2MaskedOp(1, 8, np.arange(8))
    C = dct2_matrix(8)
    for k in range(8):
        e = np.zeros((8, 1)); e[k] = 1
        assert np.allclose(op.apply(e)[:, 0], C[k, :], atol=1e-14)


@pytest.mark.parametrize("conv", [0, 1])
@pytest.mark.parametrize("rows,cols", [(8, 16), (16, 8), (32, 32)])
def test_dct_masked_vs_scipy_and_invariants(rows, cols, conv):
    rng = np.random.default_rng(rows * 100 + cols + conv)
    D = rows * cols
    N = D // 4
    obs = np.sort(rng.choice(D, N, replace=False))
    op = DCT2MaskedOp(rows, cols, obs, conv)
    V = rng.standard_normal((D, 3))
    W = rng.standard_normal((N, 3))
    for j in range(3):   # independent: scipy.fft
        assert rel(op.apply(V)[:, j], cf.dct_phi(rows, cols, obs, V[:, j], conv)) < 1e-12
        assert rel(op.apply_T(W)[:, j], cf.dct_phiT(rows, cols, obs, W[:, j], conv)) < 1e-12
    # adjoint
    assert abs(np.sum(op.apply(V) * W) - np.sum(V * op.apply_T(W))) < 1e-10 * np.sum(np.abs(V)) * np.sum(np.abs(W))
    # Phi Phi^T = I_N
    assert np.allclose(op.apply(op.apply_T(np.eye(N))), np.eye(N), atol=1e-12)
    # colsq vs definition sum_n Phi_nd^2 with Phi materialised
    phi = dense_phi(op)
    assert np.allclose(op.colsq(), np.sum(phi * phi, axis=0), atol=1e-13)


def test_dct_full_mask_orthogonal():
    op = DCT2MaskedOp(8, 8, np.arange(64))
    phi = dense_phi(op)
    assert np.allclose(phi.T @ phi, np.eye(64), atol=1e-12)
    assert np.allclose(op.colsq(), 1.0)


def test_dct_rejects_bad_mask():
    with pytest.raises(ValueError):
        DCT2MaskedOp(4, 4, np.array([3, 2]))
    with pytest.raises(ValueError):
        DCT2MaskedOp(4, 4, np.array([2, 2]))


@pytest.mark.parametrize("D", [64, 67, 200])
def test_circconv_vs_circulant_and_fft(D):
    rng = np.random.default_rng(D)
    h = rng.standard_normal(64)
    op = CircConvOp(h, D)
    # explicit circulant: Phi[i, (i - j) mod D] += h_j
    Phi = np.zeros((D, D))
    for i in range(D):
        for j in range(64):
            Phi[i, (i - j) % D] += h[j]
    V = rng.standard_normal((D, 2))
    assert rel(op.apply(V), Phi @ V) < 1e-13
    assert rel(op.apply_T(V), Phi.T @ V) < 1e-13
    hp = np.concatenate([h, np.zeros(D - 64)])
    fftconv = np.real(np.fft.ifft(np.fft.fft(hp)[:, None] * np.fft.fft(V, axis=0), axis=0))
    assert rel(op.apply(V), fftconv) < 1e-12
    assert np.allclose(op.colsq(), np.sum(Phi * Phi, axis=0))


def test_gram_apply_examples_and_assembly():
    rng = np.random.default_rng(0)
    V = rng.standard_normal((5, 2))
    assert np.allclose(gram_apply(DenseOp(np.zeros((3, 5))), 7.0, np.ones(5), V), V)
    assert np.allclose(gram_apply(DenseOp(np.eye(5)), 1.0, np.ones(5), V), 2 * V)
    phi = rng.standard_normal((4, 6))
    alpha = rng.uniform(0.5, 2, 6)
    A = 0.5 * phi.T @ phi + np.diag(alpha)
    V = rng.standard_normal((6, 3))
    assert rel(gram_apply(DenseOp(phi), 0.5, alpha, V), A @ V) < 1e-14
    # linearity
    V2 = rng.standard_normal((6, 3))
    g = lambda X: gram_apply(DenseOp(phi), 0.5, alpha, X)
    assert rel(g(2 * V - 3 * V2), 2 * g(V) - 3 * g(V2)) < 1e-13
