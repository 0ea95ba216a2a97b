"""Operator-level GPU parity: one batched Gram apply Q = A X, A = beta Phi^T Phi + diag(alpha)
(Eq. 7; the CG matrix-matrix product of §3.2) through cofem_apply -- the same
kernels the E-step runs -- against the fp64 oracle's gram_apply, column by column, for every
operator path: dense tcgen05 3xTF32 and FP32 SIMT, 1024 x 1024 DCT fast path and the generic
DCT, overlap-save FFT convolution and the direct stencil.

Bars: the fp64 mean column (column 0) <= 1e-12 relative; fp32 probe columns <= 2e-6 (the
FP32-SIMT class bound of SURVEY §8(d) note 3, the acceptance test of the 3xTF32 split).
"""
import os

import numpy as np
import pytest

import synth
from oracle.operators import CircConvOp, DCT2MaskedOp, DenseOp, gram_apply

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2202_12808_b200 import build
    build.build()
    torch.cuda.set_device(0)


def op_of(w):
    if w.kind == "dense":
        return DenseOp(w.phi)
    if w.kind == "dct2_masked":
        return DCT2MaskedOp(w.rows, w.cols, w.obs_idx, w.convention)
    return CircConvOp(w.taps, w.D)


def col_err(a, b):
    return np.linalg.norm(a - b, axis=1) / np.linalg.norm(b, axis=1)


def run_apply(w, K, blocks, apply_path=0, alpha_seed=3):
    """GPU apply of [x0 | X] (fp64 mean column + K fp32 probe columns) and the fp64 oracle.
    apply_path 1 selects the general kernels (cofem_options.apply_path)."""
    from paper_2202_12808_b200 import Context
    ctx = Context.from_workload(w, max_probes=K, cg_iters=1, apply_path=apply_path)
    rng = np.random.default_rng(alpha_seed)
    alpha = np.exp(rng.uniform(-3.0, 6.0, w.D))           # EM-like spread of precisions
    x0 = rng.standard_normal(w.D)
    X = blocks(rng, K, w.D).astype(np.float32)
    q0 = np.empty(w.D)
    Q = np.empty((K, w.D), dtype=np.float32)
    gamma = np.empty(K + 1)
    ctx.apply(alpha, x0, np.ascontiguousarray(X), q0, Q, gamma)
    V = np.concatenate([x0[:, None], X.T.astype(np.float64)], axis=1)
    ref = gram_apply(op_of(w), w.beta, alpha, V)
    got = np.concatenate([q0[:, None], Q.T.astype(np.float64)], axis=1)
    e = col_err(got.T, ref.T)
    g_ref = np.sum(V * ref, axis=0)
    return e, np.abs(gamma - g_ref) / np.abs(g_ref)


def rademacher(rng, K, D):
    return rng.choice([-1.0, 1.0], size=(K, D))


def gaussian(rng, K, D):
    return rng.standard_normal((K, D))


DENSE = [synth.preset("C2"), synth.dense(250, 1000, 20, K=8, U=1, T=1, seed=1, name="dense_ragged_250x1000"),
         synth.preset("C1")]


@pytest.mark.parametrize("w", DENSE, ids=lambda w: w.name)
@pytest.mark.parametrize("blocks", [rademacher, gaussian], ids=["rademacher", "gaussian"])
@pytest.mark.parametrize("path", ["tcgen05_3xtf32", "fp32_simt"])
def test_dense_apply(w, blocks, path):
    e, eg = run_apply(w, 16, blocks, 1 if path == "fp32_simt" else 0)
    assert e[0] <= 1e-12, e[0]
    assert e[1:].max() <= 2e-6, e[1:].max()
    assert eg.max() <= 2e-6, eg.max()


def test_dense_apply_c3_shape_tensor_cores():
    """Config 3 shape (8192 x 32768, 1 GiB Phi): the 3xTF32 error budget at full size."""
    w = synth.preset("C3")
    e, eg = run_apply(w, 8, gaussian)
    assert e[0] <= 1e-12 and e[1:].max() <= 2e-6, (e[0], e[1:].max())


@pytest.mark.parametrize("w,path", [
    (synth.dct(1024, 1024, 262144, 100, K=8, U=1, T=1, seed=4), 0),                       # fast path
    (synth.dct(1024, 1024, 262144, 100, K=8, U=1, T=1, seed=4), 1),
    (synth.dct(64, 128, 2048, 40, K=8, U=1, T=1, seed=5), 0),                             # generic, rows != cols
    (synth.dct(64, 128, 2048, 40, K=8, U=1, T=1, seed=5, convention=1), 0),               # Phi = S C2 (R11)
    (synth.dct(1024, 1024, 262144, 100, K=8, U=1, T=1, seed=4, convention=1), 0),         # conv. 1, C4 shape
], ids=["dct1024_fast", "dct1024_generic", "dct64x128", "dct64x128_conv1", "dct1024_conv1"])
def test_dct_apply(w, path):
    e, eg = run_apply(w, 8, gaussian, path)
    assert e[0] <= 1e-12 and e[1:].max() <= 2e-6, (e[0], e[1:].max())
    assert eg.max() <= 2e-6


@pytest.mark.parametrize("w,path", [
    (synth.circconv(65536, 64, 60, K=8, U=1, T=1, seed=6), 0),                            # FFT, D multiple of 896? no
    (synth.circconv(5003, 64, 5, K=8, U=1, T=1, seed=7), 0),                              # FFT, prime D: wrapped windows
    (synth.circconv(5003, 64, 5, K=8, U=1, T=1, seed=7), 1),       # direct stencil
    (synth.circconv(1500, 17, 5, K=8, U=1, T=1, seed=8), 0),                              # D < 2048: direct
], ids=["fft_65536", "fft_5003", "direct_5003", "direct_1500_T17"])
def test_conv_apply(w, path):
    e, eg = run_apply(w, 8, gaussian, path)
    assert e[0] <= 1e-12 and e[1:].max() <= 2e-6, (e[0], e[1:].max())
    assert eg.max() <= 2e-6
