"""Randomised shapes (seeded, so every run checks the same cases): E-step 1 parity of the CUDA
path against the fp64 oracle on dense (tensor-core and, for D % 4 != 0, SIMT), masked 2-D DCT
(generic lengths, rows != cols) and circular convolution (direct and FFT, ragged D) workloads
with K from 1 to 24 — shapes the named configs do not reach (odd N, K = 1, tiny grids, taps
close to D).  Bars: the north_star E-step bar, 1e-4 on mu and s."""
import numpy as np
import pytest

import synth
from oracle.cofem import estep
from oracle.operators import CircConvOp, DCT2MaskedOp, DenseOp

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2202_12808_b200 import build
    build.build()
    torch.cuda.set_device(0)


def case(i):
    rng = np.random.default_rng(1000 + i)
    kind = ("dense", "dct", "conv")[i % 3]
    K = int(rng.integers(1, 25))
    U = int(rng.integers(30, 120))
    if kind == "dense":
        # converged U: an unconverged iterate of these ill-conditioned systems (kappa ~ beta (1 +
        # sqrt(D/N))^2 ~ 1e5) amplifies fp32 rounding of the probe columns past 1e-4 (measured
        # 1.7-2.2e-4 at U < 120 on the SIMT path), the same effect DESIGN.md §4 quantifies
        N = int(rng.integers(17, 300))
        D = int(rng.integers(40, 1300))
        return synth.dense(N, D, max(1, D // 50), K=K, U=400, T=1, seed=i, name="fz%d_dense_%dx%d_K%d" % (i, N, D, K))
    if kind == "dct":
        rows = int(rng.choice([16, 32, 64, 128]))
        cols = int(rng.choice([16, 32, 64, 128]))
        D = rows * cols
        N = int(rng.integers(D // 8, D // 2))
        return synth.dct(rows, cols, N, max(1, D // 30), K=K, U=U, T=1, seed=i,
                         name="fz%d_dct_%dx%d_N%d_K%d" % (i, rows, cols, N, K))
    D = int(rng.integers(300, 9000))
    taps = int(rng.integers(1, 65))
    return synth.circconv(D, taps, max(1, D // 100), K=K, U=U, T=1, seed=i,
                          name="fz%d_conv_D%d_T%d_K%d" % (i, D, taps, K))


CASES = [case(i) for i in range(18)]


def op_of(w):
    if w.kind == "dense":
        return DenseOp(w.phi)
    if w.kind == "dct2_masked":
        return DCT2MaskedOp(w.rows, w.cols, w.obs_idx, w.convention)
    return CircConvOp(w.taps, w.D)


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("w", CASES, ids=lambda w: w.name)
def test_random_shape_estep_parity(w):
    from paper_2202_12808_b200 import Context
    ctx = Context.from_workload(w)
    a = torch.ones(w.D, dtype=torch.float64, device="cuda")
    mu, s = torch.empty_like(a), torch.empty_like(a)
    ctx.estep(a, w.K, 11, 2, mu, s)
    omu, os_, _ = estep(op_of(w), w.y, w.beta, np.ones(w.D), w.K, 11, 2, w.U)
    em, es = rel(mu.cpu().numpy(), omu), rel(s.cpu().numpy(), os_)
    assert em <= 1e-4 and es <= 1e-4, (em, es)
