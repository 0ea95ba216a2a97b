"""The exact-EM GPU baseline (tools/exact_em_gpu.py: fp64 Cholesky through cuSOLVER, the paper's EM
of Table 1 -- NEXT-3) against the CPU oracle's exact EM (oracle/exact.py, pinned by the scalar
closed forms and the evidence-monotone tests), on the dense and masked-DCT operators."""
import os
import sys

import numpy as np
import pytest

import synth
from oracle.exact import dense_phi as oracle_phi
from oracle.exact import exact_em
from oracle.operators import DCT2MaskedOp

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("w", [synth.paper_dense(256, 4, seed=1, T=8), synth.paper_dct(8, seed=2, T=8),
                               synth.dct(16, 32, 128, 10, K=1, U=1, T=8, seed=3, convention=1)],
                         ids=lambda w: w.name + "_conv%d" % w.convention)
def test_exact_em_gpu_matches_oracle(w):
    import exact_em_gpu as eg
    phi_g = eg.dense_phi(w)
    if w.kind == "dense":
        phi_o = w.phi.astype(np.float64)
    else:
        phi_o = oracle_phi(DCT2MaskedOp(w.rows, w.cols, w.obs_idx, w.convention))
    assert rel(phi_g.cpu().numpy(), phi_o) < 1e-13                 # the explicit Phi of the operator
    a, mu, sd, nr, sec = eg.exact_em(phi_g, w.y, w.beta, w.T, z_true=w.z_true)
    oa, omu, oS = exact_em(phi_o, w.beta, w.y, w.T)
    # fp64 both sides; kappa(A) ~ 1e6 at beta = 1/sigma^2 = 4e4 with unnormalised Phi: ~1e-9 after 8 EM
    assert rel(1 / a, 1 / oa) < 1e-7 and rel(mu, omu) < 1e-7 and rel(sd, np.diag(oS)) < 1e-7
    assert len(nr) == w.T and np.all(np.isfinite(nr))
