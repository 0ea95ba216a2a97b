"""Error of one dense Gram apply (tcgen05 3xTF32 vs FP32 SIMT) against fp64 as a function of
the two contraction lengths (N for Phi^T W, D for Phi P): diagnoses accumulation precision."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from oracle.operators import DenseOp, gram_apply
from paper_2202_12808_b200 import Context

def err(N, D, simt, K=8):
    w = synth.dense(N, D, 5, K=K, U=1, T=1, seed=1)
    ctx = Context.from_workload(w, max_probes=K, cg_iters=1, apply_path=1 if simt else 0)
    rng = np.random.default_rng(0)
    alpha = np.ones(D) * 1e-3
    x0 = rng.standard_normal(D)
    X = rng.standard_normal((K, D)).astype(np.float32)
    q0 = np.empty(D); Q = np.empty((K, D), np.float32)
    ctx.apply(alpha, x0, X, q0, Q)
    V = np.concatenate([x0[:, None], X.T.astype(np.float64)], 1)
    ref = gram_apply(DenseOp(w.phi), w.beta, alpha, V)
    e = np.linalg.norm(Q.T - ref[:, 1:], axis=0) / np.linalg.norm(ref[:, 1:], axis=0)
    # also W = Phi X (first GEMM) error proxy: not exposed; report q error only
    return e.max()

for N, D in [(32, 4096), (128, 4096), (512, 4096), (2048, 4096), (8192, 4096), (2048, 512), (2048, 32768)]:
    print(N, D, "tc %.2e" % err(N, D, False), "simt %.2e" % err(N, D, True), flush=True)
