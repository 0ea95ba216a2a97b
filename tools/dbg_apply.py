import os, sys, numpy as np
sys.path.insert(0, "/root/repo")
import synth
from paper_2202_12808_b200 import Context
for arg in sys.argv[1:]:
    N, D, simt = [int(v) for v in arg.split(",")]
    if simt: os.environ["COFEM_DENSE_SIMT"] = "1"
    else: os.environ.pop("COFEM_DENSE_SIMT", None)
    w = synth.dense(N, D, 5, K=8, U=1, T=1, seed=1)
    ctx = Context.from_workload(w, max_probes=8, cg_iters=1)
    rng = np.random.default_rng(0)
    alpha = np.ones(D); x0 = rng.standard_normal(D); X = rng.standard_normal((8, D)).astype(np.float32)
    q0 = np.empty(D); Q = np.empty((8, D), np.float32)
    try:
        ctx.apply(alpha, x0, X, q0, Q); print("ok", N, D, simt, flush=True)
    except Exception as e:
        print("FAIL", N, D, simt, e, flush=True); break
