import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import synth
from oracle.cofem import cofem_em
from oracle.operators import DCT2MaskedOp
from paper_2202_12808_b200 import Context
w = synth.dct(1024, 1024, 262144, 400, K=3, U=30, T=3, seed=3)
op = DCT2MaskedOp(w.rows, w.cols, w.obs_idx)
rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
for T in (1, 2):
    oa, omu, _ = cofem_em(op, w.y, w.beta, T, 3, 4, 30, warm_start=True)
    ca, cmu, _ = cofem_em(op, w.y, w.beta, T, 3, 4, 30, warm_start=False)
    for kw in ({}, {"apply_path": 1}, {"probe_precision": 1}, {"apply_path": 1, "probe_precision": 1}):
        ctx = Context.from_workload(w, max_probes=3, cg_iters=30, warm_start=True, **kw)
        a = torch.empty(w.D, dtype=torch.float64, device="cuda"); mu = torch.empty_like(a); s = torch.empty_like(a)
        ctx.em(T, 3, 4, 0, None, a, mu, s)
        print(T, kw, "vs warm oracle: 1/a %.2e mu %.2e | vs cold oracle 1/a %.2e" % (rel(1/a.cpu().numpy(), 1/oa), rel(mu.cpu().numpy(), omu), rel(1/a.cpu().numpy(), 1/ca)), flush=True)
