"""SURVEY §8(d) note 3: record that ONE tf32 MMA per product (no hi/lo split) misses the error
budget.  Run once with the default library (3xTF32) and once with the COFEM_TC_EXP_1XTF32 build
(tools/build_variant.sh op_dense_tc.cu tf32x1 -DCOFEM_TC_EXP_1XTF32) installed as libcofem.so:
    python tools/tf32x1_check.py <label>
prints the per-column apply error against fp64 (bar 2e-6, FP32-SIMT class) at the C2 shape and the
C2 E-step-1 error against the oracle's fixture (north_star bar 1e-4)."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from oracle.operators import DenseOp, gram_apply  # noqa: E402
from paper_2202_12808_b200 import Context  # noqa: E402

label = sys.argv[1] if len(sys.argv) > 1 else "default"
w = synth.preset("C2")
ctx = Context.from_workload(w, max_probes=16, cg_iters=1)
rng = np.random.default_rng(3)
alpha = np.exp(rng.uniform(-3.0, 6.0, w.D))
x0 = rng.standard_normal(w.D)
X = rng.choice([-1.0, 1.0], size=(16, w.D)).astype(np.float32)
q0, Q, g = np.empty(w.D), np.empty((16, w.D), np.float32), np.empty(17)
ctx.apply(alpha, x0, X, q0, Q, g)
V = np.concatenate([x0[:, None], X.T.astype(np.float64)], 1)
ref = gram_apply(DenseOp(w.phi), w.beta, alpha, V)
e = np.linalg.norm(Q.T - ref[:, 1:], axis=0) / np.linalg.norm(ref[:, 1:], axis=0)
f = np.load(os.path.join(ROOT, "tests", "golden", "fullcfg", "C2_full.npz"))
c2 = Context.from_workload(w)
a = torch.ones(w.D, dtype=torch.float64, device="cuda")
mu, s = torch.empty_like(a), torch.empty_like(a)
c2.estep(a, 32, 0, 0, mu, s)
rel = lambda x, y: float(np.linalg.norm(x - y) / np.linalg.norm(y))
out = {"label": label, "apply_max_col_err": float(e.max()), "apply_bar": 2e-6,
       "estep1_mu_rel": rel(mu.cpu().numpy(), f["mu1"]), "estep1_s_rel": rel(s.cpu().numpy(), f["s1"]),
       "estep1_bar": 1e-4}
print(json.dumps(out))
