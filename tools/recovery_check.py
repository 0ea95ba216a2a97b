"""Full-size EM (T_em of each config) on the GPU: NRMSE of mu against the synthetic z* and
support hits, a sanity check of the method end to end (pinned in tests/test_gpu_parity.py)."""
import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import synth
from paper_2202_12808_b200 import Context
for name in ["C4", "C3", "C5", "C2"]:
    w = synth.preset(name)
    ctx = Context.from_workload(w)
    a, mu, s = (torch.empty(w.D, dtype=torch.float64, device="cuda") for _ in range(3))
    ctx.em(w.T, w.K, 0, 0, None, a, mu, s)
    m = mu.cpu().numpy(); z = w.z_true
    nrmse = np.linalg.norm(m - z) / np.linalg.norm(z)
    sup_true = set(np.nonzero(z)[0]); sup = set(np.nonzero(np.abs(m) > 1e-3 * np.abs(m).max())[0])
    print(name, "T", w.T, "NRMSE %.4f" % nrmse, "finite", bool(np.isfinite(a.cpu().numpy()).all()),
          "true nnz", len(sup_true), "found", len(sup), "hit", len(sup & sup_true), flush=True)
