"""Sensitivity of the K = 4 EM trajectory at full size (tests/test_gpu_fullcfg.py em6 cases):
GPU parity-mode alpha_5 against the oracle's (tests/golden/fullcfg/<case>.npz alpha_in), and two
GPU parity-mode runs whose only difference is the summation order (probe groups 1 / 2 on the DCT
path; apply_path 0 / 1 on dense) -- how far fp64 rounding alone moves the trajectory.
    python tools/traj_check.py C4_ss"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2202_12808_b200 import Context  # noqa: E402

case = sys.argv[1]
f = np.load(os.path.join("tests", "golden", "fullcfg", case + ".npz"))
meta = json.loads(str(f["meta"]))
w = synth.preset(case.split("_")[0]) if not case.startswith("C5s") else \
    synth.circconv(1 << 20, 64, 1048, K=16, U=150, T=20, seed=0)
K, U = meta["K"], meta["U"]
a5o = f["alpha_in"]


def run(T, **kw):
    ctx = Context.from_workload(w, max_probes=K, cg_iters=U, probe_precision=1, **kw)
    a = torch.empty(w.D, dtype=torch.float64, device="cuda")
    mu, s = torch.empty_like(a), torch.empty_like(a)
    out = []
    for t in range(T):
        ctx.em(1, K, 0, t, None if t == 0 else a, a, mu, s)
        out.append((a.cpu().numpy().copy(), ctx.report()["frozen_at"]))
    return out


def rel(x, y):
    return float(np.linalg.norm(1 / x - 1 / y) / np.linalg.norm(1 / y))


r1 = run(5)
alt = {"probe_groups": 1} if w.kind == "dct2_masked" else {"apply_path": 1} if w.kind == "dense" else {"use_graph": False}
r2 = run(5, **alt)
for t in range(5):
    print("%s EM it %d: 1/alpha rel diff between two GPU fp64 orders %.3e; frozen_at %s | %s" % (
        case, t + 1, rel(r1[t][0], r2[t][0]), r1[t][1], r2[t][1]), flush=True)
print("%s GPU parity alpha_5 vs oracle alpha_5: 1/alpha rel %.3e" % (case, rel(r1[4][0], a5o)))
