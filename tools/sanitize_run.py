"""Small E-steps through every kernel family, for compute-sanitizer (memcheck / racecheck /
synccheck): the 1024^2 DCT fast path (fp32 probes in two groups + the fp64 mean column, U = 3),
the generic DCT passes (both conventions), the dense tcgen05 and SIMT paths, the FFT and direct
convolutions, parity mode, cofem_apply.  Graphs off (the sanitizer then sees every launch).
    compute-sanitizer --tool memcheck python tools/sanitize_run.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2202_12808_b200 import Context  # noqa: E402

cases = [
    (synth.dct(1024, 1024, 262144, 100, K=4, U=3, T=1, seed=1), {}),
    (synth.dct(64, 64, 1024, 41, K=3, U=5, T=1, seed=0), {}),
    (synth.dct(32, 64, 512, 10, K=3, U=5, T=1, seed=0, convention=1), {}),
    (synth.dense(250, 1000, 20, K=8, U=4, T=1, seed=1), {}),
    (synth.dense(250, 1000, 20, K=8, U=4, T=1, seed=1), {"apply_path": 1}),
    (synth.dense(100, 400, 10, K=4, U=4, T=1, seed=1), {"probe_precision": 1}),
    (synth.circconv(5003, 64, 5, K=4, U=4, T=1, seed=0), {}),
    (synth.circconv(5003, 64, 5, K=4, U=4, T=1, seed=0), {"apply_path": 1}),
    (synth.dct(1024, 1024, 262144, 100, K=2, U=2, T=1, seed=1), {"probe_precision": 1}),
]
for w, kw in cases:
    ctx = Context.from_workload(w, cg_iters=w.U, max_probes=w.K, use_graph=False, **kw)
    a = torch.ones(w.D, dtype=torch.float64, device="cuda")
    mu, s = torch.empty_like(a), torch.empty_like(a)
    ctx.em(2, w.K, 3, 0, None, a, mu, s)
    torch.cuda.synchronize()
    print(w.name, kw, "ok", float(mu.abs().max()), float(s.abs().max()), flush=True)
    ctx.close()
