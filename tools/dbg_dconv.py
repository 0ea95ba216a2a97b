import os, sys, time, numpy as np, torch
sys.path.insert(0, "/root/repo")
import synth
from paper_2202_12808_b200 import Context, get_unique_id
w = synth.circconv(20000, 64, 20, K=8, U=int(sys.argv[1]) if len(sys.argv) > 1 else 3, T=3, seed=4)
t0 = time.time()
ctx = Context.from_workload(w, rank=0, world=1, nccl_id=get_unique_id(), d_offset=0, D_global=w.D)
print("setup ok %.1fs" % (time.time() - t0), flush=True)
a = torch.ones(w.D, dtype=torch.float64, device="cuda"); mu = torch.empty_like(a); s = torch.empty_like(a)
ctx.estep(a, 8, 5, 0, mu, s); torch.cuda.synchronize()
print("estep ok %.1fs" % (time.time() - t0), float(mu.norm()), flush=True)
