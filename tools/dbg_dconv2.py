import os, sys, time, numpy as np, torch
sys.path.insert(0, "/root/repo")
import synth
from paper_2202_12808_b200 import OP_CIRCCONV, Context, get_unique_id
w = synth.circconv(20000, 64, 20, K=8, U=150, T=3, seed=4)
t0 = time.time()
def log(*a): print("%.1fs" % (time.time() - t0), *a, flush=True)
sh = Context.from_workload(w, rank=0, world=1, nccl_id=get_unique_id(), d_offset=0, D_global=w.D, max_probes=8)
log("sh setup")
a = torch.ones(w.D, dtype=torch.float64, device="cuda"); mu = torch.empty_like(a); s = torch.empty_like(a)
sh.estep(a, 8, 5, 0, mu, s); torch.cuda.synchronize(); log("sh estep")
ao = torch.empty_like(a)
sh.em(2, 8, 6, 0, None, ao, mu, s); torch.cuda.synchronize(); log("sh em")
d0 = 128; Dl = w.D - d0
part = Context(OP_CIRCCONV, Dl, Dl, np.ascontiguousarray(w.y[d0:]), w.beta, taps=w.taps, cg_iters=w.U, max_probes=8,
               rank=0, world=1, nccl_id=get_unique_id(), d_offset=d0, D_global=w.D)
log("part setup")
a2 = torch.ones(Dl, dtype=torch.float64, device="cuda"); m2 = torch.empty_like(a2); s2 = torch.empty_like(a2)
part.estep(a2, 8, 5, 0, m2, s2); torch.cuda.synchronize(); log("part estep")
