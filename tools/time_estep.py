"""Time E-steps at a fixed alpha so that runs with different library settings follow identical
CG trajectories (frozen columns are skipped, so the cost of an E-step depends on alpha):
    python tools/time_estep.py C4 5 [alpha.pt]
alpha.pt: if it exists it is loaded, else alpha after 3 EM iterations is computed and saved
(the steady-state regime of bench.py; alpha = 1 freezes columns early and is unrepresentative)."""
import os
import sys
import torch
sys.path.insert(0, "/root/repo")
import synth
from paper_2202_12808_b200 import Context

w = synth.preset(sys.argv[1] if len(sys.argv) > 1 else "C4")
if os.environ.get("TIME_K"):          # emulate one rank of a probe-parallel run (K / world probes)
    w.K = int(os.environ["TIME_K"])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
kw = {"probe_groups": int(os.environ["TIME_GROUPS"])} if os.environ.get("TIME_GROUPS") else {}
if os.environ.get("TIME_PATH"):       # cofem_options.apply_path (1: the general kernels)
    kw["apply_path"] = int(os.environ["TIME_PATH"])
if os.environ.get("TIME_NOGRAPH"):
    kw["use_graph"] = False
if os.environ.get("TIME_U"):          # CG iterations per E-step (use with an existing alpha file)
    w.U = int(os.environ["TIME_U"])
ctx = Context.from_workload(w, max_probes=w.K, **kw)
alpha = torch.ones(w.D, dtype=torch.float64, device="cuda")
mu, s = torch.empty_like(alpha), torch.empty_like(alpha)
ap = sys.argv[3] if len(sys.argv) > 3 else None
if ap and os.path.exists(ap):
    alpha = torch.load(ap).cuda()
elif ap:
    ctx.em(3, w.K, 0, 0, None, alpha, mu, s)
    torch.save(alpha.cpu(), ap)
for t in range(2):
    ctx.estep(alpha, w.K, 0, t, mu, s)
torch.cuda.synchronize()
ms = []
for t in range(reps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    if os.environ.get("TIME_PROBES_ONLY"):     # a probe-parallel rank that does not own the mean system
        ctx.estep_probes(alpha, w.K, 0, 2 + t, s)
    else:
        ctx.estep(alpha, w.K, 0, 2 + t, mu, s)
    b.record()
    torch.cuda.synchronize()
    ms.append(a.elapsed_time(b))
fz = ctx.report()["frozen_at"]
print("%s E-step at fixed alpha (U = %d): median %.2f ms (min %.2f) over %d; frozen_at max %d, mean %.1f, mean column %d" % (
    w.name, w.U, sorted(ms)[len(ms) // 2], min(ms), reps, max(fz), sum(fz) / len(fz), fz[0]))
