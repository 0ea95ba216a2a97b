"""How much CG work the bench's timed EM iterations really do: replays bench.py's sequence
(W warm-up EM iterations, then the timed ones) and prints, per EM iteration, the number of
probe columns that froze (R5) and the fraction of the U x K probe column-iterations executed.
    python tools/freeze_check.py C4 [W=3] [steps=3]"""
import sys
import torch
sys.path.insert(0, "/root/repo")
import synth
from paper_2202_12808_b200 import Context

w = synth.preset(sys.argv[1] if len(sys.argv) > 1 else "C4")
W = int(sys.argv[2]) if len(sys.argv) > 2 else 3
S = int(sys.argv[3]) if len(sys.argv) > 3 else 3
ctx = Context.from_workload(w, max_probes=w.K)
alpha = torch.ones(w.D, dtype=torch.float64, device="cuda")
mu, s = torch.empty_like(alpha), torch.empty_like(alpha)
for t in range(W + S):
    ctx.em(1, w.K, 0, t, alpha, alpha, mu, s)
    r = ctx.report()
    fz = r["frozen_at"][1:]
    done = sum(w.U if f < 0 else min(f + 1, w.U) for f in fz)
    print("%s t=%d %s: frozen %d/%d, mean frozen_at %s, work fraction %.4f, mean column frozen_at %d" % (
        w.name, t, "warmup" if t < W else "timed", sum(f >= 0 for f in fz), len(fz),
        (sum(f for f in fz if f >= 0) / max(1, sum(f >= 0 for f in fz))), done / float(w.U * len(fz)), r["frozen_at"][0]))
