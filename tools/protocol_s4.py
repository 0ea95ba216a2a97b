"""The paper's §4 protocol on B200, CoFEM through the C
ABI (libcofem.so) against the exact-EM GPU baseline (tools/exact_em_gpu.py).  The IRLS / AMP / VI /
Seq comparison curves stay out of scope (comparison systems).
  (a) Fig. 1a  dense, D = 1024, f = 1..8, REPS repetitions: NRMSE after T_em = 50 (CoFEM K = 20, U = 400)
  (b) Fig. 1b  dense, f = 4, D = 2^9..2^PMAX: seconds for 30 EM iterations (CoFEM vs exact EM)
  (c) Fig. 1c  dense, D = 2^PMAX: NRMSE per EM iteration (CoFEM vs exact EM)
  (d) Fig. 1d  masked 2D DCT (synth.paper_dct), D = 2^9..2^PMAX: seconds for 30 EM iterations
  (e) Fig. 1e  DCT, D = 2^PMAX: NRMSE per EM iteration
  (f) Fig. 1f  DCT with d = 0.1 D, D = 2^12..2^18: CoFEM seconds to NRMSE <= 2 % (no Seq curve)
Writes one JSON object (stdout and --out).  Times: CUDA events around the EM iterations, inputs on
the device, setup excluded (the paper's 'running time for 30 EM iterations').
    python tools/protocol_s4.py --out profiles/r02/protocol_s4.json [--reps 25] [--pmax 15]"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import exact_em_gpu as eg  # noqa: E402
import synth  # noqa: E402
from paper_2202_12808_b200 import Context  # noqa: E402


def nrmse(mu, z):
    return float(np.linalg.norm(mu - z) / np.linalg.norm(z))


def cofem_run(w, T, K=20, U=400, trace=False):
    """T EM iterations of CoFEM; returns (seconds, final NRMSE, per-iteration NRMSE or None)."""
    ctx = Context.from_workload(w, max_probes=K, cg_iters=U)
    a = torch.ones(w.D, dtype=torch.float64, device="cuda")
    mu, s = torch.empty_like(a), torch.empty_like(a)
    ctx.em(1, K, 99, 1000, a, torch.empty_like(a), mu, s)          # warm-up (different probe stream)
    a.fill_(1.0)
    torch.cuda.synchronize()
    per = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if trace:
        sec = 0.0
        for t in range(T):
            e0.record()
            ctx.em(1, K, 0, t, a, a, mu, s)
            e1.record()
            torch.cuda.synchronize()
            sec += e0.elapsed_time(e1) / 1000.0
            per.append(nrmse(mu.cpu().numpy(), w.z_true))
    else:
        e0.record()
        ctx.em(T, K, 0, 0, a, a, mu, s)
        e1.record()
        torch.cuda.synchronize()
        sec = e0.elapsed_time(e1) / 1000.0
    ctx.close()
    return sec, nrmse(mu.cpu().numpy(), w.z_true), (per if trace else None)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=25)
    ap.add_argument("--pmax", type=int, default=15)
    ap.add_argument("--pmax_f", type=int, default=18)
    ap.add_argument("--parts", default="abcdef")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    out = {"gpu": torch.cuda.get_device_name(0), "cofem": {"K": 20, "U": 400}, "parts": {}}
    if "a" in args.parts:
        rows = []
        for f in range(1, 9):
            ce, ee = [], []
            for rep in range(args.reps):
                w = synth.paper_dense(1024, f, seed=rep, T=50)
                ce.append(cofem_run(w, 50)[1])
                _, mu, _, _, _ = eg.exact_em(eg.dense_phi(w), w.y, w.beta, 50)
                ee.append(nrmse(mu, w.z_true))
            rows.append({"f": f, "cofem_nrmse_mean": float(np.mean(ce)), "em_nrmse_mean": float(np.mean(ee)),
                         "cofem_nrmse_median": float(np.median(ce)), "em_nrmse_median": float(np.median(ee))})
            print("a", rows[-1], flush=True)
        out["parts"]["a_fig1a_dense_nrmse_vs_f"] = {"D": 1024, "T_em": 50, "reps": args.reps, "rows": rows}
    for part, kind in (("b", "dense"), ("d", "dct")):
        if part not in args.parts:
            continue
        rows = []
        for p in range(9, args.pmax + 1):
            w = synth.paper_dense(1 << p, 4, seed=0, T=30) if kind == "dense" else synth.paper_dct(p, seed=0, T=30)
            trace = p == args.pmax
            cs, cn, cper = cofem_run(w, 30, trace=trace)
            phi = eg.dense_phi(w)
            _, mu, _, eper, es = eg.exact_em(phi, w.y, w.beta, 30, z_true=w.z_true)
            del phi
            torch.cuda.empty_cache()
            rows.append({"D": w.D, "N": w.N, "cofem_s": cs, "exact_em_s": es, "speedup": es / cs,
                         "cofem_nrmse": cn, "em_nrmse": nrmse(mu, w.z_true)})
            print(part, rows[-1], flush=True)
            if trace:
                key = "c_fig1c_dense_convergence" if kind == "dense" else "e_fig1e_dct_convergence"
                out["parts"][key] = {"D": w.D, "cofem_nrmse_per_iter": cper, "em_nrmse_per_iter": eper}
        key = "b_fig1b_dense_time_vs_D" if kind == "dense" else "d_fig1d_dct_time_vs_D"
        out["parts"][key] = {"f": 4, "T_em": 30, "rows": rows}
    if "f" in args.parts:
        rows = []
        for p in range(12, args.pmax_f + 1):
            w = synth.paper_dct(p, seed=0, frac=0.1, T=60)
            ctx = Context.from_workload(w, max_probes=20, cg_iters=400)
            a = torch.ones(w.D, dtype=torch.float64, device="cuda")
            mu, s = torch.empty_like(a), torch.empty_like(a)
            torch.cuda.synchronize()
            sec, it, nr = 0.0, 0, 1.0
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            while it < 60 and nr > 0.02:
                e0.record()
                ctx.em(1, 20, 0, it, a, a, mu, s)
                e1.record()
                torch.cuda.synchronize()
                sec += e0.elapsed_time(e1) / 1000.0
                nr = nrmse(mu.cpu().numpy(), w.z_true)
                it += 1
            ctx.close()
            rows.append({"D": w.D, "em_iters": it, "cofem_s_to_2pct": sec, "nrmse": nr})
            print("f", rows[-1], flush=True)
        out["parts"]["f_fig1f_dct_time_to_2pct"] = {"d": "0.1 D", "rows": rows}
    js = json.dumps(out)
    if args.out:
        os.makedirs(os.path.dirname(args.out), exist_ok=True)
        open(args.out, "w").write(js + "\n")
    print(js)


if __name__ == "__main__":
    main()
