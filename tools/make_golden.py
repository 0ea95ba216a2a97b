"""Write the full-configuration oracle fixtures under tests/golden/fullcfg/ (oracle side only).

This script calls ONLY oracle/ (the fp64 CPU implementation of Algorithm 1) and synth/ (the
seeded input generators): no value here comes from the CUDA path.  The GPU parity tests
(tests/test_gpu_fullcfg.py) read these files as the expected values at sizes whose oracle run
takes minutes to hours on the host, which is too long for a test.

Cases (BASELINE.json configs; DESIGN.md §4 "full-configuration parity"):
  C2_full   C2 at its configured K = 32, U = 200, T_em = 50 from alpha = 1: E-step 1 (mu1, s1)
            and the whole EM (alpha_in = alpha_49, mu, s of E-step 50, and its support).
  C3_e1     C3 at K = 64, U = 300: E-step 1 (alpha = 1).
  C3_ss     C3 at K = 4, U = 300: 6 EM iterations; alpha_in = alpha_5 (steady state: prior
            precisions spread over ~10 decades), mu, s of E-step 6.
  C4_ss     C4 (1024^2 masked DCT) at K = 4, U = 200: the same 6-iteration EM.
  C5s_ss    C5's filter and sparsity at D = 2^20 (the same FFT-convolution path), K = 4, U = 150:
            6-iteration EM; and C5s_k16: the configured K = 16 E-step at that alpha_5.
Probe seed 0; E-step t uses probe counter t (Algorithm 1 l.5, reading R8).

Storage: D-vectors at D >= 2^20 are stored as float32 (the bars are 1e-4 / 1e-3, rounding 6e-8),
except alpha_in, which is an INPUT and is stored exactly (fp64); support bits are computed in fp64.

    python tools/make_golden.py CASE [CASE ...]
    python tools/make_golden.py --slim      # drop the arrays the tests do not read (repo size)

Rounding sensitivity (cases <case>_pert, meta only): the oracle against ITSELF when its input is
perturbed at the rounding level -- alpha times (1 + 1e-15 r), r = +-1 seeded -- once for the
steady-state E-step (alpha_in) and once for the whole K = 4 EM from alpha = 1.  Where U leaves the
CG unconverged the iterate amplifies rounding, so two correct fp64 implementations that differ only
in summation order differ by about this much; the GPU tests use it as the floor of their bars
(reading R20).
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from oracle.cofem import cofem_em, estep, support  # noqa: E402
from oracle.operators import CircConvOp, DCT2MaskedOp, DenseOp  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "fullcfg")


def op_of(w):
    if w.kind == "dense":
        return DenseOp(w.phi)
    if w.kind == "dct2_masked":
        return DCT2MaskedOp(w.rows, w.cols, w.obs_idx, w.convention)
    return CircConvOp(w.taps, w.D)


def c5s():
    return synth.circconv(1 << 20, 64, 1048, K=16, U=150, T=20, seed=0, name="C5s_conv_2^20")


def workload(case):
    return {"C2_full": lambda: synth.preset("C2"), "C3_e1": lambda: synth.preset("C3"),
            "C3_ss": lambda: synth.preset("C3"), "C4_ss": lambda: synth.preset("C4"),
            "C5s_ss": c5s}[case]()


def vec(x, D):
    return np.asarray(x, dtype=np.float32 if D >= (1 << 20) else np.float64)


def save(case, meta, **arrays):
    os.makedirs(OUT, exist_ok=True)
    path = os.path.join(OUT, case + ".npz")
    np.savez_compressed(path, meta=json.dumps(meta), **arrays)
    print("wrote", path, {k: (v.dtype.name, v.shape) for k, v in arrays.items()}, flush=True)


def em_case(case, w, K, U, T, seed=0, extra_K=None):
    op = op_of(w)
    trace = []
    t0 = time.time()
    alpha, mu, s = cofem_em(op, w.y, w.beta, T, K, seed, U, trace=trace)
    sec = (time.time() - t0) / T
    alpha_in = trace[T - 2][0]                       # alpha after M-step T-1: input of E-step T
    meta = {"workload": w.name, "K": K, "U": U, "T": T, "seed": seed, "t_last": T - 1,
            "oracle_s_per_estep": sec, "threads": os.environ.get("OMP_NUM_THREADS", "default")}
    arrays = dict(alpha_in=alpha_in.astype(np.float64), mu=vec(mu, w.D), s=vec(s, w.D),
                  support=np.packbits(support(mu)), mu1=vec(trace[0][1], w.D), s1=vec(trace[0][2], w.D))
    save(case, meta, **arrays)
    if extra_K:
        t0 = time.time()
        mu2, s2, _ = estep(op, w.y, w.beta, alpha_in, extra_K, seed, T - 1, U)
        meta2 = dict(meta, K=extra_K, oracle_s_per_estep=time.time() - t0, from_case=case)
        save(case.replace("_ss", "_k%d" % extra_K), meta2, alpha_in=alpha_in.astype(np.float64),
             mu=vec(mu2, w.D), s=vec(s2, w.D), support=np.packbits(support(mu2)))


def slim():
    """Keep only what tests/test_gpu_fullcfg.py reads: the steady-state cases do not need their
    E-step-1 vectors, and C5s_k16 shares C5s_ss's alpha_in (the same oracle alpha_5)."""
    for name in sorted(os.listdir(OUT)):
        path = os.path.join(OUT, name)
        f = np.load(path)
        arrays = {k: f[k] for k in f.files if k != "meta"}
        meta = json.loads(str(f["meta"]))
        drop = []
        if name.endswith("_ss.npz"):
            drop = ["mu1", "s1"]
        if name.endswith("_k16.npz"):
            drop = ["alpha_in"]
            meta["alpha_in_from"] = meta.get("from_case")
        drop = [k for k in drop if k in arrays]
        if drop:
            for k in drop:
                arrays.pop(k)
            np.savez_compressed(path, meta=json.dumps(meta), **arrays)
            print("slimmed", name, "dropped", drop)


def rel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def elem(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))


def pert_case(case):
    """Oracle vs oracle at a 1e-15 relative perturbation of alpha (see the module docstring)."""
    base = case[:-len("_pert")]
    w = workload(base)
    f = np.load(os.path.join(OUT, base + ".npz"))
    meta = json.loads(str(f["meta"]))
    K, U, T, seed = meta["K"], meta["U"], meta["T"], meta["seed"]
    op = op_of(w)
    r = np.random.default_rng(12345).choice([-1.0, 1.0], size=w.D)
    a_in = f["alpha_in"] * (1.0 + 1e-15 * r)
    t0 = time.time()
    mu_p, s_p, _ = estep(op, w.y, w.beta, a_in, K, seed, T - 1, U)
    # the stored steady-state result (float32 at D >= 2^20) against the perturbed fp64 one
    out = {"workload": w.name, "K": K, "U": U, "T": T, "perturbation": "alpha * (1 + 1e-15 r), r = +-1",
           "estep_mu_rel": rel(mu_p, f["mu"]), "estep_s_rel": rel(s_p, f["s"]),
           "estep_mu_elem": elem(mu_p, f["mu"]), "estep_s_elem": elem(s_p, f["s"])}
    a_em, mu_em, s_em = cofem_em(op, w.y, w.beta, T, K, seed, U, alpha_init=np.ones(w.D) * (1.0 + 1e-15 * r))
    from oracle.cofem import mstep
    a_ref = mstep(f["mu"].astype(np.float64), f["s"].astype(np.float64))
    out.update({"em_inv_alpha_rel": rel(1 / a_em, 1 / a_ref), "em_mu_rel": rel(mu_em, f["mu"]),
                "em_inv_alpha_elem": elem(1 / a_em, 1 / a_ref), "em_mu_elem": elem(mu_em, f["mu"]),
                "em_support_flips": int(np.sum(support(mu_em) != np.unpackbits(f["support"])[:w.D].astype(bool))),
                "seconds": time.time() - t0})
    save(case, out)
    print(case, json.dumps(out), flush=True)


def main(cases):
    if cases == ["--slim"]:
        return slim()
    for case in cases:
        if case.endswith("_pert"):
            pert_case(case)
            continue
        w = workload(case)
        print(case, w.name, flush=True)
        if case == "C2_full":
            em_case(case, w, 32, 200, 50)
        elif case == "C3_e1":
            t0 = time.time()
            mu, s, _ = estep(op_of(w), w.y, w.beta, np.ones(w.D), 64, 0, 0, 300)
            save(case, {"workload": w.name, "K": 64, "U": 300, "seed": 0, "t": 0,
                        "oracle_s_per_estep": time.time() - t0}, mu=vec(mu, w.D), s=vec(s, w.D))
        elif case == "C3_ss":
            em_case(case, w, 4, 300, 6)
        elif case == "C4_ss":
            em_case(case, w, 4, 200, 6)
        elif case == "C5s_ss":
            em_case(case, w, 4, 150, 6, extra_K=16)
        else:
            raise KeyError(case)


if __name__ == "__main__":
    main(sys.argv[1:])
