"""Exact EM on the GPU in fp64 -- the paper's EM baseline (Eq. 3-4, Table 1 "EM": O(T D^3) time,
O(D^2) space), for SURVEY §8(f) NEXT-3 and the §4 protocol (tools/protocol_s4.py).

This is a COMPARISON SYSTEM, not the CoFEM product path: it forms A = beta Phi^T Phi + diag(alpha)
explicitly (D x D), factors it with cuSOLVER's Cholesky (through torch.linalg), and takes the full
inverse for diag(Sigma):
    Sigma = A^-1,  mu = beta Sigma Phi^T y                       (Eq. 3)
    alpha = 1 / (mu o mu + Sigma[diag])  (floor 1e-12, clamp 1e12; Eq. 4, R7)
Checked against the CPU oracle's exact_em (oracle/exact.py) in tests/test_gpu_exact_em.py.
D <= 2^15 (the D x D matrices take 8 GB each there)."""
import time

import numpy as np
import torch


def dense_phi(w, device="cuda"):
    """Phi of a synth workload as an explicit fp64 N x D tensor (dense: the matrix; masked 2D DCT:
    the selected rows of C_r^T (x) C_c^T, convention 0 -- reading R11)."""
    if w.kind == "dense":
        return torch.as_tensor(np.asarray(w.phi, dtype=np.float64), device=device)
    if w.kind == "dct2_masked":
        def dctm(L):
            k = torch.arange(L, dtype=torch.float64, device=device)[:, None]
            n = torch.arange(L, dtype=torch.float64, device=device)[None, :]
            C = torch.cos(np.pi * (2 * n + 1) * k / (2 * L)) * np.sqrt(2.0 / L)
            C[0, :] = np.sqrt(1.0 / L)
            return C
        Cr, Cc = dctm(w.rows), dctm(w.cols)
        obs = torch.as_tensor(w.obs_idx, device=device)
        r, c = obs // w.cols, obs % w.cols
        if w.convention == 0:   # pixel (r, c) of C2^T z: sum_{k,l} Cr[k, r] Cc[l, c] z[k, l]
            return (Cr.T[r][:, :, None] * Cc.T[c][:, None, :]).reshape(w.N, w.D)
        return (Cr[r][:, :, None] * Cc[c][:, None, :]).reshape(w.N, w.D)
    raise ValueError(w.kind)


def exact_em(phi, y, beta, T, alpha_init=None, z_true=None, den_floor=1e-12, alpha_max=1e12):
    """T exact EM iterations.  Returns (alpha, mu, diag Sigma, per-iteration NRMSE of mu vs z_true
    (or None), seconds) -- timed with CUDA events, inputs resident on the device."""
    phi = phi.to(torch.float64)
    y = torch.as_tensor(np.asarray(y, dtype=np.float64), device=phi.device)
    D = phi.shape[1]
    alpha = torch.ones(D, dtype=torch.float64, device=phi.device) if alpha_init is None else \
        torch.as_tensor(np.asarray(alpha_init, dtype=np.float64), device=phi.device).clone()
    zt = None if z_true is None else torch.as_tensor(np.asarray(z_true, dtype=np.float64), device=phi.device)
    nrmse = []
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    G = beta * (phi.T @ phi)
    b = beta * (phi.T @ y)
    mu = sd = None
    for _ in range(T):
        A = G.clone()
        A.diagonal().add_(alpha)
        L = torch.linalg.cholesky(A)
        del A
        mu = torch.cholesky_solve(b[:, None], L)[:, 0]
        sd = torch.cholesky_inverse(L).diagonal().clone()
        del L
        alpha = torch.clamp(1.0 / torch.clamp(mu * mu + sd, min=den_floor), max=alpha_max)
        if zt is not None:
            nrmse.append(float(torch.linalg.norm(mu - zt) / torch.linalg.norm(zt)))
    e1.record()
    torch.cuda.synchronize()
    return (alpha.cpu().numpy(), mu.cpu().numpy(), sd.cpu().numpy(), nrmse if zt is not None else None,
            e0.elapsed_time(e1) / 1000.0)


def wall(fn):
    t0 = time.perf_counter()
    out = fn()
    return out, time.perf_counter() - t0
