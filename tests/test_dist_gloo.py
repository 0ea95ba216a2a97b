"""Probe-parallel host logic (paper_2202_12808_b200/dist.py) on CPU with gloo, world size 2.

The E-step / M-step are the oracle's (this is a test of the sharding and the
exchange, not of the kernels): the distributed result must equal the
single-process oracle EM.
"""
import os

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2202_12808_b200.dist import em_probe_parallel, probe_split, probe_split_owner


def test_probe_split_covers_all():
    for K in (1, 2, 7, 16, 32, 33):
        for world in range(1, min(K, 8) + 1):
            parts = [probe_split(K, world, r) for r in range(world)]
            ks = [k for off, n in parts for k in range(off, off + n)]
            assert ks == list(range(K)) and min(n for _, n in parts) >= 1
    with pytest.raises(ValueError):
        probe_split(2, 4, 0)


def test_probe_split_owner_covers_all_and_balances():
    for K in (2, 7, 16, 32, 33):
        for world in range(1, min(K, 8) + 1):
            for cost in (0.0, 1.0, 6.5, 40.0):
                parts = [probe_split_owner(K, world, r, cost) for r in range(world)]
                ks = [k for off, n, _ in parts for k in range(off, off + n)]
                assert ks == list(range(K)) and min(n for _, n, _ in parts) >= 1
                assert [o for _, _, o in parts] == [True] + [False] * (world - 1)
    # C4 at 8 GPUs: the owner of a 6.5-probe mean system gets 1 probe, the others 4-5
    assert [n for _, n, _ in (probe_split_owner(32, 8, r, 6.5) for r in range(8))] == [1, 5, 5, 5, 4, 4, 4, 4]


def _worker(rank, world, port, out, mean_cost=None):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch

    import synth
    from oracle.cofem import estep, mstep
    from oracle.operators import DenseOp
    w = synth.dense(40, 120, 4, K=6, U=200, T=3, seed=1)   # converged U: see DESIGN.md §4
    op = DenseOp(w.phi)

    def estep_fn(alpha, K_local, seed, t, mu, s, k_offset, K_total):
        m, s_loc, _ = estep(op, w.y, w.beta, alpha, K_local, seed, t, w.U, k_offset=k_offset)
        mu[:] = m
        s[:] = s_loc * K_local / K_total          # partial (1/K) sum over this rank's probes

    def allreduce(s):
        t = torch.from_numpy(s)
        dist.all_reduce(t)                          # in place on the shared buffer

    def mstep_fn(mu, s, alpha):
        alpha[:] = mstep(mu, s)

    def estep_probes_fn(alpha, K_local, seed, t, s, k_offset, K_total):
        _, s_loc, _ = estep(op, w.y, w.beta, alpha, K_local, seed, t, w.U, k_offset=k_offset)
        s[:] = s_loc * K_local / K_total

    def broadcast(mu):
        dist.broadcast(torch.from_numpy(mu), src=0)

    alpha, mu, s = np.ones(w.D), np.zeros(w.D), np.zeros(w.D)
    if rank > 0 and mean_cost is not None:
        mu[:] = np.nan                              # never computed here: must arrive by broadcast
    em_probe_parallel(estep_fn, mstep_fn, allreduce, 3, 6, 9, rank, world, alpha, mu, s,
                      mean_cost=mean_cost, estep_probes=estep_probes_fn, broadcast=broadcast)
    np.save(out + ".%d.npy" % rank, np.stack([alpha, mu, s]))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,mean_cost", [(2, None), (2, 1.5), (3, 2.0)])
def test_probe_parallel_gloo_world2_equals_single(tmp_path, world, mean_cost):
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    out = str(tmp_path / "r")
    mp.start_processes(_worker, args=(world, port, out, mean_cost), nprocs=world, join=True, start_method="spawn")
    for r in range(1, world):                      # every rank ends with the same alpha, mu, s
        assert np.array_equal(np.load(out + ".%d.npy" % r), np.load(out + ".0.npy"))
    a, mu, s = np.load(out + ".0.npy")
    import synth
    from oracle.cofem import cofem_em
    from oracle.operators import DenseOp
    w = synth.dense(40, 120, 4, K=6, U=200, T=3, seed=1)   # converged U: see DESIGN.md §4
    ea, emu, es = cofem_em(DenseOp(w.phi), w.y, w.beta, 3, 6, 9, w.U)
    rel = lambda x, y: np.linalg.norm(x - y) / np.linalg.norm(y)
    assert rel(a, ea) < 1e-10 and rel(mu, emu) < 1e-10 and rel(s, es) < 1e-10, (rel(a, ea), rel(mu, emu), rel(s, es))


# ---------------------------------------------------------------- column-sharded dense mode
def test_column_shard_covers_all_aligned():
    from paper_2202_12808_b200.dist import column_shard
    for D in (256, 400, 1000, 8000, 32768):
        for world in (1, 2, 3, 4, 8):
            if (D + 127) // 128 < world:
                continue
            parts = [column_shard(D, world, r) for r in range(world)]
            assert [d for off, n in parts for d in range(off, off + n)] == list(range(D))
            assert all(off % 128 == 0 for off, _ in parts) and min(n for _, n in parts) >= 1


def _col_worker(rank, world, port, out, sr=False):
    """One rank of the column-sharded E-step, following the library's schedule exactly
    (op_dense_tc.cu + cofem.cu sharded path): local b0 / colsq / probes of the rank's global
    d range; every reduction the library sends through NCCL (rho0, W = Phi P and Phi p0,
    gamma, rho') is a gloo all-reduce here; the step lengths are then taken identically on
    every rank.  Local arithmetic is plain NumPy fp64 (this is a test of the decomposition
    and the exchange schedule, not of the kernels).  sr: the single-reduction CG (cg_variant 2,
    reading R23, the library's default in this mode) -- ONE all-reduce of (gamma, rho = r^T M^-1 r,
    delta1 = q^T M^-1 r, delta2 = q^T M^-1 q) per iteration, a = rho / gamma,
    rho' = rho - 2 a delta1 + a^2 delta2 (for b only), and no reduction after the update."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch

    import synth
    from oracle.philox import rademacher_probes
    from paper_2202_12808_b200.dist import column_shard
    w = synth.dense(60, 640, 6, K=5, U=200, T=1, seed=3)   # converged U
    d0, Dr = column_shard(w.D, world, rank)
    Phi = w.phi.astype(np.float64)[:, d0:d0 + Dr]
    alpha = np.linspace(0.5, 3.0, w.D)[d0:d0 + Dr]
    beta, K, U = w.beta, w.K, w.U

    def ar(x):
        t = torch.from_numpy(np.array(x, dtype=np.float64, copy=True))
        dist.all_reduce(t)
        return t.numpy()

    b0 = beta * Phi.T @ w.y.astype(np.float64)
    diag = beta * np.sum(Phi * Phi, axis=0) + alpha
    P = rademacher_probes(w.D, K, 11, 0)[d0:d0 + Dr]          # global d range (reading R8)
    B = np.concatenate([b0[:, None], P], axis=1)
    X = np.zeros_like(B)
    R = B.copy()
    Z = R / diag[:, None]
    Pd = Z.copy()
    rho = ar(np.sum(R * Z, axis=0))                            # k_init -> colsum -> all-reduce
    rho0 = rho.copy()
    frozen = np.zeros(K + 1, dtype=bool)
    for _ in range(U):
        W = ar(Phi @ Pd)                                       # K1 partial W -> all-reduce
        Q = beta * Phi.T @ W + alpha[:, None] * Pd             # K2 (local rows)
        if sr:                                                 # k_sr_dots + one all-reduce (mode 3)
            g4 = ar(np.concatenate([np.sum(Pd * Q, axis=0), np.sum(R * R / diag[:, None], axis=0),
                                    np.sum(Q * R / diag[:, None], axis=0), np.sum(Q * Q / diag[:, None], axis=0)]))
            gamma, rho_f, d1, d2 = (g4[i * (K + 1):(i + 1) * (K + 1)] for i in range(4))
            rho = np.where(frozen, rho, rho_f)                   # the current rho, recomputed (no drift)
        else:
            gamma = ar(np.sum(Pd * Q, axis=0))                 # gamma -> colsum -> all-reduce
        with np.errstate(all="ignore"):                        # freeze rule R5, same on every rank
            ok = np.isfinite(gamma) & np.isfinite(rho) & (gamma > 0) & (rho > 1e-30 * rho0)
        frozen |= ~ok
        act = ~frozen
        a = np.where(act, rho / np.where(act, gamma, 1.0), 0.0)
        X += a * Pd
        R -= a * Q
        Z = R / diag[:, None]
        if sr:
            rho_new = rho - 2 * a * d1 + a * a * d2             # k_sharded_finish mode 3
        else:
            rho_new = ar(np.sum(R * Z, axis=0))                # rho' -> colsum -> all-reduce
        b = np.where(act, rho_new / rho, 0.0)
        Pd = np.where(act, Z + b * Pd, Pd)
        rho = np.where(act, rho_new, rho)
    mu = X[:, 0]
    s = np.mean(P * X[:, 1:], axis=1)
    full = np.zeros(w.D)
    full[d0:d0 + Dr] = mu
    mu_full = ar(full)
    full = np.zeros(w.D)
    full[d0:d0 + Dr] = s
    s_full = ar(full)
    if rank == 0:
        np.save(out, np.stack([mu_full, s_full]))
    dist.destroy_process_group()


@pytest.mark.parametrize("sr", [False, True], ids=["two_reductions", "single_reduction"])
def test_column_sharded_gloo_world2_equals_single(tmp_path, sr):
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    out = str(tmp_path / "c0.npy")
    mp.start_processes(_col_worker, args=(2, port, out, sr), nprocs=2, join=True, start_method="spawn")
    mu, s = np.load(out)
    import synth
    from oracle.cofem import estep
    from oracle.operators import DenseOp
    w = synth.dense(60, 640, 6, K=5, U=200, T=1, seed=3)   # converged U
    alpha = np.linspace(0.5, 3.0, w.D)
    emu, es, _ = estep(DenseOp(w.phi), w.y, w.beta, alpha, w.K, 11, 0, w.U)
    rel = lambda x, y: np.linalg.norm(x - y) / np.linalg.norm(y)
    assert rel(mu, emu) < 1e-8 and rel(s, es) < 1e-8, (rel(mu, emu), rel(s, es))


# ---------------------------------------------------------------- D-sharded convolution (halo exchange)
def _halo_worker(rank, world, port, out):
    """One rank of the D-sharded Gram apply q = beta g * p + alpha o p (g = autocorr(h), 127
    taps) following comm_halo's ring schedule: send the first 64 samples to the left
    neighbour and the last 64 to the right one, receive the right / left halos, convolve the
    extended window, keep the rank's own outputs.  gloo point-to-point stands in for NCCL."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch

    import synth
    from paper_2202_12808_b200.dist import column_shard
    w = synth.circconv(3000, 64, 5, K=2, U=1, T=1, seed=5)
    d0, Dl = column_shard(w.D, world, rank)
    rng = np.random.default_rng(7)
    p_full = rng.standard_normal(w.D)
    alpha = rng.uniform(0.5, 2.0, w.D)
    p = p_full[d0:d0 + Dl]
    left, right = (rank - 1) % world, (rank + 1) % world
    send_l, send_r = torch.from_numpy(p[:64].copy()), torch.from_numpy(p[-64:].copy())
    recv_l, recv_r = torch.zeros(64, dtype=torch.float64), torch.zeros(64, dtype=torch.float64)
    reqs = [dist.isend(send_l, left), dist.isend(send_r, right), dist.irecv(recv_r, right), dist.irecv(recv_l, left)]
    for r in reqs:
        r.wait()
    ext = np.concatenate([recv_l.numpy(), p, recv_r.numpy()])      # samples d0-64 .. d0+Dl+63
    h = w.taps.astype(np.float64)
    g = np.correlate(h, h, mode="full")                             # g_l, l = -63 .. 63
    H = len(h) - 1
    q = np.array([np.dot(g, ext[64 + i - H:64 + i + H + 1]) for i in range(Dl)])
    q = w.beta * q + alpha[d0:d0 + Dl] * p
    gam = torch.tensor([np.dot(p, q)])
    dist.all_reduce(gam)                                           # gamma = p^T q over ranks
    full = torch.zeros(w.D, dtype=torch.float64)
    full[d0:d0 + Dl] = torch.from_numpy(q)
    dist.all_reduce(full)
    if rank == 0:
        np.save(out, np.concatenate([full.numpy(), gam.numpy()]))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_d_sharded_conv_halo_gloo(tmp_path, world):
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    out = str(tmp_path / "h0.npy")
    mp.start_processes(_halo_worker, args=(world, port, out), nprocs=world, join=True, start_method="spawn")
    res = np.load(out)
    q, gam = res[:-1], res[-1]
    import synth
    from oracle.operators import CircConvOp, gram_apply
    w = synth.circconv(3000, 64, 5, K=2, U=1, T=1, seed=5)
    rng = np.random.default_rng(7)
    p = rng.standard_normal(w.D)
    alpha = rng.uniform(0.5, 2.0, w.D)
    ref = gram_apply(CircConvOp(w.taps, w.D), w.beta, alpha, p[:, None])[:, 0]
    assert np.linalg.norm(q - ref) / np.linalg.norm(ref) < 1e-12
    assert abs(gam - p @ ref) / abs(p @ ref) < 1e-12
