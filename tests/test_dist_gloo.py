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

from paper_2202_12808_b200.dist import em_probe_parallel, probe_split


def test_probe_split_covers_all():
    for K in (1, 2, 7, 16, 32, 33):
        for world in range(1, min(K, 8) + 1):
            parts = [probe_split(K, world, r) for r in range(world)]
            ks = [k for off, n in parts for k in range(off, off + n)]
            assert ks == list(range(K)) and min(n for _, n in parts) >= 1
    with pytest.raises(ValueError):
        probe_split(2, 4, 0)


def _worker(rank, world, port, out):
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

    alpha, mu, s = np.ones(w.D), np.zeros(w.D), np.zeros(w.D)
    em_probe_parallel(estep_fn, mstep_fn, allreduce, 3, 6, 9, rank, world, alpha, mu, s)
    if rank == 0:
        np.save(out, np.stack([alpha, mu, s]))
    dist.destroy_process_group()


def test_probe_parallel_gloo_world2_equals_single(tmp_path):
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    out = str(tmp_path / "r0.npy")
    mp.start_processes(_worker, args=(2, port, out), nprocs=2, join=True, start_method="spawn")
    a, mu, s = np.load(out)
    import synth
    from oracle.cofem import cofem_em
    from oracle.operators import DenseOp
    w = synth.dense(40, 120, 4, K=6, U=200, T=3, seed=1)   # converged U: see DESIGN.md §4
    ea, emu, es = cofem_em(DenseOp(w.phi), w.y, w.beta, 3, 6, 9, w.U)
    rel = lambda x, y: np.linalg.norm(x - y) / np.linalg.norm(y)
    assert rel(a, ea) < 1e-10 and rel(mu, emu) < 1e-10 and rel(s, es) < 1e-10, (rel(a, ea), rel(mu, emu), rel(s, es))
