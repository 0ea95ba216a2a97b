"""Probe-parallel CoFEM over ranks (one process per GPU; BASELINE north_star multi-GPU mode).

The K probe columns of Eq. 7 are independent systems (reading R3), so rank r
solves probes [k_offset, k_offset + K_r) with their GLOBAL indices in the Philox
counter (reading R8) plus either a replica of the deterministic mean column, or (mean_cost
given) only rank 0 solves the mean system, with fewer probes, and broadcasts mu; the
exchange is one sum-allreduce of the partial s = (1/K) sum_{k in rank} p_k o x_k per
E-step (Eq. 6) (+ the mu broadcast), after which every rank applies the M-step (Eq. 8).
The collective is injected (torch.distributed NCCL on GPUs, gloo in the CPU
tests); this module holds only the host-side orchestration.  The product's multi-GPU
probe-parallel mode lives in the library itself (cofem_options.dist_mode = 1: NCCL all-reduce of s
and broadcast of mu inside cofem_estep / cofem_em); this module is its host-side model, exercised
over gloo in tests/test_dist_gloo.py.
"""
import math


def column_shard(D, world, rank, align=128):
    """Column-sharded dense mode: contiguous slice [d_offset, d_offset + D_r)
    of the D columns of Phi for `rank`, boundaries multiples of `align` (the probe counter
    block, reading R8) so every rank regenerates the same p_k[d] for its global d.
    Returns (d_offset, D_r)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    blocks = (D + align - 1) // align
    if blocks < world:
        raise ValueError("column sharding needs >= %d columns per rank" % align)
    base, extra = divmod(blocks, world)
    b0 = rank * base + min(rank, extra)
    b1 = b0 + base + (1 if rank < extra else 0)
    d0, d1 = b0 * align, min(D, b1 * align)
    return d0, d1 - d0


def probe_split(K, world, rank):
    """Contiguous split of K probes over `world` ranks: (k_offset, K_local)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    if K < world:
        raise ValueError("probe-parallel needs K >= world (every rank solves >= 1 probe)")
    base, extra = divmod(K, world)
    K_local = base + (1 if rank < extra else 0)
    k_offset = rank * base + min(rank, extra)
    return k_offset, K_local


def probe_split_owner(K, world, rank, mean_cost):
    """Probe split when rank 0 OWNS the mean system (the other ranks skip it, cofem_estep_probes,
    and receive mu by broadcast).  mean_cost = the mean system's effective cost in probe columns
    (it runs concurrently with the probes: bench.py mean_cost).  Rank 0 gets
    K0 = max(1, floor((K + mean_cost) / world - mean_cost + 1/2)) probes (the library's own split in the
    probe-parallel mode, cofem.cu pp_split, is the same rule), the other ranks split the
    remaining K - K0 contiguously (>= 1 each).  Returns (k_offset, K_local, owns_mean)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    if world == 1:
        return 0, K, True
    if K < world:
        raise ValueError("probe-parallel needs K >= world (every rank solves >= 1 probe)")
    K0 = max(1, min(K - (world - 1), int(math.floor((K + mean_cost) / world - mean_cost + 0.5))))
    if rank == 0:
        return 0, K0, True
    off, n = probe_split(K - K0, world - 1, rank - 1)
    return K0 + off, n, False


def em_probe_parallel(estep, mstep, allreduce_sum, T, K, seed, rank, world, alpha, mu, s, t0=0,
                      mean_cost=None, estep_probes=None, broadcast=None):
    """Algorithm 1 with the probes split over ranks.

    estep(alpha, K_local, seed, t, mu, s, k_offset, K_total) writes mu and this
    rank's partial s; allreduce_sum(s) sums s over ranks in place; mstep(mu, s,
    alpha) overwrites alpha.  Returns (alpha, mu, s) of the last iteration (R9).
    """
    if mean_cost is None or world == 1:          # every rank solves the (deterministic) mean system
        k_offset, K_local = probe_split(K, world, rank)
        owns = True
    else:                                        # rank 0 owns it: estep_probes elsewhere, mu broadcast
        k_offset, K_local, owns = probe_split_owner(K, world, rank, mean_cost)
    for t in range(t0, t0 + T):
        if owns:
            estep(alpha, K_local, seed, t, mu, s, k_offset, K)
        else:
            estep_probes(alpha, K_local, seed, t, s, k_offset, K)
        if world > 1:
            allreduce_sum(s)
            if mean_cost is not None:
                broadcast(mu)                    # from rank 0
        mstep(mu, s, alpha)
    return alpha, mu, s
