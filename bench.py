#!/usr/bin/env python
"""bench.py — CoFEM hot path on B200 (BASELINE.json metric: EM iters/s and CG
RHS-operator-applies/s at D = 2^20; % of HBM roofline).

A step = one EM iteration of Algorithm 1: probes, Jacobi-PCG with
U iterations on the K+1 columns, s, M-step — every row of SURVEY.md §8(a) —
on the synthetic workload of BASELINE config 4 (masked 1024 x 1024 DCT,
N = 2^18, K = 32, U = 200), with alpha carried from step to step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload C4]

N > 1 (one process per GPU; `--gpus N` re-launches itself under torch.distributed.run when
WORLD_SIZE is unset): probe-parallel inside the library (cofem_options.dist_mode = 1) — rank 0
solves the mean system and a smaller share of the K probes, the others their shares; one NCCL
all-reduce of s and one broadcast of mu per E-step; total work fixed ("strong").  The line
carries the N-rank vs 1-rank difference of mu and s (multirank_check).  --mode column: the
column-sharded dense / D-sharded convolution modes.  --impl reference times the CPU fp64 oracle
(oracle/) on a bounded sample (rank 0 only).
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "EM iters/s and CG RHS-operator-applies/s at D=2^20; % of HBM/compute roofline"
UNIT = "EM iters/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="C4")
    ap.add_argument("--mode", default="probe", choices=["probe", "column"],
                    help="multi-GPU partitioning: probe-parallel (any operator) or column-sharded dense Phi")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-conformance", action="store_true",
                    help="skip the fast-vs-parity-mode support comparison (2 extra EM iterations per mode)")
    ap.add_argument("--prof-steps", type=int, default=0,
                    help="EM iterations of the per-kernel profiled pass (0 = all timed iterations)")
    ap.add_argument("--rtol", type=float, default=0.0,
                    help="NEXT-1: the paper's CG stopping rule eps (per-column freezing, U stays the cap); "
                         "0 = the BASELINE fixed-U contract")
    return ap.parse_args()


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clock and throttle reasons sampled DURING the timed region (B200_PROFILING recipe):
    NVML polled every 5 ms from a thread (nvidia-smi -lms as the fallback)."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index):
        self.index, self.lines, self.proc, self.nvml = index, [], None, None
        self.samples, self.stop_flag = [], threading.Event()

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            bits = [pynvml.nvmlClocksEventReasonHwSlowdown, pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                    pynvml.nvmlClocksEventReasonSwThermalSlowdown, pynvml.nvmlClocksEventReasonSwPowerCap]
            self.nvml = (pynvml, h, bits, pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))

            def poll():
                while not self.stop_flag.is_set():
                    sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                    rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.samples.append((sm, [n for n, bit in zip(self.NAMES, bits) if rs & bit]))
                    time.sleep(0.005)
            self.t = threading.Thread(target=poll, daemon=True)
            self.t.start()
            return
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.nvml:
            self.stop_flag.set()
            self.t.join(timeout=1.0)
            sm = sorted(x for x, _ in self.samples)
            reasons = sorted({n for _, rs in self.samples for n in rs})
            return {"sm_mhz": float(sm[len(sm) // 2]) if sm else None, "sm_max_mhz": float(self.nvml[3]),
                    "reasons": reasons, "samples": len(sm), "source": "nvml, 5 ms"}
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 7:
                continue
            try:
                sm.append(float(p[0]))
                mx = float(p[1])
            except ValueError:
                continue
            for n, v in zip(self.NAMES, p[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "source": "nvidia-smi -lms 50"}


# ------------------------------------------------------------------ algorithmic bytes per launch
def algorithmic_bytes(cls, w, K_local, D_local=None):
    """Bytes the algorithm must move per launch of kernel class `cls`:
    4 B per fp32 probe element, D elements per column; arrays shared by all columns
    (dinv, alpha, s, probe bits) are counted once per launch.  On the 1024 x 1024 DCT
    fast path the fp64 mean column runs as its own class ("mean_column") on a second
    stream, so the probe classes count the K probe columns only."""
    D, K = (D_local or w.D), K_local
    fast = w.kind == "dct2_masked" and w.rows == 1024 and w.cols == 1024
    if cls == "dct_rows_inv":      # read r, p; write p (direction), write T^T; dinv once
        return D * (16 * K + 4) if fast else D * (16 * K + 32 + 4 + 8)
    if cls == "dct_cols":          # read T^T, write T2
        return D * 8 * K if fast else D * (8 * K + 16)
    if cls == "dct_rows_fwd":      # read T2, p; write q; alpha once
        return D * (12 * K + 4) if fast else D * (12 * K + 24 + 8)
    if cls == "pcg_update":        # r, q, p read + r write per probe; s read-modify-write, dinv, bits once
        return D * (16 * K + 16 + 4) + D * K // 8 + (0 if fast else D * 56)
    if cls == "pcg_direction":     # r, p read, p write (+dinv)
        return D * (12 * K + 24 + 12)
    if cls == "conv_apply":        # r, p read, p (direction, other buffer), q write; dinv, alpha once
        return D * (16 * K + 8)
    if cls == "dense_phiT_w":      # Phi once, p read, q write, alpha
        return w.N * D * 4 + D * (8 * K + 16 + 8)
    if cls == "dense_phi_p":
        return w.N * D * 4 + D * (4 * K + 8)
    if cls == "dense_cluster":     # the whole CG loop in one cluster: Phi and the state once per E-step
        return w.N * D * 4 + D * (12 * K + 64)
    return None


def active_bytes(cls, w, K_local, D_local, groups, frozen):
    """Algorithmic bytes class `cls` moved over the profiled E-steps, counting only the work
    the kernels execute: a column frozen at CG iteration F (R5, report frozen_at) is applied in
    iterations 0..F and updated (and, on the dense path, given a new direction) in 0..F-1; the
    per-column bytes count per active column-iteration and the arrays shared by a launch's
    columns once per launch with an active column (launch g of an iteration covers the probe
    columns [gj[g], gj[g+1]), gj[g] = 1 + K g / G, as cg_loop_split).  Returns (bytes, executed
    fraction of the U x K column-iterations)."""
    U, K = w.U, K_local
    shared = algorithmic_bytes(cls, w, 0, D_local)
    per_col = algorithmic_bytes(cls, w, 1, D_local) - shared
    lag = 0 if cls in ("pcg_update", "pcg_direction") else 1
    gj = [1 + (K * g) // groups for g in range(groups + 1)]
    tot, colit = 0.0, 0
    for fz in frozen:
        act = [U if f < 0 else min(f + lag, U) for f in fz[1:K + 1]]
        colit += sum(act)
        tot += per_col * sum(act)
        for g in range(groups):
            tot += shared * max(act[gj[g] - 1:gj[g + 1] - 1], default=0)
    return tot, colit / float(max(1, U * K * len(frozen)))


def working_set_bytes(w, K_local, D_local):
    """Bytes one E-step keeps touching: ~5 fp32 vectors per probe column (r, p, q, x, z) plus
    the operator's own storage (dense Phi; the DCT mask and conv taps are negligible)."""
    b = (K_local + 1) * D_local * 4 * 5
    if w.kind == "dense":
        b += w.N * D_local * 4
    return b


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


# ------------------------------------------------------------------ CPU oracle sample
def cpu_sample(w, seed=0):
    """Time the oracle (as it stands) on a bounded sample of one E-step of w: the
    setup part (probes, b0, Jacobi diagonal) and one PCG iteration of all K+1
    columns; E-step time = setup + U x iteration (the oracle's PCG cost is
    linear in U).  Returns (EM iters/s, description, threads)."""
    import numpy as np

    from oracle.cofem import jacobi_diag, mean_rhs, pcg
    from oracle.operators import CircConvOp, DCT2MaskedOp, DenseOp, gram_apply
    from oracle.philox import rademacher_probes
    try:
        from threadpoolctl import threadpool_info
        threads = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        threads = os.cpu_count()
    if w.kind == "dense":
        op = DenseOp(w.phi)
    elif w.kind == "dct2_masked":
        op = DCT2MaskedOp(w.rows, w.cols, w.obs_idx, w.convention)
    else:
        op = CircConvOp(w.taps, w.D)
    alpha = np.ones(w.D)
    t0 = time.perf_counter()
    b0 = mean_rhs(op, w.y, w.beta)
    diag = jacobi_diag(op, w.beta, alpha)
    P = rademacher_probes(w.D, w.K, seed, 0)
    B = np.concatenate([b0[:, None], P], axis=1)
    t1 = time.perf_counter()
    pcg(lambda V: gram_apply(op, w.beta, alpha, V), B, diag, 1)
    t2 = time.perf_counter()
    est = (t1 - t0) + w.U * (t2 - t1)
    desc = ("oracle E-step setup + 1 of U=%d PCG iterations on all %d columns of %s (%.1f s measured), "
            "E-step time extrapolated linearly in U" % (w.U, w.K + 1, w.name, t2 - t0))
    return 1.0 / est, desc, threads, t2 - t0


# ------------------------------------------------------------------ reference arm
def run_reference(args, rank):
    if rank != 0:
        return 0
    import synth
    w = synth.preset(args.workload, seed=args.seed)
    for _ in range(args.warmup):
        cpu_sample(w, args.seed)
    vals, descs, threads = [], None, 1
    t0 = time.perf_counter()
    for _ in range(args.steps):
        v, descs, threads, _ = cpu_sample(w, args.seed)
        vals.append(v)
    wall = time.perf_counter() - t0
    value = len(vals) / sum(1.0 / v for v in vals)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 / value,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": w.name, **w.config()},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": descs},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "wall_s": wall}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ our arm
def spawn_ranks(args):
    """`bench.py --gpus N` without a torchrun environment: re-launch this script as N ranks (one
    process per GPU) with torch.distributed.run on 127.0.0.1; rank 0 prints the JSON line."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(args.gpus),
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def executed_applies(frozen, U):
    """Column-iterations whose apply actually ran: a column frozen at CG iteration F (R5,
    report frozen_at) is applied in iterations 0..F (the apply of iteration F finds it frozen)."""
    return sum(sum(U if f < 0 else min(f + 1, U) for f in fz) for fz in frozen)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank)
    if args.warmup < 3:
        raise SystemExit("timing rules: --warmup must be >= 3")

    import numpy as np
    import torch

    import synth
    from paper_2202_12808_b200 import Context, get_unique_id
    from paper_2202_12808_b200.dist import column_shard
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    w = synth.preset(args.workload, seed=args.seed)
    column = args.mode == "column"
    nid = None
    if world > 1:       # the library's own NCCL communicator: one id from rank 0, broadcast
        box = [get_unique_id() if rank == 0 else None]
        torch.distributed.broadcast_object_list(box, src=0)
        nid = box[0]
    d0 = 0
    if column:
        # column-sharded dense Phi / D-sharded convolution: rank r holds the D-slice
        # [d0, d0 + Dr) of Phi (or of the signal) and of alpha, mu, s; the library all-reduces W and
        # the column dots (or exchanges the 64-sample halos) over NCCL inside the E-step
        if w.kind not in ("dense", "circconv"):
            raise SystemExit("--mode column needs a dense (C1-C3, column-sharded) or convolution (C5, D-sharded) workload")
        from paper_2202_12808_b200 import OP_CIRCCONV, OP_DENSE
        d0, Dr = column_shard(w.D, world, rank)
        if nid is None:
            nid = get_unique_id()
        if w.kind == "dense":
            ctx = Context(OP_DENSE, w.N, Dr, w.y, w.beta, phi=np.ascontiguousarray(w.phi[:, d0:d0 + Dr]),
                          cg_iters=w.U, max_probes=w.K, rank=rank, world=world, nccl_id=nid, d_offset=d0,
                          D_global=w.D, cg_rtol=args.rtol)
        else:
            ctx = Context(OP_CIRCCONV, Dr, Dr, np.ascontiguousarray(w.y[d0:d0 + Dr]), w.beta, taps=w.taps,
                          cg_iters=w.U, max_probes=w.K, rank=rank, world=world, nccl_id=nid, d_offset=d0,
                          D_global=w.D, cg_rtol=args.rtol)
        D = Dr
    elif world > 1:
        # probe-parallel inside the library (dist_mode 1): global K, owner split (rank 0 also solves
        # the mean system), one NCCL all-reduce of s and a broadcast of mu per E-step
        ctx = Context.from_workload(w, max_probes=(w.K + world - 1) // world + 2, rank=rank, world=world,
                                    nccl_id=nid, dist_mode=1, cg_rtol=args.rtol)
        D = w.D
    else:
        ctx = Context.from_workload(w, cg_rtol=args.rtol)
        D = w.D
    alpha = torch.ones(D, dtype=torch.float64, device=dev)
    mu = torch.empty_like(alpha)
    s = torch.empty_like(alpha)
    seed = args.seed

    def step(t, a_in, a_out, m_out, s_out):       # one EM iteration through the C ABI (all modes)
        ctx.em(1, w.K, seed, t, a_in, a_out, m_out, s_out)

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    t = 0
    for _ in range(args.warmup):
        step(t, alpha, alpha, mu, s)
        t += 1
    K_loc = ctx.report()["cols"] - 1            # this rank's probe columns (the library's split)
    # ---- device-timed region (inputs resident in HBM; the library replays one captured
    # CUDA graph per E-step)
    classes = ["dct_rows_inv", "dct_cols", "dct_rows_fwd", "pcg_update", "pcg_direction", "conv_apply",
               "dense_phi_p", "dense_phiT_w", "pcg_init", "probe_bits", "finalize_mstep", "mean_column",
               "dense_cluster"]
    # the profiled pass and the e2e pass below replay exactly these EM iterations (same t, same
    # starting alpha): later iterations freeze more columns and run faster
    t_timed, alpha_timed = t, alpha.clone()
    # timing rule: inputs larger than L2, or L2 flushed between timed iterations
    ws_mb = working_set_bytes(w, K_loc, D) / 1e6
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if ws_mb < 2 * 126 else None
    clk = ClockSampler(local)
    clk.start()
    barrier()
    launches0 = ctx.launches
    if flush is None:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            step(t, alpha, alpha, mu, s)
            t += 1
        e1.record()
        barrier()
        ms = e0.elapsed_time(e1)
    else:                      # per-iteration events; the 256 MB flush write sits between them
        evs = []
        for _ in range(args.steps):
            flush.fill_(t & 0xFF)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            step(t, alpha, alpha, mu, s)
            b.record()
            evs.append((a, b))
            t += 1
        barrier()
        ms = sum(a.elapsed_time(b) for a, b in evs)
    clocks = clk.stop()
    launches = ctx.launches - launches0
    ms_t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(ms_t, op=torch.distributed.ReduceOp.MAX)
    ms = float(ms_t.item())
    value = args.steps / (ms / 1000.0)
    support_cert = ctx.report()["support"]

    # ---- per-kernel-class device time: a separate profiled pass (CUDA events around every
    # launch on its stream, uncaptured) replaying the timed EM iterations
    ctx.profile_enable(classes)
    for c in classes:
        ctx.profile_read(c, reset=True)
    t = t_timed
    alpha.copy_(alpha_timed)
    if args.prof_steps <= 0:
        args.prof_steps = args.steps
    barrier()
    # after each replayed E-step the report gives every column's freeze iteration (R5): a frozen
    # column does no work in the remaining CG iterations, so the algorithmic bytes below count
    # the column-iterations actually executed, not U x K
    prof_ms, frozen = 0.0, []
    for _ in range(args.prof_steps):
        p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        p0.record()
        step(t, alpha, alpha, mu, s)
        p1.record()
        barrier()
        prof_ms += p0.elapsed_time(p1)
        frozen.append(ctx.report()["frozen_at"])
        t += 1
    busy = {c: ctx.profile_busy(c) for c in classes}
    prof = {c: ctx.profile_read(c) for c in classes}
    ctx.profile_enable([])
    # RHS-operator applies per second (BASELINE metric): executed column-iterations of this rank
    # (mean column included; frozen columns do no work) summed over ranks, over the timed time
    ex = torch.tensor([float(executed_applies(frozen, w.U))], dtype=torch.float64, device=dev)
    if world > 1 and not column:
        torch.distributed.all_reduce(ex)      # probe-parallel: ranks hold different columns
    ex_per_step = float(ex.item()) / args.prof_steps
    rhs_applies = ex_per_step * args.steps / (ms / 1000.0)
    rhs_nominal = (w.K + 1) * w.U * args.steps / (ms / 1000.0)

    # ---- end-to-end through the C ABI with pinned host buffers
    e2e = None
    if not args.no_e2e:
        a_h = torch.empty(D, dtype=torch.float64).pin_memory()
        m_h = torch.empty(D, dtype=torch.float64).pin_memory()
        s_h = torch.empty(D, dtype=torch.float64).pin_memory()
        a_h.copy_(alpha_timed.cpu())
        t = t_timed
        barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record()
        for _ in range(args.steps):
            ctx.em(1, w.K, seed, t, a_h, a_h, m_h, s_h)      # h2d alpha; d2h alpha, mu, s
            t += 1
        f1.record()
        barrier()
        ems = torch.tensor([f0.elapsed_time(f1)], dtype=torch.float64, device=dev)
        if world > 1:
            torch.distributed.all_reduce(ems, op=torch.distributed.ReduceOp.MAX)
        e2e = {"value": args.steps / (float(ems.item()) / 1000.0), "unit": UNIT,
               "h2d_bytes_per_step": D * 8, "d2h_bytes_per_step": 3 * D * 8}

    # ---- multi-rank correctness: this N-rank E-step against a 1-rank single-GPU context on rank 0
    multirank = None
    if world > 1:
        mu_n, s_n = torch.empty_like(alpha), torch.empty_like(alpha)
        ctx.estep(alpha_timed, w.K, seed, t_timed, mu_n, s_n)
        a_full, mu_f, s_f = alpha_timed, mu_n, s_n
        if column:                      # gather the D-slices (padded to the largest slice)
            sizes = [column_shard(w.D, world, r)[1] for r in range(world)]
            mx = max(sizes)

            def gather(v):
                pad = torch.zeros(mx, dtype=torch.float64, device=dev)
                pad[:v.numel()] = v
                parts = [torch.empty_like(pad) for _ in range(world)]
                torch.distributed.all_gather(parts, pad)
                return torch.cat([p[:n] for p, n in zip(parts, sizes)])
            a_full, mu_f, s_f = gather(alpha_timed), gather(mu_n), gather(s_n)
        if rank == 0:
            try:              # rank 0 alone: an error here must not leave the other ranks at the barrier
                ref = Context.from_workload(w)
                mu1, s1 = torch.empty_like(a_full), torch.empty_like(a_full)
                ref.estep(a_full, w.K, seed, t_timed, mu1, s1)
                torch.cuda.synchronize()
                mrel = lambda a, b: float((a - b).abs().max() / b.abs().max())
                multirank = {"ref": "1-rank single-GPU context on rank 0: same alpha, t and probes",
                             "mu_max_rel_diff": mrel(mu_f, mu1), "s_max_rel_diff": mrel(s_f, s1),
                             "mu_rel_l2": float((mu_f - mu1).norm() / mu1.norm()),
                             "s_rel_l2": float((s_f - s1).norm() / s1.norm())}
                ref.close()
            except Exception as e:          # reported in the line, not swallowed
                multirank = {"error": "%s: %s" % (type(e).__name__, e)}
        barrier()

    # ---- conformance: two EM iterations from the timed alpha in fast mode (fp32
    # probe columns, this bench's path) and in parity mode (every column fp64, which matches the
    # fp64 oracle to ~1e-7): support flips between them, each with its margin
    conformance = None
    if world == 1 and not args.no_conformance:
        par = Context.from_workload(w, probe_precision=1, cg_rtol=args.rtol)
        outs = []
        for cx in (ctx, par):
            ao, mo, so = torch.empty_like(alpha), torch.empty_like(alpha), torch.empty_like(alpha)
            cx.em(2, w.K, seed, t_timed, alpha_timed, ao, mo, so)
            outs.append((ao.cpu().numpy(), mo.cpu().numpy()))
        par.close()
        (af, mf), (ap, mp) = outs
        thr = 1e-3
        mxp = np.max(np.abs(mp))
        sf, sp = np.abs(mf) > thr * np.max(np.abs(mf)), np.abs(mp) > thr * mxp
        fl = np.nonzero(sf != sp)[0]
        conformance = {"vs": "parity mode (probe_precision = 1, fp64 probe columns) on this GPU, same alpha/t/probes",
                       "em_iters": 2, "support_size": int(sp.sum()), "support_flips": int(fl.size),
                       "flips": [{"d": int(d), "margin": float(abs(abs(mp[d]) / mxp - thr)),
                                  "dmu": float(abs(mf[d] - mp[d]) / mxp)} for d in fl[:10]],
                       "mu_rel_l2": float(np.linalg.norm(mf - mp) / np.linalg.norm(mp)),
                       "inv_alpha_rel_l2": float(np.linalg.norm(1 / af - 1 / ap) / np.linalg.norm(1 / ap)),
                       "library_certificate": support_cert}

    # ---- roofline of the dominant kernel (live CUDA events over the timed region)
    pk, pk_kind = peaks()
    # dominant = the class with the largest busy time (union of its launch intervals: concurrent
    # probe groups count once) among the classes with algorithmic bytes
    dom = max((c for c in classes if prof[c][1] > 0 and algorithmic_bytes(c, w, K_loc, D)),
              key=lambda c: busy[c] if busy[c] > 0 else prof[c][0])
    tot_ms, cnt = prof[dom]
    avg_ms = tot_ms / cnt
    # the probe columns may run as G concurrent groups (1024^2 DCT path): a launch then covers
    # K / G columns (G = launches per CG iteration of the class), and the G launches of one
    # iteration overlap: achieved = the class's executed bytes over its busy time (union of
    # intervals).  Executed bytes: per-column bytes x active column-iterations + the shared
    # arrays once per launch that has an active column (active_bytes)
    groups = max(1, int(round(cnt / float(w.U * args.prof_steps))))
    byt = algorithmic_bytes(dom, w, K_loc / groups, D)
    busy_ms = busy[dom] if busy[dom] > 0 else tot_ms
    dom_bytes, work_frac = active_bytes(dom, w, K_loc, D, groups, frozen)
    achieved = dom_bytes / (busy_ms / 1000.0) / 1e9
    traffic = None
    pipes = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        tdoc = json.load(open(tp))
        traffic = tdoc.get(args.workload, {}).get(dom)
        pipes = tdoc.get(args.workload + "_pipes", {}).get(dom)
    share = {c: round(prof[c][0] / prof_ms, 4) for c in classes if prof[c][1] > 0}
    busy_share = {c: round(busy[c] / prof_ms, 4) for c in classes if prof[c][1] > 0}
    # whole-step view (the classes run concurrently on the DCT path): every class's algorithmic
    # bytes per EM iteration over the device-timed step time
    step_bytes = 0.0
    for c in classes:
        b_c = algorithmic_bytes(c, w, K_loc, D) if prof[c][1] > 0 else None
        if b_c:
            g_c = max(1, int(round(prof[c][1] / float(w.U * args.prof_steps))))
            step_bytes += active_bytes(c, w, K_loc, D, g_c, frozen)[0] / args.prof_steps
    roof = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
            "frac": achieved / pk["hbm_gbs"], "traffic": traffic, "peak_source": pk_kind,
            "algorithmic_bytes_per_launch": byt, "avg_launch_ms": avg_ms, "launches": cnt,
            "columns_per_launch": K_loc / groups, "busy_ms": busy_ms,
            "work_fraction": work_frac,
            "achieved_def": "algorithmic bytes of the column-iterations executed (frozen columns, R5, do no "
                            "work; work_fraction = executed / (U x K)) / busy time (union of launch intervals)",
            "step": {"algorithmic_bytes": step_bytes, "achieved": step_bytes / (ms / args.steps / 1000.0) / 1e9,
                     "frac": step_bytes / (ms / args.steps / 1000.0) / 1e9 / pk["hbm_gbs"],
                     "def": "all classes' executed algorithmic bytes per EM iteration / device-timed ms_per_step "
                            "(probe classes; the fp64 mean column is not counted)"},
            "share_of_step": share, "busy_share_of_step": busy_share, "timed_in": "separate profiled pass of %d EM iteration(s), events per launch" %
            args.prof_steps}
    if pipes:
        # what bounds a kernel that is not HBM-bound (dct_cols: the L1TEX / shared-memory pipe), from the
        # committed steady-state ncu capture of the same kernel (like `traffic`), % of peak while active
        roof["ncu_pipes"] = dict(pipes, source="profiles/ncu_traffic.json (steady-state ncu --set full capture)")
    if dom == "dense_cluster":
        # the whole CG loop in 8-CTA clusters, state in shared memory (op_dense_cluster.cu): the
        # bound is FP32 issue and the cluster barriers, not memory.  FP32 SIMT peak = SMs x 128 lanes
        # x 2 flop x max SM clock (B200_PROFILING unit counts); the kernel runs on 8 SMs per cluster,
        # min(8, K, max(min(4, K), ceil(K / 4))) clusters (dcl_groups' default, probe_groups = 0)
        probe_ex = sum(sum(w.U if f < 0 else min(f + 1, w.U) for f in fz[1:]) for fz in frozen)
        ncl = max(1, min(8, K_loc, max(min(4, K_loc), (K_loc + 3) // 4)))
        props = torch.cuda.get_device_properties(local)
        fmax = (clocks or {}).get("sm_max_mhz") or 1965.0
        fp32_peak = props.multi_processor_count * 128 * 2 * fmax * 1e6 / 1e12
        fl = 2 * 2 * w.N * D * probe_ex
        ach = fl / (busy_ms / 1000.0) / 1e12
        roof.update({"bound": "alu", "achieved": ach, "peak": fp32_peak, "unit": "TFLOP/s",
                     "frac": ach / fp32_peak, "peak_source": "%d SMs x 128 FP32 lanes x 2 x %.0f MHz" %
                     (props.multi_processor_count, fmax),
                     "frac_of_cluster_sms": ach / (fp32_peak * 8 * ncl / props.multi_processor_count),
                     "cluster_sms": 8 * ncl,
                     "achieved_def": "FP32 flops of the probe columns' two products (2 x 2 N D per executed "
                                     "column-iteration; the fp64 mean column not counted) / busy time"})
    if w.kind == "dense" and flush is not None:
        # Phi fits in L2 (C1, C2): the dense GEMMs are bound by the tensor pipe, not HBM.  3xTF32 =
        # 3 tf32 MMAs per product, 2 N D flops per column per GEMM; tf32 peak = measured bf16 x 1/2
        # (B200_PROFILING nominal ratio)
        probe_ex = sum(sum(w.U if f < 0 else min(f + 1, w.U) for f in fz[1:]) for fz in frozen)
        tf32_peak = pk.get("bf16_tflops", 1638.5) / 2.0
        gemm_ms = busy.get("dense_phi_p", 0) + busy.get("dense_phiT_w", 0)
        fl = 3 * 2 * 2 * w.N * D * probe_ex
        if gemm_ms > 0:
            ach = fl / (gemm_ms / 1000.0) / 1e12
            roof.update({"bound": "tensor", "kernel": "dense_phi_p + dense_phiT_w", "achieved": ach,
                         "peak": tf32_peak, "unit": "TFLOP/s", "frac": ach / tf32_peak,
                         "peak_source": pk_kind + " bf16 x 1/2 (nominal tf32 ratio)",
                         "achieved_def": "3xTF32 MMA flops (3 x 2 N D per probe column per GEMM, executed "
                                         "column-iterations) / busy time of the two GEMM classes",
                         "hbm_view": {"kernel": dom, "achieved": achieved, "frac_of_hbm": achieved / pk["hbm_gbs"],
                                      "note": "Phi (%.0f MB) is L2-resident between launches" % (w.N * D * 4 / 1e6)}})

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, desc, threads, _ = cpu_sample(w, seed)
        cpu = {"value": v, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": desc,
               "extrapolated": True, "cpu_model": cpu_model()}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
                "scaling": "strong" if not column or w.kind == "dense" else "strong",
                "vs_baseline": None, "dtype": "f32 (probe columns) + f64 (mean column)",
                "data": "synthetic",
                "config": {"workload": w.name, **w.config(),
                           "parallelism": (("column-sharded x%d" if w.kind == "dense" else "D-sharded x%d") if column
                                           else "probe-parallel x%d" + (" (library-owned NCCL: all-reduce of s, "
                                                                         "broadcast of mu; rank 0 owns the mean system)"
                                                                         if world > 1 else "")) % world,
                           "K_per_rank": K_loc, "D_per_rank": D, **({"cg_rtol": args.rtol} if args.rtol > 0 else {}),
                           "l2": ("inputs larger than L2 (working set %.0f MB > 126 MB)" % ws_mb if flush is None
                                  else "working set %.1f MB fits in L2: 256 MB flush write before every timed "
                                       "EM iteration, outside its events" % ws_mb)},
                "rhs_applies_per_s": rhs_applies,
                "rhs_applies_def": "executed column-iterations (frozen columns, R5, do no work; mean column "
                                   "included) per second; nominal (K+1) U per EM iteration: %.0f/s" % rhs_nominal,
                "e2e": e2e, "roofline": roof, "cpu_baseline": cpu, "multirank_check": multirank,
                "conformance": conformance, "clocks": clocks, "gpu_launches": launches}
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
