"""Thin ctypes binding of the C ABI in include/cofem.h (argument marshalling only).

Every step of the hot path runs in libcofem.so's CUDA kernels; this module only
converts torch tensors / NumPy arrays to pointers and status codes to
exceptions.  There is no CPU fallback: importing works without a GPU, but
creating a Context needs the built library and a CUDA device, and fails loudly
otherwise.

Names follow the paper: alpha (prior precisions, Eq. 1), beta (noise precision),
mu (posterior mean), s (diagonal estimate of Sigma, Eq. 6), K probes, U CG
iterations, T_em EM iterations (Algorithm 1).
"""
import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libcofem.so")

OP_DENSE, OP_DCT2_MASKED, OP_CIRCCONV = 0, 1, 2
STATUS = {0: "OK", 1: "ERR_INVALID", 2: "ERR_CUDA", 3: "ERR_NCCL", 4: "ERR_NUMERIC", 5: "ERR_OOM",
          6: "ERR_UNSUPPORTED"}


class CofemError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__("cofem %s: %s" % (STATUS.get(status, status), msg))
        self.status = status


class _Operator(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("N", ctypes.c_int64), ("D", ctypes.c_int64),
                ("phi", ctypes.c_void_p), ("ld", ctypes.c_int64),
                ("rows", ctypes.c_int32), ("cols", ctypes.c_int32), ("obs_idx", ctypes.c_void_p),
                ("convention", ctypes.c_int32),
                ("taps", ctypes.c_void_p), ("ntaps", ctypes.c_int32),
                ("d_offset", ctypes.c_int64), ("D_global", ctypes.c_int64)]


class _Options(ctypes.Structure):
    _fields_ = [("cg_iters", ctypes.c_int32), ("precond", ctypes.c_int32), ("den_floor", ctypes.c_double),
                ("alpha_max", ctypes.c_double), ("probe_precision", ctypes.c_int32),
                ("max_probes", ctypes.c_int32), ("rank", ctypes.c_int32), ("world", ctypes.c_int32),
                ("nccl_id", ctypes.c_void_p), ("cg_rtol", ctypes.c_double), ("apply_path", ctypes.c_int32),
                ("probe_groups", ctypes.c_int32), ("use_graph", ctypes.c_int32), ("dist_mode", ctypes.c_int32),
                ("warm_start", ctypes.c_int32), ("cg_variant", ctypes.c_int32)]


class _Report(ctypes.Structure):
    _fields_ = [("cols", ctypes.c_int32), ("cg_iters", ctypes.c_int32),
                ("frozen_at", ctypes.POINTER(ctypes.c_int32)), ("rho", ctypes.POINTER(ctypes.c_double)),
                ("rho0", ctypes.POINTER(ctypes.c_double)), ("bad_col", ctypes.c_int32),
                ("bad_iter", ctypes.c_int32), ("estep_ms_last", ctypes.c_double), ("launches", ctypes.c_int64),
                ("support_count", ctypes.c_int64), ("support_adjacent", ctypes.c_int64),
                ("support_max_abs_mu", ctypes.c_double), ("support_min_margin", ctypes.c_double),
                ("support_delta", ctypes.c_double), ("collectives", ctypes.c_int64)]


# (name, restype, argtypes) — every entry point of include/cofem.h
SYMBOLS = [
    ("cofem_get_unique_id", ctypes.c_int, [ctypes.c_void_p]),
    ("cofem_default_options", None, [ctypes.POINTER(_Options)]),
    ("cofem_setup", ctypes.c_int, [ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(_Operator), ctypes.c_void_p,
                                   ctypes.c_double, ctypes.POINTER(_Options), ctypes.c_void_p]),
    ("cofem_estep", ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_uint64,
                                   ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p,
                                   ctypes.c_void_p]),
    ("cofem_estep_probes", ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_uint64,
                                          ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p]),
    ("cofem_mstep", ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    ("cofem_apply", ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p,
                                   ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    ("cofem_em", ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_uint64, ctypes.c_int32,
                                ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    ("cofem_em_multi", ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32,
                                      ctypes.c_uint64, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                      ctypes.c_void_p]),
    ("cofem_last_report", ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(_Report)]),
    ("cofem_probe_split", ctypes.c_int, [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_double,
                                         ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32),
                                         ctypes.POINTER(ctypes.c_int32)]),
    ("cofem_profile_enable", ctypes.c_int, [ctypes.c_void_p, ctypes.c_uint32]),
    ("cofem_profile_busy", ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.POINTER(ctypes.c_double)]),
    ("cofem_profile_read", ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.POINTER(ctypes.c_double),
                                          ctypes.POINTER(ctypes.c_int64), ctypes.c_int32]),
    ("cofem_kernel_class_name", ctypes.c_char_p, [ctypes.c_int32]),
    ("cofem_last_error", ctypes.c_char_p, [ctypes.c_void_p]),
    ("cofem_version", ctypes.c_char_p, []),
    ("cofem_destroy", None, [ctypes.c_void_p]),
]

_lib = None


def lib():
    """Load libcofem.so (raises if it was not built — there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError("libcofem.so is not built (python -m paper_2202_12808_b200.build); "
                               "the CoFEM path has no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        for name, res, args in SYMBOLS:
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def get_unique_id():
    """128-byte NCCL unique id for the column-sharded mode (broadcast it to every rank)."""
    buf = ctypes.create_string_buffer(128)
    st = lib().cofem_get_unique_id(buf)
    if st != 0:
        raise CofemError(st, "libnccl.so.2 could not be loaded")
    return buf.raw


def probe_split(K, world, rank, mean_cost):
    """The library's probe-parallel owner split (cofem_probe_split, host only):
    (k_offset, K_local, owns_mean)."""
    o, n, m = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    st = lib().cofem_probe_split(int(K), int(world), int(rank), float(mean_cost), ctypes.byref(o), ctypes.byref(n),
                                 ctypes.byref(m))
    if st != 0:
        raise CofemError(st, lib().cofem_last_error(None).decode())
    return o.value, n.value, bool(m.value)


def kernel_classes():
    out, i = [], 0
    while True:
        n = lib().cofem_kernel_class_name(i)
        if n is None:
            return out
        out.append(n.decode())
        i += 1


def _ptr(x, dtype, n=None, what="array"):
    """Pointer of a contiguous torch tensor (CUDA or CPU) or NumPy array of the given dtype."""
    if x is None:
        return None
    if hasattr(x, "data_ptr"):     # torch
        import torch
        want = {np.float32: torch.float32, np.float64: torch.float64, np.int64: torch.int64}[dtype]
        if x.dtype != want or not x.is_contiguous():
            raise TypeError("%s must be a contiguous %s tensor" % (what, want))
        if n is not None and x.numel() < n:
            raise ValueError("%s has %d elements, need %d" % (what, x.numel(), n))
        return ctypes.c_void_p(x.data_ptr())
    if isinstance(x, np.ndarray):
        if x.dtype != dtype or not x.flags.c_contiguous:
            raise TypeError("%s must be a C-contiguous %s array" % (what, np.dtype(dtype).name))
        if n is not None and x.size < n:
            raise ValueError("%s has %d elements, need %d" % (what, x.size, n))
        return ctypes.c_void_p(x.ctypes.data)
    raise TypeError("%s: expected a torch tensor or numpy array" % what)


class Context:
    """One cofem_ctx: an operator Phi, observations y and beta (Alg. 1 signature)."""

    def __init__(self, kind, N, D, y, beta, phi=None, rows=0, cols=0, obs_idx=None, convention=0, taps=None,
                 cg_iters=100, precond=1, probe_precision=0, max_probes=32, den_floor=1e-12, alpha_max=1e12,
                 stream=None, d_offset=0, D_global=0, rank=0, world=1, nccl_id=None, cg_rtol=0.0, apply_path=0,
                 probe_groups=0, use_graph=True, dist_mode=0, ld=None, warm_start=False, cg_variant=0):
        """Multi-GPU; nccl_id = get_unique_id() from one rank, broadcast to all.
        dist_mode 0 with nccl_id: column-sharded dense / D-sharded conv -- phi (or y) holds this
        rank's slice [d_offset, d_offset + D) of D_global; the library all-reduces W and the column
        dots (or exchanges halos) over NCCL itself.  dist_mode 1: probe-parallel -- every rank holds
        the whole operator, estep/em take the GLOBAL K, the library splits the probes, all-reduces s
        and broadcasts mu.  apply_path 1: the general kernels (tests); use_graph False: no CUDA graph.
        cg_variant (cofem.h): 0 auto, 1 standard PCG, 2 single-reduction (column-sharded dense)."""
        L = lib()
        self.N, self.D, self.kind = int(N), int(D), int(kind)
        self._keep = [y, phi, obs_idx, taps]
        op = _Operator()
        op.kind, op.N, op.D = self.kind, self.N, self.D
        if phi is not None:        # a CUDA tensor is borrowed (zero-copy, row stride ld), host data copied
            op.ld = self.D if ld is None else int(ld)
            op.phi = _ptr(phi, np.float32, (self.N - 1) * op.ld + self.D, "phi")
        op.rows, op.cols, op.convention = int(rows), int(cols), int(convention)
        op.d_offset, op.D_global = int(d_offset), int(D_global)
        if obs_idx is not None:
            op.obs_idx = _ptr(obs_idx, np.int64, self.N, "obs_idx")
        if taps is not None:
            op.taps = _ptr(taps, np.float32, None, "taps")
            op.ntaps = int(taps.numel() if hasattr(taps, "numel") else taps.size)
        opt = _Options()
        L.cofem_default_options(ctypes.byref(opt))
        opt.cg_iters, opt.precond, opt.probe_precision, opt.max_probes = int(cg_iters), int(precond), \
            int(probe_precision), int(max_probes)
        opt.den_floor, opt.alpha_max = float(den_floor), float(alpha_max)
        opt.rank, opt.world = int(rank), int(world)
        opt.cg_rtol = float(cg_rtol)
        opt.apply_path, opt.probe_groups = int(apply_path), int(probe_groups)
        opt.use_graph, opt.dist_mode = int(bool(use_graph)), int(dist_mode)
        opt.warm_start = int(bool(warm_start))
        opt.cg_variant = int(cg_variant)
        if nccl_id is not None:
            self._nid = ctypes.create_string_buffer(bytes(nccl_id), 128)
            opt.nccl_id = ctypes.cast(self._nid, ctypes.c_void_p)
        self.U, self.K_max = int(cg_iters), int(max_probes)
        self.probe_precision = int(probe_precision)
        h = ctypes.c_void_p()
        st = L.cofem_setup(ctypes.byref(h), ctypes.byref(op), _ptr(y, np.float32, self.N, "y"), float(beta),
                           ctypes.byref(opt), ctypes.c_void_p(stream) if stream else None)
        if st != 0:
            raise CofemError(st, L.cofem_last_error(None).decode())
        self._h = h

    @classmethod
    def from_workload(cls, w, **kw):
        """Build from a synth.Workload (host arrays are copied to the device by the library)."""
        kw.setdefault("cg_iters", w.U)
        kw.setdefault("max_probes", w.K)
        if w.kind == "dense":
            return cls(OP_DENSE, w.N, w.D, w.y, w.beta, phi=np.ascontiguousarray(w.phi), **kw)
        if w.kind == "dct2_masked":
            return cls(OP_DCT2_MASKED, w.N, w.D, w.y, w.beta, rows=w.rows, cols=w.cols,
                       obs_idx=np.ascontiguousarray(w.obs_idx, dtype=np.int64), convention=w.convention, **kw)
        if w.kind == "circconv":
            return cls(OP_CIRCCONV, w.N, w.D, w.y, w.beta, taps=np.ascontiguousarray(w.taps), **kw)
        raise ValueError(w.kind)

    def _check(self, st):
        if st != 0:
            raise CofemError(st, lib().cofem_last_error(self._h).decode())

    def estep(self, alpha, K, seed, t, mu, s, k_offset=0, K_total=None):
        """Simplified E-step (Alg. 1 l.3-7): writes mu and s (D fp64 each, host or device)."""
        D = self.D
        self._check(lib().cofem_estep(self._h, _ptr(alpha, np.float64, D, "alpha"), int(K), int(seed), int(t),
                                      int(k_offset), int(K if K_total is None else K_total),
                                      _ptr(mu, np.float64, D, "mu"), _ptr(s, np.float64, D, "s")))

    def estep_probes(self, alpha, K, seed, t, s, k_offset=0, K_total=None):
        """E-step for the probe columns only (the mean system is owned by another rank): s = this
        call's partial (1/K_total) sum; mu is not computed."""
        D = self.D
        self._check(lib().cofem_estep_probes(self._h, _ptr(alpha, np.float64, D, "alpha"), int(K), int(seed),
                                             int(t), int(k_offset), int(K if K_total is None else K_total),
                                             _ptr(s, np.float64, D, "s")))

    def apply(self, alpha, x0, X, q0, Q, gamma=None):
        """One Gram apply q0 = A x0, Q_k = A X_k (A = beta Phi^T Phi + diag alpha, Eq. 7) through the
        E-step's kernels; X, Q: K x D in probe precision (float32, or float64 with probe_precision=1)."""
        D = self.D
        K = int(X.shape[0])
        pdt = np.float64 if self.probe_precision else np.float32
        self._check(lib().cofem_apply(self._h, _ptr(alpha, np.float64, D, "alpha"), K, _ptr(x0, np.float64, D, "x0"),
                                      _ptr(X, pdt, K * D, "X"), _ptr(q0, np.float64, D, "q0"),
                                      _ptr(Q, pdt, K * D, "Q"), _ptr(gamma, np.float64, K + 1, "gamma")))

    def mstep(self, mu, s, alpha_out):
        """M-step, Eq. 8."""
        D = self.D
        self._check(lib().cofem_mstep(self._h, _ptr(mu, np.float64, D, "mu"), _ptr(s, np.float64, D, "s"),
                                      _ptr(alpha_out, np.float64, D, "alpha_out")))

    def em(self, iters, K, seed, t0=0, alpha_init=None, alpha_out=None, mu_out=None, s_out=None):
        """Algorithm 1 for `iters` EM iterations (probe counter t = t0 + i)."""
        D = self.D
        self._check(lib().cofem_em(self._h, int(iters), int(K), int(seed), int(t0),
                                   _ptr(alpha_init, np.float64, D, "alpha_init"),
                                   _ptr(alpha_out, np.float64, D, "alpha_out"),
                                   _ptr(mu_out, np.float64, D, "mu_out"), _ptr(s_out, np.float64, D, "s_out")))

    def em_multi(self, Y, iters, K, seed, t0=0, alpha_init=None, alpha_out=None, MU_out=None, s_out=None):
        """Multi-task EM (NEXT-4, reading R22): Y is L x N fp32 (row l = task l's y), MU_out L x D."""
        D = self.D
        L = int(Y.shape[0])
        self._check(lib().cofem_em_multi(self._h, L, _ptr(Y, np.float32, L * self.N, "Y"), int(iters), int(K),
                                         int(seed), int(t0), _ptr(alpha_init, np.float64, D, "alpha_init"),
                                         _ptr(alpha_out, np.float64, D, "alpha_out"),
                                         _ptr(MU_out, np.float64, L * D, "MU_out"), _ptr(s_out, np.float64, D, "s_out")))

    def report(self):
        r = _Report()
        self._check(lib().cofem_last_report(self._h, ctypes.byref(r)))
        n = r.cols
        return {"cols": n, "cg_iters": r.cg_iters,
                "frozen_at": [r.frozen_at[i] for i in range(n)],
                "rho": [r.rho[i] for i in range(n)], "rho0": [r.rho0[i] for i in range(n)],
                "bad_col": r.bad_col, "bad_iter": r.bad_iter, "estep_ms": r.estep_ms_last,
                "launches": r.launches, "collectives": r.collectives,
                "support": {"count": r.support_count, "adjacent": r.support_adjacent,
                            "max_abs_mu": r.support_max_abs_mu, "min_margin": r.support_min_margin,
                            "delta": r.support_delta}}

    def profile_enable(self, classes):
        names = kernel_classes()
        mask = 0
        for c in classes:
            mask |= 1 << names.index(c)
        self._check(lib().cofem_profile_enable(self._h, mask))

    def profile_read(self, cls, reset=False):
        idx = kernel_classes().index(cls)
        ms, cnt = ctypes.c_double(), ctypes.c_int64()
        self._check(lib().cofem_profile_read(self._h, idx, ctypes.byref(ms), ctypes.byref(cnt), int(reset)))
        return ms.value, cnt.value

    def profile_busy(self, cls):
        """Union of the class's launch intervals in ms (concurrent launches counted once)."""
        ms = ctypes.c_double()
        self._check(lib().cofem_profile_busy(self._h, kernel_classes().index(cls), ctypes.byref(ms)))
        return ms.value

    @property
    def launches(self):
        return self.report()["launches"]

    def close(self):
        if getattr(self, "_h", None):
            lib().cofem_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
