"""Seeded synthetic workloads shaped like the paper's experiments.

Shared by the oracle-side tests and the GPU path (the only module both use).  It
holds none of CoFEM's arithmetic: it draws the generative model of Eq. 1
 — a sparse z, a dictionary, y = Phi z + noise — with NumPy's PCG64
(`default_rng(seed)`), in fp64, and casts the inputs both sides consume (Phi, y,
h) to fp32.  y = Phi z is evaluated with library routines (matmul,
scipy.fft.idctn, numpy.fft), which is data generation, not the method.

The paper measures on simulated compressed-sensing data only (§4, P:112,
P:124-125); there is no dataset.  The five presets are BASELINE.json's
configs C1..C5; `scale` variants shrink them for parity tests.

Reading R13: nonzero count = floor(frac * D); R14: seed 0; R15: Phi ~ N(0, 1/N).
"""
import dataclasses
import math

import numpy as np
import scipy.fft as sfft

BETA = 1.0e4           # sigma = 0.01 (all configs)
SIGMA = 0.01


@dataclasses.dataclass
class Workload:
    name: str
    kind: str                  # "dense" | "dct2_masked" | "circconv"
    N: int
    D: int
    K: int
    U: int
    T: int
    beta: float
    y: np.ndarray              # fp32 [N]
    z_true: np.ndarray         # fp64 [D]
    phi: np.ndarray = None     # fp32 [N, D] row-major (dense)
    rows: int = 0              # dct grid
    cols: int = 0
    obs_idx: np.ndarray = None  # int64 [N], sorted distinct (dct)
    convention: int = 0
    taps: np.ndarray = None    # fp32 [T] (circconv)
    seed: int = 0

    def config(self):
        c = {"workload": self.name, "kind": self.kind, "N": self.N, "D": self.D, "K": self.K,
             "U": self.U, "T_em": self.T, "beta": self.beta}
        if self.kind == "dct2_masked":
            c["grid"] = [self.rows, self.cols]
        if self.kind == "circconv":
            c["taps"] = int(self.taps.size)
        return c


def _sparse_z(rng, D, nnz):
    z = np.zeros(D)
    idx = rng.choice(D, nnz, replace=False)
    z[idx] = rng.standard_normal(nnz)
    return z


def dense(N, D, nnz, K, U, T, seed=0, name=None):
    """Dense Gaussian dictionary, entries iid N(0, 1/N) (BASELINE configs 1-3)."""
    rng = np.random.default_rng(seed)
    phi = np.empty((N, D), dtype=np.float32)
    step = max(1, (1 << 24) // max(D, 1))
    for r0 in range(0, N, step):              # chunked: fp64 draw, fp32 store
        r1 = min(N, r0 + step)
        phi[r0:r1] = (rng.standard_normal((r1 - r0, D)) / math.sqrt(N)).astype(np.float32)
    z = _sparse_z(rng, D, nnz)
    y = (phi.astype(np.float64) @ z + SIGMA * rng.standard_normal(N)).astype(np.float32)
    return Workload(name or "dense_%dx%d" % (N, D), "dense", N, D, K, U, T, BETA, y, z, phi=phi, seed=seed)


def paper_dense(D, f, seed=0, sigma=0.005, K=20, U=400, T=50):
    """The paper's own dense setup (§4.1): N = D/f, Phi ~ N(0, 1)
    (unnormalised), d = floor(0.04 D) spikes of +-1, noise sigma = 0.005,
    beta = 1/sigma^2."""
    rng = np.random.default_rng(seed)
    N = D // f
    phi = rng.standard_normal((N, D)).astype(np.float32)
    nnz = int(math.floor(0.04 * D))
    z = np.zeros(D)
    z[rng.choice(D, nnz, replace=False)] = rng.choice([-1.0, 1.0], nnz)
    y = (phi.astype(np.float64) @ z + sigma * rng.standard_normal(N)).astype(np.float32)
    return Workload("paper_dense_D%d_f%d" % (D, f), "dense", N, D, K, U, T, 1.0 / sigma ** 2, y, z,
                    phi=phi, seed=seed)


def dct(rows, cols, N, nnz, K, U, T, seed=0, convention=0, name=None, sigma=SIGMA):
    """Orthonormal 2D DCT on a rows x cols grid, uniform random N-pixel mask (config 4)."""
    rng = np.random.default_rng(seed)
    D = rows * cols
    obs = np.sort(rng.choice(D, N, replace=False)).astype(np.int64)
    z = _sparse_z(rng, D, nnz)
    img = z.reshape(rows, cols)
    pix = sfft.idctn(img, norm="ortho") if convention == 0 else sfft.dctn(img, norm="ortho")
    y = (pix.ravel()[obs] + sigma * rng.standard_normal(N)).astype(np.float32)
    return Workload(name or "dct_%dx%d" % (rows, cols), "dct2_masked", N, D, K, U, T, 1.0 / sigma ** 2, y, z,
                    rows=rows, cols=cols, obs_idx=obs, convention=convention, seed=seed)


def paper_dct(p, seed=0, frac=0.04, K=20, U=400, T=30):
    """The paper's structured setup (§4.2): D = 2^p DCT coefficients on a 2^floor(p/2) x
    2^ceil(p/2) grid (reading R11: 2D), N = D/4 observed pixels, d = floor(frac D) N(0, 1)
    coefficients; the noise level is not restated in §4.2, so §4.1's sigma = 0.005 (beta = 1/sigma^2)."""
    rows, cols = 1 << (p // 2), 1 << (p - p // 2)
    D = rows * cols
    return dct(rows, cols, D // 4, int(math.floor(frac * D)), K=K, U=U, T=T, seed=seed, sigma=0.005,
               name="paper_dct_2^%d" % p)


def circconv(D, ntaps, nnz, K, U, T, seed=0, name=None):
    """Circular convolution with a length-ntaps N(0,1) filter normalised to unit L2 (config 5).
    The fp32-rounded taps are the definition (reading R12)."""
    rng = np.random.default_rng(seed)
    h = rng.standard_normal(ntaps)
    h = (h / np.linalg.norm(h)).astype(np.float32)
    z = _sparse_z(rng, D, nnz)
    hp = np.zeros(D)
    hp[:ntaps] = h.astype(np.float64)
    y = np.fft.irfft(np.fft.rfft(hp) * np.fft.rfft(z), n=D)
    y = (y + SIGMA * rng.standard_normal(D)).astype(np.float32)
    return Workload(name or "conv_%d" % D, "circconv", D, D, K, U, T, BETA, y, z, taps=h, seed=seed)


def tasks(w, L, seed=1, shared_support=True):
    """Observation vectors of L tasks on workload w's dictionary (multi-task SBL, R22): task 0 is
    w.y; tasks 1..L-1 draw new N(0, 1) values (on w's support when shared_support, the multi-task
    model's shared sparsity profile) and y_l = Phi z_l + sigma e with library routines, as above.
    Returns (Y fp32 [L, N], Z fp64 [L, D])."""
    rng = np.random.default_rng(1000 + seed)
    sigma = 1.0 / math.sqrt(w.beta)
    sup = np.nonzero(w.z_true)[0]
    Y, Z = [w.y], [w.z_true]
    for _ in range(1, L):
        z = np.zeros(w.D)
        idx = sup if shared_support else rng.choice(w.D, sup.size, replace=False)
        z[idx] = rng.standard_normal(idx.size)
        if w.kind == "dense":
            y = w.phi.astype(np.float64) @ z
        elif w.kind == "dct2_masked":
            img = z.reshape(w.rows, w.cols)
            pix = sfft.idctn(img, norm="ortho") if w.convention == 0 else sfft.dctn(img, norm="ortho")
            y = pix.ravel()[w.obs_idx]
        else:
            hp = np.zeros(w.D)
            hp[:w.taps.size] = w.taps.astype(np.float64)
            y = np.fft.irfft(np.fft.rfft(hp) * np.fft.rfft(z), n=w.D)
        Y.append((y + sigma * rng.standard_normal(y.size)).astype(np.float32))
        Z.append(z)
    return np.ascontiguousarray(np.stack(Y)), np.stack(Z)


def preset(name, seed=0):
    """BASELINE.json configs C1..C5 at full size."""
    if name == "C1":
        return dense(100, 400, 10, K=20, U=100, T=30, seed=seed, name="C1_dense_100x400")
    if name == "C2":
        return dense(2000, 8000, 160, K=32, U=200, T=50, seed=seed, name="C2_dense_2000x8000")
    if name == "C3":
        return dense(8192, 32768, 327, K=64, U=300, T=50, seed=seed, name="C3_dense_8192x32768")
    if name == "C4":
        return dct(1024, 1024, 262144, 10485, K=32, U=200, T=30, seed=seed, name="C4_dct_1024x1024")
    if name == "C5":
        return circconv(1 << 24, 64, 16777, K=16, U=150, T=20, seed=seed, name="C5_conv_2^24")
    raise KeyError(name)


def small(name, seed=0):
    """Scaled-down shapes of the presets that the oracle finishes in seconds."""
    if name == "C1":
        return preset("C1", seed)
    if name == "C2":
        return dense(250, 1000, 20, K=32, U=200, T=5, seed=seed, name="C2s_dense_250x1000")
    if name == "C3":
        return dense(512, 2048, 20, K=64, U=300, T=3, seed=seed, name="C3s_dense_512x2048")
    if name == "C4":
        return dct(64, 64, 1024, 41, K=32, U=200, T=5, seed=seed, name="C4s_dct_64x64")
    if name == "C5":
        return circconv(4099, 64, 4, K=16, U=150, T=5, seed=seed, name="C5s_conv_4099")
    raise KeyError(name)
