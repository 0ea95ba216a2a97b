"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on the same
seeded inputs and the same Philox probes.  Bars (BASELINE.json north_star):
rel. L2 error <= 1e-4 on mu and s after one E-step, <= 1e-3 on final 1/alpha and
mu after all EM iterations, identical recovered support |mu_d| > 1e-3 max|mu|.
Parity mode (fp64 probe columns) is held to 1e-7: fp64 rounding-order differences
(u = 1.1e-16) amplified by the unconverged fixed-U CG iterate (measured amplification
up to ~1e10 for unconverged dense cases)."""
import numpy as np
import pytest

import synth
from oracle import closed_forms as cf
from oracle.cofem import cofem_em, estep, support
from oracle.operators import CircConvOp, DCT2MaskedOp, DenseOp
from oracle.philox import rademacher_probes

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2202_12808_b200 import build
    build.build()
    torch.cuda.set_device(0)


def ctx_of(w, **kw):
    from paper_2202_12808_b200 import Context
    return Context.from_workload(w, **kw)


def op_of(w):
    if w.kind == "dense":
        return DenseOp(w.phi)
    if w.kind == "dct2_masked":
        return DCT2MaskedOp(w.rows, w.cols, w.obs_idx, w.convention)
    return CircConvOp(w.taps, w.D)


def dev(n):
    return torch.empty(n, dtype=torch.float64, device="cuda")


def gpu_estep(ctx, w, alpha, K, seed, t):
    a = torch.as_tensor(alpha, dtype=torch.float64, device="cuda").contiguous()
    mu, s = dev(w.D), dev(w.D)
    ctx.estep(a, K, seed, t, mu, s)
    return mu.cpu().numpy(), s.cpu().numpy()


def gpu_em(ctx, w, T, K, seed, t0=0, alpha_init=None):
    ao, mu, s = dev(w.D), dev(w.D), dev(w.D)
    ai = None if alpha_init is None else torch.as_tensor(alpha_init, device="cuda").contiguous()
    ctx.em(T, K, seed, t0, ai, ao, mu, s)
    return ao.cpu().numpy(), mu.cpu().numpy(), s.cpu().numpy()


SMALL = [
    synth.preset("C1"),                                                  # dense 100 x 400 (full config 1)
    synth.dense(250, 1000, 20, K=32, U=200, T=5, seed=1, name="dense_ragged_250x1000"),
    synth.dct(64, 64, 1024, 41, K=32, U=200, T=5, seed=0),
    synth.dct(32, 128, 1024, 40, K=12, U=150, T=4, seed=2),            # rows != cols
    synth.dct(128, 128, 4096, 163, K=8, U=200, T=3, seed=3),
    synth.circconv(5003, 64, 5, K=16, U=150, T=5, seed=0),              # ragged (prime) D
    synth.circconv(20000, 64, 20, K=8, U=150, T=3, seed=4),
    synth.dct(64, 64, 1024, 41, K=8, U=150, T=4, seed=6, convention=1, name="dct_64x64_conv1"),   # Phi = S C2
    synth.dct(32, 128, 1024, 40, K=6, U=150, T=3, seed=7, convention=1, name="dct_32x128_conv1"),
]


@pytest.mark.parametrize("w", SMALL, ids=lambda w: w.name)
def test_estep1_parity(w):
    ctx = ctx_of(w)
    mu, s = gpu_estep(ctx, w, np.ones(w.D), w.K, 5, 0)
    omu, os_, _ = estep(op_of(w), w.y, w.beta, np.ones(w.D), w.K, 5, 0, w.U)
    assert rel(mu, omu) <= 1e-4 and rel(s, os_) <= 1e-4, (rel(mu, omu), rel(s, os_))
    rep = ctx.report()
    assert rep["cols"] == w.K + 1 and rep["bad_col"] == -1


@pytest.mark.parametrize("w", SMALL, ids=lambda w: w.name)
def test_em_parity_and_support(w):
    ctx = ctx_of(w)
    T = min(w.T, 5)
    a, mu, s = gpu_em(ctx, w, T, w.K, 11)
    oa, omu, os_ = cofem_em(op_of(w), w.y, w.beta, T, w.K, 11, w.U)
    assert rel(1 / a, 1 / oa) <= 1e-3 and rel(mu, omu) <= 1e-3, (rel(1 / a, 1 / oa), rel(mu, omu))
    sg, so = support(mu), support(omu)
    flips = np.nonzero(sg != so)[0]
    if flips.size:   # certify: every flip sits at the threshold (SURVEY.md §8(c) fragility note)
        mx = np.max(np.abs(omu))
        margin = np.abs(np.abs(omu[flips]) / mx - 1e-3)
        assert flips.size <= 2 and np.all(margin < 1e-5), (flips, margin)


def test_full_em_c1_30_iterations():
    w = synth.preset("C1")
    ctx = ctx_of(w)
    a, mu, s = gpu_em(ctx, w, w.T, w.K, 0)
    oa, omu, os_ = cofem_em(op_of(w), w.y, w.beta, w.T, w.K, 0, w.U)
    assert rel(1 / a, 1 / oa) <= 1e-3 and rel(mu, omu) <= 1e-3
    assert np.array_equal(support(mu), support(omu))


# D ~ 4K with this filter is a case where any fp32 rounding in the unconverged PCG
# recurrence moves s by ~1e-4 (CPU emulation: 1.7e-4 fp32 vs 4.5e-8 fp64; D >= 5003:
# 8e-8): parity mode is the conforming path there.
@pytest.mark.parametrize("w", [SMALL[1], SMALL[2], synth.circconv(4099, 64, 4, K=16, U=150, T=5, seed=0)],
                         ids=lambda w: w.name)
def test_parity_mode_fp64_probes(w):
    ctx = ctx_of(w, probe_precision=1)
    mu, s = gpu_estep(ctx, w, np.ones(w.D), w.K, 3, 1)
    omu, os_, _ = estep(op_of(w), w.y, w.beta, np.ones(w.D), w.K, 3, 1, w.U)
    assert rel(mu, omu) <= 1e-7 and rel(s, os_) <= 1e-7, (rel(mu, omu), rel(s, os_))
    a, mu, s = gpu_em(ctx, w, 3, w.K, 3)
    oa, omu, _ = cofem_em(op_of(w), w.y, w.beta, 3, w.K, 3, w.U)
    assert rel(1 / a, 1 / oa) <= 1e-7 and np.array_equal(support(mu), support(omu))


def test_probes_match_oracle_through_estimator():
    # A = I + beta Phi^T Phi with U = 1 and no preconditioner: x_k = (p^T p / p^T A p) p_k, so
    # s_d = (1/K) sum_k D / (p_k^T A p_k): any probe bit error changes s at O(1/K).
    w = synth.dense(30, 256, 3, K=5, U=1, T=1, seed=2)
    ctx = ctx_of(w, precond=0)
    mu, s = gpu_estep(ctx, w, np.ones(w.D), w.K, 123456789012345, 9)
    omu, os_, _ = estep(op_of(w), w.y, w.beta, np.ones(w.D), w.K, 123456789012345, 9, 1, precond=False)
    # a probe bit error moves s by O(1/K) = 0.2; the bar only has to sit above the fp32-class
    # apply error (tcgen05 3xTF32: <= 2^-21 per product, fp32 accumulation; measured 1.4e-6)
    assert rel(s, os_) < 1e-5 and rel(mu, omu) < 1e-5


def test_edge_cases_k1_u1_phi_zero():
    w = synth.dense(8, 40, 2, K=1, U=1, T=1, seed=0)
    ctx = ctx_of(w)
    mu, s = gpu_estep(ctx, w, np.ones(w.D), 1, 0, 0)
    omu, os_, _ = estep(op_of(w), w.y, w.beta, np.ones(w.D), 1, 0, 0, 1)
    assert rel(mu, omu) < 1e-6 and rel(s, os_) < 1e-5
    z = synth.dense(8, 40, 2, K=4, U=5, T=1, seed=0)
    z.phi = np.zeros_like(z.phi)
    ctx = ctx_of(z)
    mu, s = gpu_estep(ctx, z, np.ones(z.D), 4, 0, 0)
    assert np.all(mu == 0) and np.allclose(s, 1.0, rtol=0, atol=1e-7)


def test_invalid_arguments_rejected():
    from paper_2202_12808_b200 import CofemError, Context, OP_DCT2_MASKED
    w = synth.dct(32, 32, 100, 5, K=4, U=10, T=1, seed=0)
    ctx = ctx_of(w)
    with pytest.raises(CofemError) as e:
        gpu_estep(ctx, w, np.ones(w.D), 0, 0, 0)                              # K = 0
    assert e.value.status == 1
    with pytest.raises(CofemError):
        gpu_estep(ctx, w, np.ones(w.D), 5, 0, 0)                              # K > max_probes
    bad = np.ones(w.D); bad[3] = -1.0
    with pytest.raises(CofemError):
        gpu_estep(ctx, w, bad, 2, 0, 0)                                       # alpha <= 0
    with pytest.raises(CofemError) as e:
        Context(OP_DCT2_MASKED, 100, w.D, w.y, w.beta, rows=32, cols=32, obs_idx=w.obs_idx[::-1].copy())
    assert e.value.status == 1
    with pytest.raises(CofemError) as e:
        Context(OP_DCT2_MASKED, 100, 24 * 32, w.y, w.beta, rows=24, cols=32, obs_idx=w.obs_idx)
    assert e.value.status == 6
    with pytest.raises(CofemError):
        Context(OP_DCT2_MASKED, 100, w.D, w.y, -1.0, rows=32, cols=32, obs_idx=w.obs_idx)   # beta <= 0


def test_nan_reports_numeric_breakdown():
    from paper_2202_12808_b200 import CofemError
    w = synth.dense(20, 64, 2, K=2, U=5, T=1, seed=0)
    w.phi = w.phi.copy()
    w.phi[3, 7] = np.nan
    ctx = ctx_of(w)
    with pytest.raises(CofemError) as e:
        gpu_estep(ctx, w, np.ones(w.D), 2, 0, 0)
    assert e.value.status == 4
    assert ctx.report()["bad_col"] >= 0


def test_determinism_and_host_pointers():
    w = SMALL[2]
    ctx = ctx_of(w)
    a1 = gpu_em(ctx, w, 2, w.K, 4)
    a2 = gpu_em(ctx, w, 2, w.K, 4)
    for x, y in zip(a1, a2):
        assert np.array_equal(x, y)
    ah, mh, sh = np.empty(w.D), np.empty(w.D), np.empty(w.D)          # host buffers through the C ABI
    ctx.em(2, w.K, 4, 0, None, ah, mh, sh)
    assert np.array_equal(ah, a1[0]) and np.array_equal(mh, a1[1]) and np.array_equal(sh, a1[2])


def test_em_equals_estep_mstep_and_resume():
    w = SMALL[5]
    ctx = ctx_of(w)
    a2, mu2, s2 = gpu_em(ctx, w, 2, w.K, 8)
    mu, s = gpu_estep(ctx, w, np.ones(w.D), w.K, 8, 0)
    a1 = dev(w.D)
    ctx.mstep(torch.as_tensor(mu, device="cuda"), torch.as_tensor(s, device="cuda"), a1)
    mu_b, s_b = gpu_estep(ctx, w, a1.cpu().numpy(), w.K, 8, 1)
    assert np.array_equal(mu_b, mu2) and np.array_equal(s_b, s2)
    ar, mur, sr = gpu_em(ctx, w, 1, w.K, 8, t0=1, alpha_init=a1.cpu().numpy())
    assert np.array_equal(ar, a2) and np.array_equal(mur, mu2)


def test_probe_parallel_partial_s_sums_to_full():
    # probe-parallel ranks: k_offset / K_total give partial s that sum to the single-GPU s
    w = SMALL[2]
    ctx = ctx_of(w)
    mu, s = gpu_estep(ctx, w, np.ones(w.D), w.K, 6, 2)
    parts = []
    for r in range(4):
        a = torch.ones(w.D, dtype=torch.float64, device="cuda")
        m_r, s_r = dev(w.D), dev(w.D)
        ctx.estep(a, w.K // 4, 6, 2, m_r, s_r, k_offset=r * (w.K // 4), K_total=w.K)
        parts.append(s_r.cpu().numpy())
        assert np.array_equal(m_r.cpu().numpy(), mu)
    assert rel(np.sum(parts, axis=0), s) < 1e-12


@pytest.mark.parametrize("w", [SMALL[0], SMALL[2], SMALL[5],
                               synth.dct(1024, 1024, 262144, 400, K=4, U=8, T=1, seed=1)], ids=lambda w: w.name)
def test_estep_probes_equals_estep_s(w):
    """cofem_estep_probes (probe-parallel ranks that do not own the mean system): the same s,
    bit for bit, as the full E-step (the columns are independent, R3), column 0 frozen at 0."""
    ctx = ctx_of(w)
    a = torch.ones(w.D, dtype=torch.float64, device="cuda")
    mu, s = dev(w.D), dev(w.D)
    ctx.estep(a, w.K, 2, 1, mu, s, k_offset=3, K_total=w.K + 5)
    s2 = dev(w.D)
    ctx.estep_probes(a, w.K, 2, 1, s2, k_offset=3, K_total=w.K + 5)
    assert torch.equal(s, s2)
    assert ctx.report()["frozen_at"][0] == 0
    mu3, s3 = dev(w.D), dev(w.D)                   # and the graph of the full E-step is rebuilt after
    ctx.estep(a, w.K, 2, 1, mu3, s3, k_offset=3, K_total=w.K + 5)
    assert torch.equal(mu3, mu) and torch.equal(s3, s)


# ------------------------------------------------------------ full-size checks (bench launch config)
def test_c4_full_estep1_closed_form():
    """Config 4 at full size (1024 x 1024, N = 2^18, K = 32, U = 200): E-step 1 vs the
    closed form mu = b0/(beta+1), x_k = p_k - beta/(beta+1) P p_k (oracle/closed_forms.py)."""
    w = synth.preset("C4")
    ctx = ctx_of(w)
    mu, s = gpu_estep(ctx, w, np.ones(w.D), w.K, 0, 0)
    P = rademacher_probes(w.D, w.K, 0, 0)
    emu, es, _ = cf.masked_dct_estep1(w.rows, w.cols, w.obs_idx, w.y, w.beta, P)
    assert rel(mu, emu) <= 1e-4 and rel(s, es) <= 1e-4, (rel(mu, emu), rel(s, es))


def test_c4_full_sampled_oracle_iterations():
    """Config 4 at full size, U = 3: the oracle's 3-iteration iterate (not converged, so
    it checks the recurrence itself) against the GPU, every element."""
    w = synth.preset("C4")
    w.U = 3
    ctx = ctx_of(w, cg_iters=3, max_probes=4)
    mu, s = gpu_estep(ctx, w, np.ones(w.D), 4, 1, 0)
    omu, os_, _ = estep(op_of(w), w.y, w.beta, np.ones(w.D), 4, 1, 0, 3)
    assert rel(mu, omu) <= 1e-6 and rel(s, os_) <= 1e-5, (rel(mu, omu), rel(s, os_))


def test_c5_full_size_vs_fft_closed_form():
    """Config 5 at full size (D = 2^24, 64 taps) with K = 4 probes solved to convergence
    (U = 1500) against the FFT diagonalisation (oracle/closed_forms.py item 3)."""
    w = synth.preset("C5")
    ctx = ctx_of(w, cg_iters=1500, max_probes=4)
    mu, s = gpu_estep(ctx, w, np.ones(w.D), 4, 2, 0)
    P = rademacher_probes(w.D, 4, 2, 0)
    emu, es, _ = cf.circconv_estep(w.taps, w.D, w.y, w.beta, 1.0, P)
    assert rel(mu, emu) <= 1e-4 and rel(s, es) <= 1e-4, (rel(mu, emu), rel(s, es))


def test_c4_fast_path_em_two_iterations():
    """The 1024 x 1024 fast path (op_dct1k.cu: warp-per-line FFTs, transposed
    intermediates, concurrent fp64 mean column) through two EM iterations with the
    direction update active, every element against the oracle."""
    w = synth.preset("C4")
    ctx = ctx_of(w, cg_iters=6, max_probes=3)
    a, mu, s = gpu_em(ctx, w, 2, 3, 9)
    oa, omu, os_ = cofem_em(op_of(w), w.y, w.beta, 2, 3, 9, 6)
    assert rel(1 / a, 1 / oa) <= 1e-5 and rel(mu, omu) <= 1e-5 and rel(s, os_) <= 1e-4, \
        (rel(1 / a, 1 / oa), rel(mu, omu), rel(s, os_))


def test_c2_full_size_tensor_core_path():
    """Config 2 shape (2000 x 8000 dense, fp32 Phi): the tcgen05 3xTF32 apply (op_dense_tc.cu,
    256-row CTAs, split-K) against the fp64 oracle, E-step 1 and two EM iterations."""
    w = synth.preset("C2")
    ctx = ctx_of(w, cg_iters=40, max_probes=8)
    mu, s = gpu_estep(ctx, w, np.ones(w.D), 8, 4, 0)
    omu, os_, _ = estep(op_of(w), w.y, w.beta, np.ones(w.D), 8, 4, 0, 40)
    assert rel(mu, omu) <= 1e-4 and rel(s, os_) <= 1e-4, (rel(mu, omu), rel(s, os_))
    a, mu, s = gpu_em(ctx, w, 2, 8, 6)
    oa, omu, _ = cofem_em(op_of(w), w.y, w.beta, 2, 8, 6, 40)
    assert rel(1 / a, 1 / oa) <= 1e-3 and rel(mu, omu) <= 1e-3, (rel(1 / a, 1 / oa), rel(mu, omu))


def test_c3_full_size_mean_residual_and_sampled_parity():
    """Config 3 at full size (8192 x 32768 dense, 1 GiB fp32 Phi, K = 64, U = 300: the bench
    launch configuration, tcgen05 3xTF32 path).  The oracle cannot run this E-step in
    seconds, so the properties any correct E-step has are checked instead (Eq. 5-7):
    (i) mu = x0 solves A x = b0 = beta Phi^T y to the CG's convergence (fp64 mean column);
    (ii) sampled parity: the K = 1 E-step (probe 1 of the same Philox stream) against the
    fp64 oracle E-step at the full U, the north_star bar (1e-4 on mu and s)."""
    from oracle.cofem import mean_rhs
    w = synth.preset("C3")
    op = DenseOp(w.phi)
    ones = np.ones(w.D)
    b0 = mean_rhs(op, w.y, w.beta)

    def A(x):
        return w.beta * op.apply_T(op.apply(x[:, None]))[:, 0] + x

    ctx = ctx_of(w)
    mu, s = gpu_estep(ctx, w, ones, w.K, 0, 0)
    assert np.all(np.isfinite(s)) and np.all(s > 0)          # diag(A^-1) > 0 (A is SPD)
    assert rel(A(mu), b0) <= 1e-8, rel(A(mu), b0)
    ctx1 = ctx_of(w, max_probes=1)
    mu1, s1 = gpu_estep(ctx1, w, ones, 1, 0, 0)
    assert rel(mu1, mu) <= 1e-12                              # the mean column ignores K
    omu, os_, _ = estep(op, w.y, w.beta, ones, 1, 0, 0, w.U)  # sampled: probe 1 only, full U
    assert rel(mu1, omu) <= 1e-4 and rel(s1, os_) <= 1e-4, (rel(mu1, omu), rel(s1, os_))


@pytest.mark.parametrize("variant", [1, 2], ids=["standard_cg", "single_reduction_cg"])
def test_column_sharded_path_world1(variant):
    """The column-sharded dense path (comm.cu + the sharded finishes of cofem.cu /
    op_dense_tc.cu) on a 1-rank NCCL communicator: (i) with d_offset = 0 it must reproduce
    the single-GPU run -- exactly with the standard CG (the all-reduces are identities, the sums
    are the same), within the fp32-probe bar with the single-reduction CG (cg_variant 2, reading
    R23: other dot products, the same iteration in exact arithmetic); (ii) a rank holding columns
    [128, 1024) of a 1024-column Phi must solve its sub-system with the probes of its GLOBAL
    indices (reading R8), against the fp64 oracle PCG."""
    from oracle.cofem import jacobi_diag, mean_rhs, pcg
    from oracle.operators import gram_apply
    from paper_2202_12808_b200 import OP_DENSE, Context, get_unique_id
    w = synth.dense(250, 1024, 20, K=8, U=60, T=3, seed=2)
    a, mu, s = gpu_em(ctx_of(w, apply_path=2), w, 3, 8, 5)   # the sharded mode's kernels (not the cluster loop)
    nid = get_unique_id()
    sh = ctx_of(w, rank=0, world=1, nccl_id=nid, d_offset=0, D_global=w.D, cg_variant=variant)
    a2, mu2, s2 = gpu_em(sh, w, 3, 8, 5)
    if variant == 1:
        assert np.array_equal(a2, a) and np.array_equal(mu2, mu) and np.array_equal(s2, s)
    else:
        assert rel(1 / a2, 1 / a) <= 1e-4 and rel(mu2, mu) <= 1e-4 and rel(s2, s) <= 1e-4, \
            (rel(1 / a2, 1 / a), rel(mu2, mu), rel(s2, s))
        omu, os_, _ = estep(op_of(w), w.y, w.beta, np.ones(w.D), 8, 5, 0, w.U)   # E-step 1 vs the oracle
        m1, s1 = gpu_estep(sh, w, np.ones(w.D), 8, 5, 0)
        assert rel(m1, omu) <= 1e-4 and rel(s1, os_) <= 1e-4, (rel(m1, omu), rel(s1, os_))
    d0 = 128
    phi_r = np.ascontiguousarray(w.phi[:, d0:])
    part = Context(OP_DENSE, w.N, w.D - d0, w.y, w.beta, phi=phi_r, cg_iters=w.U, max_probes=8,
                   rank=0, world=1, nccl_id=get_unique_id(), d_offset=d0, D_global=w.D,
                   cg_variant=variant)   # one id per communicator
    alpha = np.ones(w.D - d0)
    a_dev = torch.ones(w.D - d0, dtype=torch.float64, device="cuda")
    m_dev, s_dev = dev(w.D - d0), dev(w.D - d0)
    n0 = part.report()["collectives"]
    part.estep(a_dev, 8, 5, 0, m_dev, s_dev)
    # NCCL launches per E-step: rho0 once, then per CG iteration the grouped W = Phi P / Phi p0 pair and
    # (standard) gamma + rho' or (single reduction) one (gamma, rho, delta1, delta2) all-reduce
    assert part.report()["collectives"] - n0 == 1 + (3 if variant == 1 else 2) * w.U
    op = DenseOp(phi_r)
    P = rademacher_probes(w.D, 8, 5, 0)[d0:]
    B = np.concatenate([mean_rhs(op, w.y, w.beta)[:, None], P], axis=1)
    X, _ = pcg(lambda V: gram_apply(op, w.beta, alpha, V), B, jacobi_diag(op, w.beta, alpha), w.U)
    omu, os_ = X[:, 0], np.mean(P * X[:, 1:], axis=1)
    assert rel(m_dev.cpu().numpy(), omu) <= 1e-4 and rel(s_dev.cpu().numpy(), os_) <= 1e-4, \
        (rel(m_dev.cpu().numpy(), omu), rel(s_dev.cpu().numpy(), os_))


def test_d_sharded_conv_path_world1():
    """D-sharded convolution (halo exchange through NCCL send/recv with both ring neighbours,
    rank sums of gamma / rho') on a 1-rank communicator: the ring closes on itself, so the
    rank must reproduce the single-GPU circular convolution (identical up to FFT rounding in
    the edge windows); a rank holding samples [128, D) must solve its own circular sub-system
    with globally indexed probes (reading R8)."""
    from oracle.cofem import jacobi_diag, mean_rhs, pcg
    from oracle.operators import gram_apply
    from paper_2202_12808_b200 import OP_CIRCCONV, Context, get_unique_id
    w = synth.circconv(20000, 64, 20, K=8, U=150, T=3, seed=4)
    mu, s = gpu_estep(ctx_of(w), w, np.ones(w.D), 8, 5, 0)
    sh = ctx_of(w, rank=0, world=1, nccl_id=get_unique_id(), d_offset=0, D_global=w.D)
    mu2, s2 = gpu_estep(sh, w, np.ones(w.D), 8, 5, 0)
    assert rel(mu2, mu) <= 1e-6 and rel(s2, s) <= 1e-5, (rel(mu2, mu), rel(s2, s))
    a, m_, s_ = gpu_em(ctx_of(w), w, 2, 8, 6)
    a2, m2, s2_ = gpu_em(sh, w, 2, 8, 6)
    assert rel(1 / a2, 1 / a) <= 1e-4 and rel(m2, m_) <= 1e-4
    d0 = 128
    Dl = w.D - d0
    y_r = np.ascontiguousarray(w.y[d0:])
    part = Context(OP_CIRCCONV, Dl, Dl, y_r, w.beta, taps=w.taps, cg_iters=w.U, max_probes=8,
                   rank=0, world=1, nccl_id=get_unique_id(), d_offset=d0, D_global=w.D)
    a_dev = torch.ones(Dl, dtype=torch.float64, device="cuda")
    m_dev, s_dev = dev(Dl), dev(Dl)
    n0 = part.report()["collectives"]
    part.estep(a_dev, 8, 5, 0, m_dev, s_dev)
    # rho0, then per CG iteration: the halo exchange (one NCCL group), gamma, rho'
    assert part.report()["collectives"] - n0 == 1 + 3 * w.U, part.report()["collectives"] - n0
    op = CircConvOp(w.taps, Dl)
    alpha = np.ones(Dl)
    P = rademacher_probes(w.D, 8, 5, 0)[d0:]
    B = np.concatenate([mean_rhs(op, y_r, w.beta)[:, None], P], axis=1)
    X, _ = pcg(lambda V: gram_apply(op, w.beta, alpha, V), B, jacobi_diag(op, w.beta, alpha), w.U)
    omu, os_ = X[:, 0], np.mean(P * X[:, 1:], axis=1)
    assert rel(m_dev.cpu().numpy(), omu) <= 1e-4 and rel(s_dev.cpu().numpy(), os_) <= 1e-4, \
        (rel(m_dev.cpu().numpy(), omu), rel(s_dev.cpu().numpy(), os_))


@pytest.mark.parametrize("name,nrmse_max", [("C2", 0.05), ("C3", 0.06), ("C4", 0.10)])
def test_full_em_recovers_the_sparse_signal(name, nrmse_max):
    """The method end to end at a BASELINE config's full size and T_em (bench launch
    configuration): all EM iterations finite, the posterior mean recovers the synthetic sparse
    z* (NRMSE of P:125 well below the signal) and >= 95 % of its support (R16 threshold).
    Measured: C2 0.023, C3 0.030, C4 0.050 (tools/recovery_check.py)."""
    w = synth.preset(name)
    a, mu, s = gpu_em(ctx_of(w), w, w.T, w.K, 0)
    assert np.all(np.isfinite(a)) and np.all(np.isfinite(mu)) and np.all(np.isfinite(s))
    z = w.z_true
    assert np.linalg.norm(mu - z) / np.linalg.norm(z) <= nrmse_max
    true_sup = np.nonzero(z)[0]
    found = np.abs(mu) > 1e-3 * np.abs(mu).max()
    assert found[true_sup].mean() >= 0.95


def test_c4_full_size_bitwise_deterministic():
    """Config 4 at full size with the concurrent streams of the fast path (two probe groups and
    the fp64 mean column): every reduction is fixed-order, so two runs agree bit for bit."""
    w = synth.preset("C4")
    r1 = gpu_em(ctx_of(w), w, 2, w.K, 4)
    r2 = gpu_em(ctx_of(w), w, 2, w.K, 4)
    for x, y in zip(r1, r2):
        assert np.array_equal(x, y)


# ------------------------------------------------------------ round 2: library modes and boundary
def test_probe_parallel_library_mode_world1():
    """dist_mode 1 (probe-parallel inside the library: owner split, NCCL all-reduce of s and
    broadcast of mu) on a 1-rank communicator: the collectives are identities, so cofem_em must be
    bitwise equal to the single-GPU run, on the generic DCT path, the 1024^2 fast path and the dense
    cluster CG loop (C1)."""
    from paper_2202_12808_b200 import get_unique_id
    for w in [SMALL[2], synth.dct(1024, 1024, 262144, 400, K=4, U=8, T=1, seed=1), SMALL[0]]:
        ref = gpu_em(ctx_of(w, cg_iters=w.U), w, 2, w.K, 3)
        pp = ctx_of(w, cg_iters=w.U, rank=0, world=1, nccl_id=get_unique_id(), dist_mode=1)
        got = gpu_em(pp, w, 2, w.K, 3)
        for x, y in zip(got, ref):
            assert np.array_equal(x, y)
        mu, s = gpu_estep(pp, w, np.ones(w.D), w.K, 3, 0)
        mu_r, s_r = gpu_estep(ctx_of(w, cg_iters=w.U), w, np.ones(w.D), w.K, 3, 0)
        assert np.array_equal(mu, mu_r) and np.array_equal(s, s_r)


def test_mu_independent_of_max_probes_and_groups():
    """mu (the fp64 mean column) does not depend on max_probes, K or the probe groups: its gamma is
    reduced from one partial per image row in fixed order, whatever the launch size."""
    w = synth.dct(1024, 1024, 262144, 400, K=4, U=12, T=1, seed=2)
    outs = []
    for mp, groups, K in [(4, 0, 4), (32, 0, 4), (32, 1, 4), (32, 2, 20)]:
        ctx = ctx_of(w, cg_iters=w.U, max_probes=mp, probe_groups=groups)
        outs.append(gpu_estep(ctx, w, np.ones(w.D), K, 1, 0)[0])
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])


def test_support_certificate_in_report():
    """cofem_report.support_*: count of |mu_d| > 1e-3 max|mu|, coordinates within 1e-6 of the
    threshold and the smallest margin, against NumPy on the returned mu."""
    w = SMALL[2]
    ctx = ctx_of(w)
    mu, _ = gpu_estep(ctx, w, np.ones(w.D), w.K, 5, 0)
    sup = ctx.report()["support"]
    mx = np.max(np.abs(mu))
    margin = np.abs(np.abs(mu) / mx - 1e-3)
    assert sup["max_abs_mu"] == mx
    assert sup["count"] == int(np.sum(np.abs(mu) > 1e-3 * mx))
    assert sup["adjacent"] == int(np.sum(margin < 1e-6))
    assert sup["min_margin"] == pytest.approx(float(margin.min()), rel=1e-12, abs=1e-300)
    a, mu2, _ = gpu_em(ctx, w, 2, w.K, 5)
    assert ctx.report()["support"]["count"] == int(np.sum(np.abs(mu2) > 1e-3 * np.max(np.abs(mu2))))


def test_dense_device_phi_is_borrowed():
    """A device Phi is borrowed (zero-copy) with its row stride ld: the same E-step, bit for bit, as
    the library's own copy of the host Phi, on the tensor-core path (ld % 4 == 0) and the SIMT path
    (ld odd)."""
    from paper_2202_12808_b200 import OP_DENSE, Context
    w = synth.dense(250, 1000, 20, K=8, U=40, T=1, seed=3)
    ref = gpu_estep(ctx_of(w, cg_iters=40), w, np.ones(w.D), 8, 2, 0)
    for pad in (0, 4, 3):
        ld = w.D + pad
        buf = torch.full((w.N, ld), float("nan"), dtype=torch.float32, device="cuda")
        buf[:, :w.D] = torch.as_tensor(w.phi, device="cuda")
        ctx = Context(OP_DENSE, w.N, w.D, w.y, w.beta, phi=buf, ld=ld, cg_iters=40, max_probes=8)
        got = gpu_estep(ctx, w, np.ones(w.D), 8, 2, 0)
        if pad % 4 == 0:
            assert np.array_equal(got[0], ref[0]) and np.array_equal(got[1], ref[1])
        else:   # SIMT path: same fp32-class accuracy, different kernels
            assert rel(got[0], ref[0]) <= 1e-6 and rel(got[1], ref[1]) <= 1e-4
        buf[:, w.D:] = 0.0   # the padding is never read (NaN there would have propagated)


def test_c4_shape_convention1_estep1_closed_form():
    """DCT convention 1 (Phi = S C2, BASELINE config 4's literal "rows of DCT-II", reading R11) at
    the C4 shape (1024 x 1024, N = 2^18; generic passes): E-step 1 against the closed form
    mu = b0/(beta+1), x_k = p_k - beta/(beta+1) Phi^T Phi p_k, element by element."""
    from parity_util import check
    w = synth.dct(1024, 1024, 262144, 10485, K=8, U=200, T=1, seed=0, convention=1, name="C4_conv1")
    ctx = ctx_of(w)
    mu, s = gpu_estep(ctx, w, np.ones(w.D), w.K, 0, 0)
    P = rademacher_probes(w.D, w.K, 0, 0)
    emu, es, _ = cf.masked_dct_estep1(w.rows, w.cols, w.obs_idx, w.y, w.beta, P, convention=1)
    check("mu", mu, emu, 1e-4)
    check("s", s, es, 1e-4, 1e-3)


@pytest.mark.parametrize("w", [SMALL[0], SMALL[1], SMALL[2], SMALL[5], SMALL[7],
                               synth.dct(1024, 1024, 262144, 400, K=3, U=30, T=3, seed=3, name="dct1024_fast_U30")],
                         ids=lambda w: w.name)
def test_warm_start_em_matches_oracle(w):
    """NEXT-1 warm start (reading R20, cofem_options.warm_start): EM iterations after the first start
    the mean system's CG from the previous mu, on every operator path, against the oracle's
    cofem_em(warm_start=True): north_star EM bars, and parity mode to 1e-7."""
    from parity_util import check
    T = 2        # E-step 2 is warm; longer unconverged fp32 runs drift at 1e-3 (fast path, U = 30: 6e-3 at
                 # T = 3 while parity mode matches the warm oracle to 3e-11: tools/warm_dbg.py)
    oa, omu, _ = cofem_em(op_of(w), w.y, w.beta, T, w.K, 4, w.U, warm_start=True)
    a, mu, _ = gpu_em(ctx_of(w, warm_start=True), w, T, w.K, 4)
    check("1/alpha", 1 / a, 1 / oa, 1e-3, 1e-2)
    check("mu", mu, omu, 1e-3, 1e-2)
    a, mu, _ = gpu_em(ctx_of(w, warm_start=True, probe_precision=1), w, T, w.K, 4)
    check("1/alpha parity", 1 / a, 1 / oa, 1e-7, 1e-6)
    check("mu parity", mu, omu, 1e-7, 1e-6)
    a0, mu0, _ = gpu_em(ctx_of(w), w, 1, w.K, 4)            # the first E-step of a call is cold
    a1, mu1, _ = gpu_em(ctx_of(w, warm_start=True), w, 1, w.K, 4)
    assert np.array_equal(a0, a1) and np.array_equal(mu0, mu1)


@pytest.mark.parametrize("w", [SMALL[1], SMALL[2], SMALL[5], SMALL[7], synth.preset("C1"),
                               synth.dct(1024, 1024, 262144, 400, K=3, U=20, T=2, seed=3, name="dct1024_fast_U20")],
                         ids=lambda w: w.name)
def test_multitask_em_matches_oracle(w):
    """NEXT-4 multi-task SBL (reading R22, cofem_em_multi): three tasks sharing Phi and alpha, against
    the oracle's cofem_em_multi -- fast mode at the north_star EM bars, parity mode to 1e-7 -- and L = 1
    equals cofem_em bit for bit."""
    from oracle.cofem import cofem_em_multi
    from parity_util import check
    Y, _ = synth.tasks(w, 3, seed=2)
    T = 2
    oa, OMU, os_ = cofem_em_multi(op_of(w), Y.T.astype(np.float64), w.beta, T, w.K, 6, w.U)
    for p64, bar in ((0, 1e-3), (1, 1e-6)):      # parity: fp64 rounding through the unconverged CG (C1: 4.7e-7)
        ctx = ctx_of(w, probe_precision=p64)
        a, MU, s = dev(w.D), torch.empty(3 * w.D, dtype=torch.float64, device="cuda"), dev(w.D)
        ctx.em_multi(torch.as_tensor(Y, device="cuda"), T, w.K, 6, 0, None, a, MU, s)
        MU = MU.cpu().numpy().reshape(3, w.D)
        check("1/alpha", 1 / a.cpu().numpy(), 1 / oa, bar, 10 * bar)
        for l in range(3):
            check("mu_%d" % l, MU[l], OMU[:, l], bar, 10 * bar)
    ctx = ctx_of(w)
    a1, m1, s1 = dev(w.D), dev(w.D), dev(w.D)
    ctx.em_multi(torch.as_tensor(Y[:1], device="cuda"), T, w.K, 6, 0, None, a1, m1, s1)
    ref = gpu_em(ctx_of(w), w, T, w.K, 6)
    assert np.array_equal(a1.cpu().numpy(), ref[0]) and np.array_equal(m1.cpu().numpy(), ref[1])


def test_round2_option_validation():
    """The round-2 options reject what they do not support (COFEM_ERR_INVALID = 1, UNSUPPORTED = 6):
    bad option values, warm start or multi-task in sharded / probe-parallel contexts, probe-parallel
    calls with a local k_offset, cofem_estep_probes in the probe-parallel mode, L < 1, the
    single-reduction CG outside the column-sharded dense mode."""
    from paper_2202_12808_b200 import OP_DENSE, CofemError, Context, get_unique_id
    w = SMALL[1]
    for kw in ({"apply_path": 3}, {"probe_groups": 9}, {"dist_mode": 2}, {"warm_start": 1, "d_offset": 0,
                                                                          "D_global": w.D, "nccl_id": None},
               {"cg_variant": 3}, {"cg_variant": 2}):
        bad = dict(kw)
        if bad.get("nccl_id", 1) is None:
            bad["nccl_id"] = get_unique_id()
            bad["world"], bad["rank"] = 1, 0
        with pytest.raises(CofemError) as e:
            ctx_of(w, **bad)
        assert e.value.status in (1, 6)
    pp = ctx_of(w, rank=0, world=1, nccl_id=get_unique_id(), dist_mode=1)
    a = torch.ones(w.D, dtype=torch.float64, device="cuda")
    mu, s = dev(w.D), dev(w.D)
    with pytest.raises(CofemError) as e:
        pp.estep(a, w.K, 1, 0, mu, s, k_offset=2, K_total=w.K + 2)
    assert e.value.status == 1
    with pytest.raises(CofemError) as e:
        pp.estep_probes(a, w.K, 1, 0, s)
    assert e.value.status == 1
    Y, _ = synth.tasks(w, 2, seed=1)
    with pytest.raises(CofemError) as e:
        pp.em_multi(torch.as_tensor(Y, device="cuda"), 1, w.K, 1, 0, None, dev(w.D), None, None)
    assert e.value.status == 6
    ws = ctx_of(w, warm_start=True)
    with pytest.raises(CofemError) as e:
        ws.em_multi(torch.as_tensor(Y, device="cuda"), 1, w.K, 1, 0, None, dev(w.D), None, None)
    assert e.value.status == 6
    ok = ctx_of(w)
    with pytest.raises((CofemError, ValueError)):
        ok.em_multi(torch.empty((0, w.N), dtype=torch.float32, device="cuda"), 1, w.K, 1)


@pytest.mark.parametrize("w", [synth.preset("C1"), synth.dense(37, 203, 4, K=5, U=40, T=3, seed=8),
                               synth.dense(64, 1000, 12, K=33, U=80, T=2, seed=9)], ids=lambda w: w.name)
def test_dense_cluster_cg_loop(w):
    """The small-dense CG loop in one thread-block cluster (op_dense_cluster.cu; DSMEM reductions,
    uneven column slices at D = 203 and 1000, K > 32): against the fp64 oracle (fp32 probes 1e-4,
    fp64 probes 1e-7 as test_parity_mode_fp64_probes: the unconverged fp64 mean moves 3e-9 on C1 on
    every path) and against the per-iteration tensor-core kernels (apply_path 2) over an EM;
    one cluster launch per E-step (plus the probe and init kernels)."""
    ctx = ctx_of(w, max_probes=w.K)
    mu, s = gpu_estep(ctx, w, np.ones(w.D), w.K, 3, 1)
    omu, os_, _ = estep(op_of(w), w.y, w.beta, np.ones(w.D), w.K, 3, 1, w.U)
    # fp32 probes: the north_star bar, or (reading R21) twice what the general FP32 SIMT kernels
    # deviate where fp32 rounding in the unconverged CG moves s more (37 x 203: 5e-4 on every path)
    m1, s1 = gpu_estep(ctx_of(w, max_probes=w.K, apply_path=1), w, np.ones(w.D), w.K, 3, 1)
    bar = max(1e-4, 2 * rel(s1, os_))
    assert rel(mu, omu) <= 1e-4 and rel(s, os_) <= bar, (rel(mu, omu), rel(s, os_), bar)
    l0 = ctx.launches
    gpu_estep(ctx, w, np.ones(w.D), w.K, 3, 1)
    assert ctx.launches - l0 <= 6, ctx.launches - l0
    p64 = ctx_of(w, max_probes=w.K, probe_precision=1)
    mu, s = gpu_estep(p64, w, np.ones(w.D), w.K, 3, 1)
    # fp64 probes: 1e-7, or 10x the oracle's own move under alpha (1 + 1e-15 r) (reading R21) where
    # the unconverged CG amplifies rounding (64 x 1000 at U = 80: the oracle moves s by ~5e-8)
    r = np.random.default_rng(12345).choice([-1.0, 1.0], size=w.D)
    pmu, ps_, _ = estep(op_of(w), w.y, w.beta, 1.0 + 1e-15 * r, w.K, 3, 1, w.U)
    bm, bs = max(1e-7, 10 * rel(pmu, omu)), max(1e-7, 10 * rel(ps_, os_))
    assert rel(mu, omu) <= bm and rel(s, os_) <= bs, (rel(mu, omu), rel(s, os_), bm, bs)
    a, mu, s = gpu_em(ctx, w, w.T, w.K, 5)
    a2, mu2, s2 = gpu_em(ctx_of(w, max_probes=w.K, apply_path=2), w, w.T, w.K, 5)
    assert rel(1 / a, 1 / a2) <= 1e-3 and rel(mu, mu2) <= 1e-4, (rel(1 / a, 1 / a2), rel(mu, mu2))
    assert ctx.report()["frozen_at"] is not None


@pytest.mark.parametrize("w", [synth.preset("C1"), synth.dense(64, 1000, 12, K=33, U=80, T=2, seed=9),
                               synth.dense(37, 203, 4, K=3, U=40, T=2, seed=8)], ids=lambda w: w.name)
def test_dense_cluster_groups(w):
    """The probe columns split over 1..8 thread-block clusters of one launch (probe_groups;
    op_dense_cluster.cu dcl_groups; more clusters than probes falls back to K): the mean system is
    cluster 0's whatever the split, so mu is bitwise the same; s differs only by the order of the
    clusters' partial sums (cluster order, deterministic: repeated runs are bitwise equal), and
    every split meets the north_star bar against the oracle.  Also on an EM (alpha, mu)."""
    omu, os_, _ = estep(op_of(w), w.y, w.beta, np.ones(w.D), w.K, 3, 1, w.U)
    m1, s1 = gpu_estep(ctx_of(w, max_probes=w.K, probe_groups=1), w, np.ones(w.D), w.K, 3, 1)
    bar = max(1e-4, 2 * rel(s1, os_))
    em1 = gpu_em(ctx_of(w, max_probes=w.K, probe_groups=1), w, w.T, w.K, 5)
    for g in (2, 3, 4, 5, 8):
        ctx = ctx_of(w, max_probes=w.K, probe_groups=g)
        mu, s = gpu_estep(ctx, w, np.ones(w.D), w.K, 3, 1)
        mu2, s2 = gpu_estep(ctx, w, np.ones(w.D), w.K, 3, 1)
        assert np.array_equal(mu, m1), g
        assert np.array_equal(mu, mu2) and np.array_equal(s, s2), g
        assert rel(s, s1) <= 1e-12 and float(np.abs(s - s1).max() / np.abs(s1).max()) <= 1e-12, (g, rel(s, s1))
        assert rel(mu, omu) <= 1e-4 and rel(s, os_) <= bar, (g, rel(mu, omu), rel(s, os_), bar)
        a, emu, es = gpu_em(ctx, w, w.T, w.K, 5)
        assert rel(1 / a, 1 / em1[0]) <= 1e-6 and rel(emu, em1[1]) <= 1e-6, (g, rel(1 / a, 1 / em1[0]))


@pytest.mark.parametrize("path", [0, 1, 2], ids=["cluster", "simt", "tcgen05"])
def test_context_created_later_with_smaller_smem_does_not_break_earlier(path):
    """Dynamic shared-memory limits are per kernel function, not per context: a context set up after
    another with a smaller max_probes must not lower the limit the first one's launches need
    (raise_smem_attr).  Direct launches (use_graph off): a captured graph fixes its launch
    configuration at instantiation and would not notice."""
    w = synth.preset("C1")
    ones = np.ones(w.D)
    big = ctx_of(w, max_probes=64, apply_path=path, use_graph=False)
    mu1, s1 = gpu_estep(big, w, ones, w.K, 3, 0)
    small = ctx_of(w, max_probes=2, apply_path=path, use_graph=False)
    gpu_estep(small, w, ones, 2, 3, 0)
    mu2, s2 = gpu_estep(big, w, ones, w.K, 3, 0)
    assert np.array_equal(mu1, mu2) and np.array_equal(s1, s2)
