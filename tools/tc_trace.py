"""(Pair protocol: MMA events 0/2/3 are indexed by the pair p, not the step.)
Pipeline trace of the dense tcgen05 k_tc_phiTW mainloop (CTA 0): run with the
COFEM_TC_EXP_TRACE build in place of libcofem.so (tools/build_tc_variants.sh VARIANTS=TRACE).
Events per K step kt (clock64): 0 MMA after chunk_free, 1 after full, 2 after split_done,
3 after issue+commits; 4/5/6 splitter (q=0 warp of group kt%4) after full / tfree / arrive;
7 promote(c) of group g after chunk_full (row 4c+g); 8 producer after empty."""
import ctypes, sys
import numpy as np
sys.path.insert(0, "/root/repo")
import synth
from paper_2202_12808_b200 import Context, cofem

w = synth.preset(sys.argv[1] if len(sys.argv) > 1 else "C3")
ctx = Context.from_workload(w, max_probes=w.K, cg_iters=1)
rng = np.random.default_rng(0)
D, K = w.D, w.K
alpha = np.ones(D); x0 = rng.standard_normal(D); X = rng.standard_normal((K, D)).astype(np.float32)
q0 = np.empty(D); Q = np.empty((K, D), np.float32); g = np.empty(K + 1)
for _ in range(3):
    ctx.apply(alpha, x0, X, q0, Q, g)
L = ctypes.CDLL(cofem.LIB_PATH)
if not hasattr(L, "cofem_tc_trace_dump"):   # regular build (e.g. under ncu): the applies were the point
    sys.exit(0)
buf = np.zeros((1024, 10), dtype=np.int64)
assert L.cofem_tc_trace_dump(buf.ctypes.data_as(ctypes.c_void_p)) == 0
nk = int((buf[:, 3] > 0).sum())
t0 = buf[0, 8]
T = (buf - t0).astype(np.float64)
print("nk traced", nk, " total cycles", T[nk - 1, 3])
print("kt   chunkfree full  splitdone issued | spl_full spl_tfree spl_arrive | prod_empty")
for kt in list(range(0, 12)) + list(range(100, 116)):
    r = T[kt]
    print("%3d %9.0f %6.0f %9.0f %7.0f | %8.0f %9.0f %10.0f | %9.0f" % (kt, r[0], r[1], r[2], r[3], r[4], r[5], r[6], r[8]))
iss = np.diff(T[:nk, 3])
print("issue interval: median %.0f mean %.0f" % (np.median(iss), iss[10:].mean()))
wait_cf = T[:nk, 0] - np.r_[0, T[:nk - 1, 3]]
wait_full = T[:nk, 1] - T[:nk, 0]
wait_sd = T[:nk, 2] - T[:nk, 1]
iss_t = T[:nk, 3] - T[:nk, 2]
for kin in (0, 1):
    sel = np.arange(10, nk) % 2 == kin
    print("kin=%d: chunk_free wait %.0f  full %.0f  split_done %.0f  issue %.0f" % (kin, wait_cf[10:][sel].mean(),
          wait_full[10:][sel].mean(), wait_sd[10:][sel].mean(), iss_t[10:][sel].mean()))
print("MMA thread per step: chunk_free wait %.0f, full wait %.0f, split_done wait %.0f, issue %.0f" %
      tuple(x[10:].mean() for x in (wait_cf, wait_full, wait_sd, iss_t)))
sp_tf = T[:nk, 5] - T[:nk, 4]
sp_work = T[:nk, 6] - T[:nk, 5]
print("splitter per step: tfree wait %.0f, split+arrive %.0f" % (sp_tf[10:].mean(), sp_work[10:].mean()))
lat = T[:nk, 6] - T[:nk, 4]
print("tfree(kt) observed - MMA(kt-4) issued: %.0f" % (T[14:nk, 5] - T[10:nk - 4, 3]).mean())

# pair-protocol summary (MMA events indexed by pair)
npair = int((buf[:, 3] > 0).sum())
P = T[:npair]
iss = P[8:, 3] - P[8:, 2]
gap = P[9:, 0] - P[8:-1, 3]
wsd = P[8:, 2] - P[8:, 0]
print("PAIR: period %.0f cycles, issue %.0f, chunk_free gap %.0f, split_done wait %.0f" %
      (np.diff(P[8:, 3]).mean(), iss.mean(), gap.mean(), wsd.mean()))

print("pair  e3(p-1)->e0  e0->e2  e2->e3")
for p in range(40, 52):
    print("%4d %10.0f %7.0f %7.0f" % (p, T[p, 0] - T[p - 1, 3], T[p, 2] - T[p, 0], T[p, 3] - T[p, 2]))
