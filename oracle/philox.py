"""Philox4x32-10 and the Rademacher probe mapping (oracle side; test infrastructure only).

Paper: the probes p_k have iid entries drawn from the "Randemacher" (Rademacher)
distribution, +1 or -1 with equal probability (§3.1), freshly drawn inside
every EM iteration (Algorithm 1 line 5).  The paper does not name an RNG;
DESIGN.md reading R8 fixes a counter-based Philox4x32-10 so that the oracle and
the GPU draw bit-identical probes without sharing code (each side implements the
generator itself).

Philox4x32-10 (Salmon et al., "Parallel random numbers: as easy as 1, 2, 3",
SC'11): 10 rounds of
    (hi0, lo0) = mulhilo(0xD2511F53, c0);  (hi1, lo1) = mulhilo(0xCD9E8D57, c2)
    c = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0)
    k = (k0 + 0x9E3779B9, k1 + 0xBB67AE85)
Pinned by the published known-answer vectors (tests/golden/philox_kat.txt).

Probe mapping (reading R8):
    key     = (seed mod 2^32, seed >> 32)
    counter = (floor(d / 128), k, t, 0x50524F42)
    word    = Philox(counter, key)[floor((d mod 128) / 32)]
    p_k[d]  = +1 if bit (d mod 32) of word is 0 else -1
"""
import numpy as np

_M0 = np.uint64(0xD2511F53)
_M1 = np.uint64(0xCD9E8D57)
_W0 = np.uint64(0x9E3779B9)
_W1 = np.uint64(0xBB67AE85)
_MASK = np.uint64(0xFFFFFFFF)
_S32 = np.uint64(32)

PROBE_TAG = 0x50524F42  # "PROB"


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Philox4x32-10 on (broadcastable) arrays of 32-bit counters; returns 4 uint32 arrays."""
    c = [np.asarray(x, dtype=np.uint64) & _MASK for x in (c0, c1, c2, c3)]
    k0 = np.asarray(k0, dtype=np.uint64) & _MASK
    k1 = np.asarray(k1, dtype=np.uint64) & _MASK
    for _ in range(10):
        p0 = _M0 * c[0]
        p1 = _M1 * c[2]
        hi0, lo0 = p0 >> _S32, p0 & _MASK
        hi1, lo1 = p1 >> _S32, p1 & _MASK
        c = [hi1 ^ c[1] ^ k0, lo1, hi0 ^ c[3] ^ k1, lo0]
        k0 = (k0 + _W0) & _MASK
        k1 = (k1 + _W1) & _MASK
    return [x.astype(np.uint32) for x in c]


def rademacher_probes(D, K, seed, t, k_offset=0):
    """D x K fp64 matrix of +-1 probes p_k for EM iteration t.

    Column j holds the probe with global index k = k_offset + j (probe-parallel
    ranks pass their first global k).
    """
    if K < 1:
        raise ValueError("K must be >= 1 (S:148)")
    d = np.arange(D, dtype=np.uint64)
    blk = d // np.uint64(128)
    word_sel = (d % np.uint64(128)) // np.uint64(32)
    bit = d % np.uint64(32)
    seed = int(seed)
    k0, k1 = seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF
    out = np.empty((D, K), dtype=np.float64)
    for j in range(K):
        k = k_offset + j
        w = philox4x32_10(blk, k, t, PROBE_TAG, k0, k1)
        words = np.choose(word_sel.astype(np.int64), w).astype(np.uint64)
        bits = (words >> bit) & np.uint64(1)
        out[:, j] = np.where(bits == 0, 1.0, -1.0)
    return out
