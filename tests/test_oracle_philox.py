"""Pins for oracle/philox.py (reading R8)."""
import os

import numpy as np
import pytest

from oracle.philox import PROBE_TAG, philox4x32_10, rademacher_probes

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "philox_kat.txt")


def _kat():
    rows = []
    for line in open(GOLDEN):
        line = line.strip()
        if line and not line.startswith("#"):
            v = [int(x, 16) for x in line.split()]
            rows.append((v[:4], v[4:6], v[6:10]))
    return rows


@pytest.mark.parametrize("ctr,key,out", _kat())
def test_philox_known_answers(ctr, key, out):
    got = philox4x32_10(*ctr, *key)
    assert [int(x) for x in got] == out


def test_probe_mapping_by_hand():
    # p_k[d] for d = 128*3 + 32*2 + 5: word 2 of Philox((3, k, t, TAG), key), bit 5.
    seed, t, k = (7 << 32) | 11, 4, 2
    D = 128 * 4
    P = rademacher_probes(D, 3, seed, t)
    w = philox4x32_10(3, k, t, PROBE_TAG, 11, 7)
    d = 128 * 3 + 32 * 2 + 5
    bit = (int(w[2]) >> 5) & 1
    assert P[d, k] == (1.0 if bit == 0 else -1.0)


def test_probes_support_determinism_and_mean():
    P = rademacher_probes(10_000, 10, seed=123, t=0)
    assert set(np.unique(P)) == {-1.0, 1.0}
    assert abs(P.mean()) < 0.05
    assert np.array_equal(P, rademacher_probes(10_000, 10, seed=123, t=0))
    assert not np.array_equal(P, rademacher_probes(10_000, 10, seed=123, t=1))  # fresh per EM step
    # columns independent-looking: off-diagonal correlations ~ 1/sqrt(D)
    C = P.T @ P / P.shape[0]
    assert np.max(np.abs(C - np.eye(10))) < 0.05


def test_probe_k_offset_consistent():
    a = rademacher_probes(1000, 6, seed=5, t=3)
    b = rademacher_probes(1000, 2, seed=5, t=3, k_offset=4)
    assert np.array_equal(a[:, 4:], b)


def test_probe_rejects_k0():
    with pytest.raises(ValueError):
        rademacher_probes(10, 0, 0, 0)
