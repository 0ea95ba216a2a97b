"""Comparison helpers of the GPU parity tests (host-side NumPy only).

Bars (BASELINE.json north_star; readings R16/R17 in DESIGN.md §3):
  rel. L2  ||g - o||_2 / ||o||_2 per vector (1/alpha compared as 1/alpha)
  element  max_d |g_d - o_d| / max_d |o_d|  -- beside every L2 check, so that a single wrong
           element at large D (which moves the L2 error by ~1/sqrt(D)) cannot hide
  support  |mu_d| > 1e-3 max|mu| on each side's own mu; a flip is certified when the oracle's
           coordinate sits within `adj` of the threshold (SURVEY.md §8(c) fragility note)
"""
import numpy as np


def rel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def elem(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))


def check(tag, got, ref, bar, elem_bar=None):
    """Relative L2 <= bar and max-normalised per-element error <= elem_bar (default bar)."""
    e2, ee = rel(got, ref), elem(got, ref)
    eb = bar if elem_bar is None else elem_bar
    assert e2 <= bar and ee <= eb, "%s: rel L2 %.3e (bar %.1e), elem %.3e (bar %.1e)" % (tag, e2, bar, ee, eb)
    return e2, ee


def support(mu, thr=1e-3):
    mu = np.asarray(mu, dtype=np.float64)
    return np.abs(mu) > thr * np.max(np.abs(mu))


def flips(mu_gpu, mu_ref, sup_ref=None, thr=1e-3):
    """Support flips with their certificate: for each flipped d, the oracle's margin
    | |mu_d|/max|mu| - thr | and the GPU-oracle difference |dmu_d| / max|mu|."""
    g = support(mu_gpu, thr)
    o = support(mu_ref, thr) if sup_ref is None else sup_ref
    idx = np.nonzero(g != o)[0]
    mx = np.max(np.abs(np.asarray(mu_ref, dtype=np.float64)))
    margin = np.abs(np.abs(np.asarray(mu_ref, dtype=np.float64)[idx]) / mx - thr)
    dmu = np.abs(np.asarray(mu_gpu, dtype=np.float64)[idx] - np.asarray(mu_ref, dtype=np.float64)[idx]) / mx
    return idx, margin, dmu
