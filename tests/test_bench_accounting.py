"""Host logic of bench.py's roofline accounting (CPU): the algorithmic bytes a kernel class
executed when columns freeze (reading R5; DESIGN §8 "Correction").  A column frozen at CG
iteration F is applied in iterations 0..F and updated in 0..F-1; the arrays shared by a
launch's columns are counted once per launch that still has an active column."""
import os
import sys
import types

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import bench  # noqa: E402  (plain-Python module: argparse, json, subprocess at import)


def _w(D=1000, U=10, kind="circconv"):
    return types.SimpleNamespace(D=D, U=U, kind=kind, N=D, rows=0, cols=0)


def test_no_freezing_counts_u_times_k():
    w = _w()
    K = 4
    per_launch = bench.algorithmic_bytes("conv_apply", w, K)
    tot, frac = bench.active_bytes("conv_apply", w, K, w.D, 1, [[-1] * (K + 1)])
    assert frac == 1.0
    assert tot == per_launch * w.U


def test_frozen_columns_apply_f_plus_one_update_f():
    w = _w(U=10)
    K = 2
    frozen = [[0, 3, -1]]           # column 0 = mean (ignored), column 1 froze at 3, column 2 never
    shared = bench.algorithmic_bytes("conv_apply", w, 0)
    per_col = bench.algorithmic_bytes("conv_apply", w, 1) - shared
    tot, frac = bench.active_bytes("conv_apply", w, K, w.D, 1, frozen)
    assert tot == per_col * (4 + 10) + shared * 10       # applied in 0..3 and 0..9; one launch per iteration
    assert abs(frac - 14 / 20.0) < 1e-12
    shared_u = bench.algorithmic_bytes("pcg_update", w, 0)
    per_u = bench.algorithmic_bytes("pcg_update", w, 1) - shared_u
    tot_u, _ = bench.active_bytes("pcg_update", w, K, w.D, 1, frozen)
    assert tot_u == per_u * (3 + 10) + shared_u * 10     # updated in 0..2 and 0..9


def test_groups_count_shared_arrays_per_group_launch():
    w = _w(U=10, kind="dct2_masked")
    w.rows = w.cols = 1024
    K, G = 4, 2                      # groups cover probe columns [1, 3) and [3, 5)
    frozen = [[0, 1, 1, 5, -1]]      # group 0 active in iterations 0..1, group 1 in 0..9
    shared = bench.algorithmic_bytes("dct_rows_inv", w, 0)
    per_col = bench.algorithmic_bytes("dct_rows_inv", w, 1) - shared
    tot, _ = bench.active_bytes("dct_rows_inv", w, K, w.D, G, frozen)
    assert tot == per_col * (2 + 2 + 6 + 10) + shared * (2 + 10)


def test_all_frozen_at_zero_executes_one_apply_and_no_update():
    w = _w(U=50)
    K = 3
    frozen = [[0, 0, 0, 0]]
    tot_u, frac_u = bench.active_bytes("pcg_update", w, K, w.D, 1, frozen)
    assert tot_u == 0 and frac_u == 0.0
    tot_a, frac_a = bench.active_bytes("conv_apply", w, K, w.D, 1, frozen)
    assert abs(frac_a - 1 / 50.0) < 1e-12 and tot_a > 0


def test_executed_applies_counts_frozen_columns():
    """rhs_applies_per_s counts executed column-iterations: a column frozen at CG iteration F is
    applied in iterations 0..F (the apply of F finds it frozen), one never frozen in all U."""
    assert bench.executed_applies([[-1, 3, 0]], 10) == 10 + 4 + 1
    assert bench.executed_applies([[-1, -1], [9, 12]], 10) == 20 + 10 + 10


def test_every_profiled_class_with_work_has_bytes():
    """The dominant-kernel pick only considers classes with algorithmic bytes: every kernel class
    that carries the E-step's work on some path (incl. the cluster CG loop of small dense problems)
    must have them, or a path whose only heavy class lacks them would have no roofline."""
    dense = types.SimpleNamespace(D=400, U=10, kind="dense", N=100, rows=0, cols=0)
    dct = types.SimpleNamespace(D=1 << 20, U=10, kind="dct2_masked", N=1 << 18, rows=1024, cols=1024)
    conv = _w()
    for cls, w in [("dense_phi_p", dense), ("dense_phiT_w", dense), ("dense_cluster", dense),
                   ("pcg_update", dense), ("pcg_direction", dense), ("dct_rows_inv", dct), ("dct_cols", dct),
                   ("dct_rows_fwd", dct), ("conv_apply", conv)]:
        assert bench.algorithmic_bytes(cls, w, 4) > 0, cls
    # the cluster loop reads Phi and the state once per E-step: more columns, more bytes
    assert bench.algorithmic_bytes("dense_cluster", dense, 8) > bench.algorithmic_bytes("dense_cluster", dense, 4)
