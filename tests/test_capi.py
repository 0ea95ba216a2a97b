"""The C-ABI library builds, loads and exports every entry point include/cofem.h declares
(no compute: runs without a GPU)."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2202_12808_b200 import build
    build.build()
    from paper_2202_12808_b200 import cofem
    return cofem.lib()


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "cofem.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(cofem_[a-z_]+)\s*\(", txt)))


def test_every_header_symbol_exported_and_bound(L):
    from paper_2202_12808_b200 import cofem
    syms = header_symbols()
    assert len(syms) >= 12
    bound = {n for n, _, _ in cofem.SYMBOLS}
    for s in syms:
        assert hasattr(L, s), s
        assert s in bound, s


def test_host_only_calls(L):
    from paper_2202_12808_b200 import cofem
    assert b"sm_100a" in L.cofem_version()
    names = cofem.kernel_classes()
    assert "dct_cols" in names and "pcg_update" in names
    o = cofem._Options()
    L.cofem_default_options(o)
    assert o.cg_iters == 100 and o.precond == 1 and o.den_floor == 1e-12 and o.alpha_max == 1e12


def test_library_is_sm100a(L):
    import subprocess
    from paper_2202_12808_b200.build import OUT
    r = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", OUT], capture_output=True, text=True)
    assert "sm_100a" in r.stdout


def test_no_oracle_in_product():
    pkg = os.path.join(ROOT, "paper_2202_12808_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert "oracle" not in re.sub(r"(#|//).*", "", txt).lower().replace("oracle/", ""), f


def test_default_options_new_fields(L):
    from paper_2202_12808_b200 import cofem
    o = cofem._Options()
    L.cofem_default_options(o)
    assert (o.apply_path, o.probe_groups, o.use_graph, o.dist_mode) == (0, 0, 1, 0)
    assert o.world == 1 and o.rank == 0 and not o.nccl_id


@pytest.mark.parametrize("mean_cost", [0.0, 1.0, 2.0, 3.5])
def test_probe_split_matches_host_model(L, mean_cost):
    """The library's probe-parallel split (cofem_probe_split, used by dist_mode 1) equals the host
    model dist.probe_split_owner, covers [0, K) exactly once and gives every rank >= 1 probe."""
    from paper_2202_12808_b200 import probe_split
    from paper_2202_12808_b200.dist import probe_split_owner
    for world in range(1, 9):
        for K in range(world, 70):
            seen = []
            for r in range(world):
                got = probe_split(K, world, r, mean_cost)
                assert got == probe_split_owner(K, world, r, mean_cost), (K, world, r)
                off, n, owns = got
                assert n >= 1 and owns == (r == 0)
                seen.extend(range(off, off + n))
            assert seen == list(range(K))


def test_probe_split_rejects_bad_arguments(L):
    from paper_2202_12808_b200 import CofemError, probe_split
    for args in [(3, 4, 0, 0.0), (8, 2, 2, 0.0), (8, 0, 0, 0.0), (8, 2, -1, 0.0)]:
        with pytest.raises(CofemError):
            probe_split(*args)
