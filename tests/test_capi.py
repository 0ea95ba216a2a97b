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
