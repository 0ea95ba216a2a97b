"""Pin the oracle's Philox4x32-10 against cuRAND's independent implementation on the GPU."""
import os
import subprocess

import numpy as np
import pytest

from oracle.philox import PROBE_TAG, philox4x32_10

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def test_oracle_philox_equals_curand(tmp_path):
    exe = str(tmp_path / "philox_curand")
    r = subprocess.run(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-o", exe,
                        os.path.join(HERE, "gpu_helpers", "philox_curand.cu")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    rng = np.random.default_rng(0)
    rows = [(b, k, t, PROBE_TAG, s & 0xFFFFFFFF, s >> 32)
            for b, k, t, s in zip(rng.integers(0, 1 << 17, 200), rng.integers(0, 64, 200), rng.integers(0, 50, 200),
                                  rng.integers(0, 1 << 63, 200, dtype=np.uint64).astype(object))]
    rows += [(0, 0, 0, 0, 0, 0), (0xFFFFFFFF,) * 6]
    inp = "\n".join(" ".join("%x" % int(v) for v in row) for row in rows)
    out = subprocess.run([exe], input=inp, capture_output=True, text=True, check=True).stdout.split("\n")
    for row, line in zip(rows, out):
        got = [int(x, 16) for x in line.split()]
        want = [int(x) for x in philox4x32_10(*row)]
        assert got == want, (row, got, want)
