"""The shared input generators: determinism, shapes, counts (reading R13-R15)."""
import numpy as np

import synth


def test_presets_small_shapes_and_determinism():
    for name in ["C1", "C2", "C3", "C4", "C5"]:
        a, b = synth.small(name), synth.small(name)
        assert np.array_equal(a.y, b.y) and a.y.dtype == np.float32 and a.y.shape == (a.N,)
        assert a.z_true.shape == (a.D,)
    w = synth.small("C4")
    assert w.obs_idx.size == w.N and np.all(np.diff(w.obs_idx) > 0)
    assert np.count_nonzero(w.z_true) == 41
    w = synth.small("C5")
    assert np.isclose(np.linalg.norm(w.taps.astype(np.float64)), 1.0, atol=1e-6)
    c1 = synth.preset("C1")
    assert c1.phi.shape == (100, 400) and np.count_nonzero(c1.z_true) == 10
    assert abs(c1.phi.std() - 0.1) < 0.01
    assert not np.array_equal(synth.dense(10, 20, 2, 1, 1, 1, seed=1).y, synth.dense(10, 20, 2, 1, 1, 1, seed=2).y)
