"""The reference's dense solver (fusion.py:253-325): the oracle restatement
against the reference's own output (CPU), and the GPU dense_fuse -- the
grid run as a full tree -- against the same fixture bit for bit."""
import numpy as np
import pytest

from oracle import oracle as orc
from tests.conftest import has_gpu
from tests.goldens import load


def test_oracle_dense_matches_reference():
    z = load("dense")
    p = orc.Params(iterations=6, lam=0.4)
    u = orc.dense_fuse(z["u0"], list(z["fs"]), list(z["ws"]), p)
    assert np.array_equal(u, z["u"])


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
def test_gpu_dense_fuse_matches_reference():
    from paper_1608_07411_b200 import fusion
    z = load("dense")
    p = fusion.FusionParams(iterations=6, lam=0.4)
    u, stats = fusion.dense_fuse(z["u0"], list(z["fs"]), list(z["ws"]), p)
    assert np.array_equal(u, z["u"])
    np.testing.assert_allclose([s.energy for s in stats], z["energies"],
                               rtol=1e-12)
    one = fusion.dense_step(z["u0"], list(z["fs"]), list(z["ws"]), p, p.xi0)
    want = orc.dense_step(z["u0"], list(z["fs"]), list(z["ws"]),
                          orc.Params(iterations=6, lam=0.4), 0.1)
    assert np.array_equal(one, want)
    e = fusion.dense_energy(z["u"], list(z["fs"]), list(z["ws"]), p)
    assert abs(e - z["energies"][-1]) <= 1e-12 * abs(z["energies"][-1])
