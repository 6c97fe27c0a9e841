"""BASELINE config 4 (solver microbenchmark) at test size: a random adaptive
tree refined around a random implicit surface, N=32 per-leaf samples given
per slot (no view trees), restructuring off.  The oracle sees the same
samples as view trees with the tree's structure."""
import numpy as np
import pytest
import torch

from oracle import oracle as orc
from tests.conftest import has_gpu

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]


@pytest.fixture(scope="module")
def cfg5_small():
    from paper_1608_07411_b200 import scenes
    u0, (F, W), info = scenes.cfg5_inputs(60_000, nviews=32, d_max=9,
                                          device="cuda")
    h = u0.to_host()
    Fh = F.cpu().numpy()
    ones = np.ones(h.used, dtype=np.float32)
    views = [orc.Pool(Fh[v].copy(), h.child, h.state.copy(), h.d_max,
                      weight=ones) for v in range(F.shape[0])]
    u0h = orc.Pool(h.value, h.child, h.state.copy(), h.d_max)
    return u0, (F, W), u0h, views, info


def test_tree_shape(cfg5_small):
    _, _, u0h, _, info = cfg5_small
    hist = info["leaves_per_level"]
    n = info["leaves"]
    assert n == int((u0h.child < 0).sum())
    assert 0.4 < hist[9] / n < 0.8 and hist[8] / n > 0.1   # finest levels dominate
    assert len(orc.leaves(u0h)) == n


def test_descent_with_per_leaf_samples_bitexact(cfg5_small):
    from paper_1608_07411_b200 import fusion
    u0, samples, u0h, views, _ = cfg5_small
    p = fusion.FusionParams(iterations=5, tau=-1.0, tau_split=0.0,
                            tau_join=1.5, lam=0.3)
    res = fusion.fuse(u0, None, p, samples=samples)
    ref = orc.fuse(u0h, views, orc.Params(iterations=5, tau_split=0.0,
                                           tau_join=1.5, lam=0.3))
    got = res.field.to_host().value
    assert np.array_equal(got, ref.field.value[:ref.field.used])
    np.testing.assert_allclose([s.energy for s in res.stats],
                               [s.energy for s in ref.stats], rtol=1e-12)
    r32 = fusion.fuse(u0, None, p, samples=samples, precision="fp32")
    assert np.max(np.abs(r32.field.to_host().value - got)) <= 1e-4


def test_pd_with_per_leaf_samples_bitexact(cfg5_small):
    from paper_1608_07411_b200 import fusion
    u0, samples, u0h, views, _ = cfg5_small
    p = fusion.FusionParams(iterations=4, lam=0.3, tau_split=0.0,
                            tau_join=1.5)
    s = fusion.PDSolver(u0, None, p, precision="fp64", samples=samples)
    s.run(0, 4)
    u, ub, px, py, pz, en = orc.pd_fuse(u0h, views, 0.3, 1e-4, 4)
    got = [t[:u0h.used].cpu().numpy() for t in s.state]
    for g, w in zip(got, (u, ub, px, py, pz)):
        assert np.array_equal(g, w)
    np.testing.assert_allclose([st.energy for st in s.stats[:-1]], en[1:],
                               rtol=1e-12)


def test_samples_path_equals_view_path(cfg5_small):
    from paper_1608_07411_b200 import fusion
    from paper_1608_07411_b200.octree import OctreeField
    u0, samples, u0h, views, _ = cfg5_small
    dv = [OctreeField.from_host(v.value, v.child, v.state, v.d_max,
                                weight=v.weight) for v in views]
    p = fusion.FusionParams(iterations=3, tau=-1.0, tau_split=0.0,
                            tau_join=1.5, lam=0.3)
    a = fusion.fuse(u0, dv, p, precision="fp32").field.to_host().value
    b = fusion.fuse(u0, None, p, samples=samples,
                    precision="fp32").field.to_host().value
    assert np.array_equal(a, b)


def test_fused_propagate_equals_per_level(cfg5_small, monkeypatch):
    """The primal-dual kernel's fused bottom propagate level (five fields)
    gives the per-level launches' pools bit for bit (fp32 and fp64, every
    field including inner nodes)."""
    from paper_1608_07411_b200 import fusion
    u0, samples, _, _, _ = cfg5_small
    p = fusion.FusionParams(iterations=3, tau=-1.0, tau_split=0.0,
                            tau_join=1.5, lam=0.3)

    def run():
        out = []
        for prec in ("fp32", "fp64"):
            s = fusion.PDSolver(u0, None, p, precision=prec, samples=samples)
            s.run(0, 3)
            out += [t.cpu().numpy() for t in s.state]
        return out

    fused = run()
    monkeypatch.setenv("OCTF_NO_FUSED_PARENT", "1")
    plain = run()
    for a, b in zip(fused, plain):
        assert np.array_equal(a, b)
