"""solver='pd' has no reference counterpart (its oracle, pd_oracle.c, is a
written definition), but the functional it reports is the reference's: the
reference energy (_kernels.pyx:466-578, restated in octfuse_oracle.c and
pinned bit for bit to the reference's fixtures) with its smoothing eps -> 0
is the TV-L1 energy sum_leaves [sum w|u - f| / (gamma + sum w) +
lam |grad+ u|] h^3.  These tests tie the pd mode's energies to that pinned
code: on the states the pd oracle / the GPU pd solver visits, the pd energy
equals the reference energy evaluated at eps = 1e-9."""
import numpy as np
import pytest

from oracle import oracle as orc
from tests.conftest import has_gpu


def _scene(seed=3, d=4, nviews=6):
    rng = np.random.default_rng(seed)
    n = 1 << d
    base = np.kron(rng.choice([-0.6, 0.0, 0.6], (4, 4, 4)),
                   np.ones((n // 4,) * 3))
    views = []
    for _ in range(nviews):
        f = np.clip(base + rng.standard_normal((n, n, n)) * 0.2, -1,
                    1).astype(np.float32)
        w = (rng.random((n, n, n)) < 0.8).astype(np.uint8)
        f[w == 0] = -1.0
        views.append(orc.build_octree(f, w, tau=0.5, dtype=np.float32))
    g = base * 0.5 + rng.integers(0, 3, (n, n, n)) * 0.1 - 0.1
    g[:, :, n // 2:] = base[:, :, n // 2:] * 0.5
    return views, orc.build_octree(g, tau=0.15)


def _ref_energy(u, child, views, d_max, lam, gamma, eps=1e-9):
    return orc.tree_energy(np.ascontiguousarray(u, dtype=np.float64), child,
                           [v.value for v in views], [v.weight for v in views],
                           [v.child for v in views], d_max, lam, eps, gamma)


def test_pd_oracle_energy_is_the_reference_energy_at_eps_zero():
    views, u0 = _scene()
    lam, gamma = 0.4, 1e-4
    used = u0.used
    # the energy before pass k is that of the state after k passes
    for k in (0, 1, 5):
        u, *_, en = orc.pd_fuse(u0, views, lam, gamma, k + 1)
        uk = (u0.value[:used].astype(np.float64) if k == 0
              else orc.pd_fuse(u0, views, lam, gamma, k)[0])
        want = _ref_energy(uk, u0.child[:used], views, u0.d_max, lam, gamma)
        assert en[k] == pytest.approx(want, rel=1e-7)
    assert en[5] < en[0]


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
def test_gpu_pd_energy_is_the_reference_energy_at_eps_zero():
    """The GPU pd solver's reported energies against the GPU energy kernel
    of the descent path (fusion.tree_energy, bit-pinned to the reference) at
    eps = 1e-9, on the pd solver's own states."""
    from paper_1608_07411_b200 import fusion
    from paper_1608_07411_b200.octree import OctreeField
    views_h, u0h = _scene()

    def dev(p):
        return OctreeField.from_host(p.value, p.child, p.state, p.d_max,
                                     weight=p.weight)
    views = [dev(v) for v in views_h]
    lam = 0.4
    for iters in (1, 6):
        p = fusion.FusionParams(lam=lam, iterations=iters, tau_split=0.0,
                                tau_join=1.5)
        res = fusion.fuse(dev(u0h), views, p, solver="pd", precision="fp64")
        pe = fusion.FusionParams(lam=lam, eps=1e-9, iterations=1,
                                 tau_split=0.0, tau_join=1.5)
        want = fusion.tree_energy(res.field, views, pe)
        assert res.stats[-1].energy == pytest.approx(want, rel=1e-7)


def test_pd_oracle_prox_minimises_its_objective():
    """The pd oracle's prox (pd_oracle.c wmedian_prox) on a single-cell tree,
    where a pass is u' = prox_{tau D}(u) with D(x) = sum w|x - f| / (gamma +
    sum w): u' minimises (x - u)^2 / 2 + tau D(x) -- checked against the
    objective at every kink f_i, every stationary point of a linear piece
    and a fine grid (random weights, ties, zero weights, u outside the
    samples' range)."""
    rng = np.random.default_rng(0)
    gamma, tau = 1e-4, 0.7

    def leaf(v, w=None):
        return orc.Pool(np.array([v], np.float32 if w is not None else np.float64),
                        np.full(1, -1, np.int32), np.array([1, -1, 1], np.int64),
                        0, weight=None if w is None else np.array([w], np.float32))
    for trial in range(200):
        n = int(rng.integers(1, 9))
        f = np.round(rng.uniform(-1, 1, n) * 8) / 8 if trial % 3 == 0 \
            else rng.uniform(-1, 1, n)
        w = rng.choice([0.0, 0.25, 0.5, 1.0], n) if trial % 2 else np.ones(n)
        if not w.any():
            w[0] = 1.0
        f32, w32 = f.astype(np.float32), w.astype(np.float32)
        u = float(rng.uniform(-1.5, 1.5)) if trial % 5 else float(f32[0])
        views = [leaf(a, b) for a, b in zip(f32, w32)]
        out = orc.pd_fuse(leaf(u), views, 0.3, gamma, 1, tau=tau, sigma=0.1,
                          clamp=False)
        x = float(out[0][0])
        fd, wd = f32.astype(np.float64), w32.astype(np.float64)
        c = tau / (wd.sum() + gamma)

        def obj(y):
            return 0.5 * (y - u) ** 2 + c * float((wd * np.abs(y - fd)).sum())
        order = np.argsort(fd, kind="stable")
        S = np.concatenate([[0.0], np.cumsum(wd[order])])
        cands = list(fd) + [u - c * (2 * s - wd.sum()) for s in S] \
            + list(np.linspace(-2, 2, 401))
        best = min(obj(y) for y in cands)
        assert obj(x) <= best + 1e-12
