"""Sharded solving on one GPU: the ranks of a plan run in lock-step in one
process (each rank's kernels complete before the next starts; no kernel
waits on another), the halo exchange is a device copy between the ranks'
buffers.  fp64 results must equal the single-GPU run bit for bit."""
import numpy as np
import pytest
import torch

from oracle import oracle as orc
from tests.conftest import has_gpu

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]


class _NoExchange:
    def exchange(self, values, group=None):
        pass


def _dev(pool):
    from paper_1608_07411_b200.octree import OctreeField
    return OctreeField.from_host(pool.value, pool.child, pool.state, pool.d_max,
                                 weight=pool.weight)


def _scene(full: bool, d=5, seed=3):
    rng = np.random.default_rng(seed)
    n = 1 << d
    views = []
    for _ in range(4):
        f = np.clip(rng.standard_normal((n, n, n)) * 0.4, -1, 1).astype(np.float32)
        w = (rng.random((n, n, n)) < 0.85).astype(np.uint8)
        f[w == 0] = -1.0
        views.append(orc.build_octree(f, w, tau=-1.0 if full else 0.5,
                                      dtype=np.float32))
    g = rng.integers(0, 3, (n, n, n)).astype(np.float64) * 0.3 - 0.3
    u0 = orc.build_octree(g, tau=-1.0 if full else 0.2)
    return u0, views


@pytest.mark.parametrize("full,world", [(True, 2), (False, 2), (False, 3)])
def test_lockstep_shards_match_single_gpu(full, world):
    from paper_1608_07411_b200 import fusion, shard
    u0h, views_h = _scene(full)
    p = fusion.FusionParams(iterations=6, tau=-1.0, tau_split=0.0,
                            tau_join=1.5, lam=0.4)
    views = [_dev(v) for v in views_h]
    ref = fusion.fuse(_dev(u0h), views, p)
    rh = ref.field.to_host()
    pl = shard.plan(u0h.child, u0h.d_max, world, used=u0h.used, k=2)
    ranks = [shard.ShardedSolver(_dev(u0h), views, p, pl, r, precision="fp64",
                                 exchange=_NoExchange()) for r in range(world)]
    for t in range(p.iterations):
        for s in ranks:
            s.compute(t)
        for (src, dst), idx in pl.send.items():
            if idx.size:
                ii = torch.as_tensor(idx, device="cuda")
                ranks[dst].s.nxt[ii] = ranks[src].s.nxt[ii]
        for s in ranks:
            s.finish()
    leaves = np.nonzero(rh.child < 0)[0]
    for r, s in enumerate(ranks):
        mine = leaves[pl.owner[leaves] == r]
        got = s.values[:s.s.u.used].cpu().numpy()
        assert np.array_equal(got[mine], rh.value[mine]), r
    # energies: per-rank partial sums add up to the single-GPU energies
    e = sum(s.energies(reduce=False).cpu().numpy() for s in ranks)
    want = [st.energy for st in ref.stats]
    np.testing.assert_allclose(e[1:], want[:-1], rtol=1e-12, atol=0)


@pytest.mark.parametrize("full,world", [(True, 2), (False, 3)])
def test_lockstep_overlapped_shards_match_single_gpu(full, world):
    """The overlapped pass (interior tiles before the halo of the previous
    pass arrives, boundary tiles after) gives the single-GPU values bit for
    bit; interior and boundary tile ranges both non-empty."""
    from paper_1608_07411_b200 import fusion, shard
    u0h, views_h = _scene(full, d=6)
    p = fusion.FusionParams(iterations=5, tau=-1.0, tau_split=0.0,
                            tau_join=1.5, lam=0.4)
    views = [_dev(v) for v in views_h]
    ref = fusion.fuse(_dev(u0h), views, p)
    rh = ref.field.to_host()
    pl = shard.plan(u0h.child, u0h.d_max, world, used=u0h.used, k=2)
    assert all(ti > 0 for ti in pl.interior_tiles)
    ranks = [shard.ShardedSolver(_dev(u0h), views, p, pl, r, precision="fp64",
                                 exchange=_NoExchange()) for r in range(world)]
    assert any(s.tiles > pl.interior_tiles[r] for r, s in enumerate(ranks))

    def halo_copy():   # the previous pass's values, into every halo
        for (src, dst), idx in pl.send.items():
            if idx.size:
                ii = torch.as_tensor(idx, device="cuda")
                ranks[dst].s.cur[ii] = ranks[src].s.cur[ii]
    for t in range(p.iterations):
        for s in ranks:
            s.interior(t)
        halo_copy()
        for s in ranks:
            s.boundary(t)
    halo_copy()
    for s in ranks:
        s.s.kern.propagate_levels(s.s.cur, s.s.u.child, 0, pl.top_levels,
                                  ctx=s.s.ctx)
    used = u0h.used
    leaves = np.nonzero(rh.child[:used] < 0)[0]
    for r, s in enumerate(ranks):
        got = s.values[:used].cpu().numpy()
        mine = leaves[pl.owner[leaves] == r]
        assert mine.size and np.array_equal(got[mine], rh.value[mine]), r
        halo = pl.halo[r]          # and the halo after the final exchange
        assert np.array_equal(got[halo], rh.value[halo]), r
    e = sum(s.energies(reduce=False).cpu().numpy() for s in ranks)
    want = [st.energy for st in ref.stats]
    np.testing.assert_allclose(e[1:], want[:-1], rtol=1e-12, atol=0)


@pytest.mark.parametrize("full,world", [(True, 2), (False, 3)])
def test_lockstep_pd_shards_match_single_gpu(full, world):
    """solver='pd' sharded (five fields in the halo): fp64 u, ubar, px, py,
    pz of every owned leaf equal the single-GPU PDSolver bit for bit."""
    from paper_1608_07411_b200 import fusion, shard
    u0h, views_h = _scene(full)
    p = fusion.FusionParams(iterations=5, tau=-1.0, tau_split=0.0,
                            tau_join=1.5, lam=0.4)
    views = [_dev(v) for v in views_h]
    ref = fusion.PDSolver(_dev(u0h), views, p, precision="fp64")
    ref.run(0, p.iterations)
    want = [t[:u0h.used].cpu().numpy() for t in ref.state]
    ref.close()
    pl = shard.plan(u0h.child, u0h.d_max, world, used=u0h.used, k=2)
    ranks = [shard.ShardedPDSolver(_dev(u0h), views, p, pl, r,
                                   precision="fp64", exchange=_NoExchange())
             for r in range(world)]
    for t in range(p.iterations):
        for s in ranks:
            s.compute(t)
        for (src, dst), idx in pl.send.items():
            if idx.size:
                ii = torch.as_tensor(idx, device="cuda")
                for k in range(5):
                    ranks[dst].state[k][ii] = ranks[src].state[k][ii]
        for s in ranks:
            s.finish()
    leaves = np.nonzero(u0h.child[:u0h.used] < 0)[0]
    for r, s in enumerate(ranks):
        mine = leaves[pl.owner[leaves] == r]
        assert mine.size
        for k in range(5):
            got = s.state[k][:u0h.used].cpu().numpy()
            assert np.array_equal(got[mine], want[k][mine]), (r, k)


def test_lockstep_sample_shards_match_single_gpu():
    """BASELINE config 4's per-slot samples path sharded (descent and pd):
    each rank gathers only its own leaves' samples, values equal the
    single-GPU run bit for bit (fp64)."""
    from paper_1608_07411_b200 import fusion, scenes, shard
    u0, samples, info = scenes.cfg5_inputs(40_000, nviews=8, d_max=8,
                                           device="cuda")
    p = fusion.FusionParams(iterations=4, tau=-1.0, tau_split=0.0,
                            tau_join=1.5, lam=0.3)
    h = u0.to_host(scratch=False)
    pl = shard.plan(h.child, h.d_max, 2, used=h.used)
    leaves = np.nonzero(h.child < 0)[0]
    # descent
    ref = fusion.fuse(u0, None, p, samples=samples).field.to_host().value
    ranks = [shard.ShardedSolver(u0, None, p, pl, r, precision="fp64",
                                 exchange=_NoExchange(), samples=samples)
             for r in range(2)]
    # each rank's sample store covers only its own leaf tiles
    full = fusion.Solver(u0, None, p, precision="fp64", samples=samples)
    ntiles = full.ctx.info()["tiles"]
    full.close()
    assert all(s.s.ctx.info()["tiles"] < ntiles for s in ranks)
    for t in range(p.iterations):
        for s in ranks:
            s.compute(t)
        for (src, dst), idx in pl.send.items():
            if idx.size:
                ii = torch.as_tensor(idx, device="cuda")
                ranks[dst].s.nxt[ii] = ranks[src].s.nxt[ii]
        for s in ranks:
            s.finish()
    for r, s in enumerate(ranks):
        mine = leaves[pl.owner[leaves] == r]
        got = s.values[:h.used].cpu().numpy()
        assert np.array_equal(got[mine], ref[mine]), r
        s.close()
    # pd
    rp = fusion.PDSolver(u0, None, p, precision="fp64", samples=samples)
    rp.run(0, p.iterations)
    want = [t[:h.used].cpu().numpy() for t in rp.state]
    rp.close()
    ranks = [shard.ShardedPDSolver(u0, None, p, pl, r, precision="fp64",
                                   exchange=_NoExchange(), samples=samples)
             for r in range(2)]
    for t in range(p.iterations):
        for s in ranks:
            s.compute(t)
        for (src, dst), idx in pl.send.items():
            if idx.size:
                ii = torch.as_tensor(idx, device="cuda")
                for k in range(5):
                    ranks[dst].state[k][ii] = ranks[src].state[k][ii]
        for s in ranks:
            s.finish()
    for r, s in enumerate(ranks):
        mine = leaves[pl.owner[leaves] == r]
        for k in range(5):
            assert np.array_equal(s.state[k][:h.used].cpu().numpy()[mine],
                                  want[k][mine]), (r, k)
        s.close()


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_halo_staging_kernel(dtype):
    """octf_halo_pack: field-major gather of up to five fields at a slot
    list, and the scatter back, equal torch indexing."""
    from paper_1608_07411_b200 import _kernels
    g = torch.Generator(device="cuda").manual_seed(5)
    fields = [torch.rand(1000, device="cuda", generator=g).to(dtype)
              for _ in range(5)]
    idx = torch.randperm(1000, device="cuda")[:300].to(torch.int32)
    for nf in (1, 5):
        buf = torch.empty(nf * 300, dtype=dtype, device="cuda")
        _kernels.halo_pack(fields[:nf], idx, buf)
        want = torch.cat([f[idx.long()] for f in fields[:nf]])
        assert torch.equal(buf, want)
        dst = [torch.zeros_like(f) for f in fields[:nf]]
        _kernels.halo_pack(dst, idx, buf, unpack=True)
        for d, f in zip(dst, fields):
            assert torch.equal(d[idx.long()], f[idx.long()])
            mask = torch.ones(1000, dtype=torch.bool, device="cuda")
            mask[idx.long()] = False
            assert torch.all(d[mask] == 0)
