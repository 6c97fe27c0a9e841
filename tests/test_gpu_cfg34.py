"""BASELINE configs 2 and 3 (cfg3 adaptive object, cfg4 room) at reduced
scale, end to end: sphere-traced depth maps -> TSDF -> view trees -> u0 ->
fuse with split/join every pass, GPU (through the C ABI) against the CPU
oracle on the same depth maps.  Full scale is infeasible for the oracle
(SURVEY.md §8(d)); tools/cfg3_bench.py measures it on the GPU alone."""
import numpy as np
import pytest
import torch

from oracle import oracle as orc
from tests.conftest import has_gpu

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]


def oracle_prepare(sc, p):
    n = sc.resolution
    wf = np.zeros((n, n, n))
    ws = np.zeros((n, n, n))
    views = []
    for d, c in zip(sc.depths, sc.cameras):
        f, w = orc.build_view_tsdf(d, c, sc.origin, sc.voxel_size, n, p.delta,
                                   p.eta)
        wf += f.astype(np.float64) * w
        ws += w
        views.append(orc.build_octree(f, w, tau=p.tau, dtype=np.float32))
    ub = orc.initial_field(wf, ws, p.gamma)
    return views, orc.build_octree(ub, tau=p.tau)


def run_case(sc, iterations):
    from paper_1608_07411_b200 import fusion, volume
    kw = dict(sc.params, iterations=iterations)
    p_gpu = fusion.FusionParams(**kw)
    p_orc = orc.Params(**kw)
    dom = volume.VolumeDomain(sc.origin, sc.voxel_size, sc.resolution)
    views, u0, seen = fusion.prepare(sc.depths, sc.cameras, dom, p_gpu)
    oviews, ou0 = oracle_prepare(sc, p_orc)
    # view trees and u0: bit-exact
    for g, r in zip(views, oviews):
        h = g.to_host()
        assert np.array_equal(h.child, r.child)
        assert np.array_equal(h.value, r.value)
        assert np.array_equal(h.weight, r.weight)
    hu = u0.to_host()
    assert np.array_equal(hu.child, ou0.child)
    assert np.array_equal(hu.value, ou0.value)
    # the solver with split/join every pass, fp64: the reference's pools
    res = fusion.fuse(u0, views, p_gpu, precision="fp64", log_joins=True)
    ref = orc.fuse(ou0, oviews, p_orc, log_joins=True)
    got = res.field.to_host()
    used = int(ref.field.state[0])
    assert list(got.state) == list(ref.field.state)
    assert np.array_equal(got.child[:used], ref.field.child[:used])
    assert np.array_equal(got.value[:used], ref.field.value[:used])
    assert [(s.splits, s.joins) for s in res.stats] == \
        [(s.splits, s.joins) for s in ref.stats]
    np.testing.assert_allclose([s.energy for s in res.stats],
                               [s.energy for s in ref.stats], rtol=1e-12)
    assert np.array_equal(res.join_log, ref.join_log)
    return res, ref, seen


def test_cfg3_reduced_end_to_end():
    from paper_1608_07411_b200 import scenes
    sc = scenes.make_cfg3(d_max=7, n_views=16, width=320, height=240,
                          focal=262.5, device="cuda")
    res, ref, seen = run_case(sc, 6)
    assert sum(s.splits + s.joins for s in ref.stats) > 0   # restructures
    assert bool(seen.any())


def test_cfg4_reduced_end_to_end():
    from paper_1608_07411_b200 import scenes
    sc = scenes.make_cfg4(d_max=7, n_frames=12, width=320, height=240,
                          focal=262.5, device="cuda")
    res, ref, _ = run_case(sc, 4)
    assert sum(s.splits + s.joins for s in ref.stats) > 0


def test_incremental_regather_equals_full_gather(monkeypatch):
    """After a restructuring pass the context keeps unchanged leaves' samples
    and gathers only new leaves (ctx_regather); forcing full gathers
    (OCTF_FULL_GATHER=1) must give the same trajectory bit for bit."""
    from paper_1608_07411_b200 import fusion, scenes, volume
    sc = scenes.make_cfg3(d_max=6, n_views=8, width=160, height=120,
                          focal=131.25, device="cuda")
    p = fusion.FusionParams(**dict(sc.params, iterations=6))
    dom = volume.VolumeDomain(sc.origin, sc.voxel_size, sc.resolution)
    views, u0, _ = fusion.prepare(sc.depths, sc.cameras, dom, p)
    outs = []
    for full in ("0", "1"):
        monkeypatch.setenv("OCTF_FULL_GATHER", full)
        s = fusion.Solver(u0, views, p, precision="fp32")
        s.ctx.profile(True)
        s.run(0, 6)
        prof = s.ctx.profile(False)
        r = s.result()
        outs.append((r.field.to_host(), [(q.splits, q.joins) for q in r.stats],
                     prof))
        s.close()
    (a, sa, pa), (b, sb, pb) = outs
    assert sa == sb and sum(x + y for x, y in sa) > 0
    assert np.array_equal(a.child[:a.used], b.child[:b.used])
    assert np.array_equal(a.value[:a.used], b.value[:b.used])
    assert pa["gathers"] >= 2   # restructured passes were regathered


def test_cfg3_reduced_pd_with_restructure():
    """solver='pd' with split/join every pass on the reduced cfg3 scene
    against pd_oracle.c (unpinned definition): same per-pass splits/joins,
    child array and pool state, live values bit-exact in fp64."""
    from paper_1608_07411_b200 import fusion, scenes, volume
    sc = scenes.make_cfg3(d_max=6, n_views=8, width=160, height=120,
                          focal=131.25, device="cuda")
    kw = dict(sc.params, iterations=5)
    p = fusion.FusionParams(**kw)
    dom = volume.VolumeDomain(sc.origin, sc.voxel_size, sc.resolution)
    views, u0, _ = fusion.prepare(sc.depths, sc.cameras, dom, p)
    oviews, ou0 = oracle_prepare(sc, orc.Params(**kw))
    s = fusion.PDSolver(u0, views, p, precision="fp64")
    s.run(0, 5)
    u, ub, px, py, pz, en, child, state, sj = orc.pd_fuse(
        ou0, oviews, p.lam, p.gamma, 5, tau_split=p.tau_split,
        tau_join=p.tau_join, cap=s.u.capacity)
    assert [(st.splits, st.joins) for st in s.stats] == sj
    assert sum(a + b for a, b in sj) > 0
    assert list(s.u.state) == list(state)
    used = int(state[0])
    assert np.array_equal(s.u.child[:used].cpu().numpy(), child[:used])
    live = [n for n, *_ in orc.leaves(orc.Pool(np.zeros(used), child[:used],
                                                state, ou0.d_max))]
    got = [t[:used].cpu().numpy() for t in s.state]
    for g, w in zip(got, (u, ub, px, py, pz)):
        assert np.array_equal(g[live], w[:used][live])


class _ThreadComm:
    """In-process stand-in for torch.distributed between Python threads (one
    GPU, one process): mailboxes for send/recv, a shared slot + barrier for
    broadcast.  No kernel waits on another rank's kernel."""

    def __init__(self, rank, world, box):
        self.rank, self.world, self.box = rank, world, box

    def send(self, t, dst):
        self.box["q"][(self.rank, dst)].put(t.clone())

    def recv(self, t, src):
        t.copy_(self.box["q"][(src, self.rank)].get(timeout=120))

    def broadcast(self, t, src):
        b = self.box["bar"]
        if self.rank == src:
            self.box["slot"] = t.clone()
        b.wait()
        if self.rank != src:
            t.copy_(self.box["slot"])
        b.wait()


def test_frame_split_prepare_equals_single_gpu():
    """fusion.prepare with the frames split over 3 ranks (threads on one GPU,
    in-process mailboxes): views, u0 and seen equal the single-GPU prepare
    bit for bit on every rank."""
    import queue
    import threading
    from paper_1608_07411_b200 import fusion, scenes, volume
    sc = scenes.make_cfg3(d_max=6, n_views=7, width=160, height=120,
                          focal=131.25, device="cuda")
    p = fusion.FusionParams(**dict(sc.params, iterations=1))
    dom = volume.VolumeDomain(sc.origin, sc.voxel_size, sc.resolution)
    ref_views, ref_u0, ref_seen = fusion.prepare(sc.depths, sc.cameras, dom, p)
    world = 3
    box = {"q": {(a, b): queue.Queue() for a in range(world)
                 for b in range(world)},
           "bar": threading.Barrier(world), "slot": None}
    out, errs = [None] * world, []

    def run(r):
        try:
            torch.cuda.set_device(0)
            out[r] = fusion.prepare(sc.depths, sc.cameras, dom, p,
                                    comm=_ThreadComm(r, world, box))
            torch.cuda.synchronize()
        except Exception as exc:          # pragma: no cover - reported below
            errs.append(exc)
            box["bar"].abort()
    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not errs, errs
    hu = ref_u0.to_host()
    for views, u0, seen in out:
        assert torch.equal(seen, ref_seen)
        g = u0.to_host()
        assert np.array_equal(g.child[:g.used], hu.child[:hu.used])
        assert np.array_equal(g.value[:g.used], hu.value[:hu.used])
        for a, b in zip(views, ref_views):
            ah, bh = a.to_host(), b.to_host()
            assert np.array_equal(ah.child, bh.child)
            assert np.array_equal(ah.value, bh.value)
            assert np.array_equal(ah.weight, bh.weight)


def test_cfg3_many_views_ell_store_end_to_end():
    """40 views, ELL forced: the descent reads the ELL sample store (observed views only,
    per-tile rows) -- through restructuring passes (in-place list patches
    with warp-gathered new leaves) the fp64 pools equal the oracle's, and a
    forced full regather gives the same trajectory."""
    from paper_1608_07411_b200 import fusion, scenes, volume
    import os
    sc = scenes.make_cfg3(d_max=6, n_views=40, width=160, height=120,
                          focal=131.25, device="cuda")
    os.environ["OCTF_FORCE_ELL"] = "1"
    try:
        res, ref, _ = run_case(sc, 6)
    finally:
        del os.environ["OCTF_FORCE_ELL"]
    assert sum(s.splits + s.joins for s in ref.stats) > 0
    p = fusion.FusionParams(**dict(sc.params, iterations=6))
    dom = volume.VolumeDomain(sc.origin, sc.voxel_size, sc.resolution)
    views, u0, _ = fusion.prepare(sc.depths, sc.cameras, dom, p)
    s = fusion.Solver(u0, views, p, precision="fp32")
    s.ctx.set_options(2)               # ELL from 33 views
    s.run(0, 1)
    assert s.ctx.info()["ell"] == 1
    s.run(1, 5)
    a = s.result().field.to_host()
    s.close()
    os.environ["OCTF_FULL_GATHER"] = "1"
    try:
        s2 = fusion.Solver(u0, views, p, precision="fp32")
        s2.ctx.set_options(2)
        s2.run(0, 6)
        b = s2.result().field.to_host()
        s2.close()
    finally:
        del os.environ["OCTF_FULL_GATHER"]
    assert np.array_equal(a.child[:a.used], b.child[:b.used])
    assert np.array_equal(a.value[:a.used], b.value[:b.used])


@pytest.mark.parametrize("case", ["cfg1", "cfg3", "cfg4"])
def test_boxed_prepare_equals_dense(case):
    """fusion.prepare_boxed (the volume as eight octant boxes, no (2^d)^3
    grid: how BASELINE config 3 runs at depth 11) gives prepare's view
    trees and u0 bit for bit, and the observed-mask tree of w_sum > 0."""
    from paper_1608_07411_b200 import fusion, mesh, scenes, volume
    if case == "cfg1":
        sc = scenes.make_cfg1()
        depths, cams = sc.depths, sc.cameras
        p = fusion.FusionParams(delta=sc.delta, eta=sc.eta, lam=sc.lam)
        dom = volume.VolumeDomain(sc.origin, sc.voxel_size, sc.resolution)
    else:
        sc = (scenes.make_cfg3(d_max=7, n_views=12, width=320, height=240,
                               focal=262.5, device="cuda") if case == "cfg3"
              else scenes.make_cfg4(d_max=7, n_frames=12, width=320,
                                    height=240, focal=262.5, device="cuda"))
        depths, cams = sc.depths, sc.cameras
        p = fusion.FusionParams(**sc.params)
        dom = volume.VolumeDomain(sc.origin, sc.voxel_size, sc.resolution)
    views, u0, seen = fusion.prepare(depths, cams, dom, p)

    def same(a, b):
        ha, hb = a.to_host(), b.to_host()
        assert list(ha.state) == list(hb.state)
        assert np.array_equal(ha.child, hb.child)
        assert np.array_equal(ha.value, hb.value)
        if ha.weight is not None:
            assert np.array_equal(ha.weight, hb.weight)
    st = mesh.seen_tree(seen)
    d = dom.resolution.bit_length() - 1
    for bd in (d - 1, d - 2, d - 4):   # 8, 64 and 4096 boxes
        bviews, bu0, bseen = fusion.prepare_boxed(depths, cams, dom, p,
                                                  box_depth=bd)
        for a, b in zip(views, bviews):
            same(a, b)
        same(u0, bu0)
        same(st, bseen)


def test_trace_kernels_match_array_program():
    """The ray-marching kernels (octf_trace_blob / octf_trace_room) give the
    depth maps of the array program in scenes.py (torch ops on the device,
    which produced the maps the golden fixtures' reference runs consumed) bit
    for bit: hits, misses and the bisected depths.  (On the CPU torch's
    vectorised f64 sqrt is not correctly rounded, so the comparison is made
    on the device, where it is.)"""
    from paper_1608_07411_b200 import scenes
    # blob: an off-centre camera so part of the image misses
    tabs = [scenes._lattice(3 * 7 + o, 4 * (1 << o) + 2, "cuda")
            for o in range(3)]
    c = torch.tensor([0.5, 0.5, 0.5], dtype=torch.float64, device="cuda")

    def blob(p):
        return scenes._norm3(p - c) - (0.35 + 0.03 * scenes.value_noise(
            p, tabs))

    centre = np.array([0.5, 0.5, 0.5])
    for k, dvec in enumerate(scenes.fibonacci_hemisphere(5)[::2]):
        pos = centre + 1.2 * dvec
        cam = scenes.PinholeCamera(80.0, 80.0, 47.5, 31.5, 96, 64,
                                   scenes.look_at(pos, centre + 0.2 * k), pos)
        want = scenes.sphere_trace(blob, cam, lipschitz=1.7, t_max=3.0,
                                   device="cuda").cpu().numpy()
        got = scenes.trace_blob(cam, tabs, lipschitz=1.7,
                                t_max=3.0).cpu().numpy()
        assert (want > 0).any() and (want == 0).any()
        assert np.array_equal(got, want)
    # room: boxes, spheres and walls
    objs = scenes._room_objects(5, 40, 4.0)
    room = scenes.room_sdf_fn(objs, "cuda", 4.0)
    arr, nb, ns = scenes.room_objects_array(objs, "cuda")
    rng = np.random.default_rng(1)
    done = 0
    while done < 3:
        pos = rng.uniform(0.4, 3.6, 3)
        if float(room(torch.tensor(pos[None], device="cuda"))[0]) < 0.2:
            continue
        cam = scenes.PinholeCamera(70.0, 70.0, 47.5, 31.5, 96, 64,
                                   scenes.look_at(pos, rng.uniform(0, 4, 3)),
                                   pos)
        want = scenes.sphere_trace(room, cam, lipschitz=1.0, t_max=8.0,
                                   device="cuda", eps=1e-6).cpu().numpy()
        got = scenes.trace_room(cam, arr, nb, ns, size=4.0, lipschitz=1.0,
                                t_max=8.0, eps=1e-6).cpu().numpy()
        assert (want > 0).any()
        assert np.array_equal(got, want)
        done += 1


def test_trace_kernels_against_closed_forms():
    """Edge cases of the ray marcher with known answers: a blob without
    noise octaves is a sphere (the exact ray/sphere depth of
    scenes.sphere_depth, reference synth.py:80-109, to the bisection's
    resolution; same hit mask), and a room without objects is its six walls
    (depth of the wall the ray meets)."""
    from paper_1608_07411_b200 import scenes
    centre = np.array([0.5, 0.5, 0.5])
    pos = centre + 1.2 * np.array([0.3, -0.5, 0.81])
    cam = scenes.PinholeCamera(90.0, 90.0, 47.5, 31.5, 96, 64,
                               scenes.look_at(pos, centre), pos)
    empty = [torch.zeros((2, 2, 2), dtype=torch.float64, device="cuda")]
    got = scenes.trace_blob(cam, empty, amp=0.0, lipschitz=1.0,
                            t_max=3.0).cpu().numpy()
    want = scenes.sphere_depth(cam, centre, 0.35)
    # (sphere tracing stops 1e-7 off the surface: a ray grazing the limb
    # stops up to sqrt(2 R 1e-7) early or misses; compare where both hit,
    # and require the masks to agree but for a thin rim)
    both = (got > 0) & (want > 0)
    assert both.sum() > 500
    err = np.abs(got[both] - want[both])
    assert np.quantile(err, 0.99) < 1e-5 and err.max() < 2e-3
    assert ((got > 0) != (want > 0)).sum() <= 0.02 * both.sum()
    # walls only: from an interior point every ray hits a wall
    size = 4.0
    p0 = np.array([1.0, 2.5, 1.5])
    cam = scenes.PinholeCamera(70.0, 70.0, 47.5, 31.5, 96, 64,
                               scenes.look_at(p0, np.array([3.5, 0.5, 2.0])),
                               p0)
    objs = torch.zeros(1, dtype=torch.float64, device="cuda")
    z = scenes.trace_room(cam, objs, 0, 0, size=size, lipschitz=1.0,
                          t_max=8.0, eps=1e-6).cpu().numpy()
    R = np.asarray(cam.rotation)
    px = (np.arange(96) - cam.cx) / cam.fx
    py = (np.arange(64) - cam.cy) / cam.fy
    d = (R[:, 0][None, None, :] * px[None, :, None]
         + R[:, 1][None, None, :] * py[:, None, None] + R[:, 2][None, None, :])
    with np.errstate(divide="ignore", invalid="ignore"):
        t_hi = np.where(d > 0, (size - p0) / d, np.inf)
        t_lo = np.where(d < 0, (0.0 - p0) / d, np.inf)
    t_wall = np.minimum(t_hi, t_lo).min(axis=2)
    assert (z > 0).all()
    err = np.abs(z - t_wall)
    assert np.quantile(err, 0.99) < 1e-5 and err.max() < 1e-3
