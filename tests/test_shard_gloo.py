"""Multi-rank sharding on CPU: world_size 2 (and 3) over gloo.

Each rank owns a Morton range of subtrees (paper_1608_07411_b200.shard).  To
test the decomposition without a GPU, every rank runs the CPU oracle's pass
over its replicated pool, then *forgets* every value it does not own (NaN),
receives its halo over gloo and recomputes the replicated top.  If the plan
is right, the next pass's owned leaves read only owned/halo/top values, so
after K passes the owned leaves equal the single-process result bit for bit
(and any missing halo entry shows up as a NaN)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as orc
from paper_1608_07411_b200 import shard

K_PASSES = 4


def scene(seed=7, d=5, nviews=3):
    rng = np.random.default_rng(seed)
    n = 1 << d
    views = []
    for _ in range(nviews):
        f = (rng.integers(-2, 3, (n, n, n)) * 0.45).astype(np.float32)
        w = (rng.random((n, n, n)) < 0.8).astype(np.uint8)
        f[w == 0] = -1.0
        views.append(orc.build_octree(f, w, tau=0.3, dtype=np.float32))
    g = rng.integers(0, 3, (n, n, n)).astype(np.float64) * 0.3 - 0.3
    u0 = orc.build_octree(g, tau=0.2)        # mixed leaf depths
    p = orc.Params(iterations=K_PASSES, tau_split=0.0, tau_join=1.5, lam=0.4)
    return u0, views, p


def top_propagate(u, plan_):
    """Recompute the replicated inner nodes above the partition level
    (sequential child sums, _kernels.pyx:104-110)."""
    st = shard.structure(u.child, u.d_max, u.used)
    for L in range(plan_.k - 1, -1, -1):
        nodes = np.nonzero((st.level == L) & (u.child[:u.used] >= 0))[0]
        for n in nodes:
            b = u.child[n]
            acc = 0.0
            for c in range(8):
                acc += u.value[b + c]
            u.value[n] = acc / 8.0


def run_pass(u, views, p, t):
    vv = [v.value for v in views]
    vw = [v.weight for v in views]
    vc = [v.child for v in views]
    orc.iterate_pass(u.value, u.snap, u.child, u.joined, u.state, vv, vw, vc,
                     u.d_max, p.lam, p.eps, p.gamma, orc.step_scale(t, p),
                     p.tau_split, p.tau_join, p.clamp, False, None)
    orc.propagate(u.value, u.child)


def worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        u0, views, p = scene()
        u = orc.solver_pool(u0, cap=u0.used)
        pl = shard.plan(u.child, u.d_max, world, used=u.used, k=2)
        ex = shard.HaloExchange(pl, rank, torch.device("cpu"), torch.float64)
        owned = pl.owner[:u.used] == rank
        top = (pl.owner[:u.used] < 0)
        vals = torch.from_numpy(u.value)       # shares memory with the pool
        for t in range(p.iterations):
            run_pass(u, views, p, t)
            keep = owned | top
            u.value[:u.used][~keep] = np.nan
            ex.exchange(vals[:u.used])
            top_propagate(u, pl)
        leaves = np.nonzero(u.child[:u.used] < 0)[0]
        mine = leaves[owned[leaves]]
        q.put((rank, mine, u.value[mine].copy(), pl.leaves_per_rank))
    finally:
        dist.destroy_process_group()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def scatter_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        u0, _, _ = scene()
        u = orc.solver_pool(u0, cap=u0.used)
        full = shard.plan(u.child, u.d_max, world, used=u.used, k=2)
        got = shard.plan_scattered(u.child if rank == 0 else None, u.d_max,
                                   world, rank, used=u.used, k=2)
        ok = (np.array_equal(got.sel[rank], full.sel[rank])
              and np.array_equal(got.masks[rank], full.masks[rank])
              and np.array_equal(got.halo[rank], full.halo[rank])
              and got.interior_tiles == full.interior_tiles
              and got.top_levels == full.top_levels
              and np.array_equal(got.leaves_per_rank, full.leaves_per_rank)
              and set(got.send) == {k for k in full.send if rank in k}
              and all(np.array_equal(got.send[k], full.send[k])
                      for k in got.send)
              and all(got.sel[r].size == 0 for r in range(world) if r != rank))
        # the exchange built from the received part works as from the full plan
        shard.HaloExchange(got, rank, torch.device("cpu"), torch.float64)
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


def test_plan_scattered_gives_each_rank_its_part():
    """bench.py --gpus N: the plan is built on rank 0 only and every rank
    receives exactly its own leaf blocks, masks, halo and send lists."""
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=scatter_worker, args=(r, world, port, q))
             for r in range(world)]
    for pr in procs:
        pr.start()
    out = dict(q.get(timeout=300) for _ in procs)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert out == {0: True, 1: True, 2: True}


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_passes_match_single_process(world):
    u0, views, p = scene()
    ref = orc.fuse(u0, views, p).field
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, q))
             for r in range(world)]
    for pr in procs:
        pr.start()
    out = [q.get(timeout=300) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    covered = []
    for rank, mine, vals, counts in out:
        assert np.all(np.isfinite(vals)), f"rank {rank} read a missing halo value"
        assert np.array_equal(vals, ref.value[mine])
        covered.append(mine)
        assert counts.min() > 0
    allv = np.sort(np.concatenate(covered))
    leaves = np.nonzero(ref.child[:ref.used] < 0)[0]
    assert np.array_equal(allv, leaves)      # every leaf owned exactly once


def test_plan_is_balanced_and_disjoint():
    u0, _, _ = scene(d=6)
    pl = shard.plan(u0.child, u0.d_max, 4, used=u0.used)
    leaves = np.nonzero(u0.child < 0)[0]
    own = pl.owner[leaves]
    assert (own >= 0).all()
    counts = np.bincount(own, minlength=4)
    assert counts.max() <= 1.5 * counts.mean()
    # selected leaf blocks' masks cover each owned leaf once
    st = shard.structure(u0.child, u0.d_max)
    total = sum(int(np.unpackbits(m[:, None], axis=1).sum()) for m in pl.masks)
    assert total == leaves.size
    # halo never contains own or top nodes
    for r in range(4):
        h = pl.halo[r]
        assert (pl.owner[h] != r).all() and (pl.owner[h] >= 0).all()


def test_host_tables_match_reference_descent():
    """shard.structure's neighbour tables == root descents of the oracle."""
    u0, _, _ = scene(d=4)
    st = shard.structure(u0.child, u0.d_max)
    child = u0.child
    for i, b in enumerate(st.lblocks):
        if b == 0:
            continue
        L = int(st.level[b])
        par = st.parent[b]
        for d in range(12):
            qx, qy, qz = (st.x[par] + shard.DIRS[d, 0], st.y[par] + shard.DIRS[d, 1],
                          st.z[par] + shard.DIRS[d, 2])
            m = 1 << (L - 1)
            if not (0 <= qx < m and 0 <= qy < m and 0 <= qz < m):
                assert st.nbr[i, d] == -1
                continue
            node, lvl = 0, 0
            while lvl < L - 1 and child[node] >= 0:
                s = L - 1 - lvl - 1
                node = child[node] + ((((qx >> s) & 1) << 2) | (((qy >> s) & 1) << 1)
                                      | ((qz >> s) & 1))
                lvl += 1
            want = child[node] if (lvl == L - 1 and child[node] >= 0) else -node - 2
            assert st.nbr[i, d] == want


def test_plan_interior_and_boundary_ranges():
    """The plan orders each rank's leaf blocks interior-first: blocks in the
    leading interior tiles read (own slots, neighbour blocks, coarse
    neighbours) only nodes the rank computes itself; the padding to a whole
    tile is -1 with an empty mask; every owned leaf appears exactly once."""
    u0, views, p = scene()
    st = shard.structure(u0.child, u0.d_max, u0.used)
    for world in (2, 3):
        pl = shard.plan(u0.child, u0.d_max, world, used=u0.used, k=2)
        seen = np.zeros(u0.used, dtype=int)
        for r in range(world):
            sel, msk, ti = pl.sel[r], pl.masks[r], pl.interior_tiles[r]
            assert sel.size == msk.size and ti * 32 <= sel.size
            pad = sel < 0
            assert not msk[pad].any()
            for j, (i, m) in enumerate(zip(sel, msk)):
                if i < 0:
                    continue
                b = int(st.lblocks[i])
                for c in range(8):
                    if (m >> c) & 1:
                        seen[b + c] += 1
                        assert pl.owner[b + c] == r
                if j < ti * 32:          # interior: every read is owned
                    reads = [b + c for c in range(8) if b != 0 or c == 0]
                    for ref in st.nbr[i]:
                        if ref >= 0:
                            reads += [int(ref) + c for c in range(8)]
                        elif ref <= -2:
                            reads.append(int(-ref - 2))
                    assert all(pl.owner[x] == r for x in reads)
        leaves = np.nonzero(u0.child[:u0.used] < 0)[0]
        assert (seen[leaves] == 1).all()


def test_halo_exchange_start_complete_equals_exchange():
    world = 2
    port = free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_start_complete_worker, args=(r, world, port, q))
             for r in range(world)]
    for pr in procs:
        pr.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
    assert all(ok for _, ok in out)


def _start_complete_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        u0, views, p = scene()
        pl = shard.plan(u0.child, u0.d_max, world, used=u0.used, k=2)
        ex = shard.HaloExchange(pl, rank, torch.device("cpu"), torch.float64)
        base = torch.arange(u0.used, dtype=torch.float64)
        owned = torch.from_numpy(pl.owner[:u0.used] == rank)
        a = torch.where(owned, base, torch.full_like(base, -7.0))
        b = a.clone()
        ex.exchange(a)
        works = ex.start(b)
        b.mul_(1.0)                 # work between post and completion
        ex.complete(works, b)
        halo = torch.as_tensor(pl.halo[rank], dtype=torch.int64)
        ok = torch.equal(a, b) and torch.equal(a[halo], base[halo])
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


# ---------------------------------------------------- frame-split TSDF ----

def _oracle_backend(depths, cams, origin, vox, n, p):
    def build(k):
        f, w = orc.build_view_tsdf(depths[k], cams[k], origin, vox, n, p.delta,
                                   p.eta)
        return (torch.from_numpy(f), torch.from_numpy(w),
                orc.build_octree(f, w, tau=p.tau, dtype=np.float32))

    def grid():
        return torch.zeros((n, n, n), dtype=torch.float64)

    def accumulate(wf, ws, f, w):
        wf.add_(f.double() * w.double())
        ws.add_(w.double())

    def pack(t):
        meta = torch.tensor([t.value.shape[0], *[int(s) for s in t.state],
                             t.d_max, 0, 0, 0], dtype=torch.int64)
        return meta, [torch.from_numpy(np.ascontiguousarray(t.value)),
                      torch.from_numpy(np.ascontiguousarray(t.weight)),
                      torch.from_numpy(np.ascontiguousarray(t.child))]

    def unpack(meta):
        cap, s0, s1, s2, d = (int(x) for x in meta[:5].tolist())
        arrays = [torch.zeros(cap, dtype=torch.float32),
                  torch.zeros(cap, dtype=torch.float32),
                  torch.zeros(cap, dtype=torch.int32)]

        def finish(a):
            return orc.Pool(a[0].numpy(), a[2].numpy(),
                            np.array([s0, s1, s2], np.int64), d,
                            weight=a[1].numpy())
        return arrays, finish
    return build, grid, accumulate, pack, unpack


def _frame_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1608_07411_b200 import fusion
        from tests.goldens import cfg1_inputs
        depths, cams, origin, vox, n, p = cfg1_inputs()
        be = _oracle_backend(depths, cams, origin, vox, n, p)
        trees, wf, ws = fusion.frame_split(len(depths), *be,
                                           fusion.TorchFrameComm())
        q.put((rank, wf.numpy(), ws.numpy(),
               [(t.value.copy(), t.weight.copy(), t.child.copy(),
                 t.state.copy()) for t in trees]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_frame_split_tsdf_matches_single_process(world):
    """Frames split in contiguous blocks across gloo ranks: the wf/w sums
    (accumulated in frame order along the ranks) and every view tree equal
    the single-process frame-order result bit for bit, on every rank."""
    from tests.goldens import cfg1_inputs
    depths, cams, origin, vox, n, p = cfg1_inputs()
    wf0 = np.zeros((n, n, n))
    ws0 = np.zeros((n, n, n))
    ref = []
    for d, c in zip(depths, cams):
        f, w = orc.build_view_tsdf(d, c, origin, vox, n, p.delta, p.eta)
        wf0 += f.astype(np.float64) * w
        ws0 += w
        ref.append(orc.build_octree(f, w, tau=p.tau, dtype=np.float32))
    port = free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_frame_worker, args=(r, world, port, q))
             for r in range(world)]
    for pr in procs:
        pr.start()
    out = [q.get(timeout=300) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
    for rank, wf, ws, trees in out:
        assert np.array_equal(wf, wf0) and np.array_equal(ws, ws0), rank
        assert len(trees) == len(ref)
        for (v, w, c, st), t in zip(trees, ref):
            used = int(t.state[0])
            assert np.array_equal(c[:used], t.child[:used])
            assert np.array_equal(v[:used], t.value[:used])
            assert np.array_equal(w[:used], t.weight[:used])
            assert list(st) == list(t.state)


# ------------------------------------------------ solver="pd" sharded ----

def pd_worker(rank, world, port, q):
    """As ``worker`` for the primal-dual mode: the five pd fields are
    forgotten off the rank's ownership, exchanged in one halo message per
    peer (HaloExchange, nfields=5) and their top recomputed."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        u0, views, p = scene()
        used = u0.used
        tau, sigma = orc.pd_steps(p.lam)
        pl = shard.plan(u0.child, u0.d_max, world, used=used, k=2)
        ex = shard.HaloExchange(pl, rank, torch.device("cpu"), torch.float64,
                                nfields=5)
        keep = (pl.owner[:used] == rank) | (pl.owner[:used] < 0)
        u = u0.value[:used].astype(np.float64)
        fields = [u, u.copy(), np.zeros(used), np.zeros(used), np.zeros(used)]
        child = u0.child[:used].copy()
        for _ in range(p.iterations):
            fields, _ = orc.pd_pass(fields, child, used, views, u0.d_max,
                                    p.lam, tau, sigma, p.gamma)
            for f in fields:
                f[~keep] = np.nan
            ex.exchange([torch.from_numpy(f) for f in fields])
            for f in fields:
                top_propagate(orc.Pool(f, child, u0.state, u0.d_max), pl)
        leaves = np.nonzero(child < 0)[0]
        mine = leaves[(pl.owner[leaves] == rank)]
        q.put((rank, mine, [f[mine].copy() for f in fields]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_pd_passes_match_single_process(world):
    u0, views, p = scene()
    want = orc.pd_fuse(u0, views, p.lam, p.gamma, p.iterations)[:5]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=pd_worker, args=(r, world, port, q))
             for r in range(world)]
    for pr in procs:
        pr.start()
    out = [q.get(timeout=300) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    covered = []
    for rank, mine, vals in out:
        for k in range(5):
            assert np.all(np.isfinite(vals[k])), (rank, k)
            assert np.array_equal(vals[k], want[k][mine]), (rank, k)
        covered.append(mine)
    leaves = np.nonzero(u0.child[:u0.used] < 0)[0]
    assert np.array_equal(np.sort(np.concatenate(covered)), leaves)
