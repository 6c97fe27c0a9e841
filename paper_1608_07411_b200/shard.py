"""Morton-range sharding of a fixed-structure octree across ranks
(SURVEY.md §8(e)).

Ownership is by subtree: the *units* are the nodes at a partition level k
(plus leaves above k).  Units are ordered by Morton key and cut into
contiguous runs of roughly equal leaf count, one run per rank; a rank owns
every node of its units' subtrees.  The few inner nodes above level k (the
*top*) are replicated: every rank recomputes them from the unit roots.

Per pass each rank updates the leaves it owns (the same leaf kernel over a
rank-local leaf-block list whose leaf masks keep only owned leaves),
propagates, then receives the *halo*: values of nodes its stencils read (or
the top recomputation needs) that other ranks own.  Per-node arithmetic does
not depend on the partition, so structure and values stay bit-identical to
a single GPU; only the order of the final energy sum changes.

This module is host-side numpy (plans are built once per structure) plus
the exchange itself, written against torch.distributed so the same code
runs over NCCL on GPUs and over gloo in the CPU tests.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

__all__ = ["Structure", "structure", "ShardPlan", "plan", "rank_view",
           "plan_scattered", "ShardedSolver",
           "ShardedPDSolver", "HaloExchange"]

# direction table of the 13-point stencil (octf_common.cuh dir_offset)
DIRS = np.array([[-1, 0, 0], [1, 0, 0], [0, -1, 0], [0, 1, 0], [0, 0, -1],
                 [0, 0, 1], [-1, 1, 0], [-1, 0, 1], [1, -1, 0], [0, -1, 1],
                 [1, 0, -1], [0, 1, -1]], dtype=np.int64)


def _spread3(v: np.ndarray) -> np.ndarray:
    v = v.astype(np.uint64) & np.uint64(0x1fffff)
    for shift, mask in ((32, 0x1f00000000ffff), (16, 0x1f0000ff0000ff),
                        (8, 0x100f00f00f00f00f), (4, 0x10c30c30c30c30c3),
                        (2, 0x1249249249249249)):
        v = (v | (v << np.uint64(shift))) & np.uint64(mask)
    return v


def morton(x, y, z) -> np.ndarray:
    """x-major Morton key (child index c = x<<2|y<<1|z at every level)."""
    return (_spread3(x) << np.uint64(2)) | (_spread3(y) << np.uint64(1)) | _spread3(z)


@dataclass
class Structure:
    """Per-node geometry of a reference-layout pool, and its leaf blocks."""
    d_max: int
    level: np.ndarray       # int8 per slot (-1: not a live node)
    x: np.ndarray
    y: np.ndarray
    z: np.ndarray
    parent: np.ndarray      # int64 per slot (-1 root / free)
    leaf: np.ndarray        # bool per slot
    lblocks: np.ndarray     # ascending base slots of blocks with >=1 leaf
    nbr: np.ndarray         # [nlb, 12] neighbour refs (csrc/ctx.cu encoding)


def structure(child: np.ndarray, d_max: int, used: int | None = None) -> Structure:
    """Level, cell, parent of every live node (top-down BFS) and the leaf
    blocks with their 12-entry neighbour tables -- the host restatement of
    ctx_prepare / k_leaf_tables (csrc/ctx.cu)."""
    child = np.asarray(child)
    n = child.shape[0] if used is None else used
    child = child[:n].astype(np.int64)
    level = np.full(n, -1, dtype=np.int8)
    x = np.zeros(n, dtype=np.int64)
    y = np.zeros(n, dtype=np.int64)
    z = np.zeros(n, dtype=np.int64)
    parent = np.full(n, -1, dtype=np.int64)
    level[0] = 0
    frontier = np.array([0], dtype=np.int64)
    for L in range(d_max):
        cb = child[frontier]
        inner = frontier[cb >= 0]
        if inner.size == 0:
            break
        base = child[inner]
        kids = (base[:, None] + np.arange(8)[None, :]).ravel()
        par = np.repeat(inner, 8)
        c = np.tile(np.arange(8), inner.size)
        level[kids] = L + 1
        parent[kids] = par
        x[kids] = 2 * x[par] + ((c >> 2) & 1)
        y[kids] = 2 * y[par] + ((c >> 1) & 1)
        z[kids] = 2 * z[par] + (c & 1)
        frontier = kids
    live = level >= 0
    leaf = live & (child < 0)
    # leaf blocks: base slots of blocks holding a leaf (root pseudo-block 0)
    lslots = np.nonzero(leaf)[0]
    bases = np.where(lslots == 0, 0, ((lslots - 1) & ~7) + 1)
    lblocks = np.unique(bases)
    nbr = _tables(child, level, x, y, z, parent, lblocks)
    return Structure(d_max, level, x, y, z, parent, leaf, lblocks, nbr)


def _descend(child, L, qx, qy, qz):
    node = np.zeros(qx.shape, dtype=np.int64)
    lvl = np.zeros(qx.shape, dtype=np.int64)
    for l in range(int(L.max()) if L.size else 0):
        go = (l < L) & (child[node] >= 0)
        if not go.any():
            break
        s = (L - l - 1).clip(min=0)
        sel = (((qx >> s) & 1) << 2) | (((qy >> s) & 1) << 1) | ((qz >> s) & 1)
        node = np.where(go, child[node] + sel, node)
        lvl = np.where(go, lvl + 1, lvl)
    return node, lvl


def _tables(child, level, x, y, z, parent, lblocks):
    nlb = lblocks.size
    nbr = np.full((nlb, 12), -1, dtype=np.int64)
    real = lblocks != 0
    b = lblocks[real]
    L = level[b].astype(np.int64)            # level of the block's nodes
    par = parent[b]
    px, py, pz = x[par], y[par], z[par]
    m = (1 << (L - 1))
    out = np.full((b.size, 12), -1, dtype=np.int64)
    for d in range(12):
        qx, qy, qz = px + DIRS[d, 0], py + DIRS[d, 1], pz + DIRS[d, 2]
        ok = (qx >= 0) & (qy >= 0) & (qz >= 0) & (qx < m) & (qy < m) & (qz < m)
        q, lq = _descend(child, np.where(ok, L - 1, 0), np.where(ok, qx, 0),
                         np.where(ok, qy, 0), np.where(ok, qz, 0))
        qb = child[q]
        ref = np.where((lq == L - 1) & (qb >= 0), qb, -q - 2)
        out[:, d] = np.where(ok, ref, -1)
    nbr[real] = out
    return nbr.astype(np.int32)


@dataclass
class ShardPlan:
    nranks: int
    k: int                      # partition level
    owner: np.ndarray           # per slot: owning rank, -1 top / not live
    leaves_per_rank: np.ndarray
    sel: list = field(default_factory=list)     # per rank: leaf-block indices
    masks: list = field(default_factory=list)   # per rank: owned-leaf masks (u8)
    halo: list = field(default_factory=list)    # per rank: slots to receive
    send: dict = field(default_factory=dict)    # (src, dst) -> slots
    top_levels: int = 0                         # propagate levels [0, k)
    # per rank: leading tiles of sel whose stencils read only values the
    # rank computes itself (interior); sel is ordered interior blocks, -1
    # padding to a whole tile, boundary blocks
    interior_tiles: list = field(default_factory=list)


def _unit_of(st: Structure, k: int) -> np.ndarray:
    """Unit (level-k ancestor, or the node itself if a leaf above k) of every
    live node; -1 for inner nodes above k (the replicated top)."""
    n = st.level.shape[0]
    unit = np.full(n, -1, dtype=np.int64)
    live = st.level >= 0
    lvl = st.level.astype(np.int64)
    atk = live & (lvl == k)
    unit[atk] = np.nonzero(atk)[0]
    shallow_leaf = st.leaf & (lvl < k)
    unit[shallow_leaf] = np.nonzero(shallow_leaf)[0]
    for L in range(k + 1, st.d_max + 1):          # inherit top-down
        at = np.nonzero(live & (lvl == L))[0]
        unit[at] = unit[st.parent[at]]
    return unit


def _interior(st: Structure, slots, valid, owner, idx, r, chunk=1 << 16):
    """Leaf blocks (indices into st.lblocks) whose stencil reads -- their own
    eight slots, the twelve neighbour blocks' slots, coarse neighbours --
    are all nodes rank r computes itself (no halo, no replicated top)."""
    out = np.zeros(idx.size, dtype=bool)
    for lo in range(0, idx.size, chunk):
        j = idx[lo:lo + chunk]
        refs = st.nbr[j].astype(np.int64)                       # (n, 12)
        same = np.where(refs[:, :, None] >= 0,
                        refs[:, :, None] + np.arange(8)[None, None, :], -1)
        coarse = np.where(refs <= -2, -refs - 2, -1)
        own = np.where(valid[j], slots[j], -1)
        reads = np.concatenate([own, same.reshape(len(j), -1), coarse], axis=1)
        ok = (reads < 0) | (owner[np.maximum(reads, 0)] == r)
        out[lo:lo + chunk] = ok.all(axis=1)
    return out


def plan(child, d_max: int, nranks: int, used: int | None = None,
         k: int | None = None, st: Structure | None = None) -> ShardPlan:
    st = st if st is not None else structure(child, d_max, used)
    if k is None:  # enough units to balance: ~64 per rank
        k = 0
        while k < d_max and 8 ** k < 64 * nranks:
            k += 1
    unit = _unit_of(st, k)
    n = st.level.shape[0]
    units = np.unique(unit[unit >= 0])
    lvl_u = st.level[units].astype(np.int64)
    shift = (st.d_max - lvl_u).astype(np.uint64) * np.uint64(3)
    key = morton(st.x[units], st.y[units], st.z[units]) << shift
    order = np.argsort(key, kind="stable")
    units = units[order]
    # leaves per unit
    leaf_slots = np.nonzero(st.leaf)[0]
    pos = np.empty(n, dtype=np.int64)
    pos[units] = np.arange(units.size)
    counts = np.bincount(pos[unit[leaf_slots]], minlength=units.size)
    cum = np.cumsum(counts)
    total = cum[-1] if cum.size else 0
    cuts = np.searchsorted(cum, (np.arange(1, nranks) * total) / nranks,
                           side="left")
    urank = np.zeros(units.size, dtype=np.int64)
    for r, cidx in enumerate(cuts):
        urank[cidx + 1:] = r + 1
    owner = np.full(n, -1, dtype=np.int64)
    has = unit >= 0
    owner[has] = urank[pos[unit[has]]]
    p = ShardPlan(nranks, k, owner, np.bincount(owner[leaf_slots],
                                                minlength=nranks), top_levels=k)
    # per-rank leaf blocks and owned masks
    lb = st.lblocks
    slots = np.where(lb[:, None] == 0, np.array([0] + [-1] * 7)[None, :],
                     lb[:, None] + np.arange(8)[None, :])
    valid = slots >= 0
    sl = np.where(valid, slots, 0)
    isleaf = valid & st.leaf[sl]
    for r in range(nranks):
        own = isleaf & (owner[sl] == r)
        m = (own * (1 << np.arange(8))[None, :]).sum(axis=1).astype(np.uint8)
        idx = np.nonzero(m)[0]
        inner = _interior(st, slots, valid, owner, idx, r)
        ii, bb = idx[inner], idx[~inner]
        pad = (-ii.size) % 32          # 32 leaf blocks = one 256-leaf tile
        sel = np.concatenate([ii, np.full(pad, -1), bb]).astype(np.int32)
        msk = np.concatenate([m[ii], np.zeros(pad, np.uint8), m[bb]])
        p.sel.append(sel)
        p.masks.append(msk.astype(np.uint8))
        p.interior_tiles.append((ii.size + pad) // 32)
    # halo: every slot the rank's stencils can read (whole neighbour blocks,
    # coarse leaves, all siblings of processed blocks) plus the unit roots
    # the top recomputation needs, minus what it owns
    top = (owner < 0) & (st.level >= 0)
    roots = units
    for r in range(nranks):
        idx = p.sel[r][p.sel[r] >= 0]
        need = [slots[idx][valid[idx]]]
        refs = st.nbr[idx].astype(np.int64).ravel()
        same = refs[refs >= 0]
        need.append((same[:, None] + np.arange(8)[None, :]).ravel())
        need.append(-refs[refs <= -2] - 2)
        need.append(roots)
        need = np.unique(np.concatenate(need))
        need = need[(owner[need] != r) & ~top[need]]
        p.halo.append(need)
        for q in range(nranks):
            if q != r:
                p.send[(q, r)] = need[owner[need] == q]
    return p


def rank_view(p: ShardPlan, rank: int) -> ShardPlan:
    """The part of a plan rank ``rank`` needs to run (its leaf blocks, masks,
    halo and the send lists it takes part in); the other ranks' entries are
    empty and ``owner`` is dropped."""
    e32, e8, e64 = (np.zeros(0, np.int32), np.zeros(0, np.uint8),
                    np.zeros(0, np.int64))
    only = lambda lst, e: [a if r == rank else e for r, a in enumerate(lst)]
    return ShardPlan(p.nranks, p.k, None, p.leaves_per_rank,
                     sel=only(p.sel, e32), masks=only(p.masks, e8),
                     halo=only(p.halo, e64),
                     send={k: v for k, v in p.send.items() if rank in k},
                     top_levels=p.top_levels,
                     interior_tiles=list(p.interior_tiles))


def plan_scattered(child, d_max: int, nranks: int, rank: int, *,
                   used: int | None = None, k: int | None = None, group=None,
                   src: int = 0) -> ShardPlan:
    """``plan`` built once, on rank ``src``, and each rank's ``rank_view`` sent
    to it (torch.distributed scatter): the planner's numpy tables of a
    100M-leaf tree take tens of GB of host memory and minutes of one core, so
    the ranks of a node must not all build them side by side.  ``child`` is
    only read on ``src``."""
    import torch.distributed as dist
    parts = None
    if rank == src:
        full = plan(child, d_max, nranks, used=used, k=k)
        parts = [rank_view(full, r) for r in range(nranks)]
        del full
    out = [None]
    dist.scatter_object_list(out, parts, src=src, group=group)
    return out[0]


class ShardedSolver:
    """Frozen-structure descent on one rank's shard.

    Every rank keeps the (cheap) pool replicated and updates only the leaves
    it owns: the context's leaf-block list is cut to the rank's blocks with
    owned-leaf masks before any sample is gathered (``defer``), so samples --
    the dominant memory -- are gathered and streamed for owned leaves only.
    Per pass: leaf kernel + propagate (``compute``), halo exchange of the
    post-pass values, recomputation of the replicated top (``finish``).
    Energies stay per rank on the device until ``energies()`` sums them.
    ``samples`` = per-slot sample arrays (BASELINE config 5) instead of views.
    """

    def __init__(self, u0, views, params, plan: ShardPlan, rank: int, *,
                 precision: str = "fp32", exchange=None, group=None,
                 samples=None):
        import torch
        from . import fusion
        if not (params.tau_split <= 0 and params.clamp and params.tau_join >= 1):
            raise ValueError("sharded solving needs a frozen structure "
                             "(tau_split <= 0, tau_join >= 1, clamp)")
        self.params = params
        self.plan = plan
        self.rank = rank
        self.group = group
        self.s = fusion.Solver(u0, views, params, precision=precision,
                               samples=samples, defer=True)
        s = self.s
        if samples is None:   # structure only (deferred gather)
            s.kern.ctx_prepare(s.ctx, s.u.child, s.u.state, s.u.d_max,
                               s.vvals, s.vws, s.vchilds)
        s.kern.ctx_select(s.ctx, plan.sel[rank], plan.masks[rank])
        self.tiles = s.ctx.info()["tiles"]
        self.exchange = exchange if exchange is not None else HaloExchange(
            plan, rank, s.u.value.device, s.u.value.dtype)
        self.e = torch.zeros(max(params.iterations, 1), dtype=torch.float64,
                             device=s.u.value.device)
        self.t = 0

    @property
    def values(self):
        """Buffer holding the latest values (after ``finish``)."""
        return self.s.cur

    def compute(self, t: int) -> None:
        from .fusion import step_scale
        s, p, u = self.s, self.params, self.s.u
        if t >= self.e.shape[0]:
            import torch
            self.e = torch.cat([self.e, torch.zeros_like(self.e)])
        s.kern.fuse_passes_frozen(s.cur, s.nxt, u.child, u.state, s.vvals,
                                  s.vws, s.vchilds, u.d_max, p.lam, p.eps,
                                  p.gamma, p.tau_split, p.tau_join, p.clamp,
                                  [step_scale(t, p)], ctx=s.ctx,
                                  energies_out=self.e[t:t + 1])
        self.t = t + 1

    def finish(self) -> None:
        s, u = self.s, self.s.u
        s.kern.propagate_levels(s.nxt, u.child, 0, self.plan.top_levels,
                                ctx=s.ctx)
        s.cur, s.nxt = s.nxt, s.cur

    def run(self, t0: int, k: int, overlap: bool = True) -> None:
        if not overlap:
            for t in range(t0, t0 + k):
                self.compute(t)
                self.exchange.exchange(self.s.nxt[:self.s.u.used], self.group)
                self.finish()
            return
        # overlapped: pass t's interior tiles run while the previous pass's
        # halo is in flight; same values as above
        for t in range(t0, t0 + k):
            works = self.exchange.start(self.s.cur[:self.s.u.used], self.group)
            self.interior(t)
            self.exchange.complete(works, self.s.cur[:self.s.u.used])
            self.boundary(t)
        self.flush()

    # ---- the overlapped pass in its three stages (driven by ``run``, or
    # in lock-step by a single-GPU test)
    def interior(self, t: int) -> None:
        """Leaf tiles whose stencils read only this rank's values: may run
        before the previous pass's halo has arrived."""
        from .fusion import step_scale
        s, p, u = self.s, self.params, self.s.u
        ti = self.plan.interior_tiles[self.rank]
        if ti:
            s.kern.pass_tiles(s.cur, s.nxt, u.child, u.state, s.vvals, s.vws,
                              s.vchilds, u.d_max, p.lam, p.eps, p.gamma,
                              step_scale(t, p), p.clamp, 0, ti, ctx=s.ctx)

    def boundary(self, t: int) -> None:
        """After the halo of the previous pass is in ``cur``: recompute the
        replicated top, update the remaining tiles, propagate, energy."""
        import torch
        from .fusion import step_scale
        s, p, u = self.s, self.params, self.s.u
        s.kern.propagate_levels(s.cur, u.child, 0, self.plan.top_levels,
                                ctx=s.ctx)
        ti = self.plan.interior_tiles[self.rank]
        nt = self.tiles - ti
        if nt:
            s.kern.pass_tiles(s.cur, s.nxt, u.child, u.state, s.vvals, s.vws,
                              s.vchilds, u.d_max, p.lam, p.eps, p.gamma,
                              step_scale(t, p), p.clamp, ti, nt, ctx=s.ctx)
        if t >= self.e.shape[0]:
            self.e = torch.cat([self.e, torch.zeros_like(self.e)])
        s.kern.pass_finish(s.nxt, u.child, self.e[t:t + 1], ctx=s.ctx)
        s.cur, s.nxt = s.nxt, s.cur
        self.t = t + 1

    def flush(self) -> None:
        """Exchange and top recomputation after the last overlapped pass, so
        ``values`` holds the halo and top of the final state."""
        s, u = self.s, self.s.u
        self.exchange.exchange(s.cur[:u.used], self.group)
        s.kern.propagate_levels(s.cur, u.child, 0, self.plan.top_levels,
                                ctx=s.ctx)

    def energies(self, reduce: bool = True):
        """Energy before each pass run so far, summed over ranks."""
        import torch.distributed as dist
        e = self.e[:self.t].clone()
        if reduce and dist.is_available() and dist.is_initialized():
            dist.all_reduce(e, group=self.group)
        return e

    def close(self):
        self.s.close()


class ShardedPDSolver:
    """The north_star's TV-L1 primal-dual iteration (solver='pd') on one
    rank's shard of a frozen tree: the same ownership, leaf-block selection
    and halo as ``ShardedSolver``, with the five pd fields (u, ubar, px, py,
    pz) exchanged and their replicated top recomputed.  Per pass: pd kernel
    + propagate of the five fields over the rank's leaves, halo exchange,
    top.  Values equal the single-GPU PDSolver bit for bit (per-node
    arithmetic does not depend on the partition)."""

    def __init__(self, u0, views, params, plan: ShardPlan, rank: int, *,
                 precision: str = "fp32", exchange=None, group=None,
                 samples=None):
        import torch
        from . import fusion
        if not (params.tau_split <= 0 and params.clamp and params.tau_join >= 1):
            raise ValueError("sharded solving needs a frozen structure "
                             "(tau_split <= 0, tau_join >= 1, clamp)")
        self.params = params
        self.plan = plan
        self.rank = rank
        self.group = group
        self.s = fusion.PDSolver(u0, views, params, precision=precision,
                                 samples=samples, defer=True)
        s = self.s
        if samples is None:
            s.kern.ctx_prepare(s.ctx, s.u.child, s.u.state, s.u.d_max,
                               s.vvals, s.vws, s.vchilds)
        s.kern.ctx_select(s.ctx, plan.sel[rank], plan.masks[rank])
        self.exchange = exchange if exchange is not None else HaloExchange(
            plan, rank, s.u.value.device, s.u.value.dtype, nfields=5)
        self.e = torch.zeros(max(params.iterations, 1), dtype=torch.float64,
                             device=s.u.value.device)
        self.t = 0

    @property
    def state(self):
        return self.s.state

    def compute(self, t: int) -> None:
        import torch
        s, p, u = self.s, self.params, self.s.u
        if t >= self.e.shape[0]:
            self.e = torch.cat([self.e, torch.zeros_like(self.e)])
        s.kern.pd_passes(s.a, s.b, u.child, u.state, s.vvals, s.vws,
                         s.vchilds, u.d_max, p.lam, s.tau, s.sigma, p.gamma,
                         p.clamp, 1, ctx=s.ctx, energies_out=self.e[t:t + 1])
        s.a, s.b = s.b, s.a
        self.t = t + 1

    def finish(self) -> None:
        s, u = self.s, self.s.u
        for f in s.a:
            s.kern.propagate_levels(f, u.child, 0, self.plan.top_levels,
                                    ctx=s.ctx)

    def run(self, t0: int, k: int) -> None:
        used = self.s.u.used
        for t in range(t0, t0 + k):
            self.compute(t)
            self.exchange.exchange([f[:used] for f in self.s.a], self.group)
            self.finish()

    def energies(self, reduce: bool = True):
        import torch.distributed as dist
        e = self.e[:self.t].clone()
        if reduce and dist.is_available() and dist.is_initialized():
            dist.all_reduce(e, group=self.group)
        return e

    def close(self):
        self.s.close()


class HaloExchange:
    """Per-pass exchange of owned values into the other ranks' halos
    (torch.distributed point-to-point; NCCL on GPUs, gloo on CPU).  One
    message per peer carries every field (``nfields``: 1 for the descent, 5
    for pd), packed field-major.  On CUDA tensors the staging is the
    library's gather/scatter kernel (``octf_halo_pack``); CPU tensors (the
    gloo tests) use torch indexing."""

    def __init__(self, plan: ShardPlan, rank: int, device, dtype,
                 nfields: int = 1):
        import torch
        self.rank = rank
        self.nranks = plan.nranks
        self.nfields = nfields
        self.cuda = torch.device(device).type == "cuda"
        itype = torch.int32 if self.cuda else torch.int64
        self.sends = {}
        self.recvs = {}
        for q in range(plan.nranks):
            if q == rank:
                continue
            s = plan.send.get((rank, q))
            r = plan.send.get((q, rank))
            if s is not None and s.size:
                idx = torch.as_tensor(s, dtype=itype, device=device)
                self.sends[q] = (idx, torch.empty(nfields * s.size, dtype=dtype,
                                                  device=device))
            if r is not None and r.size:
                idx = torch.as_tensor(r, dtype=itype, device=device)
                self.recvs[q] = (idx, torch.empty(nfields * r.size, dtype=dtype,
                                                  device=device))

    def _fields(self, values):
        fields = list(values) if isinstance(values, (list, tuple)) else [values]
        if len(fields) != self.nfields:
            raise ValueError(f"expected {self.nfields} fields")
        return fields

    def _stage(self, fields, idx, buf, unpack):
        import torch
        if self.cuda:
            from . import _kernels
            _kernels.halo_pack(fields, idx, buf, unpack=unpack)
            return
        n = idx.shape[0]
        for k, f in enumerate(fields):
            if unpack:
                f.index_copy_(0, idx, buf[k * n:(k + 1) * n])
            else:
                torch.index_select(f, 0, idx, out=buf[k * n:(k + 1) * n])

    def start(self, values, group=None):
        """Post the sends of this rank's values and the receives of its halo;
        returns the pending works (with NCCL the transfer runs on its own
        stream, concurrent with kernels launched next)."""
        import torch.distributed as dist
        fields = self._fields(values)
        ops = []
        for q, (idx, buf) in self.sends.items():
            self._stage(fields, idx, buf, False)
            ops.append(dist.P2POp(dist.isend, buf, q, group))
        for q, (idx, buf) in self.recvs.items():
            ops.append(dist.P2POp(dist.irecv, buf, q, group))
        return dist.batch_isend_irecv(ops) if ops else []

    def complete(self, works, values):
        """Wait for ``start``'s works (device-side for NCCL) and scatter the
        received halo into ``values``."""
        fields = self._fields(values)
        for w in works:
            w.wait()
        for q, (idx, buf) in self.recvs.items():
            self._stage(fields, idx, buf, True)

    def exchange(self, values, group=None):
        self.complete(self.start(values, group), values)
