"""Variational fusion of per-view truncated signed distances on the GPU
(reference ``fusion.py``).

Same energy, schedule and restructuring as the reference: Jacobi descent on
a smoothed-L1 data term plus smoothed total variation, with in-pass leaf
splits near the zero crossing and joins of saturated constant-sign subtrees
(reference fusion.py:1-16, _kernels.pyx:256-381).  Two precisions:

``precision="fp64"`` (default) -- the parity mode: pools, statistics and the
    join log are bit-identical to the reference's compiled kernels (energies
    up to the order of the final sum).
``precision="fp32"`` -- the throughput mode: fp32 iterate and arithmetic
    (the north_star's "u within 1e-4").

The iterate stays in HBM for the whole schedule; the two value buffers
alternate roles each pass (pass-start snapshot / post-pass values), so the
reference's per-pass snapshot copy (_kernels.pyx:390-393) costs nothing.
"""

from __future__ import annotations

import os
import time
from dataclasses import dataclass, field as dc_field

import numpy as np
import torch

from . import _backend, _lib
from ._device import as_device, device, pool_empty, ptr, stream_handle, to_numpy
from .octree import OctreeField, build_octree, full_tree_capacity

__all__ = [
    "prepare_boxed",
    "FusionParams",
    "IterationStats",
    "FuseResult",
    "step_scale",
    "build_view_tree",
    "view_arrays",
    "initial_field",
    "prepare",
    "FrameComm",
    "TorchFrameComm",
    "frame_split",
    "fuse",
    "Solver",
    "tree_energy",
    "write_report",
    "dense_fuse",
    "dense_step",
    "dense_energy",
    "data_term_value",
    "data_term_derivative",
    "smoothness_value",
    "smoothness_flux",
    "read_report",
]


@dataclass(frozen=True)
class FusionParams:
    """Energy weights, descent schedule and restructuring thresholds
    (reference fusion.py:51-92, same defaults and validation)."""

    delta: float = 0.004
    eta: float = 0.02
    lam: float = 0.3
    eps: float = 0.25
    gamma: float = 1e-4
    xi0: float = 0.1
    halve_every: int = 20
    iterations: int = 100
    tau: float = 0.1
    tau_split: float = 0.1
    tau_join: float = 0.5
    clamp: bool = True

    def __post_init__(self):
        if self.delta <= 0 or self.eta <= 0:
            raise ValueError("delta and eta must be positive")
        if self.eta < self.delta:
            raise ValueError("eta must not be smaller than delta")
        for name in ("lam", "eps", "gamma", "xi0"):
            if getattr(self, name) <= 0:
                raise ValueError(f"{name} must be positive")
        if self.halve_every < 1 or self.iterations < 0:
            raise ValueError("bad schedule")
        if self.tau_split < 0:
            raise ValueError("tau_split must be non-negative")
        if self.tau_split >= self.tau_join:
            raise ValueError("tau_split must be smaller than tau_join")


@dataclass
class IterationStats:
    iteration: int
    energy: float
    node_count: int
    memory_bytes: int
    splits: int
    joins: int
    wall_ms: float


@dataclass
class FuseResult:
    field: OctreeField
    stats: list = dc_field(default_factory=list)
    join_log: np.ndarray | None = None

    @property
    def mem_peak_bytes(self) -> int:
        live = self.field.node_count * (self.field.value.element_size()
                                        + self.field.snap.element_size()
                                        + self.field.child.element_size())
        return max((s.memory_bytes for s in self.stats), default=live)

    @property
    def wall_ms(self) -> float:
        return sum(s.wall_ms for s in self.stats)


def step_scale(t: int, params: FusionParams) -> float:
    """Descent step of pass t (fusion.py:124-126)."""
    return params.xi0 * 2.0 ** (-(t // params.halve_every))


# -- view preparation --------------------------------------------------------

def build_view_tree(view, tau: float = 0.1) -> OctreeField:
    """Compress one view's distance/weight grids into a float32 octree
    (fusion.py:131-137), on the GPU."""
    return build_octree(view.f, view.w, tau=tau, dtype=np.float32)


def view_arrays(views) -> tuple[list, list, list]:
    for v in views:
        if v.weight is None:
            raise ValueError("view trees must carry weights")
    return ([v.value for v in views], [v.weight for v in views],
            [v.child for v in views])


def initial_field(wf_sum, w_sum, gamma: float):
    """Weighted mean of the view distances, -1 where unobserved
    (fusion.py:149-155).  numpy in -> numpy out; CUDA in -> CUDA out."""
    host = not isinstance(wf_sum, torch.Tensor)
    wf = as_device(wf_sum, torch.float64)
    ws = as_device(w_sum, torch.float64)
    if wf.shape != ws.shape:
        raise ValueError("wf_sum and w_sum shapes differ")
    out = torch.empty_like(wf)
    _lib.call("octf_initial_field", ptr(wf), ptr(ws), float(gamma), wf.numel(),
              ptr(out), stream_handle())
    return to_numpy(out) if host else out


def prepare(depths, cameras, dom, params: FusionParams, *, comm=None):
    """Depth maps -> (view trees, u0, seen): the pre-processing loop of the
    reference's ``cli.cmd_fuse`` (cli.py:141-171) on the GPU -- per view the
    TSDF with the wf/w sums accumulated in frame order, the view tree, then
    ``initial_field`` and ``build_octree(u0_grid, tau)``.  ``seen`` is the
    (N,N,N) bool grid w_sum > 0 the reference hands to its mesher.

    With ``comm`` (a :class:`FrameComm`, e.g. ``TorchFrameComm()`` over
    torch.distributed) the frames are split across ranks (north_star: "the
    per-frame TSDF integration is split across GPUs by frame"): rank r
    builds the TSDFs and view trees of a contiguous block of frames, the
    wf/w sums are accumulated in frame order along the ranks (each rank adds
    its frames to the partial sums of the ranks before it, so the result is
    the single-GPU sum bit for bit), and the view trees and final sums are
    broadcast -- every rank returns the same views, u0 and seen."""
    from .tsdf import build_view_tsdf
    n = dom.resolution
    if comm is None or comm.world == 1:
        wf = torch.zeros((n, n, n), dtype=torch.float64, device=device())
        ws = torch.zeros_like(wf)
        trees = []
        for img, cam in zip(depths, cameras):
            vt = build_view_tsdf(img, cam, dom, params.delta, params.eta,
                                 accumulate=(wf, ws))
            trees.append(build_view_tree(vt, params.tau))
            del vt
        u0 = build_octree(initial_field(wf, ws, params.gamma), tau=params.tau)
        return trees, u0, ws > 0

    def build(k):
        vt = build_view_tsdf(depths[k], cameras[k], dom, params.delta,
                             params.eta)
        return vt.f, vt.w, build_view_tree(vt, params.tau)

    def grid():
        return torch.zeros((n, n, n), dtype=torch.float64, device=device())

    def accumulate(wf, ws, f, w):
        # k_view_tsdf's accumulation, same IEEE operations:
        # wf += f64(f) * f64(w), ws += f64(w)
        wf.add_(f.double() * w.double())
        ws.add_(w.double())

    trees, wf, ws = frame_split(len(depths), build, grid, accumulate,
                                _tree_pack, _tree_unpack(device()), comm)
    u0 = build_octree(initial_field(wf, ws, params.gamma), tau=params.tau)
    return trees, u0, ws > 0


class _BoxTree:
    """One tree of a box-wise input stage (prepare_boxed): a growable
    reference-layout pool filled box subtree by box subtree
    (octf_build_octree_box), and the top levels above the boxes assembled
    from the box roots' pyramid entries.  Depth-first ranks (the
    reference's slot order: the block of the r-th splitting node, child 7
    expanded first, at slot 1 + 8r) are kept as a running count; a top node
    is opened as if it split, and if its assembled statistics say it does
    not, the count rolls back to its rank and its boxes' subtrees -- written
    past what the tree keeps -- are overwritten by later subtrees or lie
    beyond the final ``used``."""

    def __init__(self, d_max, weighted, dtype, cap=1 << 16):
        self.d, self.weighted, self.dtype = d_max, weighted, dtype
        self.cap = cap
        self.value = pool_empty(cap, dtype)
        self.child = pool_empty(cap, torch.int32)
        self.weight = pool_empty(cap, torch.float32) if weighted else None
        self.running = 0   # splitting nodes so far, in depth-first order
        self.stack = []    # open top nodes: [slot, rank, level, stats[8]]
        self.nsplit_root = 0

    def _grow(self, need=0):
        cap = max(2 * self.cap, need)

        def g(t):
            out = pool_empty(cap, t.dtype)
            out[:self.cap].copy_(t[:self.cap])
            return out
        self.value, self.child = g(self.value), g(self.child)
        if self.weight is not None:
            self.weight = g(self.weight)
        self.cap = cap

    def _child_slot(self, c):
        return 0 if not self.stack else 1 + 8 * self.stack[-1][1] + c

    def open(self, c, level):
        """A top node (child c of the current one; the root: c ignored)."""
        slot = self._child_slot(c)
        self.stack.append([slot, self.running, level, [None] * 8])
        self.running += 1
        if 1 + 8 * self.running > self.cap:
            self._grow(2 + 8 * self.running)

    def box(self, c, f, w, tau, propagate, level0):
        """The subtree of box c of the current top node from its grid."""
        d_box = self.d - level0
        ns = np.zeros(1, dtype=np.int64)
        st = np.zeros(8, dtype=np.float64)
        code = _lib.OCTF_F32 if self.dtype == torch.float32 else _lib.OCTF_F64
        slot = self._child_slot(c)
        while True:
            try:
                _lib.call("octf_build_octree_box", ptr(f),
                          _lib.OCTF_F32 if f.dtype == torch.float32
                          else _lib.OCTF_F64, ptr(w), d_box, level0, self.d,
                          float(tau), ptr(self.value), code, ptr(self.weight),
                          ptr(self.child), self.cap, self.running, slot,
                          1 if propagate else 0, ns.ctypes.data,
                          st.ctypes.data, stream_handle())
                break
            except RuntimeError as exc:
                if "capacity" not in str(exc):
                    raise
                self._grow()
        self.running += int(ns[0])
        if self.stack:
            self.stack[-1][3][c] = st
        return st, int(ns[0])

    def close(self, tau):
        """Assemble the current top node from its children's statistics
        (the pyramid's next level in numpy's order; the split rule,
        _kernels.pyx:58-63) and write it."""
        slot, rank, level, s = self.stack.pop()

        def mean8(k):
            b = [s[c][k] for c in range(8)]
            return ((((b[0] + b[1]) + (b[2] + b[3])) + (b[4] + b[5]))
                    + (b[6] + b[7])) / 8.0
        mn = min(q[0] for q in s)
        mx = max(q[1] for q in s)
        wmn = min(q[3] for q in s)
        wmx = max(q[4] for q in s)
        wm, wf, pl = mean8(5), mean8(6), mean8(7)
        if self.weighted:
            mean = wf / wm if wm > 0.0 else pl
            split = level < self.d and (mx - mn > tau or wmn != wmx)
        else:
            mean = mean8(2)
            split = level < self.d and mx - mn > tau
        st = np.array([mn, mx, mean, wmn, wmx, wm, wf, pl])
        if not split:
            self.running = rank        # drop the node and its subtrees
        self.child[slot] = 1 + 8 * rank if split else -1
        val = mean
        if split and not self.weighted:   # propagate_means: sequential sum
            acc = 0.0
            for v in self.value[1 + 8 * rank:9 + 8 * rank].double().tolist():
                acc += v
            val = acc / 8.0
            st[2] = mean            # (the pyramid entry stays the mean)
        self.value[slot] = val
        if self.weight is not None:
            self.weight[slot] = wm
        if self.stack:
            parent = self.stack[-1]
            parent[3][(slot - 1) % 8] = st
        return st

    def finish(self) -> OctreeField:
        used = 1 + 8 * self.running
        from .octree import _trim
        state = np.array([used, -1, used], dtype=np.int64)
        out = OctreeField(_trim(self.value, used), _trim(self.child, used),
                          state, self.d,
                          weight=None if self.weight is None
                          else _trim(self.weight, used))
        self.value = self.child = self.weight = None   # the grown pools
        return out


def prepare_boxed(depths, cameras, dom, params: FusionParams, *,
                  box_depth: int = 9):
    """``prepare`` without any (2^d)^3 grid: the volume is processed as
    boxes of (2^box_depth)^3 voxels in the depth-first order of the
    reference's build (child 7 first, _kernels.pyx:21-77): per box every
    frame's TSDF (octf_view_tsdf_box, with the box's wf / w sums in frame
    order) and its subtree of every view tree (octf_build_octree_box), then
    the box's initial field and its subtrees of u0 and of the observed-mask
    tree; the levels above the boxes are assembled from the box roots'
    pyramid entries.  The result is ``prepare``'s bit for bit (views, u0;
    ``seen`` as the tree mesh.seen_tree(w_sum > 0) would build), with one
    box's grids in memory -- BASELINE config 3's depth 11 (2048^3 cells)
    runs on one GPU."""
    n = dom.resolution
    d = n.bit_length() - 1
    bd = max(0, min(box_depth, d - 1))
    top = d - bd                 # levels assembled above the boxes (>= 1)
    h = 1 << bd
    from .tsdf import _camera_params
    org = np.ascontiguousarray(np.asarray(dom.origin, dtype=np.float64))
    views = [_BoxTree(d, True, torch.float32) for _ in depths]
    u0 = _BoxTree(d, False, torch.float64)
    seen = _BoxTree(d, False, torch.float64)
    trees = views + [u0, seen]
    dev = device()
    ds = [as_device(img.depth if hasattr(img, "depth") else img, torch.float32)
          for img in depths]
    cps = [np.ascontiguousarray(_camera_params(cam)) for cam in cameras]
    f = torch.empty((h, h, h), dtype=torch.float32, device=dev)
    w = torch.empty((h, h, h), dtype=torch.uint8, device=dev)

    def do_box(c, cell):
        box = np.array([cell[0] * h, cell[1] * h, cell[2] * h, h],
                       dtype=np.int32)
        wf = torch.zeros((h, h, h), dtype=torch.float64, device=dev)
        ws = torch.zeros_like(wf)
        for v in range(len(ds)):
            _lib.call("octf_view_tsdf_box", ptr(ds[v]), int(ds[v].shape[1]),
                      int(ds[v].shape[0]), cps[v].ctypes.data, org.ctypes.data,
                      float(dom.voxel_size), n, box.ctypes.data,
                      float(params.delta), float(params.eta), ptr(f), ptr(w),
                      ptr(wf), ptr(ws), stream_handle())
            views[v].box(c, f, w, params.tau, False, top)
        ub = initial_field(wf, ws, params.gamma)
        del wf
        u0.box(c, ub, None, params.tau, True, top)
        del ub
        seen.box(c, (ws > 0).double(), None, 0.0, True, top)

    def rec(level, c, cell):
        if level == top:
            do_box(c, cell)
            return
        for t in trees:
            t.open(c, level)
        for cc in range(7, -1, -1):
            rec(level + 1, cc, (2 * cell[0] + ((cc >> 2) & 1),
                                2 * cell[1] + ((cc >> 1) & 1),
                                2 * cell[2] + (cc & 1)))
        for t in trees:
            t.close(0.0 if t is seen else params.tau)

    rec(0, 0, (0, 0, 0))
    del rec          # (the recursive closure is a reference cycle)
    return [v.finish() for v in views], u0.finish(), seen.finish()


class FrameComm:
    """The point-to-point and broadcast operations ``frame_split`` needs
    (rank, world, send, recv, broadcast); see ``TorchFrameComm``."""
    rank = 0
    world = 1

    def send(self, t, dst):
        raise NotImplementedError

    def recv(self, t, src):
        raise NotImplementedError

    def broadcast(self, t, src):
        raise NotImplementedError


class TorchFrameComm(FrameComm):
    """torch.distributed (NCCL on GPUs, gloo on CPU tensors)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def _g(self, r):   # group rank -> global rank
        return r if self.group is None else \
            self.dist.get_global_rank(self.group, r)

    def send(self, t, dst):
        self.dist.send(t, self._g(dst), group=self.group)

    def recv(self, t, src):
        self.dist.recv(t, self._g(src), group=self.group)

    def broadcast(self, t, src):
        self.dist.broadcast(t, self._g(src), group=self.group)


def frame_blocks(nframes: int, world: int):
    """Contiguous frame ranges [lo, hi) per rank, sizes within one."""
    return [(r * nframes // world, (r + 1) * nframes // world)
            for r in range(world)]


def frame_split(nframes, build, grid, accumulate, pack, unpack, comm):
    """The frame-split protocol, backend-agnostic (tests drive it with the
    CPU oracle over gloo).  build(k) -> (f, w, tree) for an owned frame;
    grid() -> zero accumulator; accumulate(wf, ws, f, w) adds one frame;
    pack(tree) -> (int64 meta tensor[8], [arrays]); unpack(meta) -> (empty
    arrays to receive into, finish(arrays) -> tree).  Returns (trees in
    frame order, wf, ws), identical on every rank."""
    r, world = comm.rank, comm.world
    lo, hi = frame_blocks(nframes, world)[r]
    own = [build(k) for k in range(lo, hi)]        # in parallel on all ranks
    wf, ws = grid(), grid()
    if r > 0:                                      # frames before ours
        comm.recv(wf, r - 1)
        comm.recv(ws, r - 1)
    for f, w, _ in own:                            # ours, in frame order
        accumulate(wf, ws, f, w)
    if r < world - 1:
        comm.send(wf, r + 1)
        comm.send(ws, r + 1)
    comm.broadcast(wf, world - 1)                  # the complete sums
    comm.broadcast(ws, world - 1)
    trees = []
    owner = [q for q, (a, b) in enumerate(frame_blocks(nframes, world))
             for _ in range(a, b)]
    for k in range(nframes):
        o = owner[k]
        if o == r:
            meta, arrays = pack(own[k - lo][2])
            comm.broadcast(meta, o)
            for a in arrays:
                comm.broadcast(a, o)
            trees.append(own[k - lo][2])
        else:
            meta = torch.zeros(8, dtype=torch.int64, device=wf.device)
            comm.broadcast(meta, o)
            arrays, finish = unpack(meta)
            for a in arrays:
                comm.broadcast(a, o)
            trees.append(finish(arrays))
    return trees, wf, ws


def _tree_pack(t: OctreeField):
    meta = torch.tensor([t.capacity, int(t.state[0]), int(t.state[1]),
                         int(t.state[2]), t.d_max, 0, 0, 0],
                        dtype=torch.int64, device=t.value.device)
    return meta, [t.value, t.weight, t.child]


def _tree_unpack(dev):
    def unpack(meta):
        cap, s0, s1, s2, d = (int(x) for x in meta[:5].tolist())
        arrays = [pool_empty(cap, torch.float32), pool_empty(cap, torch.float32),
                  pool_empty(cap, torch.int32)]

        def finish(a):
            return OctreeField(a[0], a[2], np.array([s0, s1, s2], np.int64), d,
                               weight=a[1])
        return arrays, finish
    return unpack


# -- octree solver ------------------------------------------------------------

_FULL_CAP_LIMIT = 1 << 25


def _solver_capacity(u0: OctreeField) -> int:
    full = full_tree_capacity(u0.d_max)
    if full <= _FULL_CAP_LIMIT:
        return full          # the reference's policy (fusion.py:160-174)
    want = max(2 * u0.used, u0.used + 8 * 4096)
    return min(full, ((want + 7) // 8) * 8 + 1)


def _solver_field(u0: OctreeField, dtype: torch.dtype) -> OctreeField:
    cap = _solver_capacity(u0)
    used = u0.used
    value = pool_empty(cap, dtype, fill=0)
    value[:used].copy_(u0.value[:used])
    child = pool_empty(cap, torch.int32, fill=-1)
    child[:used].copy_(u0.child[:used])
    f = OctreeField(value, child, u0.state.copy(), u0.d_max)
    f.ensure_scratch()
    return f


def _grow(u: OctreeField) -> None:
    full = full_tree_capacity(u.d_max)
    if u.capacity >= full:
        raise RuntimeError("node pool capacity exhausted")
    u.ensure_capacity(min(full, 2 * u.capacity))


def tree_energy(u: OctreeField, views, params: FusionParams, *,
                ctx=None) -> float:
    """Leaf-summed energy of an octree iterate (fusion.py:177-183)."""
    vvals, vws, vchilds = view_arrays(views)
    return float(_backend.get().tree_energy(
        u.value, u.child, vvals, vws, vchilds, u.d_max, params.lam,
        params.eps, params.gamma, state=u.state, ctx=ctx))


def _pack() -> bool:
    """Packed sample positions on frozen trees (OCTF_NO_PACK=1: slot
    positions, for A/B runs)."""
    return os.environ.get("OCTF_NO_PACK", "0") != "1"


class Solver:
    """The descent schedule as a stepping object (reference fusion.py:218-236).

    One pass = iterate + propagate; the energy of a pass's result is
    evaluated by the next pass's leaf kernel from the same stencil and sample
    reads (``octf_fuse_pass``) -- or, after the last pass, by ``finish()``.
    With a frozen structure (tau_split <= 0, tau_join >= 1, clamp: no split
    or join can happen) ``run`` issues many passes in one call with no host
    round trip (``octf_fuse_passes_frozen``).  Used by ``fuse`` and the
    benchmark.
    """

    def __init__(self, u0: OctreeField, views, params: FusionParams, *,
                 log_joins: bool = False, reverse: bool = False,
                 precision: str = "fp64", samples=None, defer: bool = False):
        if not views and samples is None:
            raise ValueError("at least one view is required")
        for v in views or ():
            if v.d_max != u0.d_max:
                raise ValueError("view and iterate depths differ")
        if precision not in ("fp64", "fp32"):
            raise ValueError("precision must be 'fp64' or 'fp32'")
        self.params = params
        self.reverse = reverse
        self.log_joins = log_joins
        self.frozen = (params.tau_split <= 0.0 and params.clamp
                       and params.tau_join >= 1.0)
        self.dtype = torch.float64 if precision == "fp64" else torch.float32
        self.kern = _backend.get()
        self.u = _solver_field(u0, self.dtype)
        self.vvals, self.vws, self.vchilds = view_arrays(views or [])
        self.ctx = _lib.Ctx()
        # a shard: samples are gathered by ctx_select; a frozen tree: each
        # leaf's samples at its rank among its tile's leaves (CTX_PACKED)
        opts = ((_lib.CTX_DEFER if defer else 0)
                | (_lib.CTX_PACKED if self.frozen and _pack() else 0))
        if opts:
            self.ctx.set_options(opts)
        self.samples = samples
        if samples is not None:
            # per-slot samples (BASELINE config 5): frozen trees only
            if not self.frozen:
                raise ValueError("per-leaf samples need a frozen structure")
            self.kern.ctx_prepare(self.ctx, self.u.child, self.u.state,
                                  self.u.d_max, [], [], [])
            self.kern.ctx_set_samples(self.ctx, *samples)
        self.jbuf = None
        self.chunks: list[np.ndarray] = []
        self.stats: list[IterationStats] = []
        # `cur` holds the latest values; `nxt` receives the next pass
        self.cur, self.nxt = self.u.value, self.u.snap

    def _itemsize(self) -> int:
        return 2 * self.u.value.element_size() + self.u.child.element_size()

    def _settle(self, energy_pre: float) -> None:
        if self.stats and self.stats[-1].energy is None:
            self.stats[-1].energy = energy_pre

    def step(self, t: int) -> IterationStats:
        p, u = self.params, self.u
        xi = step_scale(t, p)
        t0 = time.perf_counter()
        while True:
            if self.log_joins and (self.jbuf is None
                                   or self.jbuf.shape[0] < u.capacity // 8 + 8):
                self.jbuf = torch.zeros((u.capacity // 8 + 8, 12),
                                        dtype=torch.float64, device=device())
            try:
                splits, joins, jrows, e_pre = self.kern.fuse_pass(
                    self.cur, self.nxt, u.child, u.joined, u.state, self.vvals,
                    self.vws, self.vchilds, u.d_max, p.lam, p.eps, p.gamma, xi,
                    p.tau_split, p.tau_join, p.clamp, self.reverse, self.jbuf,
                    ctx=self.ctx)
                break
            except RuntimeError as exc:
                if "capacity" not in str(exc):
                    raise
                u.value, u.snap = self.cur, self.nxt
                _grow(u)
                self.cur, self.nxt = u.value, u.snap
                self.ctx.invalidate()
        self._settle(e_pre)
        wall_ms = (time.perf_counter() - t0) * 1e3
        if self.jbuf is not None:
            if jrows != joins:
                raise RuntimeError("join log truncated")
            if jrows:
                self.chunks.append(to_numpy(self.jbuf[:jrows]).copy())
        self.cur, self.nxt = self.nxt, self.cur
        st = IterationStats(t + 1, None, u.node_count,
                            u.node_count * self._itemsize(), splits, joins,
                            wall_ms)
        self.stats.append(st)
        return st

    def run(self, t0: int, k: int) -> list:
        """Passes t0 .. t0+k-1; batched on the GPU when the structure is
        frozen."""
        if k <= 0:
            return []
        if self.log_joins:   # the join log is read back pass by pass
            return [self.step(t) for t in range(t0, t0 + k)]
        if not self.frozen:
            return self._run_restructuring(t0, k)
        p, u = self.params, self.u
        xis = [step_scale(t, p) for t in range(t0, t0 + k)]
        w0 = time.perf_counter()
        en = self.kern.fuse_passes_frozen(
            self.cur, self.nxt, u.child, u.state, self.vvals, self.vws,
            self.vchilds, u.d_max, p.lam, p.eps, p.gamma, p.tau_split,
            p.tau_join, p.clamp, xis, ctx=self.ctx)
        wall = (time.perf_counter() - w0) * 1e3 / k
        if k % 2:
            self.cur, self.nxt = self.nxt, self.cur
        out = []
        for j, t in enumerate(range(t0, t0 + k)):
            self._settle(float(en[j]))
            st = IterationStats(t + 1, None, u.node_count,
                                u.node_count * self._itemsize(), 0, 0, wall)
            self.stats.append(st)
            out.append(st)
        return out

    def _run_restructuring(self, t0: int, k: int, chunk: int = 32) -> list:
        """Passes with split/join, ``chunk`` at a time inside one library
        call (octf_fuse_passes: no return to Python between passes); a pass
        that exhausts the pool stops its call, the pools grow (as ``step``)
        and the run goes on from that pass."""
        p, u = self.params, self.u
        out, t = [], t0
        while t < t0 + k:
            n = min(chunk, t0 + k - t)
            xis = [step_scale(q, p) for q in range(t, t + n)]
            w0 = time.perf_counter()
            done, o3, en, err = self.kern.fuse_passes(
                self.cur, self.nxt, u.child, u.joined, u.state, self.vvals,
                self.vws, self.vchilds, u.d_max, p.lam, p.eps, p.gamma,
                p.tau_split, p.tau_join, p.clamp, self.reverse, xis,
                ctx=self.ctx)
            wall = (time.perf_counter() - w0) * 1e3 / max(done, 1)
            if done % 2:
                self.cur, self.nxt = self.nxt, self.cur
            for j in range(done):
                self._settle(float(en[j]))
                nodes = int(o3[j, 2])
                st = IterationStats(t + j + 1, None, nodes,
                                    nodes * self._itemsize(), int(o3[j, 0]),
                                    int(o3[j, 1]), wall)
                self.stats.append(st)
                out.append(st)
            t += done
            if err is not None:
                u.value, u.snap = self.cur, self.nxt
                _grow(u)
                self.cur, self.nxt = u.value, u.snap
                self.ctx.invalidate()
        return out

    def finish(self) -> None:
        """Evaluate the energy of the latest state (after the last pass)."""
        if self.stats and self.stats[-1].energy is None:
            u, p = self.u, self.params
            self.stats[-1].energy = self.kern.tree_energy(
                self.cur, u.child, self.vvals, self.vws, self.vchilds, u.d_max,
                p.lam, p.eps, p.gamma, state=u.state, ctx=self.ctx)

    def result(self) -> FuseResult:
        self.finish()
        self.u.value, self.u.snap = self.cur, self.nxt
        join_log = None
        if self.log_joins:
            join_log = (np.vstack(self.chunks) if self.chunks
                        else np.zeros((0, 12), dtype=np.float64))
        return FuseResult(field=self.u, stats=list(self.stats),
                          join_log=join_log)

    def close(self):
        self.ctx.close()
        self.kern.drop_view_cache()


def pd_steps(lam: float):
    """Default primal/dual steps for solver='pd': tau*sigma*||K||^2 < 1 with
    ||K|| <= lam*sqrt(12) at unit (finest-cell) spacing."""
    t = 0.99 / (lam * np.sqrt(12.0))
    return t, t


class PDSolver:
    """The north_star's TV-L1 primal-dual iteration (solver='pd'): dual
    ascent with projection, divergence, generalised-median prox (SURVEY.md
    §8(a) row A18; the reference has none -- its definition and CPU oracle
    are oracle/pd_oracle.c).  State: u, ubar, p = (px, py, pz) per node,
    double-buffered; p starts at 0 and ubar at u0.  Unless the structure is
    frozen (tau_split <= 0, tau_join >= 1, clamp), every pass is followed by
    the pd split/join (``octf_pd_restructure``: leaves with |u| < tau_split
    split, children carrying u/ubar/p; eight leaves past tau_join with one
    sign join), north_star item (d).  Any number of views: 4, 8, 16, 32 and
    64 use the dense sorted sample store (TMA-staged tiles), other counts
    the per-tile store of each leaf's observed views."""

    def __init__(self, u0: OctreeField, views, params: FusionParams, *,
                 precision: str = "fp32", tau: float | None = None,
                 sigma: float | None = None, samples=None,
                 defer: bool = False):
        if not views and samples is None:
            raise ValueError("at least one view is required")
        for v in views or ():
            if v.d_max != u0.d_max:
                raise ValueError("view and iterate depths differ")
        dtype = torch.float64 if precision == "fp64" else torch.float32
        self.params = params
        t, s = pd_steps(params.lam)
        self.tau = t if tau is None else tau
        self.sigma = s if sigma is None else sigma
        self.kern = _backend.get()
        self.u = _solver_field(u0, dtype)
        used, cap = self.u.used, self.u.capacity
        self.vvals, self.vws, self.vchilds = view_arrays(views or [])
        self.ctx = _lib.Ctx()
        self.restructure = not (params.tau_split <= 0.0 and params.clamp
                                and params.tau_join >= 1.0)
        # the pd kernel reads the dense layout, each leaf's samples sorted
        # once when gathered (its prox selects on them); packed positions on
        # a frozen tree
        # (view counts other than 4, 8, 16, 32, 64 -- BASELINE config 3 has
        # 300 frames: the per-tile (ELL) store of observed views, each
        # leaf's rows sorted the same way)
        nv = len(self.vvals)
        many = samples is None and nv not in (4, 8, 16, 32, 64)
        self.ctx.set_options((_lib.CTX_ELL if many else _lib.CTX_DENSE)
                             | _lib.CTX_SORTED
                             | (_lib.CTX_DEFER if defer else 0)
                             | (0 if self.restructure or not _pack()
                                else _lib.CTX_PACKED))
        self.samples = samples
        if samples is not None:
            self.kern.ctx_prepare(self.ctx, self.u.child, self.u.state,
                                  self.u.d_max, [], [], [])
            self.kern.ctx_set_samples(self.ctx, *samples)
        def z():
            return pool_empty(cap, dtype, fill=0)
        ub = z()
        ub[:used].copy_(self.u.value[:used])
        self.a = [self.u.value, ub, z(), z(), z()]
        self.b = [self.u.snap, z(), z(), z(), z()]
        self.stats: list[IterationStats] = []
        if self.restructure and samples is not None:
            raise ValueError("per-leaf samples need a frozen structure "
                             "(tau_split <= 0, tau_join >= 1, clamp)")

    def _grow(self) -> None:
        u = self.u
        full = full_tree_capacity(u.d_max)
        if u.capacity >= full:
            raise RuntimeError("node pool capacity exhausted")
        cap = min(full, 2 * u.capacity)

        def g(t, fill):
            n = pool_empty(cap, t.dtype, fill=fill)
            n[:t.shape[0]].copy_(t)
            return n
        self.a = [g(t, 0) for t in self.a]
        self.b = [g(t, 0) for t in self.b]
        u.value, u.snap = self.a[0], self.b[0]
        u.child = g(u.child, -1)
        if u.joined is not None:
            u.joined = g(u.joined, 0)
        self.ctx.invalidate()

    def _restructure(self) -> tuple:
        p, u = self.params, self.u
        while True:
            try:
                return self.kern.pd_restructure(
                    self.a, u.child, u.state, u.d_max, p.tau_split, p.tau_join,
                    ctx=self.ctx)
            except RuntimeError as exc:
                if "capacity" not in str(exc):
                    raise
                self._grow()   # the pool is untouched: grow, re-prepare, retry
                self.kern.ctx_prepare(self.ctx, u.child, u.state, u.d_max,
                                      self.vvals, self.vws, self.vchilds)

    def run(self, t0: int, k: int) -> list:
        p, u = self.params, self.u
        if self.restructure:
            out = []
            for t in range(t0, t0 + k):
                w0 = time.perf_counter()
                en = self.kern.pd_passes(self.a, self.b, u.child, u.state,
                                         self.vvals, self.vws, self.vchilds,
                                         u.d_max, p.lam, self.tau, self.sigma,
                                         p.gamma, p.clamp, 1, ctx=self.ctx)
                self.a, self.b = self.b, self.a
                splits, joins = self._restructure()
                if self.stats and self.stats[-1].energy is None:
                    self.stats[-1].energy = float(en[0])
                st = IterationStats(t + 1, None, u.node_count,
                                    u.node_count * 10 * u.value.element_size(),
                                    splits, joins,
                                    (time.perf_counter() - w0) * 1e3)
                self.stats.append(st)
                out.append(st)
            return out
        w0 = time.perf_counter()
        en = self.kern.pd_passes(self.a, self.b, u.child, u.state, self.vvals,
                                 self.vws, self.vchilds, u.d_max, p.lam,
                                 self.tau, self.sigma, p.gamma, p.clamp, k,
                                 ctx=self.ctx)
        wall = (time.perf_counter() - w0) * 1e3 / max(k, 1)
        if k % 2:
            self.a, self.b = self.b, self.a
        out = []
        for j, t in enumerate(range(t0, t0 + k)):
            if self.stats and self.stats[-1].energy is None:
                self.stats[-1].energy = float(en[j])
            st = IterationStats(t + 1, None, u.node_count,
                                u.node_count * 10 * u.value.element_size(), 0, 0,
                                wall)
            self.stats.append(st)
            out.append(st)
        return out

    def finish(self) -> None:
        """Energy of the latest u: one more evaluation pass on a scratch
        copy (the state is not advanced)."""
        if self.stats and self.stats[-1].energy is None:
            p, u = self.params, self.u
            scratch = [t.clone() for t in self.b]
            en = self.kern.pd_passes(self.a, scratch, u.child, u.state,
                                     self.vvals, self.vws, self.vchilds,
                                     u.d_max, p.lam, self.tau, self.sigma,
                                     p.gamma, p.clamp, 1, ctx=self.ctx)
            self.stats[-1].energy = float(en[0])

    def result(self) -> FuseResult:
        self.finish()
        self.u.value, self.u.snap = self.a[0], self.b[0]
        return FuseResult(field=self.u, stats=list(self.stats))

    @property
    def state(self):
        """(u, ubar, px, py, pz) after the last pass."""
        return tuple(self.a)

    def close(self):
        self.ctx.close()
        self.kern.drop_view_cache()


def fuse(u0: OctreeField, views, params: FusionParams, *,
         log_joins: bool = False, reverse: bool = False,
         precision: str = "fp64", solver: str = "descent",
         samples=None) -> FuseResult:
    """Run the full descent schedule on an octree iterate (fusion.py:186-241).

    ``u0`` is left untouched.  Statistics carry one row per pass; energies
    are those after the pass's restructuring and re-propagation.
    ``solver="pd"`` runs the north_star's TV-L1 primal-dual iteration
    instead (split/join after each pass unless frozen; no reference
    counterpart, see PDSolver).
    """
    if solver == "pd":
        pds = PDSolver(u0, views, params, precision=precision,
                       samples=samples)
        pds.run(0, params.iterations)
        res = pds.result()
        pds.close()
        return res
    if solver != "descent":
        raise ValueError("solver must be 'descent' or 'pd'")
    solver = Solver(u0, views, params, log_joins=log_joins, reverse=reverse,
                    precision=precision, samples=samples)
    solver.run(0, params.iterations)
    res = solver.result()
    solver.close()
    return res



# -- iteration reports (fusion.py:363-403) ----------------------------------

# -- dense reference solver (fusion.py:253-325) -------------------------------

def _full_tree_inputs(u0, fs, ws):
    """A dense problem as full trees: every cell a finest-level leaf (unit
    spacing), the tree path's arithmetic then equals the dense solver's."""
    u = build_octree(as_device(u0, torch.float64), tau=-1.0)
    views = [build_octree(as_device(f, torch.float32), as_device(w, torch.uint8),
                          tau=-1.0, dtype=np.float32) for f, w in zip(fs, ws)]
    return u, views


def _dense_params(params: FusionParams) -> FusionParams:
    # the dense solver never restructures
    return FusionParams(**{**params.__dict__, "tau_split": 0.0,
                           "tau_join": float("inf")})


def dense_fuse(u0, fs, ws, params: FusionParams):
    """The reference's dense solver (``fusion.dense_fuse``, fusion.py:311-325)
    on the GPU: the grid runs as a full tree (all leaves at the finest level,
    unit spacing), where the descent is the dense Jacobi step bit for bit
    (the reference's own tree == dense check, tests/test_fusion.py:121-131).
    Returns (u grid, stats) like the reference; energies are the tree's leaf
    sums (order differs from numpy's pairwise sum at the 1e-13 level)."""
    u, views = _full_tree_inputs(u0, fs, ws)
    res = fuse(u, views, _dense_params(params), precision="fp64")
    from .octree import densify
    grid = densify(res.field)
    n3 = grid.size
    stats = [IterationStats(s.iteration, s.energy, n3, n3 * 2 * 8, 0, 0,
                            s.wall_ms) for s in res.stats]
    return grid, stats


def dense_step(u, fs, ws, params: FusionParams, xi: float):
    """One Jacobi descent step on a dense grid (fusion.py:283-298)."""
    t, views = _full_tree_inputs(u, fs, ws)
    s = Solver(t, views, _dense_params(params), precision="fp64")
    s.kern.iterate_pass(s.u.value, s.u.snap, s.u.child, s.u.joined,
                        s.u.state, s.vvals, s.vws, s.vchilds, s.u.d_max,
                        params.lam, params.eps, params.gamma, xi, 0.0,
                        float("inf"), params.clamp, False, None, ctx=s.ctx)
    from .octree import densify
    out = densify(s.u)
    s.close()
    return out


def dense_energy(u, fs, ws, params: FusionParams) -> float:
    """Dense-grid energy (fusion.py:301-308) as the full tree's leaf sum."""
    t, views = _full_tree_inputs(u, fs, ws)
    return tree_energy(t, views, params)


# pointwise pieces of the energy (fusion.py:330-358; host math, exposed for
# derivative checks)
def data_term_value(u: float, f, w, eps: float, gamma: float) -> float:
    f = np.asarray(f, dtype=np.float64)
    w = np.asarray(w, dtype=np.float64)
    return float((w * np.sqrt((u - f) ** 2 + eps * eps)).sum()) / \
        (gamma + float(w.sum()))


def data_term_derivative(u: float, f, w, eps: float, gamma: float) -> float:
    f = np.asarray(f, dtype=np.float64)
    w = np.asarray(w, dtype=np.float64)
    d = u - f
    return float((w * d / np.sqrt(d * d + eps * eps)).sum()) / \
        (gamma + float(w.sum()))


def smoothness_value(g, eps: float) -> float:
    g = np.asarray(g, dtype=np.float64)
    return float(np.sqrt((g * g).sum() + eps * eps))


def smoothness_flux(g, eps: float) -> np.ndarray:
    g = np.asarray(g, dtype=np.float64)
    return g / np.sqrt((g * g).sum() + eps * eps)


REPORT_COLUMNS = ("iter", "energy", "node_count", "memory_bytes", "splits",
                  "joins", "wall_ms")


def write_report(path, stats, header: dict | None = None) -> None:
    with open(path, "w") as fp:
        for key, value in (header or {}).items():
            fp.write(f"# {key} = {value}\n")
        fp.write(",".join(REPORT_COLUMNS) + "\n")
        for s in stats:
            fp.write(f"{s.iteration},{s.energy:.17g},{s.node_count},"
                     f"{s.memory_bytes},{s.splits},{s.joins},"
                     f"{s.wall_ms:.3f}\n")


def read_report(path):
    header: dict[str, str] = {}
    stats: list[IterationStats] = []
    with open(path) as fp:
        for line in fp:
            line = line.strip()
            if not line:
                continue
            if line.startswith("#"):
                key, _, value = line[1:].partition("=")
                header[key.strip()] = value.strip()
                continue
            if line.startswith("iter,"):
                if line != ",".join(REPORT_COLUMNS):
                    raise ValueError("unexpected report columns")
                continue
            parts = line.split(",")
            if len(parts) != len(REPORT_COLUMNS):
                raise ValueError(f"bad report row: {line!r}")
            stats.append(IterationStats(int(parts[0]), float(parts[1]),
                                        int(parts[2]), int(parts[3]),
                                        int(parts[4]), int(parts[5]),
                                        float(parts[6])))
    return header, stats
