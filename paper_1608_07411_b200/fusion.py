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

import time
from dataclasses import dataclass, field as dc_field

import numpy as np
import torch

from . import _backend, _lib
from ._device import as_device, device, pool_empty, ptr, stream_handle, to_numpy
from .octree import OctreeField, build_octree, full_tree_capacity

__all__ = [
    "FusionParams",
    "IterationStats",
    "FuseResult",
    "step_scale",
    "build_view_tree",
    "view_arrays",
    "initial_field",
    "fuse",
    "tree_energy",
    "write_report",
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


def fuse(u0: OctreeField, views, params: FusionParams, *,
         log_joins: bool = False, reverse: bool = False,
         precision: str = "fp64") -> FuseResult:
    """Run the full descent schedule on an octree iterate (fusion.py:186-241).

    ``u0`` is left untouched.  Statistics carry one row per pass; energies
    are evaluated after the pass's restructuring and re-propagation.
    """
    if not views:
        raise ValueError("at least one view is required")
    for v in views:
        if v.d_max != u0.d_max:
            raise ValueError("view and iterate depths differ")
    if precision not in ("fp64", "fp32"):
        raise ValueError("precision must be 'fp64' or 'fp32'")
    dtype = torch.float64 if precision == "fp64" else torch.float32
    kern = _backend.get()
    u = _solver_field(u0, dtype)
    vvals, vws, vchilds = view_arrays(views)
    ctx = _lib.Ctx()
    jbuf = None
    chunks: list[np.ndarray] = []
    stats: list[IterationStats] = []
    itemsize = 2 * u.value.element_size() + u.child.element_size()
    # `cur` holds the latest values; `nxt` receives the next pass
    cur, nxt = u.value, u.snap
    for t in range(params.iterations):
        xi = step_scale(t, params)
        t0 = time.perf_counter()
        while True:
            if log_joins and (jbuf is None or jbuf.shape[0] < u.capacity // 8 + 8):
                jbuf = torch.zeros((u.capacity // 8 + 8, 12), dtype=torch.float64,
                                   device=device())
            try:
                splits, joins, jrows = kern.iterate_pass(
                    nxt, cur, u.child, u.joined, u.state, vvals, vws, vchilds,
                    u.d_max, params.lam, params.eps, params.gamma, xi,
                    params.tau_split, params.tau_join, params.clamp, reverse,
                    jbuf, ctx=ctx, snapshot=False)
                break
            except RuntimeError as exc:
                if "capacity" not in str(exc):
                    raise
                u.value, u.snap = cur, nxt
                _grow(u)
                cur, nxt = u.value, u.snap
                ctx.invalidate()
        kern.propagate(nxt, u.child, state=u.state, d_max=u.d_max, ctx=ctx)
        energy = kern.tree_energy(nxt, u.child, vvals, vws, vchilds, u.d_max,
                                  params.lam, params.eps, params.gamma,
                                  state=u.state, ctx=ctx)
        wall_ms = (time.perf_counter() - t0) * 1e3
        if jbuf is not None:
            if jrows != joins:
                raise RuntimeError("join log truncated")
            if jrows:
                chunks.append(to_numpy(jbuf[:jrows]).copy())
        cur, nxt = nxt, cur
        stats.append(IterationStats(t + 1, energy, u.node_count,
                                    u.node_count * itemsize, splits, joins,
                                    wall_ms))
    u.value, u.snap = cur, nxt
    join_log = None
    if log_joins:
        join_log = (np.vstack(chunks) if chunks
                    else np.zeros((0, 12), dtype=np.float64))
    ctx.close()
    return FuseResult(field=u, stats=stats, join_log=join_log)


# -- iteration reports (fusion.py:363-403) ----------------------------------

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
