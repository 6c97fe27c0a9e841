"""Device-resident octree fields (reference ``octree.py``).

Same model as the reference: a complete-children octree in flat pools
(node 0 = root, eight contiguous children per inner node, free-list block
recycling), here held in HBM as CUDA tensors.  ``state`` stays a host
int64[3] array {slots used, free-list head, live nodes}.  Pools keep the
reference layout bit for bit, so ``to_host()`` hands the reference's own
tools (``serialize``, ``quantization_error``, ``densify``) an identical pool.

Construction (pyramids + spread-rule build) and readout run on the GPU
through the C ABI; the structural queries (``locate``, ``leaves``,
``serialize``) are host-side conveniences over a downloaded copy.
"""

from __future__ import annotations

from typing import IO, Iterator

import numpy as np
import torch

from . import _backend, _lib
from ._device import (as_device, device, npdtype, pool_empty, ptr,
                      stream_handle, tdtype, to_numpy, to_pool)

__all__ = [
    "OctreeField",
    "full_tree_capacity",
    "build_octree",
    "propagate_means",
    "lookup_at_level",
    "densify",
    "densify_weight",
    "split_node",
    "join_node",
    "quantization_error",
    "serialize",
    "mean_pyramid",
]


def full_tree_capacity(d_max: int) -> int:
    """Node count of a complete octree of depth ``d_max`` (octree.py:44-46)."""
    return (8 ** (d_max + 1) - 1) // 7


class HostPool:
    """Numpy copy of a pool in the reference layout (for interop)."""

    def __init__(self, value, child, state, d_max, weight=None, snap=None,
                 joined=None):
        self.value, self.child, self.state = value, child, state
        self.d_max, self.weight, self.snap, self.joined = d_max, weight, snap, joined

    @property
    def used(self):
        return int(self.state[0])

    @property
    def node_count(self):
        return int(self.state[2])


class OctreeField:
    """Pooled octree on the GPU holding one scalar per node (octree.py:49-71).

    value   per-node scalar, CUDA float32/float64
    weight  optional per-node view weight, CUDA float32
    child   first of eight contiguous children or -1, CUDA int32
    state   host int64 [slots used, free-list head, live nodes]
    snap / joined: solver scratch (CUDA), allocated on demand.
    """

    __slots__ = ("value", "weight", "child", "state", "d_max", "snap",
                 "joined")

    def __init__(self, value, child, state, d_max, weight=None):
        self.value = value
        self.weight = weight
        self.child = child
        self.state = np.asarray(state, dtype=np.int64).copy()
        self.d_max = int(d_max)
        self.snap = None
        self.joined = None

    # -- bookkeeping (octree.py:75-144) -----------------------------------
    @property
    def capacity(self) -> int:
        return self.value.shape[0]

    @property
    def used(self) -> int:
        return int(self.state[0])

    @property
    def node_count(self) -> int:
        return int(self.state[2])

    @property
    def resolution(self) -> int:
        return 1 << self.d_max

    @property
    def nbytes_per_node(self) -> int:
        n = self.value.element_size() + self.child.element_size()
        if self.weight is not None:
            n += self.weight.element_size()
        if self.snap is not None:
            n += self.snap.element_size()
        return n

    @property
    def nbytes(self) -> int:
        return self.node_count * self.nbytes_per_node

    def ensure_capacity(self, needed: int) -> None:
        if needed <= self.capacity:
            return
        cap = max(needed, 2 * self.capacity)
        self.value = _grown(self.value, cap)
        self.child = _grown(self.child, cap, fill=-1)
        if self.weight is not None:
            self.weight = _grown(self.weight, cap)
        if self.snap is not None:
            self.snap = _grown(self.snap, cap)
        if self.joined is not None:
            self.joined = _grown(self.joined, cap)

    def ensure_scratch(self) -> None:
        if self.snap is None:
            snap = pool_empty(self.capacity, self.value.dtype, fill=0)
            snap[:self.used].copy_(self.value[:self.used])
            self.snap = snap
        if self.joined is None:
            self.joined = pool_empty(self.capacity, torch.uint8, fill=0)

    def alloc_block(self) -> int:
        free = int(self.state[1])
        if free >= 0:
            self.state[1] = int(self.child[free].item())
            b = free
        else:
            b = int(self.state[0])
            self.ensure_capacity(b + 8)
            self.state[0] = b + 8
        self.child[b:b + 8] = -1
        self.state[2] += 8
        return b

    def free_block(self, b: int) -> None:
        self.child[b:b + 8] = -1
        self.child[b] = int(self.state[1])
        self.state[1] = b
        self.state[2] -= 8

    # -- traversal ---------------------------------------------------------
    def locate(self, level: int, cell) -> tuple[int, int]:
        """Deepest node on the path to ``cell`` at ``level`` (octree.py:148)."""
        x, y, z = (int(c) for c in cell)
        if not 0 <= level <= self.d_max:
            raise ValueError(f"level {level} outside [0, {self.d_max}]")
        m = 1 << level
        if not (0 <= x < m and 0 <= y < m and 0 <= z < m):
            raise ValueError(f"cell {cell!r} invalid at level {level}")
        node, lvl = self.locate_many(level, [(x, y, z)])
        pair = torch.stack([node, lvl]).cpu()      # one device-to-host read
        return int(pair[0, 0]), int(pair[1, 0])

    def locate_many(self, level: int, cells):
        """``locate`` for (n, 3) cells of one level on the device
        (octf_locate): CUDA int32 tensors (nodes, levels)."""
        if not 0 <= level <= self.d_max:
            raise ValueError(f"level {level} outside [0, {self.d_max}]")
        c = as_device(cells, torch.int32).reshape(-1, 3).contiguous()
        n = c.shape[0]
        node = torch.empty(n, dtype=torch.int32, device=device())
        lvl = torch.empty(n, dtype=torch.int32, device=device())
        _lib.call("octf_locate", ptr(self.child), self.d_max, int(level),
                  ptr(c), n, ptr(node), ptr(lvl), stream_handle())
        return node, lvl

    def leaves(self) -> Iterator[tuple[int, int, int, int, int]]:
        """(node, level, x, y, z) of every leaf in Morton order
        (octree.py:168-181), ordered on the device (radix sort of the
        leaves' preorder keys, octf_node_order)."""
        slots, lvl, x, y, z = self.node_order(leaves_only=True)
        return iter(zip(*(to_numpy(t).tolist() for t in (slots, lvl, x, y,
                                                          z))))

    def node_order(self, leaves_only: bool = False):
        """Slots, levels and cell coordinates (CUDA tensors) of every live
        node -- or leaf -- in the reference's canonical depth-first order
        (octree.py:168-181, :413-431), sorted on the device."""
        from . import _kernels
        slots, keys = _kernels.node_order(self.child[:self.used], self.state,
                                          self.d_max, leaves_only=leaves_only)
        lvl, x, y, z = _kernels.decode_keys(keys, self.d_max)
        return slots, lvl, x, y, z

    def to_host(self, scratch: bool = True) -> HostPool:
        """Download the pool (reference layout, trimmed to ``used``) through
        pinned staging buffers; ``scratch=False`` skips the solver scratch
        (snap, joined)."""
        u = self.used

        def dl(t):
            if t is None:
                return None
            t = t[:u]
            h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
            h.copy_(t, non_blocking=True)
            return h
        parts = [dl(self.value), dl(self.child), dl(self.weight),
                 dl(self.snap) if scratch else None,
                 dl(self.joined) if scratch else None]
        torch.cuda.current_stream().synchronize()
        v, c, w, sn, j = (None if h is None else h.numpy() for h in parts)
        return HostPool(v, c, self.state.copy(), self.d_max, weight=w, snap=sn,
                        joined=j)

    @classmethod
    def from_host(cls, value, child, state, d_max, weight=None,
                  cap: int | None = None, dtype=None) -> "OctreeField":
        if not isinstance(value, torch.Tensor):
            value = np.asarray(value)
        if not isinstance(child, torch.Tensor):
            child = np.asarray(child, dtype=np.int32)
        if weight is not None and not isinstance(weight, torch.Tensor):
            weight = np.asarray(weight, np.float32)
        cap = value.shape[0] if cap is None else cap
        v = to_pool(value, dtype=dtype, cap=cap, fill=0)
        c = to_pool(child, dtype=np.int32, cap=cap, fill=-1)
        w = None if weight is None else to_pool(weight, dtype=np.float32,
                                                cap=cap, fill=0)
        return cls(v, c, state, d_max, weight=w)


def _grown(t: torch.Tensor, cap: int, fill=0) -> torch.Tensor:
    out = pool_empty(cap, t.dtype)
    out[:t.shape[0]].copy_(t)
    out[t.shape[0]:].fill_(fill)
    return out


def _leaves(child: np.ndarray):
    out = []
    stack = [(0, 0, 0, 0, 0)]
    while stack:
        node, lvl, x, y, z = stack.pop()
        b = int(child[node])
        if b < 0:
            out.append((node, lvl, x, y, z))
        else:
            for c in range(7, -1, -1):
                stack.append((b + c, lvl + 1, 2 * x + ((c >> 2) & 1),
                              2 * y + ((c >> 1) & 1), 2 * z + (c & 1)))
    return out


# -- construction -----------------------------------------------------------

def _grid_depth(f) -> int:
    shape = tuple(f.shape)
    n = shape[0] if shape else 0
    if len(shape) != 3 or shape != (n, n, n) or n < 1 or (n & (n - 1)) != 0:
        raise ValueError("field must be cubic with a power-of-two resolution")
    d = n.bit_length() - 1
    if d > _lib.MAX_DEPTH:
        raise ValueError("tree depth out of range")
    return d


def build_octree(f, w=None, tau: float = 0.1, dtype=np.float64) -> OctreeField:
    """Octree-ify a dense grid by the spread rule (octree.py:243-306), on the
    GPU: fused pyramids + parallel depth-first-order build (+ propagate when
    unweighted).  ``f`` / ``w`` may be numpy arrays or CUDA tensors."""
    d = _grid_depth(f)
    fd = as_device(f)
    if fd.dtype not in (torch.float32, torch.float64):
        fd = fd.to(torch.float64)
    wd = None
    if w is not None:
        if tuple(w.shape) != tuple(f.shape):
            raise ValueError("weight grid shape mismatch")
        wd = as_device(w).to(torch.uint8).contiguous()
    vdt = npdtype(dtype)
    if vdt not in (np.dtype(np.float32), np.dtype(np.float64)):
        raise TypeError("value dtype must be float32 or float64")
    cap = full_tree_capacity(d)
    value = pool_empty(cap, vdt)
    child = pool_empty(cap, torch.int32)
    weight = pool_empty(cap, torch.float32) if wd is not None else None
    state = np.zeros(3, dtype=np.int64)
    _lib.call("octf_build_octree", ptr(fd),
              _lib.OCTF_F32 if fd.dtype == torch.float32 else _lib.OCTF_F64,
              ptr(wd), d, float(tau), ptr(value),
              _lib.OCTF_F32 if vdt == np.float32 else _lib.OCTF_F64,
              ptr(weight), ptr(child), state.ctypes.data, cap, stream_handle())
    used = int(state[0])
    field = OctreeField(_trim(value, used), _trim(child, used), state, d,
                        weight=None if weight is None else _trim(weight, used))
    return field


def _trim(t: torch.Tensor, used: int) -> torch.Tensor:
    out = pool_empty(used, t.dtype)
    out.copy_(t[:used])
    return out


def propagate_means(field: OctreeField) -> OctreeField:
    """Recompute inner values (and weights) as child means (octree.py:309)."""
    kern = _backend.get()
    kern.propagate(field.value, field.child, state=field.state,
                   d_max=field.d_max)
    if field.weight is not None:
        kern.propagate(field.weight, field.child, state=field.state,
                       d_max=field.d_max)
    return field


def lookup_at_level(field: OctreeField, cell, level: int, *,
                    snap: bool = False) -> float:
    node, _ = field.locate(level, cell)
    arr = field.snap if snap else field.value
    return float(arr[node].item())


def densify_device(field: OctreeField, *, snap: bool = False,
                   weight: bool = False) -> torch.Tensor:
    """(2^d)^3 float64 CUDA tensor of the leaf values (_kernels.pyx:116)."""
    n = field.resolution
    out = torch.empty((n, n, n), dtype=torch.float64, device=device())
    arr = field.weight if weight else (field.snap if snap else field.value)
    _backend.get().densify(arr, field.child, field.d_max, out)
    return out


def densify(field: OctreeField, *, snap: bool = False) -> np.ndarray:
    """Expand the tree to its dense finest-level grid (octree.py:327-333)."""
    return to_numpy(densify_device(field, snap=snap))


def densify_weight(field: OctreeField) -> np.ndarray:
    if field.weight is None:
        raise ValueError("field carries no weights")
    return to_numpy(densify_device(field, weight=True))


# -- restructuring primitives (octree.py:347-388) ----------------------------

def split_node(field: OctreeField, level: int, cell) -> int:
    node, lvl = field.locate(level, cell)
    if lvl != level or int(field.child[node].item()) >= 0:
        raise ValueError(f"no leaf at level {level}, cell {tuple(cell)}")
    if level >= field.d_max:
        raise ValueError("cannot split a finest-level leaf")
    field.ensure_scratch()
    field.ensure_capacity(field.used + 8)
    field.snap[node] = field.value[node].to(field.snap.dtype)
    b = field.alloc_block()
    field.value[b:b + 8] = field.value[node]
    field.snap[b:b + 8] = field.snap[node]
    if field.weight is not None:
        field.weight[b:b + 8] = field.weight[node]
    field.child[node] = b
    return b


def join_node(field: OctreeField, level: int, cell) -> None:
    node, lvl = field.locate(level, cell)
    b = int(field.child[node].item())
    if lvl != level or b < 0:
        raise ValueError(f"no inner node at level {level}, cell {tuple(cell)}")
    if bool((field.child[b:b + 8] >= 0).any()):
        raise ValueError("join requires all eight children to be leaves")
    vals = to_numpy(field.value[b:b + 8]).astype(np.float64)
    total = 0.0
    for v in vals:
        total += float(v)
    field.value[node] = total / 8.0
    if field.weight is not None:
        ws = to_numpy(field.weight[b:b + 8]).astype(np.float64)
        wt = 0.0
        for v in ws:
            wt += float(v)
        field.weight[node] = wt / 8.0
    field.child[node] = -1
    field.free_block(b)


# -- metrics and serialization -----------------------------------------------

def mean_pyramid(grid) -> list:
    """Per-level 2x2x2 means of a cubic grid, root first, computed on the GPU
    in numpy's summation order (octree.py:193-214).  Returns numpy arrays."""
    d = _grid_depth(grid)
    g = as_device(grid)
    if g.dtype not in (torch.float32, torch.float64):
        g = g.to(torch.float64)
    total = sum(8 ** l for l in range(d + 1))
    mn = torch.empty(total, dtype=torch.float64, device=device())
    mx = torch.empty_like(mn)
    mean = torch.empty_like(mn)
    _lib.call("octf_pyramids", ptr(g),
              _lib.OCTF_F32 if g.dtype == torch.float32 else _lib.OCTF_F64,
              None, d, ptr(mn), ptr(mx), ptr(mean), None, None, None, None,
              None, stream_handle())
    flat = to_numpy(mean)
    out, off = [], 0
    for l in range(d + 1):
        n = 1 << l
        out.append(flat[off:off + n ** 3].reshape(n, n, n))
        off += n ** 3
    return out


def quantization_error(field: OctreeField, dense_u) -> tuple[float, float]:
    """Summed |leaf value - dense subvolume mean| (octree.py:393-410)."""
    dense_u = np.asarray(dense_u, dtype=np.float64)
    if dense_u.shape != (field.resolution,) * 3:
        raise ValueError("dense grid resolution mismatch")
    pyr = mean_pyramid(dense_u)
    host = field.to_host()
    n3 = float(field.resolution ** 3)
    total = 0.0
    weighted = 0.0
    for node, lvl, x, y, z in _leaves(host.child):
        diff = abs(float(host.value[node]) - float(pyr[lvl][x, y, z]))
        total += diff
        weighted += diff * (8.0 ** (field.d_max - lvl)) / n3
    return total, weighted


def serialize(field, fp: IO[str]) -> int:
    """Pre-order dump, one ``level cx cy cz is_leaf value weight`` line per
    node (octree.py:413-431).  A device field is ordered and gathered on the
    device (octf_node_order); only the text formatting runs on the host."""
    if isinstance(field, OctreeField):
        slots, lvl, x, y, z = field.node_order()
        sl = slots.long()
        leaf = field.child[:field.used][sl] < 0
        val = field.value[:field.used][sl].double()
        wt = (field.weight[:field.used][sl].double() if field.weight is not None
              else torch.zeros_like(val))
        cols = [to_numpy(t).tolist() for t in (lvl, x, y, z, leaf.int(), val,
                                               wt)]
        for L, cx, cy, cz, lf, v, w in zip(*cols):
            fp.write(f"{L} {cx} {cy} {cz} {lf} {v:.17g} {w:.17g}\n")
        return len(cols[0])
    host = field
    count = 0
    stack = [(0, 0, 0, 0, 0)]
    while stack:
        node, lvl, x, y, z = stack.pop()
        b = int(host.child[node])
        wt = float(host.weight[node]) if host.weight is not None else 0.0
        fp.write(f"{lvl} {x} {y} {z} {int(b < 0)} "
                 f"{float(host.value[node]):.17g} {wt:.17g}\n")
        count += 1
        if b >= 0:
            for c in range(7, -1, -1):
                stack.append((b + c, lvl + 1, 2 * x + ((c >> 2) & 1),
                              2 * y + ((c >> 1) & 1), 2 * z + (c & 1)))
    return count
