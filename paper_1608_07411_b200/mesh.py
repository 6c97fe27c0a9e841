"""Zero-isosurface readout (reference ``mesh.py``).

``marching_cubes(values, seen, dom)`` runs on the GPU (``octf_marching_cubes``,
``csrc/mesh.cu``) and returns the reference's mesh bit for bit: the same case
tables, vertex order (ascending grid-edge key), face order (cube order, then
table order) and f64 vertex arithmetic.  The case tables are generated here
from the rule the reference documents (``_mctables.py``): per inside/outside
corner pattern, crossed edges are paired face by face -- two crossings pair
up, four crossings pair around each inside corner -- the pairs are walked
into closed loops, each loop is oriented so its normal points from inside to
outside, and fan-triangulated.  ``tests/test_mesh.py`` checks the tables and
meshes against fixtures generated from the reference.

Mesh file I/O and mesh-to-mesh comparisons are host utilities outside the
accelerated path and are not part of this package.
"""

from __future__ import annotations

import ctypes
from typing import NamedTuple

import numpy as np
import torch

from . import _lib
from ._device import as_device, device, ptr, stream_handle

__all__ = ["TriMesh", "extract_zero_surface", "marching_cubes", "case_tables",
           "tree_zero_surface", "marching_cubes_tree", "seen_tree", "MeshDiff",
           "nearest_vertex_distances", "vertex_diff"]

# corner c of a cube sits at offset (c>>2 & 1, c>>1 & 1, c & 1) (x, y, z),
# the octree child numbering; edges 0-3 run along x, 4-7 along y, 8-11
# along z, each given as its (low, high) corner pair
_CORNER = np.array([((c >> 2) & 1, (c >> 1) & 1, c & 1) for c in range(8)])
_EDGE = [(c, c | 4) for c in (0, 1, 2, 3)] + \
        [(c, c | 2) for c in (0, 1, 4, 5)] + \
        [(c, c | 1) for c in (0, 2, 4, 6)]
_EDGE_AXIS = np.array([0] * 4 + [1] * 4 + [2] * 4, dtype=np.int8)
_EDGE_OFF = np.array([_CORNER[lo] for lo, _ in _EDGE], dtype=np.int8)


def _faces():
    """The six faces as (corner list, edge list), x-low, x-high, y-low, ..."""
    out = []
    for axis in range(3):
        bit = 4 >> axis
        for side in (0, bit):
            corners = [c for c in range(8) if (c & bit) == side]
            edges = [e for e, (a, b) in enumerate(_EDGE)
                     if a in corners and b in corners]
            out.append((corners, edges))
    return out


def _loops(mask: int, faces):
    inside = [bool((mask >> c) & 1) for c in range(8)]
    cut = [inside[a] != inside[b] for a, b in _EDGE]
    partners = {e: [] for e in range(12) if cut[e]}

    def link(a, b):
        partners[a].append(b)
        partners[b].append(a)
    for corners, edges in faces:
        hit = [e for e in edges if cut[e]]
        if len(hit) == 2:
            link(hit[0], hit[1])
        elif len(hit) == 4:          # ambiguous face: pair around inside corners
            for c in corners:
                if inside[c]:
                    around = [e for e in hit if c in _EDGE[e]]
                    link(around[0], around[1])
    loops, done = [], set()
    for start in partners:           # ascending edge id
        if start in done:
            continue
        loop, prev, cur = [start], -1, start
        while True:
            first, second = partners[cur]
            step = second if first == prev else first
            if step == start:
                break
            loop.append(step)
            prev, cur = cur, step
        done.update(loop)
        loops.append(loop)
    return inside, loops


def _orient(loop, inside):
    """Loop order whose (Newell) normal points from inside to outside."""
    mid = [(_CORNER[_EDGE[e][0]] + _CORNER[_EDGE[e][1]]) / 2.0 for e in loop]
    nrm = np.zeros(3)
    for i, p in enumerate(mid):
        nrm += np.cross(p, mid[(i + 1) % len(mid)])
    out = np.zeros(3)
    for e in loop:
        a, b = _EDGE[e]
        lo, hi = (b, a) if inside[b] else (a, b)   # inside -> outside
        out += _CORNER[hi] - _CORNER[lo]
    return loop if float(nrm @ out) > 0 else loop[::-1]


def case_tables():
    """(tri_table int8[256, 32] padded with -1, tri_count int8[256],
    edge_axis int8[12], edge_offset int8[12, 3])."""
    faces = _faces()
    table = np.full((256, 32), -1, dtype=np.int8)
    count = np.zeros(256, dtype=np.int8)
    for mask in range(256):
        inside, loops = _loops(mask, faces)
        tri = []
        for loop in loops:
            loop = _orient(loop, inside)
            for i in range(1, len(loop) - 1):
                tri += [loop[0], loop[i], loop[i + 1]]
        table[mask, :len(tri)] = tri
        count[mask] = len(tri) // 3
    return table, count, _EDGE_AXIS.copy(), _EDGE_OFF.copy()


_TABLES = None


def _tables():
    global _TABLES
    if _TABLES is None:
        _TABLES = tuple(np.ascontiguousarray(t) for t in case_tables())
    return _TABLES


class TriMesh(NamedTuple):
    """The readout's result: float64 vertex positions (V, 3) and int32
    triangle corner indices (F, 3), both numpy."""

    vertices: np.ndarray
    faces: np.ndarray


def _copy_mesh(h, nv, nf):
    try:
        verts = torch.empty((nv, 3), dtype=torch.float64, device=device())
        faces = torch.empty((nf, 3), dtype=torch.int32, device=device())
        _lib.call("octf_mesh_copy", h, ptr(verts) if nv else None,
                  ptr(faces) if nf else None, stream_handle())
    finally:
        _lib.lib().octf_mesh_free(h)
    return verts.cpu().numpy(), faces.cpu().numpy()


def _extract_tree(field, seen, origin=None, voxel=1.0, world=False,
                  slab=(-1, -1)):
    from .octree import OctreeField
    if not isinstance(field, OctreeField):
        raise TypeError("field must be a device OctreeField")
    if seen is not None and seen.d_max != field.d_max:
        raise ValueError("seen tree depth differs from the field's")
    tri, cnt, eax, eoff = _tables()
    org = np.ascontiguousarray(np.asarray(origin if origin is not None
                                          else (0.0, 0.0, 0.0), np.float64))
    st = np.ascontiguousarray(field.state[:3], dtype=np.int64)

    def code(t):
        return _lib.OCTF_F64 if t.dtype == torch.float64 else _lib.OCTF_F32
    if field.value.dtype not in (torch.float32, torch.float64):
        raise TypeError("field values must be float32 or float64")
    h = ctypes.c_void_p()
    nv, nf = ctypes.c_int64(), ctypes.c_int64()
    _lib.call("octf_marching_cubes_tree", None, code(field.value),
              ptr(field.value), ptr(field.child), st.ctypes.data,
              field.child.shape[0], field.d_max,
              code(seen.value) if seen is not None else _lib.OCTF_F64,
              ptr(seen.value) if seen is not None else None,
              ptr(seen.child) if seen is not None else None,
              tri.ctypes.data, cnt.ctypes.data, eax.ctypes.data,
              eoff.ctypes.data, org.ctypes.data, float(voxel), int(world),
              int(slab[0]), int(slab[1]), ctypes.byref(h), ctypes.byref(nv),
              ctypes.byref(nf), stream_handle())
    return _copy_mesh(h, nv.value, nf.value)


def tree_zero_surface(field, seen=None, slab=(-1, -1)):
    """extract_zero_surface(densify(field), seen) read straight from the leaf
    store (octf_marching_cubes_tree): grid index coordinates; ``seen`` an
    observed-mask tree (seen_tree) or None; ``slab`` = (b0, b1) reads only
    the cubes with x in [8 b0, 8 b1) (a mesh too large for one call)."""
    return _extract_tree(field, seen, slab=slab)


def marching_cubes_tree(field, seen, dom) -> TriMesh:
    """marching_cubes(densify(field), seen, dom) (mesh.py:114-125) without the
    dense grid: the same mesh, bit for bit."""
    if field.resolution != dom.resolution:
        raise ValueError("field does not match the domain resolution")
    return TriMesh(*_extract_tree(field, seen, dom.origin, dom.voxel_size,
                                  True))


def seen_tree(seen):
    """An observed-mask tree of a dense boolean grid (tau = 0: leaves are
    exactly the constant regions; node values 0 / 1)."""
    from .octree import build_octree
    return build_octree(as_device(seen, torch.float64), tau=0.0)


def _extract(values, mask, origin=None, voxel=1.0, world=False):
    v = as_device(values, torch.float64).contiguous()
    n = v.shape[0]
    if v.dim() != 3 or tuple(v.shape) != (n, n, n) or n < 2:
        raise ValueError("values must be a cubic grid with edge >= 2")
    m = None
    if mask is not None:
        m = as_device(mask, torch.bool)
        if tuple(m.shape) != tuple(v.shape):
            raise ValueError("mask shape mismatch")
        m = m.to(torch.uint8).contiguous()
    tri, cnt, eax, eoff = _tables()
    org = np.ascontiguousarray(np.asarray(origin if origin is not None
                                          else (0.0, 0.0, 0.0), np.float64))
    h = ctypes.c_void_p()
    nv, nf = ctypes.c_int64(), ctypes.c_int64()
    _lib.call("octf_marching_cubes", ptr(v), ptr(m) if m is not None else None,
              n, tri.ctypes.data, cnt.ctypes.data, eax.ctypes.data,
              eoff.ctypes.data, org.ctypes.data, float(voxel), int(world),
              ctypes.byref(h), ctypes.byref(nv), ctypes.byref(nf),
              stream_handle())
    try:
        verts = torch.empty((nv.value, 3), dtype=torch.float64, device=device())
        faces = torch.empty((nf.value, 3), dtype=torch.int32, device=device())
        _lib.call("octf_mesh_copy", h, ptr(verts) if nv.value else None,
                  ptr(faces) if nf.value else None, stream_handle())
    finally:
        _lib.lib().octf_mesh_free(h)
    return verts.cpu().numpy(), faces.cpu().numpy()


def extract_zero_surface(values, mask=None):
    """Zero level set in grid index coordinates (mesh.py:63-111): a cube is
    skipped unless ``mask`` is true at all eight corners.  Returns
    (vertices, faces) numpy arrays."""
    return _extract(values, mask)


def marching_cubes(values, seen, dom) -> TriMesh:
    """The implicit surface in world coordinates (mesh.py:114-125): grid
    samples at voxel centres, index i -> origin + (i + 1/2) * voxel_size."""
    if tuple(values.shape) != (dom.resolution,) * 3:
        raise ValueError("grid does not match the domain resolution")
    return TriMesh(*_extract(values, seen, dom.origin, dom.voxel_size, True))


class MeshDiff(NamedTuple):
    """Nearest-vertex distances of two meshes, each way (numpy float64), with
    the reference's summary statistics over both directions together
    (mesh.py:143-159)."""

    d_ab: np.ndarray
    d_ba: np.ndarray

    def _both(self) -> np.ndarray:
        return np.concatenate([self.d_ab, self.d_ba])

    @property
    def mean(self) -> float:
        return float(self._both().mean())

    @property
    def std(self) -> float:
        return float(self._both().std())

    @property
    def max(self) -> float:
        return float(self._both().max())


def nearest_vertex_distances(a, b):
    """Distance from every row of ``a`` (V_a, 3) to its nearest row of ``b``
    on the device (octf_nearest_vertex: uniform-grid search, the k-d tree's
    f64 arithmetic).  Returns a CUDA float64 tensor."""
    va = as_device(a, torch.float64).contiguous()
    vb = as_device(b, torch.float64).contiguous()
    if va.dim() != 2 or vb.dim() != 2 or va.shape[1] != 3 or vb.shape[1] != 3:
        raise ValueError("vertices must be (V, 3) arrays")
    if va.shape[0] == 0 or vb.shape[0] == 0:
        raise ValueError("cannot compare empty meshes")
    out = torch.empty(va.shape[0], dtype=torch.float64, device=device())
    _lib.call("octf_nearest_vertex", ptr(va), va.shape[0], ptr(vb),
              vb.shape[0], ptr(out), stream_handle())
    return out


def vertex_diff(a: TriMesh, b: TriMesh) -> MeshDiff:
    """Symmetric nearest-vertex comparison of two meshes (mesh.py:162-167)
    computed on the GPU."""
    return MeshDiff(
        nearest_vertex_distances(a.vertices, b.vertices).cpu().numpy(),
        nearest_vertex_distances(b.vertices, a.vertices).cpu().numpy())
