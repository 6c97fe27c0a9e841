"""CPU oracle for the octfuse hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this module, and only as the checker.
The product package (``paper_1608_07411_b200``) never imports it.

Two halves:
  * the native part (build_tree / propagate / densify / iterate_pass /
    tree_energy) is the plain-C restatement in ``octfuse_oracle.c`` loaded
    through ctypes;
  * the numpy part restates the reference's dense pre-processing:
    per-view TSDF (reference ``tsdf.py:87-120``), pyramids
    (``octree.py:193-225``), the octree build driver (``octree.py:243-306``),
    ``initial_field`` (``fusion.py:149-155``) and the ``fuse`` loop
    (``fusion.py:186-241``).

Parity pin: ``tests/test_oracle_golden.py`` checks every function here
against fixtures produced by the reference itself (``tests/golden/``, made by
``tests/golden/make_golden.py`` which imports /root/reference and its
compiled kernels from ``oracle/_ref``).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboctfuse_oracle.so")

ORC_ERRORS = {1: (ValueError, "tree depth out of range"),
              2: (MemoryError, "oracle scratch allocation failed"),
              3: (RuntimeError, "node pool capacity exhausted")}

_lib = None


def build_lib(force: bool = False) -> str:
    if force or not os.path.exists(_LIB_PATH):
        subprocess.check_call(["make", "-s", "-C", _HERE, "oracle"])
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build_lib()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        i64, i32, dbl = ctypes.c_int64, ctypes.c_int, ctypes.c_double
        L.orc_build_tree.argtypes = [P, P, P, P, i32, P, P, P, dbl, P, i32, P,
                                     P, P, i32]
        for nm in ("orc_propagate_f64", "orc_propagate_f32"):
            getattr(L, nm).argtypes = [P, P, i64]
        for nm in ("orc_densify_f64", "orc_densify_f32"):
            getattr(L, nm).argtypes = [P, P, i32, P]
        L.orc_iterate_pass.argtypes = [P, P, P, P, P, i64, i32, P, P, P, i32,
                                       dbl, dbl, dbl, dbl, dbl, dbl, i32, i32,
                                       P, i64, P]
        L.orc_tree_energy.argtypes = [P, P, i32, P, P, P, i32, dbl, dbl, dbl,
                                      P]
        L.orc_pd_pass.argtypes = [P] * 10 + [P, i64, i32, P, P, P, i32, dbl,
                                             dbl, dbl, dbl, i32, P]
        L.orc_pd_restructure.argtypes = [P] * 5 + [P, P, i64, i32, dbl, dbl, P]
        _lib = L
    return _lib


def _check(rc):
    if rc:
        exc, msg = ORC_ERRORS.get(rc, (RuntimeError, f"oracle error {rc}"))
        raise exc(msg)


def _ptr(a: np.ndarray):
    return a.ctypes.data if a is not None and a.size else None


def _ptr_array(arrs):
    return (ctypes.c_void_p * max(len(arrs), 1))(*[a.ctypes.data for a in arrs])


# ---------------------------------------------------------------- pools ----

def full_tree_capacity(d_max: int) -> int:
    """Node count of a complete octree of depth d_max (octree.py:44-46)."""
    return (8 ** (d_max + 1) - 1) // 7


@dataclass
class Pool:
    """A reference-layout node pool (octree.py:49-71)."""
    value: np.ndarray
    child: np.ndarray
    state: np.ndarray
    d_max: int
    weight: np.ndarray | None = None
    snap: np.ndarray | None = None
    joined: np.ndarray | None = None

    @property
    def used(self) -> int:
        return int(self.state[0])

    @property
    def node_count(self) -> int:
        return int(self.state[2])

    @property
    def resolution(self) -> int:
        return 1 << self.d_max


# ------------------------------------------------------------ pyramids ----

def reduce_pyramid(grid: np.ndarray, op: str) -> list:
    """Per-level 2x2x2 reduction, root first (octree.py:193-210).

    numpy's reduction over axes (1,3,5) of the (h,2,h,2,h,2) view sums the
    eight children c = x<<2|y<<1|z as ((((b0+b1)+(b2+b3))+(b4+b5))+(b6+b7));
    tests/test_oracle_golden.py pins that order on the running numpy.
    """
    g = np.asarray(grid)
    if op == "mean":
        g = g.astype(np.float64)
    out = [g]
    while out[-1].shape[0] > 1:
        a = out[-1]
        h = a.shape[0] // 2
        out.append(getattr(a.reshape(h, 2, h, 2, h, 2), op)(axis=(1, 3, 5)))
    return out[::-1]


def flatten_pyramid(levels):
    offs = np.zeros(len(levels), dtype=np.int64)
    acc = 0
    for i, lv in enumerate(levels):
        offs[i] = acc
        acc += lv.size
    return np.concatenate([lv.ravel() for lv in levels]), offs


def build_octree(f, w=None, tau: float = 0.1, dtype=np.float64) -> Pool:
    """Spread-rule build from a dense grid (octree.py:243-306)."""
    f = np.asarray(f)
    n = f.shape[0]
    if f.ndim != 3 or f.shape != (n, n, n) or (n & (n - 1)) != 0:
        raise ValueError("field must be cubic with a power-of-two resolution")
    d_max = n.bit_length() - 1
    f64 = f.astype(np.float64)
    minf, offs = flatten_pyramid(reduce_pyramid(f64, "min"))
    maxf, _ = flatten_pyramid(reduce_pyramid(f64, "max"))
    has_w = w is not None
    if has_w:
        w = np.asarray(w)
        if w.shape != f.shape:
            raise ValueError("weight grid shape mismatch")
        wminf, _ = flatten_pyramid(reduce_pyramid(w.astype(np.uint8), "min"))
        wmaxf, _ = flatten_pyramid(reduce_pyramid(w.astype(np.uint8), "max"))
        wm_l = reduce_pyramid(w.astype(np.float64), "mean")
        wf_l = reduce_pyramid(f64 * w, "mean")
        pl_l = reduce_pyramid(f, "mean")
        val_l = [np.where(wm > 0, wf / np.where(wm > 0, wm, 1.0), pl)
                 for wm, wf, pl in zip(wm_l, wf_l, pl_l)]
        meanf, _ = flatten_pyramid(val_l)
        wmeanf, _ = flatten_pyramid(wm_l)
    else:
        meanf, _ = flatten_pyramid(reduce_pyramid(f, "mean"))
        wminf = wmaxf = np.zeros(1, dtype=np.uint8)
        wmeanf = np.zeros(1, dtype=np.float64)
    cap = full_tree_capacity(d_max)
    value = np.zeros(cap, dtype=dtype)
    weight = np.zeros(cap, dtype=np.float32) if has_w else np.zeros(1, np.float32)
    child = np.full(cap, -1, dtype=np.int32)
    state = np.array([1, -1, 1], dtype=np.int64)
    _check(lib().orc_build_tree(
        _ptr(meanf), _ptr(minf), _ptr(maxf), _ptr(offs), int(has_w),
        _ptr(wminf), _ptr(wmaxf), _ptr(wmeanf), float(tau), _ptr(value),
        int(value.dtype == np.float32), _ptr(weight), _ptr(child),
        _ptr(state), d_max))
    used = int(state[0])
    p = Pool(value[:used].copy(), child[:used].copy(), state.copy(), d_max,
             weight=weight[:used].copy() if has_w else None)
    if not has_w:
        propagate(p.value, p.child)
    return p


def propagate(value: np.ndarray, child: np.ndarray) -> None:
    fn = lib().orc_propagate_f32 if value.dtype == np.float32 else lib().orc_propagate_f64
    _check(fn(_ptr(value), _ptr(child), child.shape[0]))


def densify(value: np.ndarray, child: np.ndarray, d_max: int) -> np.ndarray:
    n = 1 << d_max
    out = np.empty((n, n, n), dtype=np.float64)
    fn = lib().orc_densify_f32 if value.dtype == np.float32 else lib().orc_densify_f64
    _check(fn(_ptr(value), _ptr(child), d_max, _ptr(out)))
    return out


def iterate_pass(uval, usnap, uchild, ujoined, ustate, vvals, vws, vchilds,
                 d_max, lam, eps, gamma, xi, tau_s, tau_j, clamp, reverse,
                 jlog):
    """_kernels.pyx:384-461 restated; same argument list and return."""
    out3 = np.zeros(3, dtype=np.int64)
    jcap = 0 if jlog is None else jlog.shape[0]
    _check(lib().orc_iterate_pass(
        _ptr(uval), _ptr(usnap), _ptr(uchild), _ptr(ujoined), _ptr(ustate),
        uval.shape[0], len(vvals), _ptr_array(vvals), _ptr_array(vws),
        _ptr_array(vchilds), d_max, lam, eps, gamma, xi, tau_s, tau_j,
        int(bool(clamp)), int(bool(reverse)),
        _ptr(jlog) if jcap else None, jcap, _ptr(out3)))
    return int(out3[0]), int(out3[1]), int(out3[2])


def tree_energy(uval, uchild, vvals, vws, vchilds, d_max, lam, eps, gamma):
    out = np.zeros(1, dtype=np.float64)
    _check(lib().orc_tree_energy(
        _ptr(uval), _ptr(uchild), len(vvals), _ptr_array(vvals),
        _ptr_array(vws), _ptr_array(vchilds), d_max, lam, eps, gamma,
        _ptr(out)))
    return float(out[0])


# --------------------------------------------------------------- solver ----

@dataclass(frozen=True)
class Params:
    """FusionParams defaults (fusion.py:66-77)."""
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


def step_scale(t: int, p) -> float:
    """fusion.py:124-126"""
    return p.xi0 * 2.0 ** (-(t // p.halve_every))


def initial_field(wf_sum, w_sum, gamma):
    """fusion.py:149-155"""
    u = np.full(wf_sum.shape, -1.0, dtype=np.float64)
    seen = w_sum > 0
    u[seen] = wf_sum[seen] / (w_sum[seen] + gamma)
    return u


def solver_pool(u0: Pool, cap: int | None = None) -> Pool:
    """fusion.py:160-174: full-capacity f64 pool plus snap/joined scratch."""
    cap = full_tree_capacity(u0.d_max) if cap is None else cap
    used = u0.used
    value = np.zeros(cap, dtype=np.float64)
    value[:used] = u0.value[:used]
    child = np.full(cap, -1, dtype=np.int32)
    child[:used] = u0.child[:used]
    snap = np.zeros(cap, dtype=np.float64)
    snap[:used] = value[:used]
    return Pool(value, child, u0.state.copy(), u0.d_max, snap=snap,
                joined=np.zeros(cap, dtype=np.uint8))


@dataclass
class Stat:
    iteration: int
    energy: float
    node_count: int
    memory_bytes: int
    splits: int
    joins: int


@dataclass
class FuseOut:
    field: Pool
    stats: list = field(default_factory=list)
    join_log: np.ndarray | None = None


def fuse(u0: Pool, views: list, p, *, log_joins=False, reverse=False,
         cap: int | None = None) -> FuseOut:
    """fusion.py:186-241 driven through the C restatement."""
    u = solver_pool(u0, cap)
    vv = [v.value for v in views]
    vw = [v.weight for v in views]
    vc = [v.child for v in views]
    jbuf = np.zeros((u.value.shape[0] // 8 + 8, 12)) if log_joins else None
    stats, chunks = [], []
    for t in range(p.iterations):
        xi = step_scale(t, p)
        s, j, r = iterate_pass(u.value, u.snap, u.child, u.joined, u.state,
                               vv, vw, vc, u.d_max, p.lam, p.eps, p.gamma, xi,
                               p.tau_split, p.tau_join, p.clamp, reverse, jbuf)
        propagate(u.value, u.child)
        e = tree_energy(u.value, u.child, vv, vw, vc, u.d_max, p.lam, p.eps,
                        p.gamma)
        if jbuf is not None and r:
            chunks.append(jbuf[:r].copy())
        stats.append(Stat(t + 1, e, u.node_count, u.node_count * 20, s, j))
    jl = None
    if log_joins:
        jl = np.vstack(chunks) if chunks else np.zeros((0, 12))
    return FuseOut(u, stats, jl)


# ------------------------------------------------- primal-dual (unpinned) ----

def pd_steps(lam: float):
    """Default primal/dual step sizes: tau*sigma*||K||^2 < 1 with
    ||K|| <= lam*sqrt(12) at unit spacing."""
    t = 0.99 / (lam * np.sqrt(12.0))
    return t, t


def pd_pass(fields, child, used: int, views: list, d_max: int, lam: float,
            tau: float, sigma: float, gamma: float, clamp: bool = True):
    """One primal-dual pass (pd_oracle.c orc_pd_pass) on the five f64 pools
    (u, ubar, px, py, pz) followed by the propagate of each output.
    Returns (outputs, energy of the incoming u)."""
    vv = [v.value for v in views]
    vw = [v.weight for v in views]
    vc = [v.child for v in views]
    outs = [np.array(a, dtype=np.float64, copy=True) for a in fields]
    e = np.zeros(1)
    _check(lib().orc_pd_pass(
        *[_ptr(a) for a in fields], *[_ptr(o) for o in outs], _ptr(child),
        int(used), len(views), _ptr_array(vv), _ptr_array(vw),
        _ptr_array(vc), d_max, float(lam), float(tau), float(sigma),
        float(gamma), int(bool(clamp)), _ptr(e)))
    for o in outs:
        propagate(o, child)
    return outs, float(e[0])


def pd_fuse(u0: Pool, views: list, lam: float, gamma: float, iterations: int,
            tau: float | None = None, sigma: float | None = None,
            clamp: bool = True, tau_split: float | None = None,
            tau_join: float | None = None, cap: int | None = None):
    """TV-L1 primal-dual schedule (pd_oracle.c definition, PARITY UNPINNED).
    Frozen tree unless tau_split/tau_join are given: then every pass is
    followed by orc_pd_restructure (split/join, pd_oracle.c).  Returns
    (u, ubar, px, py, pz, energies_pre) -- arrays over the pool's slots --
    and, when restructuring, also (child, state, [(splits, joins)])."""
    if tau is None or sigma is None:
        tau, sigma = pd_steps(lam)
    used = u0.used
    rs = tau_split is not None or tau_join is not None
    n = (cap or full_tree_capacity(u0.d_max)) if rs else used
    def pool(a):
        out = np.zeros(n)
        out[:used] = a
        return out
    u = pool(u0.value[:used].astype(np.float64))
    ub = u.copy()
    px, py, pz = pool(0.0), pool(0.0), pool(0.0)
    child = np.full(n, -1, dtype=np.int32)
    child[:used] = u0.child[:used]
    state = np.array(u0.state[:3], dtype=np.int64)
    energies, sj = [], []
    out2 = np.zeros(2, dtype=np.int64)
    for _ in range(iterations):
        outs, en = pd_pass((u, ub, px, py, pz), child, int(state[0]), views,
                           u0.d_max, lam, tau, sigma, gamma, clamp)
        energies.append(en)
        u, ub, px, py, pz = outs
        if rs:
            _check(lib().orc_pd_restructure(
                _ptr(u), _ptr(ub), _ptr(px), _ptr(py), _ptr(pz), _ptr(child),
                _ptr(state), n, u0.d_max,
                float(-1.0 if tau_split is None else tau_split),
                float(2.0 if tau_join is None else tau_join), _ptr(out2)))
            sj.append((int(out2[0]), int(out2[1])))
    if rs:
        return u, ub, px, py, pz, energies, child, state, sj
    return u, ub, px, py, pz, energies


# ------------------------------------------------------------ traversal ----

def leaves(pool: Pool):
    """(node, level, x, y, z) in the canonical order (octree.py:168-181):
    ascending x-major Morton order."""
    stack = [(0, 0, 0, 0, 0)]
    ch = pool.child
    out = []
    while stack:
        n, l, x, y, z = stack.pop()
        b = int(ch[n])
        if b < 0:
            out.append((n, l, x, y, z))
        else:
            for c in range(7, -1, -1):
                stack.append((b + c, l + 1, 2 * x + ((c >> 2) & 1),
                              2 * y + ((c >> 1) & 1), 2 * z + (c & 1)))
    return out


def serialize_lines(pool: Pool) -> list:
    """octree.py:413-431 as a list of lines (pre-order, %.17g)."""
    lines = []
    stack = [(0, 0, 0, 0, 0)]
    while stack:
        n, l, x, y, z = stack.pop()
        b = int(pool.child[n])
        wt = float(pool.weight[n]) if pool.weight is not None else 0.0
        lines.append(f"{l} {x} {y} {z} {int(b < 0)} "
                     f"{float(pool.value[n]):.17g} {wt:.17g}")
        if b >= 0:
            for c in range(7, -1, -1):
                stack.append((b + c, l + 1, 2 * x + ((c >> 2) & 1),
                              2 * y + ((c >> 1) & 1), 2 * z + (c & 1)))
    return lines


# ----------------------------------------------------------------- TSDF ----

def build_view_tsdf(depth, cam, origin, voxel_size, n, delta, eta):
    """Per-voxel projective TSDF (tsdf.py:87-120), numpy op order.

    ``cam`` is any object with fx, fy, cx, cy, width, height, rotation (3x3
    camera-to-world) and translation (camera centre).
    Returns (f float32, w uint8).
    """
    if delta <= 0 or eta <= 0:
        raise ValueError("delta and eta must be positive")
    ax = [origin[a] + (np.arange(n) + 0.5) * voxel_size for a in range(3)]
    t = np.asarray(cam.translation, dtype=np.float64)
    r = np.asarray(cam.rotation, dtype=np.float64)
    xs = ax[0][:, None, None] - t[0]
    ys = ax[1][None, :, None] - t[1]
    zs = ax[2][None, None, :] - t[2]
    xc = xs * r[0, 0] + ys * r[1, 0] + zs * r[2, 0]
    yc = xs * r[0, 1] + ys * r[1, 1] + zs * r[2, 1]
    zc = xs * r[0, 2] + ys * r[1, 2] + zs * r[2, 2]
    front = zc > 0
    zs_ = np.where(front, zc, 1.0)
    u = cam.fx * xc / zs_ + cam.cx
    v = cam.fy * yc / zs_ + cam.cy
    inside = front & (u >= 0) & (u < cam.width) & (v >= 0) & (v < cam.height)
    pu = np.clip(np.floor(u + 0.5), 0, cam.width - 1).astype(np.intp)
    pv = np.clip(np.floor(v + 0.5), 0, cam.height - 1).astype(np.intp)
    d = np.asarray(depth, dtype=np.float32)[pv, pu].astype(np.float64)
    obs = inside & (d > 0)
    uu = (np.arange(cam.width) - cam.cx) / cam.fx
    vv = (np.arange(cam.height) - cam.cy) / cam.fy
    norms = np.sqrt(1.0 + uu[None, :] ** 2 + vv[:, None] ** 2)[pv, pu]
    dist = np.sqrt(xc * xc + yc * yc + zc * zc)
    phi = d * norms - dist
    f = np.clip(phi / delta, -1.0, 1.0)
    w = obs & (phi >= -eta)
    f = np.where(w, f, -1.0).astype(np.float32)
    return f, w.astype(np.uint8)


# ------------------------------------------------------------ mesh readout --

def extract_zero_surface(values, mask, tables):
    """mesh.py:63-111 restated (numpy): per 2x2x2 cube of the cell-centred
    grid, the inside pattern (value < 0, bit c = corner (c>>2&1, c>>1&1,
    c&1)); cubes with all corners observed emit their case's triangles; each
    triangle corner is a grid edge keyed ((axis*n + x)*n + y)*n + z;
    vertices are the sorted unique keys, faces their ranks, positions the
    linear zero crossing along the edge.  ``tables`` = (tri_table,
    tri_count, edge_axis, edge_cell_offset)."""
    tri, cnt, eax, eoff = (np.asarray(t) for t in tables)
    v = np.asarray(values, dtype=np.float64)
    n = v.shape[0]
    m = n - 1
    case = np.zeros((m, m, m), dtype=np.int64)
    ok = np.ones((m, m, m), dtype=bool)
    for c in range(8):
        dx, dy, dz = (c >> 2) & 1, (c >> 1) & 1, c & 1
        case |= (v[dx:dx + m, dy:dy + m, dz:dz + m] < 0).astype(np.int64) << c
        if mask is not None:
            ok &= np.asarray(mask)[dx:dx + m, dy:dy + m, dz:dz + m]
    ntri = cnt.astype(np.int64)[case] * ok
    cx, cy, cz = np.nonzero(ntri)
    if cx.size == 0:
        return np.zeros((0, 3)), np.zeros((0, 3), dtype=np.int32)
    k3 = 3 * ntri[cx, cy, cz]
    cube = np.repeat(np.arange(cx.size), k3)
    slot = np.arange(cube.size) - np.repeat(np.cumsum(k3) - k3, k3)
    e = tri.astype(np.int64)[case[cx, cy, cz][cube], slot]
    ax = eax.astype(np.int64)[e]
    off = eoff.astype(np.int64)[e]
    key = ((ax * n + cx[cube] + off[:, 0]) * n + cy[cube] + off[:, 1]) * n \
        + cz[cube] + off[:, 2]
    ukey, inv = np.unique(key, return_inverse=True)
    gz, gy, gx = ukey % n, (ukey // n) % n, (ukey // (n * n)) % n
    ga = ukey // (n * n * n)
    v0 = v[gx, gy, gz]
    v1 = v[gx + (ga == 0), gy + (ga == 1), gz + (ga == 2)]
    t = v0 / (v0 - v1)
    verts = np.column_stack([gx + t * (ga == 0), gy + t * (ga == 1),
                             gz + t * (ga == 2)])
    return verts, inv.reshape(-1, 3).astype(np.int32)


# ------------------------------------------------------------ dense solver --

def dense_step(u, fs, ws, p, xi):
    """fusion.py:283-298 restated: forward differences (0 at the far
    border), flux g/sqrt(|g|^2+eps^2), backward-difference divergence, data
    term summed in view order, Jacobi step, clamp."""
    eps2 = p.eps * p.eps
    g = [np.zeros_like(u) for _ in range(3)]
    g[0][:-1] = u[1:] - u[:-1]
    g[1][:, :-1] = u[:, 1:] - u[:, :-1]
    g[2][:, :, :-1] = u[:, :, 1:] - u[:, :, :-1]
    gn = np.sqrt(g[0] * g[0] + g[1] * g[1] + g[2] * g[2] + eps2)
    q = [gi / gn for gi in g]
    div = (np.diff(q[0], axis=0, prepend=0.0) + np.diff(q[1], axis=1, prepend=0.0)
           + np.diff(q[2], axis=2, prepend=0.0))
    num = np.zeros_like(u)
    den = np.full_like(u, p.gamma)
    for f, w in zip(fs, ws):
        wv = w.astype(np.float64)
        d = u - f.astype(np.float64)
        num += np.where(wv != 0.0, wv * d / np.sqrt(d * d + eps2), 0.0)
        den += wv
    un = u + xi * (p.lam * div - num / den)
    return np.clip(un, -1.0, 1.0) if p.clamp else un


def dense_fuse(u0, fs, ws, p):
    u = np.array(u0, dtype=np.float64)
    for t in range(p.iterations):
        u = dense_step(u, fs, ws, p, step_scale(t, p))
    return u
