"""Seeded synthetic inputs for BASELINE.json's configs (host-side numpy).

Input generation is outside the accelerated path; these
generators exist so the GPU path, the CPU oracle and the reference all see
the same bytes.  Assumptions the BASELINE config text leaves open are the
ones SURVEY.md §8(d) / Appendix B lists, restated next to each generator.

Cameras follow the reference conventions: ``look_at`` builds a
camera-to-world rotation whose columns are (right, down, forward)
(reference ``volume.py:154-170``), depths are camera-frame z
(``volume.py:1-7``), and the principal point is ((W-1)/2, (H-1)/2)
(``synth.py:131``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

__all__ = ["look_at", "PinholeCamera", "sphere_depth", "Cfg1Scene",
           "make_cfg1", "torus_sdf", "make_cfg2_samples", "cfg5_tree",
           "cfg5_inputs", "DepthScene", "value_noise", "sphere_trace",
           "trace_blob", "trace_room", "room_objects_array", "make_cfg3",
           "make_cfg4"]


def look_at(position, target, up=(0.0, 0.0, 1.0)) -> np.ndarray:
    """Camera-to-world rotation looking from ``position`` at ``target``."""
    pos = np.asarray(position, dtype=np.float64)
    fwd = np.asarray(target, dtype=np.float64) - pos
    fwd = fwd / np.linalg.norm(fwd)
    up = np.asarray(up, dtype=np.float64)
    if abs(float(np.dot(fwd, up)) / np.linalg.norm(up)) > 0.999:
        up = np.array([1.0, 0.0, 0.0])
    right = np.cross(fwd, up)
    right = right / np.linalg.norm(right)
    down = np.cross(fwd, right)
    return np.column_stack([right, down, fwd])


@dataclass
class PinholeCamera:
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    rotation: np.ndarray      # 3x3 camera-to-world
    translation: np.ndarray   # camera centre, world

    @property
    def center(self):
        return self.translation


def sphere_depth(cam: PinholeCamera, center, radius) -> np.ndarray:
    """Camera-frame z of the first hit of each pixel ray on a sphere, 0 on a
    miss (the exact ray/sphere depth of reference ``synth.py:80-109``)."""
    c = np.asarray(center, dtype=np.float64)
    px = (np.arange(cam.width, dtype=np.float64) - cam.cx) / cam.fx
    py = (np.arange(cam.height, dtype=np.float64) - cam.cy) / cam.fy
    dirs = np.empty((cam.height, cam.width, 3))
    dirs[..., 0] = px[None, :]
    dirs[..., 1] = py[:, None]
    dirs[..., 2] = 1.0
    d = dirs @ cam.rotation.T          # world directions with unit cam-z
    oc = cam.translation - c
    a = np.sum(d * d, axis=-1)
    b = 2.0 * np.sum(d * oc, axis=-1)
    k = float(oc @ oc) - radius * radius
    disc = b * b - 4.0 * a * k
    hit = disc >= 0.0
    root = (-b - np.sqrt(np.where(hit, disc, 0.0))) / (2.0 * a)
    return np.where(hit & (root > 0.0), root, 0.0)


@dataclass
class Cfg1Scene:
    origin: tuple
    voxel_size: float
    resolution: int
    cameras: list
    depths: list              # float32 (H, W)
    delta: float
    eta: float
    lam: float
    iterations: int


def make_cfg1(seed: int = 0, n_views: int = 8, width: int = 160,
              height: int = 120, focal: float = 150.0, d_max: int = 6,
              noise: float = 1e-3) -> Cfg1Scene:
    """BASELINE config 0 ("CPU-oracle scene").

    Sphere r=0.3 at the centre of the unit cube, ``n_views`` cameras on a
    horizontal ring of radius 1.0 in the z=0.5 plane (assumed) at angles
    2*pi*k/n, looking at the centre; fx=fy=150; depth noise N(0, noise) drawn
    per view in view order from ``default_rng(seed)`` and added to hit pixels
    only, negatives clamped to 0; misses stay 0 (no background sphere).
    delta=0.05, eta=0.25 (assumed 5*delta), lambda=0.5, 50 iterations.
    """
    rng = np.random.default_rng(seed)
    centre = np.array([0.5, 0.5, 0.5])
    cams, depths = [], []
    for k in range(n_views):
        ang = 2.0 * math.pi * k / n_views
        pos = centre + np.array([math.cos(ang), math.sin(ang), 0.0])
        cam = PinholeCamera(focal, focal, (width - 1) / 2.0,
                            (height - 1) / 2.0, width, height,
                            look_at(pos, centre), pos)
        z = sphere_depth(cam, centre, 0.3)
        eps = rng.normal(0.0, noise, z.shape)
        z = np.where(z > 0, np.maximum(z + eps, 0.0), 0.0)
        cams.append(cam)
        depths.append(z.astype(np.float32))
    n = 1 << d_max
    return Cfg1Scene((0.0, 0.0, 0.0), 1.0 / n, n, cams, depths,
                     delta=0.05, eta=0.25, lam=0.5, iterations=50)


def torus_sdf(p, centre=(0.5, 0.5, 0.5), R=0.3, r=0.1):
    """Signed distance to a torus around the z axis through ``centre``."""
    x = p[..., 0] - centre[0]
    y = p[..., 1] - centre[1]
    z = p[..., 2] - centre[2]
    q = np.sqrt(x * x + y * y) - R
    return np.sqrt(q * q + z * z) - r


def make_cfg2_samples(d_max: int = 8, n_samples: int = 16, seed: int = 0,
                      p_invalid: float = 0.1):
    """BASELINE config 1 ("fixed-structure solver test") per-leaf samples.

    Full tree at depth ``d_max``; leaf centres (i+0.5)/2^d.  For sample v:
    f_v = clip(sd + N(0, 0.01), -0.04, 0.04) as float32 (noise added to the
    torus signed distance: assumed), w_v ~ Bernoulli(1-p_invalid) per
    (leaf, sample), f_v = -1 where w_v = 0.  Draw order: for v in 0..N-1 the
    noise grid then the validity grid, from ``default_rng(seed)``.
    Returns (fs, ws): lists of dense (n,n,n) float32 / uint8 grids.
    """
    n = 1 << d_max
    rng = np.random.default_rng(seed)
    c = (np.arange(n) + 0.5) / n
    p = np.stack(np.meshgrid(c, c, c, indexing="ij"), axis=-1)
    sd = torus_sdf(p)
    del p
    fs, ws = [], []
    for _ in range(n_samples):
        f = np.clip(sd + rng.normal(0.0, 0.01, sd.shape), -0.04, 0.04)
        w = (rng.random(sd.shape) >= p_invalid).astype(np.uint8)
        f = np.where(w > 0, f, -1.0).astype(np.float32)
        fs.append(f)
        ws.append(w)
    return fs, ws


def cfg5_tree(n_target: int = 100_000_000, d_max: int = 12, seed: int = 0,
              n_spheres: int | None = None, device="cpu",
              radius_scale: float | None = None):
    """BASELINE config 4 ("solver microbenchmark") structure: a random adaptive
    octree refined around a random implicit surface (union of ``n_spheres``
    spheres, assumed; default 256 at 100M leaves / depth 12, scaled with the
    leaf count per finest-level area so radii stay comparable), built
    directly as a reference-layout pool.

    A cell at level L < d_max splits iff |sd(centre)| < a_L * h_L * sqrt(3)/2
    (h_L = cell edge), with a_L = 1 above level d_max-2 (every cell the
    surface may cross) and thinner bands a = 0.55 / 0.24 at the last two
    levels, which puts roughly 60/30/10 % of the leaves at depths 12/11/10
    (the real histogram is returned).  ``radius_scale`` (default: calibrated
    from a depth-9 pilot) sets the surface area and so the leaf count.
    Slots are assigned breadth-first (children of the k-th inner node of the
    whole tree at 1 + 8k) -- a valid pool layout in which every level is in
    Morton order.  Returns (child int32 tensor, d_max, level histogram dict).
    """
    import torch
    if n_spheres is None:
        n_spheres = int(min(256, max(8, round(
            256 * n_target / 1e8 * 4.0 ** (12 - d_max)))))
    g = torch.Generator().manual_seed(seed)
    centres = (torch.rand((n_spheres, 3), generator=g, dtype=torch.float64)
               * 0.8 + 0.1).to(device)
    radii0 = (torch.rand(n_spheres, generator=g, dtype=torch.float64)
              * 0.04 + 0.02).to(device)

    def build(scale, depth):
        radii = radii0 * scale
        levels = []   # per level: split flags (bool tensor)
        x = torch.zeros(1, dtype=torch.int64, device=device)
        y = torch.zeros_like(x)
        z = torch.zeros_like(x)
        hist = {}
        for L in range(depth + 1):
            n = x.numel()
            if L == depth:
                levels.append(torch.zeros(n, dtype=torch.bool, device=device))
                hist[L] = n
                break
            h = 1.0 / (1 << L)
            a = 1.0 if L < depth - 2 else (0.55 if L == depth - 2 else 0.24)
            split = torch.empty(n, dtype=torch.bool, device=device)
            for lo in range(0, n, 1 << 20):   # bound the [cells, spheres] temp
                hi = min(n, lo + (1 << 20))
                p = torch.stack([(x[lo:hi].double() + 0.5) * h,
                                 (y[lo:hi].double() + 0.5) * h,
                                 (z[lo:hi].double() + 0.5) * h], dim=1)
                dist = ((p[:, None, :] - centres[None, :, :]) ** 2).sum(-1).sqrt()
                sd = (dist - radii[None, :]).min(dim=1).values
                split[lo:hi] = sd.abs() < a * h * 0.8660254037844386
            levels.append(split)
            hist[L] = int((~split).sum())
            px, py, pz = x[split], y[split], z[split]
            c = torch.arange(8, device=device)
            x = (2 * px[:, None] + ((c >> 2) & 1)).reshape(-1)
            y = (2 * py[:, None] + ((c >> 1) & 1)).reshape(-1)
            z = (2 * pz[:, None] + (c & 1)).reshape(-1)
        return levels, hist

    if radius_scale is None:
        # pilot at depth d_max-3 (leaf count ~ area * 4^depth), then secant
        # steps at full depth on log(count) vs log(scale): overlapping
        # spheres make the count grow slower than radius^2
        _, hp = build(1.0, d_max - 3)
        s0 = (n_target / (sum(hp.values()) * 64.0)) ** 0.5
        _, h0 = build(s0, d_max)
        n0 = sum(h0.values())
        s1 = s0 * (n_target / n0) ** 0.5
        for _ in range(2):
            _, h1 = build(s1, d_max)
            n1 = sum(h1.values())
            if abs(n1 - n_target) < 0.01 * n_target or n1 == n0:
                break
            alpha = math.log(n1 / n0) / math.log(s1 / s0)
            alpha = min(max(alpha, 1.0), 2.5)
            s0, n0 = s1, n1
            s1 = s1 * min(max((n_target / n1) ** (1.0 / alpha), 0.5), 2.0)
        radius_scale = s1
    levels, hist = build(radius_scale, d_max)
    # breadth-first slots: level-L nodes sit at 1 + 8*R_{L-1} + j
    used = 1 + 8 * sum(int(s.sum()) for s in levels)
    child = torch.full((used,), -1, dtype=torch.int32, device=device)
    start, inner_before = 0, 0
    for L, split in enumerate(levels):
        n = split.numel()
        slots = torch.arange(start, start + n, device=device)
        k = torch.cumsum(split.to(torch.int64), 0) - 1 + inner_before
        child[slots[split]] = (1 + 8 * k[split]).to(torch.int32)
        inner_before += int(split.sum())
        # the next level's nodes are the children of this level's inner
        # nodes: their blocks start at 1 + 8 * (inner nodes before level L)
        start = 1 + 8 * (inner_before - int(split.sum()))
    return child, d_max, {"leaves_per_level": hist,
                          "leaves": sum(hist.values()), "nodes": used,
                          "radius_scale": radius_scale}


def cfg5_inputs(n_target: int = 100_000_000, nviews: int = 32, seed: int = 0,
                device="cuda", d_max: int = 12, radius_scale=None):
    """Config 4's solver microbenchmark inputs on ``device``: the tree of
    ``cfg5_tree``, N = ``nviews`` per-leaf fp32 samples U(-1, 1), all valid,
    as a per-slot [nviews, nodes] array (the solver's ``samples=``), and
    u0 = the initial field (sum f / (N + gamma), reference fusion.py:149-155)
    with inner nodes propagated.  Returns (u0 OctreeField, (F_slot, None),
    info)."""
    import torch
    from .octree import OctreeField, propagate_means
    from ._device import pool_empty
    child, d, info = cfg5_tree(n_target, d_max, seed, device=device,
                               radius_scale=radius_scale)
    used = child.numel()
    g = torch.Generator(device=device).manual_seed(seed + 1)
    F = torch.empty((nviews, used), dtype=torch.float32, device=device)
    F.uniform_(-1.0, 1.0, generator=g)
    fsum = torch.zeros(used, dtype=torch.float64, device=device)
    for v in range(nviews):          # view order, f64 (cli.py:148-149)
        fsum += F[v].double()
    u = fsum / (nviews + 1e-4)
    value = pool_empty(used, torch.float64)
    value.copy_(u)
    ch = pool_empty(used, torch.int32)
    ch.copy_(child)
    state = np.array([used, -1, used], dtype=np.int64)
    u0 = OctreeField(value, ch, state, d)
    propagate_means(u0)
    return u0, (F, None), info



# ------------------------------------------------------------------ cfg3/cfg4
# Depth-map configs rendered by sphere tracing (the reference renders only
# spheres, synth.py:80-109; SURVEY.md §8(d) notes that cfg3/cfg4 need a
# tracer).  Rendering is input generation, outside the accelerated path: it
# runs as torch f64 array code on ``device`` so the GPU and the CPU oracle
# consume the same depth maps.

@dataclass
class DepthScene:
    """Depth maps + cameras + volume + solver settings of one config."""
    name: str
    origin: tuple
    voxel_size: float
    resolution: int
    cameras: list             # PinholeCamera
    depths: list              # float32 (H, W), camera-frame z, 0 = no return
    params: dict              # FusionParams keyword arguments

    @property
    def d_max(self) -> int:
        return self.resolution.bit_length() - 1


def _lattice(seed: int, n: int, device):
    import torch
    g = torch.Generator().manual_seed(seed)
    return (torch.rand((n, n, n), generator=g, dtype=torch.float64) * 2.0
            - 1.0).to(device)


def value_noise(p, tables, base_freq: float = 4.0):
    """Lattice value noise: per octave o (frequency base_freq*2^o, amplitude
    2^-o) trilinear interpolation with smoothstep fade of U(-1,1) lattice
    values; octave sum divided by the amplitude sum, so n(p) in [-1, 1]
    (assumed form of BASELINE config 2's '3-octave value noise')."""
    import torch
    out = torch.zeros(p.shape[:-1], dtype=torch.float64, device=p.device)
    amp, total = 1.0, 0.0
    for o, tab in enumerate(tables):
        fr = base_freq * (1 << o)
        q = p.clamp(0.0, 1.0) * fr
        i0 = q.floor().clamp(max=tab.shape[0] - 2).long()
        t = q - i0
        t = t * t * (3.0 - 2.0 * t)
        acc = torch.zeros_like(out)
        for c in range(8):
            dx, dy, dz = (c >> 2) & 1, (c >> 1) & 1, c & 1
            wgt = ((t[..., 0] if dx else 1.0 - t[..., 0])
                   * (t[..., 1] if dy else 1.0 - t[..., 1])
                   * (t[..., 2] if dz else 1.0 - t[..., 2]))
            acc = acc + wgt * tab[i0[..., 0] + dx, i0[..., 1] + dy, i0[..., 2] + dz]
        out = out + amp * acc
        total += amp
        amp *= 0.5
    return out * (1.0 / total)


def _norm3(v):
    """|v| over the last axis (size 3) as ((x*x + y*y) + z*z).sqrt()."""
    return ((v[..., 0] * v[..., 0] + v[..., 1] * v[..., 1])
            + v[..., 2] * v[..., 2]).sqrt()


def sphere_trace(sdf, cam: PinholeCamera, *, lipschitz: float, t_max: float,
                 device, steps: int = 400, eps: float = 1e-7):
    """Camera-frame z of the first surface hit of each pixel ray (0 = miss)
    for a signed distance bound ``sdf`` with Lipschitz constant <=
    ``lipschitz``: conservative steps sd/L, then 40 bisection steps on the
    last bracket.  Rays have unit camera-z component (as sphere_depth), so
    the ray parameter is the depth."""
    import torch
    H, W = cam.height, cam.width
    # (x - c) * (1 / f): what torch's CUDA division by a host scalar computes
    # (the golden depth maps were made with it), written out so that every
    # device and the CUDA kernels evaluate the same expression
    px = (torch.arange(W, dtype=torch.float64, device=device) - cam.cx) * (1.0 / cam.fx)
    py = (torch.arange(H, dtype=torch.float64, device=device) - cam.cy) * (1.0 / cam.fy)
    dirs = torch.stack(torch.broadcast_tensors(px[None, :], py[:, None],
                                               torch.ones((), dtype=torch.float64,
                                                          device=device)), -1)
    R = np.asarray(cam.rotation, dtype=np.float64)
    dr = dirs.reshape(-1, 3)
    # world directions R @ dir as separate IEEE ops (no matmul / reduction
    # kernels, whose order differs between devices and runs): the maps are
    # reproducible on any GPU, and the CUDA kernels (trace_blob / trace_room)
    # give the same bits.  (torch's CPU f64 sqrt is not correctly rounded, so
    # a CPU trace may differ in the last place; the golden fixtures' depth
    # maps were dumped from the device, tools/dump_depths.py.)
    d = torch.stack([(dr[:, 0] * float(R[j, 0]) + dr[:, 1] * float(R[j, 1]))
                     + dr[:, 2] * float(R[j, 2]) for j in range(3)], 1)
    o = torch.as_tensor(cam.translation, dtype=torch.float64, device=device)
    nrm = _norm3(d)
    t = torch.zeros(d.shape[0], dtype=torch.float64, device=device)
    alive = torch.ones_like(t, dtype=torch.bool)
    hit = torch.zeros_like(alive)
    t_prev = t.clone()
    idx = alive.nonzero().squeeze(1)
    for it in range(steps):
        if it % 16 == 0:   # re-compact the live rays now and then (host sync)
            idx = alive.nonzero().squeeze(1)
            if idx.numel() == 0:
                break
        sd = sdf(o + t[idx, None] * d[idx])
        a = alive[idx]
        h = a & (sd < eps)
        go = a & ~h
        hit[idx] = hit[idx] | h
        tp = t[idx]
        tn = torch.where(go, tp + sd / (lipschitz * nrm[idx]), tp)
        t_prev[idx] = torch.where(go, tp, t_prev[idx])
        t[idx] = tn
        alive[idx] = go & (tn <= t_max)
    # bisection between the last outside point and the hit point
    idx = hit.nonzero().squeeze(1)
    lo, hi = t_prev[idx], t[idx]
    for _ in range(40):
        mid = 0.5 * (lo + hi)
        inside = sdf(o + mid[:, None] * d[idx]) < 0.0
        hi = torch.where(inside, mid, hi)
        lo = torch.where(inside, lo, mid)
    z = torch.zeros_like(t)
    z[idx] = hi
    return z.reshape(H, W)


def _is_cuda(device) -> bool:
    import torch
    return torch.device(device).type == "cuda"


def _cam_params(cam: PinholeCamera) -> np.ndarray:
    return np.ascontiguousarray(np.concatenate([
        [cam.fx, cam.fy, cam.cx, cam.cy],
        np.asarray(cam.rotation, dtype=np.float64).ravel(),
        np.asarray(cam.translation, dtype=np.float64).ravel()]))


def trace_blob(cam: PinholeCamera, tables, *, centre=(0.5, 0.5, 0.5),
               radius: float = 0.35, amp: float = 0.03,
               base_freq: float = 4.0, lipschitz: float, t_max: float,
               steps: int = 400, eps: float = 1e-7):
    """``sphere_trace`` of the noisy blob as one CUDA kernel, a thread per
    pixel ray (``octf_trace_blob``, csrc/scenes.cu): the same f64 operations
    in the same order, so the map equals the array program's bit for bit
    (``tests/test_gpu_cfg34.py::test_trace_kernels_match_array_program``)."""
    import torch
    from . import _lib
    from ._device import ptr, stream_handle
    z = torch.empty((cam.height, cam.width), dtype=torch.float64,
                    device=tables[0].device)
    tabs = [t.contiguous() for t in tables]
    lat = _lib.ptr_table([ptr(t) for t in tabs])
    lat_n = np.array([t.shape[0] for t in tabs], dtype=np.int32)
    cp = _cam_params(cam)
    c = np.ascontiguousarray(np.asarray(centre, dtype=np.float64))
    _lib.call("octf_trace_blob", cp.ctypes.data, cam.width, cam.height,
              c.ctypes.data, float(radius), float(amp), float(base_freq), lat,
              lat_n.ctypes.data, len(tabs), float(lipschitz), float(t_max),
              int(steps), float(eps), ptr(z), stream_handle())
    return z


def trace_room(cam: PinholeCamera, objects, n_box: int, n_sph: int, *,
               size: float = 4.0, lipschitz: float = 1.0, t_max: float,
               steps: int = 400, eps: float = 1e-7):
    """``sphere_trace`` of the room (``octf_trace_room``): ``objects`` is the
    device array of ``room_objects_array``; the object list is staged in
    shared memory once per CTA."""
    import torch
    from . import _lib
    from ._device import ptr, stream_handle
    z = torch.empty((cam.height, cam.width), dtype=torch.float64,
                    device=objects.device)
    cp = _cam_params(cam)
    _lib.call("octf_trace_room", cp.ctypes.data, cam.width, cam.height,
              ptr(objects), int(n_box), int(n_sph), float(size),
              float(lipschitz), float(t_max), int(steps), float(eps), ptr(z),
              stream_handle())
    return z


def room_objects_array(objs, device):
    """Boxes {centre, half extents} then spheres {centre, radius} as one flat
    f64 device array, and the two counts."""
    import torch
    boxes = [np.concatenate([c, h]) for k, c, h in objs if k == "box"]
    sph = [np.concatenate([c, [r]]) for k, c, r in objs if k == "sphere"]
    flat = np.concatenate([np.ravel(boxes), np.ravel(sph)]).astype(np.float64)
    return (torch.tensor(flat, dtype=torch.float64, device=device),
            len(boxes), len(sph))


def fibonacci_hemisphere(n: int) -> np.ndarray:
    """n unit directions with z > 0 on a Fibonacci spiral (assumed viewpoint
    layout of config 2's 'hemisphere of viewpoints')."""
    k = np.arange(n) + 0.5
    z = 1.0 - k / n                       # (0, 1]: upper hemisphere
    r = np.sqrt(np.maximum(0.0, 1.0 - z * z))
    phi = k * math.pi * (3.0 - math.sqrt(5.0))
    return np.stack([r * np.cos(phi), r * np.sin(phi), z], axis=1)


def _add_noise(z, sigma, rng):
    """N(0, sigma) on returns (sigma may be an array), negatives -> 0."""
    eps = rng.normal(0.0, 1.0, z.shape) * sigma
    return np.where(z > 0, np.maximum(z + eps, 0.0), 0.0).astype(np.float32)


def make_cfg3(d_max: int = 9, n_views: int = 64, width: int = 640,
              height: int = 480, focal: float = 525.0, seed: int = 0,
              device="cuda") -> DepthScene:
    """BASELINE config 2 ("adaptive single object").

    Unit cube, blob sd(p) = |p - c| - (0.35 + 0.03 n(p)), c = (.5,.5,.5), n =
    3-octave value noise (base frequency 4, lattices from ``seed``); 64
    cameras at distance 1.2 from c along Fibonacci directions of the upper
    hemisphere, looking at c (assumed); 640x480, fx = fy = 525, principal
    point (319.5, 239.5) (assumed); depth noise N(0, 2e-3) on returns,
    drawn per view in view order from ``default_rng(seed)``; delta = 0.02,
    eta = 0.1 (assumed), lambda = 0.3 (assumed default), tau_split = 0.1,
    tau_join = 0.5 (split/join every pass), 300 iterations.
    """
    import torch
    tables = [_lattice(seed * 7 + o, 4 * (1 << o) + 2, device) for o in range(3)]
    c = torch.tensor([0.5, 0.5, 0.5], dtype=torch.float64, device=device)

    def sdf(p):
        return _norm3(p - c) - (0.35 + 0.03 * value_noise(p, tables))

    # |grad n| <= sum_o a_o * 1.5 * 2 * f_o / sum_o a_o (smoothstep slope 1.5,
    # lattice range 2) = 20.6; L = 1 + 0.03 * 20.6 < 1.7
    rng = np.random.default_rng(seed)
    cams, depths = [], []
    centre = np.array([0.5, 0.5, 0.5])
    for k, dvec in enumerate(fibonacci_hemisphere(n_views)):
        pos = centre + 1.2 * dvec
        cam = PinholeCamera(focal, focal, (width - 1) / 2.0, (height - 1) / 2.0,
                            width, height, look_at(pos, centre), pos)
        if _is_cuda(device):
            z = trace_blob(cam, tables, lipschitz=1.7, t_max=3.0)
        else:   # no device: the array program
            z = sphere_trace(sdf, cam, lipschitz=1.7, t_max=3.0, device=device)
        cams.append(cam)
        depths.append(_add_noise(z.cpu().numpy(), 2e-3, rng))
    n = 1 << d_max
    return DepthScene("cfg3", (0.0, 0.0, 0.0), 1.0 / n, n, cams, depths,
                      dict(delta=0.02, eta=0.1, lam=0.3, tau_split=0.1,
                           tau_join=0.5, iterations=300))


def _room_objects(seed: int, n_objects: int, size: float):
    """200 axis-aligned boxes and spheres (50/50, assumed), extent U(0.1,
    0.8) m (box edges drawn independently, sphere diameter), fully inside
    the ``size`` m cube."""
    rng = np.random.default_rng(seed)
    objs = []
    for _ in range(n_objects):
        if rng.random() < 0.5:
            e = rng.uniform(0.1, 0.8, 3)
            lo = rng.uniform(0.0, size - e)
            objs.append(("box", lo + e / 2.0, e / 2.0))
        else:
            dia = rng.uniform(0.1, 0.8)
            ctr = rng.uniform(dia / 2.0, size - dia / 2.0, 3)
            objs.append(("sphere", ctr, dia / 2.0))
    return objs


def room_sdf_fn(objs, device, size: float = 4.0):
    """Union SDF of the objects and the room's six walls (the inside of the
    ``size`` m cube; exact for boxes, spheres and walls)."""
    import torch
    boxes = [(c, h) for k, c, h in objs if k == "box"]
    sph = [(c, r) for k, c, r in objs if k == "sphere"]
    bc = torch.tensor(np.array([b[0] for b in boxes]), dtype=torch.float64, device=device)
    bh = torch.tensor(np.array([b[1] for b in boxes]), dtype=torch.float64, device=device)
    sc = torch.tensor(np.array([s[0] for s in sph]), dtype=torch.float64, device=device)
    sr = torch.tensor(np.array([s[1] for s in sph]), dtype=torch.float64, device=device)

    def sdf(p):
        if p.shape[0] == 0:
            return torch.zeros(0, dtype=torch.float64, device=p.device)
        out = None
        for lo in range(0, p.shape[0], 1 << 16):
            q = p[lo:lo + (1 << 16)]
            dq = (q[:, None, :] - bc[None]).abs() - bh[None]
            outside = _norm3(dq.clamp(min=0.0))
            inside = dq.max(dim=-1).values.clamp(max=0.0)
            db = (outside + inside).min(dim=1).values
            ds = (_norm3(q[:, None, :] - sc[None]) - sr[None]).min(dim=1).values
            walls = torch.minimum(q, size - q).min(dim=1).values
            r = torch.minimum(torch.minimum(db, ds), walls)
            out = r if out is None else torch.cat([out, r])
        return out
    return sdf


def _catmull_rom(pts, n):
    """n points along a closed Catmull-Rom spline through ``pts``, and unit
    tangents."""
    m = len(pts)
    s = np.linspace(0.0, m, n, endpoint=False)
    i = np.floor(s).astype(int)
    t = (s - i)[:, None]
    p0, p1 = pts[(i - 1) % m], pts[i % m]
    p2, p3 = pts[(i + 1) % m], pts[(i + 2) % m]
    pos = 0.5 * ((2 * p1) + (-p0 + p2) * t + (2 * p0 - 5 * p1 + 4 * p2 - p3) * t * t
                 + (-p0 + 3 * p1 - 3 * p2 + p3) * t ** 3)
    tan = 0.5 * ((-p0 + p2) + 2 * (2 * p0 - 5 * p1 + 4 * p2 - p3) * t
                 + 3 * (-p0 + 3 * p1 - 3 * p2 + p3) * t * t)
    return pos, tan / np.linalg.norm(tan, axis=1, keepdims=True)


def make_cfg4(d_max: int = 11, n_frames: int = 300, width: int = 640,
              height: int = 480, focal: float = 525.0, seed: int = 0,
              n_objects: int = 200, device="cuda",
              depths_in=None) -> DepthScene:
    """BASELINE config 3 ("large room"): a 4 m cube (origin 0, d_max 11 =
    1.95 mm voxels at full size) with ``n_objects`` random boxes/spheres;
    ``n_frames`` depth maps along a closed Catmull-Rom path through 8 random
    waypoints at least 0.3 m clear of every object and the walls, looking
    along the tangent (assumed); the room's walls are part of the scene
    (assumed); intrinsics as cfg3; depth noise
    sigma = 0.0015 z^2; delta = 0.03, eta = 0.15 (assumed), tau_split /
    tau_join defaults, 500 iterations.  ``depths_in`` (the maps of an earlier
    call with the same arguments) skips the sphere tracing."""
    import torch
    size = 4.0
    objs = _room_objects(seed, n_objects, size)
    sdf = room_sdf_fn(objs, device, size)
    rng = np.random.default_rng(seed + 1)
    way = []
    while len(way) < 8:
        q = rng.uniform(0.3, size - 0.3, 3)
        if float(sdf(torch.tensor(q[None], dtype=torch.float64, device=device))[0]) > 0.3:
            way.append(q)
    pos, tan = _catmull_rom(np.array(way), n_frames)
    cams, depths = [], []
    given = depths_in
    if given is None and _is_cuda(device):
        objs_dev, n_box, n_sph = room_objects_array(objs, device)
    noise = np.random.default_rng(seed + 2)
    for k in range(n_frames):
        cam = PinholeCamera(focal, focal, (width - 1) / 2.0, (height - 1) / 2.0,
                            width, height, look_at(pos[k], pos[k] + tan[k]), pos[k])
        cams.append(cam)
        if given is not None:
            continue
        if _is_cuda(device):
            z = trace_room(cam, objs_dev, n_box, n_sph, size=size,
                           lipschitz=1.0, t_max=8.0, eps=1e-6)
        else:   # no device: the array program
            z = sphere_trace(sdf, cam, lipschitz=1.0, t_max=8.0,
                             device=device, eps=1e-6)
        z = z.cpu().numpy()
        depths.append(_add_noise(z, 0.0015 * z * z, noise))
    if given is not None:
        depths = [np.asarray(d, dtype=np.float32) for d in given]
    n = 1 << d_max
    return DepthScene("cfg4", (0.0, 0.0, 0.0), size / n, n, cams, depths,
                      dict(delta=0.03, eta=0.15, iterations=500))
