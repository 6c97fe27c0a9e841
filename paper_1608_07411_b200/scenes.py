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
           "make_cfg1", "torus_sdf", "make_cfg2_samples"]


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

