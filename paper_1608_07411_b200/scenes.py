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
