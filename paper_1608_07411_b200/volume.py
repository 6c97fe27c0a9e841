"""Reconstruction volume, pinhole cameras and range images (reference
``volume.py``).  Host-side plumbing: the GPU kernels consume these as a
handful of doubles (``Camera.packed()``).  Dataset file I/O is out of scope
(SURVEY.md §8(f) row 3)."""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

__all__ = ["VolumeDomain", "Camera", "RangeImage", "project", "look_at",
           "voxel_center"]


@dataclass(frozen=True)
class VolumeDomain:
    """Axis-aligned cubic volume: minimum corner, voxel edge, voxels/axis
    (a power of two) -- reference volume.py:34-69."""

    origin: tuple
    voxel_size: float
    resolution: int

    def __post_init__(self):
        if self.voxel_size <= 0:
            raise ValueError("voxel_size must be positive")
        n = self.resolution
        if n < 1 or (n & (n - 1)) != 0:
            raise ValueError(f"resolution must be a power of two, got {n}")
        object.__setattr__(self, "origin", tuple(float(c) for c in self.origin))

    @property
    def depth(self) -> int:
        return self.resolution.bit_length() - 1

    @property
    def extent(self) -> float:
        return self.resolution * self.voxel_size

    def axis_centers(self, axis: int) -> np.ndarray:
        return self.origin[axis] + (np.arange(self.resolution) + 0.5) * self.voxel_size


def voxel_center(idx, dom: VolumeDomain) -> np.ndarray:
    idx = np.asarray(idx)
    if np.any(idx < 0) or np.any(idx >= dom.resolution):
        raise ValueError(f"voxel index {idx!r} outside [0, {dom.resolution})")
    return np.asarray(dom.origin) + (idx + 0.5) * dom.voxel_size


class Camera:
    """Pinhole camera with a camera-to-world pose (reference volume.py:80-128)."""

    def __init__(self, fx, fy, cx, cy, width, height, rotation, translation):
        self.fx, self.fy = float(fx), float(fy)
        self.cx, self.cy = float(cx), float(cy)
        self.width, self.height = int(width), int(height)
        self.rotation = np.asarray(rotation, dtype=np.float64).reshape(3, 3)
        self.translation = np.asarray(translation, dtype=np.float64).reshape(3)
        r = self.rotation
        if not np.allclose(r @ r.T, np.eye(3), atol=1e-9):
            raise ValueError("camera rotation is not orthonormal")
        if abs(np.linalg.det(r) - 1.0) > 1e-9:
            raise ValueError("camera rotation must have determinant +1")

    @property
    def center(self) -> np.ndarray:
        return self.translation

    def world_to_cam(self, x) -> np.ndarray:
        return (np.asarray(x, dtype=np.float64) - self.translation) @ self.rotation

    def packed(self) -> np.ndarray:
        """{fx, fy, cx, cy, R row-major, t} as the C ABI expects."""
        return np.concatenate([[self.fx, self.fy, self.cx, self.cy],
                               self.rotation.ravel(), self.translation])


def project(x, cam: Camera):
    xc = cam.world_to_cam(x)
    z = xc[2]
    if z <= 0:
        return None
    u = cam.fx * xc[0] / z + cam.cx
    v = cam.fy * xc[1] / z + cam.cy
    if u < 0 or u >= cam.width or v < 0 or v >= cam.height:
        return None
    return (u, v)


def look_at(position, target, up=(0.0, 0.0, 1.0)) -> np.ndarray:
    from .scenes import look_at as _la
    return _la(position, target, up)


class RangeImage:
    """One depth frame: camera-frame z in metres, 0 = invalid."""

    def __init__(self, depth):
        d = np.asarray(depth, dtype=np.float32)
        if d.ndim != 2:
            raise ValueError("depth must be a 2-D array")
        if not np.all(np.isfinite(d)) or np.any(d < 0):
            raise ValueError("depths must be finite and non-negative")
        self.depth = d

    @property
    def height(self) -> int:
        return self.depth.shape[0]

    @property
    def width(self) -> int:
        return self.depth.shape[1]
