"""Per-view truncated signed distances on the GPU (reference ``tsdf.py``).

``build_view_tsdf`` evaluates the projective TSDF at every voxel centre in
f64 with numpy's operand order (bit-identical to the reference's
vectorised numpy, tsdf.py:87-120) and can fold the view into the running
weighted sums of reference cli.py:148-149 in the same kernel.  The scalar
contract (signed_distance / truncate / visibility_weight, tsdf.py:48-84) is
kept as host functions.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._device import as_device, device, ptr, stream_handle
from .volume import Camera, RangeImage, VolumeDomain, project

__all__ = ["ViewTsdf", "signed_distance", "truncate", "visibility_weight",
           "build_view_tsdf"]


@dataclass
class ViewTsdf:
    """Dense TSDF and weight grid of one view, resident on the GPU."""

    f: torch.Tensor      # (N, N, N) float32 in [-1, 1]
    w: torch.Tensor      # (N, N, N) uint8 in {0, 1}
    delta: float
    eta: float

    @property
    def nbytes_per_voxel(self) -> int:
        return self.f.element_size() + self.w.element_size()


def signed_distance(x, img: RangeImage, cam: Camera):
    uv = project(x, cam)
    if uv is None:
        return None
    pu = min(int(math.floor(uv[0] + 0.5)), cam.width - 1)
    pv = min(int(math.floor(uv[1] + 0.5)), cam.height - 1)
    z = float(img.depth[pv, pu])
    if z <= 0:
        return None
    du = (pu - cam.cx) / cam.fx
    dv = (pv - cam.cy) / cam.fy
    return z * math.sqrt(1.0 + du * du + dv * dv) - float(
        np.linalg.norm(np.asarray(x, float) - cam.center))


def truncate(phi: float, delta: float) -> float:
    if delta <= 0:
        raise ValueError("delta must be positive")
    if phi > delta:
        return 1.0
    if phi < -delta:
        return -1.0
    return phi / delta


def visibility_weight(phi, eta: float) -> int:
    if eta <= 0:
        raise ValueError("eta must be positive")
    if phi is None or phi < -eta:
        return 0
    return 1


def build_view_tsdf(img, cam, dom: VolumeDomain, delta: float, eta: float, *,
                    accumulate=None) -> ViewTsdf:
    """TSDF + weight of one depth frame at every voxel centre.

    ``img``: RangeImage / (H, W) array / CUDA tensor of z-depths.
    ``accumulate``: optional (wf_sum, w_sum) float64 CUDA grids updated in
    place with f*w and w (reference cli.py:148-149).
    """
    if delta <= 0 or eta <= 0:
        raise ValueError("delta and eta must be positive")
    depth = img.depth if isinstance(img, RangeImage) else img
    d = as_device(depth, torch.float32)
    n = dom.resolution
    f = torch.empty((n, n, n), dtype=torch.float32, device=device())
    w = torch.empty((n, n, n), dtype=torch.uint8, device=device())
    cp = np.ascontiguousarray(_camera_params(cam))
    org = np.ascontiguousarray(np.asarray(dom.origin, dtype=np.float64))
    wf = ws = None
    if accumulate is not None:
        wf, ws = accumulate
        for g in (wf, ws):
            if g.dtype != torch.float64 or tuple(g.shape) != (n, n, n):
                raise ValueError("accumulators must be (N,N,N) float64 CUDA grids")
    _lib.call("octf_view_tsdf", ptr(d), int(d.shape[1]), int(d.shape[0]),
              cp.ctypes.data, org.ctypes.data, float(dom.voxel_size), n,
              float(delta), float(eta), ptr(f), ptr(w), ptr(wf), ptr(ws),
              stream_handle())
    return ViewTsdf(f=f, w=w, delta=float(delta), eta=float(eta))


def _camera_params(cam) -> np.ndarray:
    return np.concatenate([[cam.fx, cam.fy, cam.cx, cam.cy],
                           np.asarray(cam.rotation, dtype=np.float64).ravel(),
                           np.asarray(cam.translation, dtype=np.float64).ravel()])
