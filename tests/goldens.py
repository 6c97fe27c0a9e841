"""Helpers that turn the committed fixtures back into oracle inputs."""
import hashlib
import json
import os

import numpy as np

from oracle import oracle as orc
from paper_1608_07411_b200 import scenes

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def load(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


def load_json(name):
    with open(os.path.join(GOLDEN, name + ".json")) as fp:
        return json.load(fp)


def cameras_from(z):
    fx, fy, cx, cy, w, h = z["intrinsics"]
    return [scenes.PinholeCamera(fx, fy, cx, cy, int(w), int(h), r, t)
            for r, t in zip(z["rotations"], z["translations"])]


def cfg1_inputs():
    """(depths, cameras, origin, voxel, n, params) of the cfg1 fixture."""
    z = load("cfg1")
    sc = scenes.make_cfg1()
    p = orc.Params(delta=sc.delta, eta=sc.eta, lam=sc.lam,
                   iterations=sc.iterations)
    return (list(z["depths"]), cameras_from(z), sc.origin, sc.voxel_size,
            sc.resolution, p)


def small_views(z):
    out = []
    i = 0
    while f"view{i}_value" in z:
        out.append(orc.Pool(z[f"view{i}_value"], z[f"view{i}_child"],
                            z[f"view{i}_state"], int(np.log2(int(z["resolution"]))),
                            weight=z[f"view{i}_weight"]))
        i += 1
    return out
