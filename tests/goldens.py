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


def live_nodes(child) -> np.ndarray:
    """Slots of every node reachable from the root, ascending (free-listed
    blocks excluded)."""
    child = np.asarray(child)
    out = [np.zeros(1, dtype=np.int64)]
    front = out[0]
    while front.size:
        c = child[front]
        c = c[c >= 0].astype(np.int64)
        front = (c[:, None] + np.arange(8)).ravel()
        if front.size:
            out.append(front)
    return np.sort(np.concatenate(out))


def live_digest(child, value) -> dict:
    """sha256 of the child array and of the values of all live nodes."""
    live = live_nodes(child)
    return {"child": sha(np.asarray(child)),
            "live_value": sha(np.asarray(value)[live]),
            "live": int(live.size)}


def blocky_scene(seed, n=16, nviews=3):
    """A seeded scene whose descent passes split and join: a blocky field
    (4^3 blocks at -0.8 / 0 / +0.8) seen by ``nviews`` noisy views, u0 = 0.9 x
    the field with fine steps in half of the volume (mixed leaf depths).
    Blocks of one sign join, the zero blocks' coarse leaves split.  Returns
    (oracle view pools, oracle u0 pool)."""
    import numpy as np
    from oracle import oracle as orc
    rng = np.random.default_rng(seed)
    base = np.kron(rng.choice([-0.8, 0.0, 0.8], (4, 4, 4)),
                   np.ones((n // 4,) * 3))
    views = []
    for _ in range(nviews):
        f = np.clip(base + rng.standard_normal((n, n, n)) * 0.2, -1,
                    1).astype(np.float32)
        w = (rng.random((n, n, n)) < 0.8).astype(np.uint8)
        f[w == 0] = -1.0
        views.append(orc.build_octree(f, w, tau=0.3, dtype=np.float32))
    g = base * 0.9 + rng.integers(0, 3, (n, n, n)) * 0.1 - 0.1
    g[:, :, n // 2:] = base[:, :, n // 2:] * 0.9
    return views, orc.build_octree(g, tau=0.15)
