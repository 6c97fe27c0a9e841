"""Mesh readout fixtures from the reference itself (run in the build
container, like make_golden.py):

    python tests/golden/make_golden_mesh.py

* mc_tables.npz -- the reference's marching-cubes case tables
  (octfuse/_mctables.py, generated at its import);
* mesh.npz -- octfuse.mesh.marching_cubes on (a) the cfg1 final field,
  densified by the reference, masked by the reference's w_sum > 0, and (b) a
  seeded random 20^3 grid without a mask (every case class appears).
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from tests.golden.make_golden import load_reference  # noqa: E402


def main():
    load_reference()
    from octfuse import _mctables, mesh, octree, tsdf, volume
    from paper_1608_07411_b200 import scenes
    np.savez_compressed(os.path.join(HERE, "mc_tables.npz"),
                        tri_table=_mctables.TRI_TABLE,
                        tri_count=_mctables.TRI_COUNT,
                        edge_axis=_mctables.EDGE_AXIS,
                        edge_cell_offset=_mctables.EDGE_CELL_OFFSET)
    z = np.load(os.path.join(HERE, "cfg1.npz"))
    sc = scenes.make_cfg1()
    dom = volume.VolumeDomain(sc.origin, sc.voxel_size, sc.resolution)
    n = sc.resolution
    ws = np.zeros((n, n, n))
    for c, d in zip(sc.cameras, sc.depths):
        cam = volume.Camera(c.fx, c.fy, c.cx, c.cy, c.width, c.height,
                            c.rotation, c.translation)
        vt = tsdf.build_view_tsdf(volume.RangeImage(d), cam, dom, sc.delta,
                                  sc.eta)
        ws += vt.w
    field = octree.OctreeField(z["final_value"].astype(np.float64),
                               z["final_child"].astype(np.int32),
                               z["final_state"].astype(np.int64), 6)
    dense = octree.densify(field)
    m1 = mesh.marching_cubes(dense, ws > 0, dom)
    rng = np.random.default_rng(7)
    rnd = rng.standard_normal((20, 20, 20))
    v2, f2 = mesh.extract_zero_surface(rnd, None)
    np.savez_compressed(os.path.join(HERE, "mesh.npz"),
                        cfg1_seen=(ws > 0), cfg1_vertices=m1.vertices,
                        cfg1_faces=m1.faces, rnd_values=rnd,
                        rnd_vertices=v2, rnd_faces=f2)
    print("cfg1 mesh", m1.vertices.shape, m1.faces.shape, "random",
          v2.shape, f2.shape)


if __name__ == "__main__" and len(sys.argv) == 1:
    main()


def dense_solver_fixture():
    """dense.npz -- the reference's dense solver (fusion.dense_fuse,
    fusion.py:253-325) on a seeded 16^3 grid with 4 views, 6 iterations."""
    load_reference()
    from octfuse import fusion
    rng = np.random.default_rng(21)
    n = 16
    fs, ws = [], []
    for _ in range(4):
        f = np.clip(rng.standard_normal((n, n, n)) * 0.5, -1, 1).astype(np.float32)
        w = (rng.random((n, n, n)) < 0.8).astype(np.uint8)
        f[w == 0] = -1.0
        fs.append(f)
        ws.append(w)
    u0 = np.clip(rng.standard_normal((n, n, n)) * 0.3, -1, 1)
    p = fusion.FusionParams(iterations=6, lam=0.4)
    u, stats = fusion.dense_fuse(u0, fs, ws, p)
    np.savez_compressed(os.path.join(HERE, "dense.npz"), fs=np.stack(fs),
                        ws=np.stack(ws), u0=u0, u=u,
                        energies=np.array([s.energy for s in stats]))
    print("dense", u.shape)


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "dense":
    dense_solver_fixture()
