"""Full-schedule golden fixtures from the reference itself (heavy: run once,
in the build container, each config in its own process):

    python tests/golden/make_golden_full.py cfg2d8    # ~45 min, 6 GB
    python tests/golden/make_golden_full.py cfg2d5    # seconds
    python tests/golden/make_golden_full.py cfg3      # hours, ~25 GB peak
    python tests/golden/make_golden_full.py cfg4d8    # BASELINE cfg4 at d 8

Each writes ``full_<name>.json`` next to this script: the sha256 of the
seeded depth maps / sample grids (the GPU test regenerates them on the device
and checks the digest first -- scenes.py's generators are written as
separate IEEE operations so CPU and GPU produce the same bits), digests of
the view trees and u0, and for EVERY pass of the configuration's whole
schedule the reference's split / join counts, node count, state, energy and
sha256 digests of the child array and of the values of all live nodes
(tests/goldens.py:live_digest).  The inputs go through the reference's own
public API (tsdf.build_view_tsdf, fusion.build_view_tree,
fusion.initial_field, octree.build_octree) and its compiled kernels
(iterate_pass / propagate / tree_energy exactly as fusion.fuse calls them,
reference fusion.py:204-229).
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, HERE)

from make_golden import load_reference, pool_digest, sha  # noqa: E402


def depth_digest(depths) -> str:
    return sha(np.stack(depths).astype(np.float32))


def run_schedule(octfuse, u0, trees, p, every_pool=1, log=print):
    """The reference's fuse loop, recording every pass."""
    from octfuse import fusion
    from tests.goldens import live_digest
    kern = sys.modules["octfuse._kernels"]
    u = fusion._solver_field(u0)
    vv, vw, vc = fusion.view_arrays(trees)
    passes = []
    t_start = time.time()
    for t in range(p.iterations):
        xi = fusion.step_scale(t, p)
        s, j, _ = kern.iterate_pass(u.value, u.snap, u.child, u.joined,
                                    u.state, vv, vw, vc, u.d_max, p.lam,
                                    p.eps, p.gamma, xi, p.tau_split,
                                    p.tau_join, p.clamp, False, None)
        kern.propagate(u.value, u.child)
        e = kern.tree_energy(u.value, u.child, vv, vw, vc, u.d_max, p.lam,
                             p.eps, p.gamma)
        rec = {"splits": int(s), "joins": int(j), "energy": float(e),
               "node_count": int(u.node_count),
               "state": [int(q) for q in u.state]}
        if t % every_pool == 0 or t == p.iterations - 1:
            rec.update(live_digest(u.child[:u.used], u.value[:u.used]))
        passes.append(rec)
        if t % 10 == 0:
            log(f"  pass {t}: {s} splits {j} joins, {u.node_count} nodes, "
                f"{time.time() - t_start:.0f} s")
    return u, passes


def prepare_reference(octfuse, sc, p, log=print):
    """Reference TSDF -> view trees -> initial field -> u0 (cli.py:141-171)."""
    from octfuse import fusion, octree, tsdf, volume
    n = sc.resolution
    dom = volume.VolumeDomain(sc.origin, sc.voxel_size, n)
    wf = np.zeros((n, n, n))
    ws = np.zeros((n, n, n))
    trees = []
    t0 = time.time()
    for k, (c, d) in enumerate(zip(sc.cameras, sc.depths)):
        cam = volume.Camera(c.fx, c.fy, c.cx, c.cy, c.width, c.height,
                            c.rotation, c.translation)
        vt = tsdf.build_view_tsdf(volume.RangeImage(d), cam, dom, p.delta,
                                  p.eta)
        wf += vt.f.astype(np.float64) * vt.w
        ws += vt.w
        trees.append(fusion.build_view_tree(vt, p.tau))
        del vt
        log(f"  view {k}: {trees[-1].node_count} nodes, "
            f"{time.time() - t0:.0f} s")
    ubar = fusion.initial_field(wf, ws, p.gamma)
    del wf, ws
    u0 = octree.build_octree(ubar, tau=p.tau)
    return trees, u0, sha(ubar)


def depth_scene(name):
    from paper_1608_07411_b200 import scenes
    if name == "cfg3":
        return scenes.make_cfg3(device="cpu")
    if name == "cfg4d8":
        # the 64 room frames traced on the GPU (tools/dump_depths.py; the
        # generator is device-independent -- cfg3's CPU and GPU traces agree
        # bit for bit -- but tracing 200 objects takes hours on these cores)
        d = np.load(os.path.join(REPO, "gpurun_out", "depths_cfg4d8.npz"))
        return scenes.make_cfg4(d_max=8, n_frames=64, device="cpu",
                                depths_in=list(d["depths"]))
    raise KeyError(name)


def gen_depth_config(name, octfuse):
    from octfuse import fusion
    sc = depth_scene(name)
    dd = depth_digest(sc.depths)
    print(f"{name}: depth maps {dd[:16]}", flush=True)
    p = fusion.FusionParams(**sc.params)
    trees, u0, ubar_sha = prepare_reference(octfuse, sc, p)
    out = {"name": name, "resolution": sc.resolution,
           "n_views": len(sc.depths), "params": sc.params,
           "depth_sha": dd, "ubar": ubar_sha,
           "views": [pool_digest(t) for t in trees],
           "u0": pool_digest(u0)}
    print(f"{name}: u0 {u0.node_count} nodes", flush=True)
    u, passes = run_schedule(octfuse, u0, trees, p)
    out["passes"] = passes
    return out


def gen_cfg2(depth, octfuse):
    from octfuse import fusion, octree
    from paper_1608_07411_b200 import scenes
    fs, ws = scenes.make_cfg2_samples(d_max=depth)
    p = fusion.FusionParams(lam=1.0, iterations=200, tau=-1.0, tau_split=0.0,
                            tau_join=1.5)
    trees = [octree.build_octree(f, w, tau=-1.0, dtype=np.float32)
             for f, w in zip(fs, ws)]
    wf = np.zeros(fs[0].shape)
    wsum = np.zeros(fs[0].shape)
    for f, w in zip(fs, ws):            # cli.py:148-149 order
        wf += f.astype(np.float64) * w
        wsum += w
    u0 = octree.build_octree(fusion.initial_field(wf, wsum, p.gamma),
                             tau=-1.0)
    out = {"name": f"cfg2d{depth}", "depth": depth,
           "samples_sha": sha(np.stack(fs)) + sha(np.stack(ws)),
           "views": [pool_digest(t) for t in trees], "u0": pool_digest(u0)}
    # frozen structure: the full value digest every 10 passes suffices
    u, passes = run_schedule(octfuse, u0, trees, p,
                             every_pool=1 if depth <= 6 else 10)
    out["passes"] = passes
    if depth <= 5:
        np.savez_compressed(os.path.join(HERE, f"full_cfg2d{depth}.npz"),
                            final_value=u.value[:u.used])
    return out


def main():
    name = sys.argv[1]
    octfuse = load_reference()
    t0 = time.time()
    if name.startswith("cfg2d"):
        out = gen_cfg2(int(name[5:]), octfuse)
    else:
        out = gen_depth_config(name, octfuse)
    out.update(numpy=np.__version__, generator="tests/golden/make_golden_full.py",
               reference="/root/reference/pkg (octfuse %s)" % octfuse.__version__,
               seconds=round(time.time() - t0, 1))
    with open(os.path.join(HERE, f"full_{name}.json"), "w") as fp:
        json.dump(out, fp, indent=0)
    print(f"{name}: done in {time.time() - t0:.0f} s", flush=True)


if __name__ == "__main__":
    main()
