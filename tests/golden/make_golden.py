"""Generate the golden fixtures from the reference itself.

Run in the build container (it needs /root/reference and the compiled
reference kernels built by ``make -C oracle ref``):

    python tests/golden/make_golden.py

The reference package is imported from /root/reference/pkg/src with its
native module ``octfuse._kernels`` taken from ``oracle/_ref`` (the reference's
own _kernels.pyx compiled there), so every number below is produced by the
reference's compiled backend.  Outputs are small .npz files next to this
script; big arrays are recorded as sha256 digests of their exact bytes.
The GPU box never runs this script (it has no /root/reference).
"""

from __future__ import annotations

import glob
import hashlib
import importlib.util
import io
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg/src"


def load_reference():
    so = glob.glob(os.path.join(REPO, "oracle", "_ref", "_kernels*.so"))
    if not so:
        raise SystemExit("build the reference kernels first: make -C oracle ref")
    spec = importlib.util.spec_from_file_location("octfuse._kernels", so[0])
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    sys.modules["octfuse._kernels"] = mod
    sys.path.insert(0, REF_SRC)
    import octfuse  # noqa: F401
    from octfuse import _backend
    assert _backend.name() == "compiled"
    return sys.modules["octfuse"]


def sha(a) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.tobytes()).hexdigest()


def pool_digest(f, upto=None):
    used = f.used if upto is None else upto
    d = {"value": sha(f.value[:used]), "child": sha(f.child[:used]),
         "state": [int(s) for s in f.state]}
    if f.weight is not None:
        d["weight"] = sha(f.weight[:used])
    return d


def main():
    octfuse = load_reference()
    from octfuse import fusion, octree, tsdf, volume
    sys.path.insert(0, REPO)
    from paper_1608_07411_b200 import scenes

    meta = {"numpy": np.__version__,
            "generator": "tests/golden/make_golden.py",
            "reference": "/root/reference/pkg (octfuse %s)" % octfuse.__version__}

    # ---------------------------------------------------------------- cfg1
    sc = scenes.make_cfg1()
    dom = volume.VolumeDomain(sc.origin, sc.voxel_size, sc.resolution)
    p = fusion.FusionParams(delta=sc.delta, eta=sc.eta, lam=sc.lam,
                            iterations=sc.iterations)
    n = sc.resolution
    wf = np.zeros((n, n, n))
    ws = np.zeros((n, n, n))
    trees, tsdf_f, tsdf_w = [], [], []
    for c, d in zip(sc.cameras, sc.depths):
        cam = volume.Camera(c.fx, c.fy, c.cx, c.cy, c.width, c.height,
                            c.rotation, c.translation)
        vt = tsdf.build_view_tsdf(volume.RangeImage(d), cam, dom, p.delta,
                                  p.eta)
        tsdf_f.append(sha(vt.f))
        tsdf_w.append(sha(vt.w))
        wf += vt.f.astype(np.float64) * vt.w
        ws += vt.w
        trees.append(fusion.build_view_tree(vt, p.tau))
    ubar = fusion.initial_field(wf, ws, p.gamma)
    u0 = octree.build_octree(ubar, tau=p.tau)
    cfg1 = {
        "tsdf_f": tsdf_f, "tsdf_w": tsdf_w, "ubar": sha(ubar),
        "views": [pool_digest(t) for t in trees],
        "u0": pool_digest(u0),
    }
    # fuse, recording each pass's pools exactly as fusion.fuse leaves them
    kern = sys.modules["octfuse._kernels"]
    u = fusion._solver_field(u0)
    vv, vw, vc = fusion.view_arrays(trees)
    jbuf = np.zeros((u.capacity // 8 + 8, 12))
    passes, logs = [], []
    for t in range(p.iterations):
        xi = fusion.step_scale(t, p)
        s, j, r = kern.iterate_pass(u.value, u.snap, u.child, u.joined,
                                    u.state, vv, vw, vc, u.d_max, p.lam,
                                    p.eps, p.gamma, xi, p.tau_split,
                                    p.tau_join, p.clamp, False, jbuf)
        kern.propagate(u.value, u.child)
        e = kern.tree_energy(u.value, u.child, vv, vw, vc, u.d_max, p.lam,
                             p.eps, p.gamma)
        logs.append(jbuf[:r].copy())
        passes.append({"splits": s, "joins": j, "energy": float(e),
                       "node_count": u.node_count, **pool_digest(u),
                       "snap": sha(u.snap[:u.used]),
                       "joined": sha(u.joined[:u.used])})
    cfg1["passes"] = passes
    buf = io.StringIO()
    octree.serialize(u, buf)
    cfg1["serialize_sha"] = hashlib.sha256(buf.getvalue().encode()).hexdigest()
    # cross-check against fusion.fuse itself (same stats)
    res = fusion.fuse(u0, trees, p, log_joins=True)
    assert [s.energy for s in res.stats] == [q["energy"] for q in passes]
    np.savez_compressed(
        os.path.join(HERE, "cfg1.npz"),
        depths=np.stack(sc.depths),
        rotations=np.stack([c.rotation for c in sc.cameras]),
        translations=np.stack([c.translation for c in sc.cameras]),
        intrinsics=np.array([sc.cameras[0].fx, sc.cameras[0].fy,
                             sc.cameras[0].cx, sc.cameras[0].cy,
                             sc.cameras[0].width, sc.cameras[0].height]),
        u0_value=u0.value, u0_child=u0.child, u0_state=u0.state,
        final_value=u.value[:u.used], final_child=u.child[:u.used],
        final_state=u.state, join_log=np.vstack(logs),
        energies=np.array([q["energy"] for q in passes]))
    with open(os.path.join(HERE, "cfg1.json"), "w") as fp:
        json.dump({**meta, **cfg1}, fp, indent=1)

    # ------------------------------------------------------- small scene
    # the reference's own backend-parity scene (tests/test_backends.py:17-29)
    import tempfile
    from octfuse.synth import make_sphere_dataset
    with tempfile.TemporaryDirectory() as tmp:
        dom, cams, imgs, _ = make_sphere_dataset(tmp, n_views=3, width=96,
                                                 height=96, resolution=16,
                                                 voxel_size=0.016)
    ps = fusion.FusionParams(iterations=6)
    tsdfs = [tsdf.build_view_tsdf(im, c, dom, ps.delta, ps.eta)
             for im, c in zip(imgs, cams)]
    wf = sum(t.w.astype(np.float64) * t.f.astype(np.float64) for t in tsdfs)
    wsum = sum(t.w.astype(np.float64) for t in tsdfs)
    ub = fusion.initial_field(wf, wsum, ps.gamma)
    views = [fusion.build_view_tree(t, ps.tau) for t in tsdfs]
    st = octree.build_octree(ub, tau=ps.tau)
    res = fusion.fuse(st, views, ps, log_joins=True)
    small = dict(
        depths=np.stack([im.depth for im in imgs]),
        rotations=np.stack([c.rotation for c in cams]),
        translations=np.stack([c.translation for c in cams]),
        intrinsics=np.array([cams[0].fx, cams[0].fy, cams[0].cx, cams[0].cy,
                             cams[0].width, cams[0].height]),
        origin=np.array(dom.origin), voxel_size=np.array(dom.voxel_size),
        resolution=np.array(dom.resolution),
        tsdf_f=np.stack([t.f for t in tsdfs]),
        tsdf_w=np.stack([t.w for t in tsdfs]),
        ubar=ub, u0_value=st.value, u0_child=st.child, u0_state=st.state,
        final_value=res.field.value[:res.field.used],
        final_child=res.field.child[:res.field.used],
        final_state=res.field.state, join_log=res.join_log,
        energies=np.array([s.energy for s in res.stats]),
        counts=np.array([[s.splits, s.joins, s.node_count]
                         for s in res.stats]))
    for i, v in enumerate(views):
        small[f"view{i}_value"] = v.value
        small[f"view{i}_weight"] = v.weight
        small[f"view{i}_child"] = v.child
        small[f"view{i}_state"] = v.state
    np.savez_compressed(os.path.join(HERE, "small.npz"), **small)

    # ----------------------------------------------- octree known answers
    rng = np.random.default_rng(11)
    blocky = rng.integers(0, 4, (16, 16, 16)).astype(np.float64) * 0.5
    rng = np.random.default_rng(13)
    g = rng.standard_normal((16, 16, 16))
    for axis in range(3):
        g = (g + np.roll(g, 1, axis) + np.roll(g, -1, axis)) / 3.0
    kat = {"blocky": blocky, "smooth": g}
    for name, grid in (("blocky", blocky), ("smooth", g)):
        for tau in (-1.0, 0.0, 0.05, 0.25, 1.0):
            t = octree.build_octree(grid, tau=tau)
            key = f"{name}_{tau:g}"
            kat[key + "_value"] = t.value
            kat[key + "_child"] = t.child
            kat[key + "_state"] = t.state
            kat[key + "_dense"] = octree.densify(t)
    # weighted build (tests/test_octree.py:123-133 pattern)
    rng = np.random.default_rng(21)
    f = g.copy()
    w = np.zeros((16, 16, 16), dtype=np.uint8)
    w[:, :8] = 1
    w[:4, :4, :4] = 0
    f[w == 0] = -1.0
    f32 = f.astype(np.float32)
    tw = octree.build_octree(f32, w, tau=0.3, dtype=np.float32)
    kat.update(wf=f32, ww=w, w_value=tw.value, w_weight=tw.weight,
               w_child=tw.child, w_state=tw.state)
    np.savez_compressed(os.path.join(HERE, "octree_kat.npz"), **kat)

    # ----------------------------------------------------- cfg2 (reduced)
    cfg2 = {}
    for d in (4, 5):
        fs, wsl = scenes.make_cfg2_samples(d_max=d)
        pc = fusion.FusionParams(lam=1.0, iterations=12, tau=-1.0,
                                 tau_split=0.0, tau_join=1.5)
        vts = [octree.build_octree(fv, wv, tau=-1.0, dtype=np.float32)
               for fv, wv in zip(fs, wsl)]
        wf = sum(wv.astype(np.float64) * fv.astype(np.float64)
                 for fv, wv in zip(fs, wsl))
        wsum = sum(wv.astype(np.float64) for wv in wsl)
        ub = fusion.initial_field(wf, wsum, pc.gamma)
        st = octree.build_octree(ub, tau=-1.0)
        res = fusion.fuse(st, vts, pc)
        cfg2[f"d{d}_final_value"] = res.field.value[:res.field.used]
        cfg2[f"d{d}_energies"] = np.array([s.energy for s in res.stats])
        cfg2[f"d{d}_u0_value"] = st.value
        cfg2[f"d{d}_view_sha"] = np.array([sha(v.value) + sha(v.weight)
                                           + sha(v.child) for v in vts])
    np.savez_compressed(os.path.join(HERE, "cfg2.npz"), **cfg2)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
