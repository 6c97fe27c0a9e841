"""Pin the CPU oracle (oracle/) against fixtures made by the reference.

These run without a GPU.  Every fixture was produced by the reference's own
compiled kernels (tests/golden/make_golden.py), so equality here means the
oracle restates the reference bit for bit on those inputs.
"""
import io

import numpy as np
import pytest

from oracle import oracle as orc
from paper_1608_07411_b200 import scenes
from tests.goldens import (cameras_from, cfg1_inputs, load, load_json, sha,
                           small_views)


def test_numpy_pyramid_order_is_pairwise():
    # octree.py:193-210 mean order; the GPU pyramid kernel hard-codes it
    rng = np.random.default_rng(0)
    g = rng.standard_normal((16, 16, 16)) * np.exp(rng.uniform(-20, 20, (16,) * 3))
    m = orc.reduce_pyramid(g, "mean")[-2]
    b = [g[(c >> 2) & 1::2, (c >> 1) & 1::2, c & 1::2] for c in range(8)]
    ref = ((((b[0] + b[1]) + (b[2] + b[3])) + (b[4] + b[5])) + (b[6] + b[7])) / 8
    assert np.array_equal(m, ref)


def test_capacity_closed_form():
    assert [orc.full_tree_capacity(d) for d in range(4)] == [1, 9, 73, 585]


class TestOctreeKat:
    z = load("octree_kat")

    @pytest.mark.parametrize("name", ["blocky", "smooth"])
    @pytest.mark.parametrize("tau", [-1.0, 0.0, 0.05, 0.25, 1.0])
    def test_plain_build_bitexact(self, name, tau):
        key = f"{name}_{tau:g}"
        t = orc.build_octree(self.z[name], tau=tau)
        assert np.array_equal(t.value, self.z[key + "_value"])
        assert np.array_equal(t.child, self.z[key + "_child"])
        assert np.array_equal(t.state, self.z[key + "_state"])
        assert np.array_equal(orc.densify(t.value, t.child, t.d_max),
                              self.z[key + "_dense"])

    def test_weighted_build_bitexact(self):
        t = orc.build_octree(self.z["wf"], self.z["ww"], tau=0.3,
                             dtype=np.float32)
        assert np.array_equal(t.value, self.z["w_value"])
        assert np.array_equal(t.weight, self.z["w_weight"])
        assert np.array_equal(t.child, self.z["w_child"])
        assert np.array_equal(t.state, self.z["w_state"])

    def test_leaves_are_morton_sorted(self):
        t = orc.build_octree(self.z["smooth"], tau=0.25)
        keys = []
        for _, l, x, y, z in orc.leaves(t):
            s = t.d_max - l
            keys.append(_morton(x << s, y << s, z << s))
        assert keys == sorted(keys) and len(set(keys)) == len(keys)


def _morton(x, y, z):
    k = 0
    for b in range(21):
        k |= ((x >> b) & 1) << (3 * b + 2)
        k |= ((y >> b) & 1) << (3 * b + 1)
        k |= ((z >> b) & 1) << (3 * b)
    return k


class TestSmallScene:
    """The reference's backend-parity scene (tests/test_backends.py:17-29)."""
    z = load("small")

    def test_tsdf_bitexact(self):
        z = self.z
        cams = cameras_from(z)
        n = int(z["resolution"])
        origin = tuple(z["origin"])
        for i, (d, c) in enumerate(zip(z["depths"], cams)):
            f, w = orc.build_view_tsdf(d, c, origin, float(z["voxel_size"]),
                                       n, 0.004, 0.02)
            assert np.array_equal(f, z["tsdf_f"][i])
            assert np.array_equal(w, z["tsdf_w"][i])

    def test_view_trees_and_u0_bitexact(self):
        z = self.z
        for i, v in enumerate(small_views(z)):
            t = orc.build_octree(z["tsdf_f"][i], z["tsdf_w"][i], tau=0.1,
                                 dtype=np.float32)
            assert np.array_equal(t.value, v.value)
            assert np.array_equal(t.weight, v.weight)
            assert np.array_equal(t.child, v.child)
        wf = sum(z["tsdf_w"][i].astype(np.float64) * z["tsdf_f"][i].astype(np.float64)
                 for i in range(len(z["tsdf_f"])))
        ws = sum(z["tsdf_w"][i].astype(np.float64) for i in range(len(z["tsdf_f"])))
        ub = orc.initial_field(wf, ws, 1e-4)
        assert np.array_equal(ub, z["ubar"])
        u0 = orc.build_octree(ub, tau=0.1)
        assert np.array_equal(u0.value, z["u0_value"])
        assert np.array_equal(u0.child, z["u0_child"])

    def test_fuse_bitexact(self):
        z = self.z
        u0 = orc.Pool(z["u0_value"], z["u0_child"], z["u0_state"], 4)
        out = orc.fuse(u0, small_views(z), orc.Params(iterations=6),
                       log_joins=True)
        u = out.field
        assert np.array_equal(u.value[:u.used], z["final_value"])
        assert np.array_equal(u.child[:u.used], z["final_child"])
        assert np.array_equal(u.state, z["final_state"])
        assert np.array_equal(out.join_log, z["join_log"])
        assert [s.energy for s in out.stats] == list(z["energies"])
        assert [[s.splits, s.joins, s.node_count] for s in out.stats] == \
            z["counts"].tolist()


@pytest.fixture(scope="module")
def built():
    depths, cams, origin, vox, n, p = cfg1_inputs()
    meta = load_json("cfg1")
    wf = np.zeros((n, n, n))
    ws = np.zeros((n, n, n))
    views = []
    for i, (d, c) in enumerate(zip(depths, cams)):
        f, w = orc.build_view_tsdf(d, c, origin, vox, n, p.delta, p.eta)
        assert sha(f) == meta["tsdf_f"][i] and sha(w) == meta["tsdf_w"][i]
        wf += f.astype(np.float64) * w
        ws += w
        views.append(orc.build_octree(f, w, tau=p.tau, dtype=np.float32))
    ub = orc.initial_field(wf, ws, p.gamma)
    assert sha(ub) == meta["ubar"]
    u0 = orc.build_octree(ub, tau=p.tau)
    return views, u0, p, meta

class TestCfg1:
    """BASELINE config 0, full size (d_max 6, 8 views, 50 passes)."""

    def test_view_trees_and_u0(self, built):
        views, u0, p, meta = built
        for v, m in zip(views, meta["views"]):
            assert sha(v.value) == m["value"] and sha(v.child) == m["child"]
            assert sha(v.weight) == m["weight"]
        assert sha(u0.value) == meta["u0"]["value"]
        assert sha(u0.child) == meta["u0"]["child"]

    def test_every_pass_bitexact(self, built):
        views, u0, p, meta = built
        u = orc.solver_pool(u0)
        vv = [v.value for v in views]
        vw = [v.weight for v in views]
        vc = [v.child for v in views]
        for t, ref in enumerate(meta["passes"]):
            xi = orc.step_scale(t, p)
            s, j, _ = orc.iterate_pass(u.value, u.snap, u.child, u.joined,
                                       u.state, vv, vw, vc, u.d_max, p.lam,
                                       p.eps, p.gamma, xi, p.tau_split,
                                       p.tau_join, p.clamp, False, None)
            orc.propagate(u.value, u.child)
            e = orc.tree_energy(u.value, u.child, vv, vw, vc, u.d_max, p.lam,
                                p.eps, p.gamma)
            used = u.used
            assert (s, j) == (ref["splits"], ref["joins"]), t
            assert e == ref["energy"], t
            assert [int(q) for q in u.state] == ref["state"], t
            assert sha(u.value[:used]) == ref["value"], t
            assert sha(u.child[:used]) == ref["child"], t
            assert sha(u.snap[:used]) == ref["snap"], t
            assert sha(u.joined[:used]) == ref["joined"], t


class TestCfg2Reduced:
    z = load("cfg2")

    @pytest.mark.parametrize("d", [4, 5])
    def test_fixed_structure_bitexact(self, d):
        fs, ws = scenes.make_cfg2_samples(d_max=d)
        p = orc.Params(lam=1.0, iterations=12, tau=-1.0, tau_split=0.0,
                       tau_join=1.5)
        views = [orc.build_octree(f, w, tau=-1.0, dtype=np.float32)
                 for f, w in zip(fs, ws)]
        for v, h in zip(views, self.z[f"d{d}_view_sha"]):
            assert sha(v.value) + sha(v.weight) + sha(v.child) == h
        wf = sum(w.astype(np.float64) * f.astype(np.float64) for f, w in zip(fs, ws))
        wsum = sum(w.astype(np.float64) for w in ws)
        u0 = orc.build_octree(orc.initial_field(wf, wsum, p.gamma), tau=-1.0)
        assert np.array_equal(u0.value, self.z[f"d{d}_u0_value"])
        out = orc.fuse(u0, views, p)
        assert np.array_equal(out.field.value[:out.field.used],
                              self.z[f"d{d}_final_value"])
        assert [s.energy for s in out.stats] == list(self.z[f"d{d}_energies"])
