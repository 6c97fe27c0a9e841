"""Zero-isosurface readout (reference mesh.py).
CPU: the package's generated case tables equal the reference's, and the
oracle restatement reproduces the reference's meshes.  GPU: the CUDA
marching cubes reproduces them bit for bit, directly and after the whole
cfg1 pipeline (fuse -> densify -> mesh)."""
import numpy as np
import pytest

from oracle import oracle as orc
from tests.conftest import has_gpu
from tests.goldens import load

gpu = [pytest.mark.gpu,
       pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]


def _tables():
    z = load("mc_tables")
    return z["tri_table"], z["tri_count"], z["edge_axis"], z["edge_cell_offset"]


def test_case_tables_equal_reference():
    from paper_1608_07411_b200 import mesh
    for got, want in zip(mesh.case_tables(), _tables()):
        assert np.array_equal(got, want)


def test_oracle_matches_reference_meshes():
    z = load("mesh")
    v, f = orc.extract_zero_surface(z["rnd_values"], None, _tables())
    assert np.array_equal(v, z["rnd_vertices"])
    assert np.array_equal(f, z["rnd_faces"])


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
def test_gpu_marching_cubes_bitexact():
    import torch
    from paper_1608_07411_b200 import mesh
    z = load("mesh")
    v, f = mesh.extract_zero_surface(torch.as_tensor(z["rnd_values"]).cuda())
    assert np.array_equal(v, z["rnd_vertices"])
    assert np.array_equal(f, z["rnd_faces"])
    # a mask that drops a slab, and an all-positive grid (empty mesh)
    mk = np.ones((20, 20, 20), dtype=bool)
    mk[7:9] = False
    v2, f2 = mesh.extract_zero_surface(z["rnd_values"], mk)
    w2, g2 = orc.extract_zero_surface(z["rnd_values"], mk, _tables())
    assert np.array_equal(v2, w2) and np.array_equal(f2, g2)
    v3, f3 = mesh.extract_zero_surface(np.ones((5, 5, 5)))
    assert v3.shape == (0, 3) and f3.shape == (0, 3)


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
def test_gpu_cfg1_pipeline_mesh_equals_reference():
    """cfg1 end to end on the GPU: views + u0 (fusion.prepare), 50 fp64
    passes, densify, w_sum > 0 mask, marching cubes -- the reference's
    mesh of the same scene bit for bit."""
    from paper_1608_07411_b200 import fusion, mesh, octree, scenes, volume
    from tests.goldens import cfg1_inputs
    depths, cams, origin, vox, n, p = cfg1_inputs()
    dom = volume.VolumeDomain(origin, vox, n)
    fp = fusion.FusionParams(delta=p.delta, eta=p.eta, lam=p.lam,
                             iterations=p.iterations)
    views, u0, seen = fusion.prepare(depths, cams, dom, fp)
    res = fusion.fuse(u0, views, fp)
    dense = octree.densify(res.field)
    m = mesh.marching_cubes(dense, seen, dom)
    z = load("mesh")
    assert np.array_equal(seen.cpu().numpy(), z["cfg1_seen"])
    assert np.array_equal(m.vertices, z["cfg1_vertices"])
    assert np.array_equal(m.faces, z["cfg1_faces"])
    a, b, c = (m.vertices[m.faces[:, k]] for k in range(3))
    assert np.einsum("ij,ij->i", a, np.cross(b, c)).sum() > 0  # outward
    # the same mesh straight from the leaf store (no dense grid), with the
    # observed mask as a tree and with f32 values
    mt = mesh.marching_cubes_tree(res.field, mesh.seen_tree(seen), dom)
    assert np.array_equal(mt.vertices, z["cfg1_vertices"])
    assert np.array_equal(mt.faces, z["cfg1_faces"])


def _random_tree(seed, d=6):
    """A mixed-depth tree over random blocky values (coarse leaves of both
    signs next to fine ones), built on the device."""
    import torch
    from paper_1608_07411_b200 import octree
    rng = np.random.default_rng(seed)
    n = 1 << d
    g = np.zeros((n, n, n))
    for s in (32, 16, 8, 4, 2, 1):
        k = n // s
        blk = rng.normal(0, 1.0 / s, (k, k, k))
        g += np.kron(blk, np.ones((s, s, s)))
    g -= np.median(g)
    g = np.round(g * 4) / 4 + 0.125       # few distinct values, no zeros
    return octree.build_octree(torch.as_tensor(g).cuda(), tau=0.3), g


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
@pytest.mark.parametrize("seed", range(4))
def test_tree_readout_equals_dense_readout(seed):
    import torch
    from paper_1608_07411_b200 import mesh, octree
    t, _ = _random_tree(seed)
    dense = octree.densify(t)
    rng = np.random.default_rng(100 + seed)
    seen = np.ones(dense.shape, dtype=bool)
    seen[rng.integers(0, 64, 20), :, :] = False
    seen[:, :, rng.integers(0, 64, 5)] = False
    for sd in (None, seen):
        v, f = mesh.extract_zero_surface(dense, sd)
        vt, ft = mesh.tree_zero_surface(
            t, None if sd is None else mesh.seen_tree(torch.as_tensor(sd)))
        assert v.shape[0] > 100
        assert np.array_equal(v, vt) and np.array_equal(f, ft)
    # slab by slab: the same triangles (slab meshes index their own vertices)
    tri = {tuple(map(tuple, vt[ft[i]])) for i in range(ft.shape[0])}
    got, nf = set(), 0
    for b0 in range(0, 8, 3):
        vs, fs = mesh.tree_zero_surface(t, slab=(b0, min(b0 + 3, 8)))
        nf += fs.shape[0]
        got |= {tuple(map(tuple, vs[fs[i]])) for i in range(fs.shape[0])}
    v0, f0 = mesh.tree_zero_surface(t)
    assert nf == f0.shape[0]
    assert got == {tuple(map(tuple, v0[f0[i]])) for i in range(f0.shape[0])}
    # f32 values: the dense readout of the same f32 field
    t32 = octree.OctreeField(t.value.float(), t.child, t.state, t.d_max)
    v, f = mesh.extract_zero_surface(octree.densify(t32))
    vt, ft = mesh.tree_zero_surface(t32)
    assert np.array_equal(v, vt) and np.array_equal(f, ft)


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
def test_tree_readout_at_depth_12_without_dense_grid():
    """BASELINE config 4's depth (4096^3 cells, 550 GB dense in f64): a
    sphere-band tree read out from the leaf store; the mesh closes (every
    edge shared by two faces) and its vertices lie on the sphere."""
    import torch
    from paper_1608_07411_b200 import mesh
    from paper_1608_07411_b200.octree import OctreeField
    d, r = 12, 0.05
    n = 1 << d
    child = np.full(1, -1, dtype=np.int64)
    value = np.zeros(1)
    fx = fy = fz = np.zeros(1, dtype=np.int64)
    fslot = np.zeros(1, dtype=np.int64)   # nodes of the front (to refine)
    for L in range(d):
        h = 1.0 / (1 << (L + 1))
        b = child.shape[0] + 8 * np.arange(fslot.size)
        child[fslot] = b
        c = np.arange(8)
        cx = (2 * fx[:, None] + (c >> 2 & 1)).ravel()
        cy = (2 * fy[:, None] + (c >> 1 & 1)).ravel()
        cz = (2 * fz[:, None] + (c & 1)).ravel()
        sd = np.sqrt(((cx + .5) * h - .5) ** 2 + ((cy + .5) * h - .5) ** 2
                     + ((cz + .5) * h - .5) ** 2) - r
        child = np.concatenate([child, np.full(cx.size, -1)])
        value = np.concatenate([value, sd])
        keep = (np.abs(sd) < 0.9 * h * np.sqrt(3)) & (L + 1 < d)
        fslot = (b[:, None] + c).ravel()[keep]
        fx, fy, fz = cx[keep], cy[keep], cz[keep]
    # slot 0 root, blocks from slot 1: the reference layout
    used = child.shape[0]
    f = OctreeField.from_host(value, child.astype(np.int32),
                              np.array([used, -1, used], np.int64), d)
    v, faces = mesh.tree_zero_surface(f)
    assert faces.shape[0] > 1000
    e = np.sort(np.stack([faces[:, [0, 1]], faces[:, [1, 2]],
                          faces[:, [2, 0]]]).reshape(-1, 2), axis=1)
    _, counts = np.unique(e, axis=0, return_counts=True)
    assert (counts == 2).all()
    rad = np.linalg.norm((v + 0.5) / n - 0.5, axis=1)
    assert np.abs(rad - r).max() < 2.0 / n


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
def test_tree_readout_cfg3_reduced_equals_dense():
    """BASELINE config 2 (adaptive object) at reduced size after restructuring
    passes: the leaf-store readout equals densify + dense marching cubes."""
    from paper_1608_07411_b200 import fusion, mesh, octree, scenes, volume
    sc = scenes.make_cfg3(d_max=7, n_views=16, width=320, height=240,
                          focal=262.5, device="cuda")
    p = fusion.FusionParams(**dict(sc.params, iterations=8))
    dom = volume.VolumeDomain(sc.origin, sc.voxel_size, sc.resolution)
    views, u0, seen = fusion.prepare(sc.depths, sc.cameras, dom, p)
    res = fusion.fuse(u0, views, p)
    m = mesh.marching_cubes(octree.densify(res.field), seen, dom)
    mt = mesh.marching_cubes_tree(res.field, mesh.seen_tree(seen), dom)
    assert m.faces.shape[0] > 1000
    assert np.array_equal(m.vertices, mt.vertices)
    assert np.array_equal(m.faces, mt.faces)


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
def test_vertex_diff_equals_kdtree():
    """vertex_diff on the GPU against the reference's own method
    (mesh.py:162-167: scipy's k-d tree, queried here) -- the distances are
    equal bit for bit: surface-like sets, a volumetric cloud, far-apart
    sets, duplicates and a single target vertex."""
    from scipy.spatial import cKDTree
    from paper_1608_07411_b200 import mesh
    rng = np.random.default_rng(0)

    def sphere(n, r, c):
        v = rng.normal(size=(n, 3))
        return c + r * v / np.linalg.norm(v, axis=1, keepdims=True)

    cases = [
        (sphere(20000, 0.3, 0.5), sphere(30000, 0.31, 0.5)),
        (rng.uniform(0, 1, (5000, 3)), rng.uniform(0, 1, (7000, 3))),
        (sphere(3000, 0.1, 0.0), sphere(3000, 0.1, 5.0)),      # disjoint
        (rng.uniform(0, 1, (100, 3)), np.full((50, 3), 0.25)),  # duplicates
        (rng.uniform(-2, 2, (1000, 3)), np.array([[0.1, 0.2, 0.3]])),
        (rng.uniform(0, 1, (4000, 3)) * [1.0, 1.0, 0.0],        # planar
         rng.uniform(0, 1, (4000, 3)) * [1.0, 1.0, 0.0]),
    ]
    for a, b in cases:
        d = mesh.vertex_diff(mesh.TriMesh(a, None), mesh.TriMesh(b, None))
        want_ab = cKDTree(b).query(a)[0]
        want_ba = cKDTree(a).query(b)[0]
        assert np.array_equal(d.d_ab, want_ab)
        assert np.array_equal(d.d_ba, want_ba)
        both = np.concatenate([want_ab, want_ba])
        assert d.mean == float(both.mean()) and d.max == float(both.max())
        assert d.std == float(both.std())
    with pytest.raises(ValueError):
        mesh.vertex_diff(mesh.TriMesh(np.zeros((0, 3)), None),
                         mesh.TriMesh(np.zeros((4, 3)), None))


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
def test_vertex_diff_of_fused_meshes():
    """The comparison the reference's acceptance run makes: the tree
    solver's mesh against the mesh of the initial field (cfg1), all on the
    device, equal to the k-d tree's numbers."""
    from scipy.spatial import cKDTree
    from paper_1608_07411_b200 import fusion, mesh, volume
    from tests.goldens import cfg1_inputs
    depths, cams, origin, vox, n, p = cfg1_inputs()
    dom = volume.VolumeDomain(origin, vox, n)
    fp = fusion.FusionParams(delta=p.delta, eta=p.eta, lam=p.lam,
                             iterations=10)
    views, u0, seen = fusion.prepare(depths, cams, dom, fp)
    st = mesh.seen_tree(seen)
    m0 = mesh.marching_cubes_tree(u0, st, dom)
    res = fusion.fuse(u0, views, fp)
    m1 = mesh.marching_cubes_tree(res.field, st, dom)
    d = mesh.vertex_diff(m0, m1)
    assert np.array_equal(d.d_ab, cKDTree(m1.vertices).query(m0.vertices)[0])
    assert np.array_equal(d.d_ba, cKDTree(m0.vertices).query(m1.vertices)[0])
    assert 0.0 < d.max < 8 * vox
