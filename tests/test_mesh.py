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
