"""Time the cfg1 scene (restructuring every pass) end to end on the GPU:
TSDF + view trees + u0 on device, then fuse() for 50 passes."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_1608_07411_b200 import fusion, octree, scenes, tsdf, volume  # noqa: E402

sc = scenes.make_cfg1()
dom = volume.VolumeDomain(sc.origin, sc.voxel_size, sc.resolution)
p = fusion.FusionParams(delta=sc.delta, eta=sc.eta, lam=sc.lam,
                        iterations=sc.iterations)
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    n = sc.resolution
    wf = torch.zeros((n, n, n), dtype=torch.float64, device="cuda")
    ws = torch.zeros_like(wf)
    views = []
    for d, c in zip(sc.depths, sc.cameras):
        vt = tsdf.build_view_tsdf(d, c, dom, p.delta, p.eta, accumulate=(wf, ws))
        views.append(fusion.build_view_tree(vt, p.tau))
    u0 = octree.build_octree(fusion.initial_field(wf, ws, p.gamma), tau=p.tau)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    for prec in ("fp64", "fp32"):
        t2 = time.perf_counter()
        res = fusion.fuse(u0, views, p, precision=prec)
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        leaves = sum(s.node_count for s in res.stats)
        print(f"rep{rep} {prec}: setup {1e3*(t1-t0):.1f} ms, fuse 50 passes "
              f"{1e3*(t3-t2):.1f} ms ({1e3*(t3-t2)/50:.2f} ms/pass), "
              f"splits {sum(s.splits for s in res.stats)} joins "
              f"{sum(s.joins for s in res.stats)}")
