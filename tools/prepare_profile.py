"""Input stage of cfg3 at full depth (8 of its views, 512^3): one warm
`fusion.prepare`, then one between cudaProfilerStart/Stop for
  ncu --profile-from-start off --metrics gpu__time_duration.sum --csv ...
(profiles/r02/launches_prepare_cfg3.md).  GPU box only."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_1608_07411_b200 import fusion, scenes, volume
sc = scenes.make_cfg3(d_max=9, n_views=8, device="cuda")
p = fusion.FusionParams(**dict(sc.params, iterations=1))
dom = volume.VolumeDomain(sc.origin, sc.voxel_size, sc.resolution)
views, u0, seen = fusion.prepare(sc.depths, sc.cameras, dom, p)   # warm
torch.cuda.synchronize()
torch.cuda.profiler.start()
t = time.time()
views, u0, seen = fusion.prepare(sc.depths, sc.cameras, dom, p)
torch.cuda.synchronize()
print("prepare 8 views s", time.time() - t)
torch.cuda.profiler.stop()
