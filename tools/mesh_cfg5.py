"""Mesh readout straight from the leaf store on BASELINE config 4 (the cfg5
solver microbenchmark tree, depth 12: 550 GB as a dense f64 grid): a few
fp32 descent passes, then mesh.tree_zero_surface, timed.

  python tools/mesh_cfg5.py [--leaves 100000000] [--passes 20]"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_1608_07411_b200 import fusion, mesh, scenes  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--leaves", type=int, default=100_000_000)
ap.add_argument("--passes", type=int, default=20)
ap.add_argument("--slab", type=int, default=16,
                help="bricks (8 cells) of x per readout call")
args = ap.parse_args()
u0, samples, info = scenes.cfg5_inputs(args.leaves, nviews=32, device="cuda")
p = fusion.FusionParams(iterations=args.passes, tau=-1.0, tau_split=0.0,
                        tau_join=1.5, lam=0.3)
res = fusion.fuse(u0, None, p, precision="fp32", samples=samples)
del samples
torch.cuda.synchronize()
torch.cuda.reset_peak_memory_stats()
out = {"leaves": info["leaves"], "passes": args.passes, "d_max": 12}
nb = ((1 << 12) - 1 + 7) // 8
torch.cuda.synchronize()
t0 = time.perf_counter()
nv = nf = 0
for b0 in range(0, nb, args.slab):
    v, f = mesh.tree_zero_surface(res.field, slab=(b0, min(b0 + args.slab, nb)))
    nv += v.shape[0]
    nf += f.shape[0]
    del v, f
torch.cuda.synchronize()
out["readout_s"] = time.perf_counter() - t0
out["slabs"] = (nb + args.slab - 1) // args.slab
out.update(vertices=int(nv), faces=int(nf),
           peak_gb=torch.cuda.max_memory_allocated() / 1e9,
           dense_f64_gb=(1 << 36) * 8 / 1e9)
print(json.dumps(out))
