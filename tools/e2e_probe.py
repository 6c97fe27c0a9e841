"""Phase timing of bench.py's e2e leg (host pools -> fuse -> host), repeated,
to see where its run-to-run variance comes from.  GPU box only."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import bench  # noqa: E402
from paper_1608_07411_b200 import fusion, octree  # noqa: E402

views, u0, p = bench.build_gpu_workload(8, 16)


def pinned(t):
    h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    h.copy_(t)
    return h


hv = [(pinned(v.value), pinned(v.weight), pinned(v.child), v.state.copy())
      for v in views]
hu = (pinned(u0.value), pinned(u0.child), u0.state.copy())
pk = fusion.FusionParams(**{**p.__dict__, "iterations": 20})
for rep in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dv = [octree.OctreeField.from_host(a, c, st, u0.d_max, weight=b)
          for a, b, c, st in hv]
    du = octree.OctreeField.from_host(hu[0], hu[1], hu[2], u0.d_max)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    s = fusion.Solver(du, dv, pk, precision="fp32")
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    s.run(0, 20)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    res = s.result()
    host = res.field.to_host()
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    s.close()
    print("rep %d h2d %.1f ms  solver-setup %.1f ms  20 passes %.1f ms  "
          "result+d2h %.1f ms" % (rep, (t1 - t0) * 1e3, (t2 - t1) * 1e3,
                                  (t3 - t2) * 1e3, (t4 - t3) * 1e3), flush=True)
    del dv, du, res, host, s

# bench.py's own e2e leg, repeated
import argparse  # noqa: E402
args = argparse.Namespace(steps=20, precision="fp32")
for rep in range(4):
    r = bench.run_e2e(views, u0, p, args)
    print("bench.run_e2e rep %d: %.1f ms" % (rep, r["ms_total"]), flush=True)
