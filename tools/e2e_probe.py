"""Phase timing of bench.py's e2e leg (host pools -> fuse -> host), to see
where its time goes.  GPU box only."""
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
torch.cuda.empty_cache()
for rep in range(4):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    dv = [octree.OctreeField.from_host(a, c, st, u0.d_max, weight=b)
          for a, b, c, st in hv]
    du = octree.OctreeField.from_host(hu[0], hu[1], hu[2], u0.d_max)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    s = fusion.Solver(du, dv, pk, precision="fp32")
    torch.cuda.synchronize(); t.append(time.perf_counter())
    s.ctx.profile(True)
    s.run(0, 1)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    pr = s.ctx.profile(True)
    s.run(1, 19)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    res = s.result()
    torch.cuda.synchronize(); t.append(time.perf_counter())
    host = res.field.to_host(scratch=False)
    t.append(time.perf_counter())
    s.close()
    d = [(b - a) * 1e3 for a, b in zip(t, t[1:])]
    print("rep %d h2d %.1f solver-init %.1f first-pass %.1f (prepare %.1f gather %.1f) "
          "19 passes %.1f result %.1f d2h %.1f" % (rep, d[0], d[1], d[2],
          pr["prepare_ms"], pr["gather_ms"], d[3], d[4], d[5]), flush=True)
    del dv, du, res, host, s
