"""Phase timing of bench.py's cfg5 e2e leg (pinned host pools -> fuse ->
host): upload, solver set-up (context + packed sample store), the passes,
result, download.  GPU box only."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import bench  # noqa: E402
from paper_1608_07411_b200 import fusion, octree  # noqa: E402

sys.argv = sys.argv[:1]
args = bench.parse()
u0, samples, info = bench.build_cfg5(args)
p = bench.cfg5_params(100)


def pinned(t):
    h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    h.copy_(t)
    return h


hF = pinned(samples[0])
hu = (pinned(u0.value[:u0.used]), pinned(u0.child[:u0.used]), u0.state.copy())
del samples
torch.cuda.empty_cache()
for rep in range(3):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    dF = hF.to("cuda", non_blocking=True)
    du = octree.OctreeField.from_host(hu[0], hu[1], hu[2], u0.d_max)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    s = fusion.Solver(du, None, p, precision="fp32", samples=(dF, None))
    torch.cuda.synchronize(); t.append(time.perf_counter())
    s.run(0, 1)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    s.run(1, 99)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    res = s.result()
    torch.cuda.synchronize(); t.append(time.perf_counter())
    host = res.field.to_host(scratch=False)
    t.append(time.perf_counter())
    s.close()
    d = [(b - a) * 1e3 for a, b in zip(t, t[1:])]
    print("rep %d h2d %.1f solver-init %.1f first-pass %.1f 99 passes %.1f "
          "result %.1f d2h %.1f" % (rep, *d), flush=True)
    del dF, du, res, host, s
    torch.cuda.empty_cache()
