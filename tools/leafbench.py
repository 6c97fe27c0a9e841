"""Kernel tuning harness: cfg2 workload, batched frozen passes, leaf-kernel
time from the library's own CUDA events.  Select a library build with
OCTF_LIB_PATH=... (e.g. a LEAF_MINB variant from tools/build_variants.sh)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import torch  # noqa: E402
from paper_1608_07411_b200 import fusion  # noqa: E402

depth = int(os.environ.get("DEPTH", "8"))
views, u0, p = bench.build_gpu_workload(depth, int(os.environ.get("VIEWS", "16")))
libs = sys.argv[1:] or [None]
for prec in ("fp32",):
    s = fusion.Solver(u0, views, p, precision=prec)
    s.run(0, 3)
    s.ctx.profile(True)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    s.run(3, 30)
    e1.record()
    torch.cuda.synchronize()
    pr = s.ctx.profile(False)
    print(os.environ.get("OCTF_LIB_PATH", "default"), prec,
          "step_ms %.4f" % (e0.elapsed_time(e1) / 30),
          "leaf_ms %.4f" % (pr["leaf_ms"] / max(pr["leaf_launches"], 1)))
