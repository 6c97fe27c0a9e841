"""Propagate timing harness: the cfg2 full tree (depth 8) and, with CFG5=1, a
cfg5-style random adaptive tree; f32 values propagated through one context
repeatedly (CUDA events), value hash printed so two builds / modes can be
compared (env A/B switches of the library apply)."""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_1608_07411_b200 import _kernels, octree, scenes  # noqa: E402

depth = int(os.environ.get("DEPTH", "8"))
if os.environ.get("CFG5") == "1":
    child, d_max = scenes.cfg5_tree(int(os.environ.get("LEAVES", "10000000")),
                                    device="cuda")[:2]
    child = child.cuda()
    used = child.shape[0]
    state = np.array([used, -1, used], np.int64)
else:
    u0 = octree.build_octree(
        torch.rand((1 << depth,) * 3, dtype=torch.float64, device="cuda"),
        tau=-1.0, dtype=np.float32)
    child, d_max = u0.child, depth
    used = int(u0.state[0])
    state = np.asarray(u0.state, np.int64).copy()
g = torch.Generator(device="cuda").manual_seed(1)
val = torch.rand(child.shape[0] + 8, generator=g, device="cuda")[:child.shape[0]]
ctx = _kernels._fresh_ctx()
_kernels.propagate(val, child, state=state, d_max=d_max, ctx=ctx)
torch.cuda.synchronize()
for fields in (1,):
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    reps = 50
    e0.record()
    for _ in range(reps):
        _kernels.propagate(val, child, state=state, d_max=d_max, ctx=ctx)
    e1.record()
    torch.cuda.synchronize()
    h = hashlib.sha256(val[:used].cpu().numpy().tobytes()).hexdigest()[:16]
    print("mode", "level" if os.environ.get("OCTF_LEVEL_PROPAGATE") == "1"
          else "up", "nodes", used, "ms %.4f" % (e0.elapsed_time(e1) / reps),
          "hash", h, flush=True)
