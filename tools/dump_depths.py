"""Write the seeded depth maps of a scene generated on the GPU (float32,
compressed) for the golden generator in the build container:
  python tools/dump_depths.py cfg4d8 gpurun_out/depths_cfg4d8.npz"""
import hashlib
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1608_07411_b200 import scenes  # noqa: E402

name, out = sys.argv[1], sys.argv[2]
if name == "cfg4d8":
    sc = scenes.make_cfg4(d_max=8, n_frames=64, device="cuda")
elif name == "cfg3":
    sc = scenes.make_cfg3(device="cuda")
else:
    raise SystemExit("unknown scene")
d = np.stack(sc.depths).astype(np.float32)
np.savez_compressed(out, depths=d)
print(name, hashlib.sha256(d.tobytes()).hexdigest(), os.path.getsize(out))
