"""Short cfg5 (BASELINE config 4) solver run for ncu captures: build the
~100M-leaf tree and its samples, then ``--passes`` passes of the descent
and/or the primal-dual solver (fp32).

  python tools/profile_cfg5.py [--only descent|pd] [--passes 4] [--leaves N]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_1608_07411_b200 import fusion, scenes  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--leaves", type=int, default=100_000_000)
ap.add_argument("--passes", type=int, default=4)
ap.add_argument("--views", type=int, default=32)
ap.add_argument("--only", choices=("descent", "pd"), default=None)
args = ap.parse_args()

u0, samples, info = scenes.cfg5_inputs(args.leaves, nviews=args.views,
                                       device="cuda")
p = fusion.FusionParams(iterations=100, tau=-1.0, tau_split=0.0,
                        tau_join=1.5, lam=0.3)
for mode, cls in (("descent", fusion.Solver), ("pd", fusion.PDSolver)):
    if args.only not in (None, mode):
        continue
    s = cls(u0, None, p, precision="fp32", samples=samples)
    s.run(0, args.passes)
    torch.cuda.synchronize()
    s.close()
    del s
    torch.cuda.empty_cache()
print("ok", info["leaves"])
