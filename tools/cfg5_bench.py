"""Config-4 solver microbenchmark at full size on one GPU: random adaptive
octree of ~100M leaves (60/27/11 % at depths 12/11/10), N=32 per-leaf fp32
samples U(-1,1), restructuring off, 100 iterations in the config (a bounded
number of timed passes here).  Times the descent (fp32) and the TV-L1
primal-dual mode (fp32 u and 3-vector dual p), reporting leaf-updates/s and
the leaf kernel's fraction of measured HBM bandwidth.

  python tools/cfg5_bench.py [--leaves 100000000] [--steps 10] [--warmup 3]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_1608_07411_b200 import fusion, scenes  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--leaves", type=int, default=100_000_000)
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--views", type=int, default=32)
ap.add_argument("--only", choices=("descent", "pd"), default=None)
args = ap.parse_args()

peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(
    os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
t0 = time.time()
u0, samples, info = scenes.cfg5_inputs(args.leaves, nviews=args.views,
                                      device="cuda")
torch.cuda.synchronize()
setup_s = time.time() - t0
n = info["leaves"]
p = fusion.FusionParams(iterations=1000, tau=-1.0, tau_split=0.0,
                        tau_join=1.5, lam=0.3)
out = {"workload": "cfg5 solver microbenchmark", "leaves": n,
       "nodes": info["nodes"], "views": args.views,
       "leaves_per_level": info["leaves_per_level"], "setup_s": setup_s}


def timed(s, label, b_leaf):
    s.run(0, args.warmup)
    s.ctx.profile(True)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    s.run(args.warmup, args.steps)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    pr = s.ctx.profile(False)
    kms = pr["leaf_ms"] / max(pr["leaf_launches"], 1)
    ach = n * b_leaf / (kms / 1e3) / 1e9
    out[label] = {"value": n / (ms / 1e3), "unit": "leaf-updates/s",
                  "ms_per_step": ms, "kernel_ms": kms, "bytes_per_leaf": b_leaf,
                  "achieved_GBs": ach, "frac_of_measured_hbm": ach / peak}


if args.only in (None, "descent"):
    s = fusion.Solver(u0, None, p, precision="fp32", samples=samples)
    timed(s, "descent_fp32", 4 + 4 + 4 * args.views)
    s.close()
    del s
    torch.cuda.empty_cache()
if args.only in (None, "pd"):
    s = fusion.PDSolver(u0, None, p, precision="fp32", samples=samples)
    timed(s, "pd_fp32", 40 + 4 * args.views)
    s.close()
print(json.dumps(out))
