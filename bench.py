#!/usr/bin/env python
"""Benchmark: octree leaf-updates/s per solver iteration (BASELINE.json
metric) on BASELINE config 4, the solver microbenchmark -- the largest
configuration that fits one GPU, the one the metric's 1/2/4/8-GPU numbers
are quoted on:

  random adaptive octree of ~100M Morton-ordered leaves refined around a
  random implicit surface (59/27/11 % at depths 12/11/10), N = 32 fp32 TSDF
  samples U(-1, 1) per leaf, fp32 u (and the 3-vector dual p in pd mode),
  restructuring off, 100 iterations.

A step = one full solver pass exactly as the reference's fuse loop runs it
(reference fusion.py:218-236): iterate (update of every leaf) + propagate +
energy.  ``value`` is the reference's descent (the parity-pinned solver,
fp32 throughput mode); ``pd_mode`` is the north_star's TV-L1 primal-dual
iteration on the same tree; ``cfg2`` keeps the fixed-structure solver test
(16.8M leaves, N = 16) as an extra line.  ``parity`` holds fp32-vs-fp64
max |u| differences after each configuration's whole schedule (the fp64 mode
is bit-exact against the oracle: tests/test_gpu_cfg5.py, test_gpu_parity.py).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl cuda|reference]

Under torchrun (N > 1) the one cfg5 tree is cut into N Morton ranges
(shard.py), each rank updates its own leaves and exchanges halos over NCCL:
strong scaling, value = all leaves / the max-over-ranks pass time.

Prints ONE JSON line (rank 0).  ``--impl reference`` times the reference's
own compiled kernels (oracle/_ref, built from /root/reference/.../
_kernels.pyx) on all host cores, one independent replica per core, on a
bounded sample of the same workload (the cfg5 generator at 1M leaves).
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import statistics
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402

METRIC = "octree leaf-updates/s per TV-L1 iteration"
UNIT = "leaf-updates/s"
CONFIG_NAME = ("cfg5 solver microbenchmark: random adaptive octree, ~100M "
               "Morton-ordered leaves (depths 12/11/10), N=32 fp32 samples "
               "U(-1,1) per leaf, restructuring off, 100 iterations")
CFG2_NAME = ("cfg2 fixed-structure solver test: full octree depth 8 "
             "(256^3 leaves), N=16 fp32 samples, 10% invalid, lambda=1, "
             "split/join off, 200 iterations")


def parse():
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("cuda", "reference"), default="cuda")
    ap.add_argument("--leaves", type=int, default=100_000_000,
                    help="cfg5 target leaf count")
    ap.add_argument("--views", type=int, default=32)
    ap.add_argument("--cpu-leaves", type=int, default=1_000_000,
                    help="leaves of the bounded CPU-reference sample")
    ap.add_argument("--cpu-passes", type=int, default=3)
    ap.add_argument("--e2e-iters", type=int, default=100,
                    help="iterations of the e2e fuse() call (config: 100)")
    ap.add_argument("--cfg2-depth", type=int, default=8)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-pd", action="store_true")
    ap.add_argument("--no-cfg2", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    return ap.parse_args()


def cfg5_params(iterations=100):
    from paper_1608_07411_b200.fusion import FusionParams
    return FusionParams(lam=0.3, iterations=iterations, tau=-1.0,
                        tau_split=0.0, tau_join=1.5)


def cfg2_params(iterations=200):
    from paper_1608_07411_b200.fusion import FusionParams
    return FusionParams(lam=1.0, iterations=iterations, tau=-1.0,
                        tau_split=0.0, tau_join=1.5)


# ----------------------------------------------------------------- clocks --
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", "-i", str(self.index),
                     f"--query-gpu={self.Q}", "--format=csv,noheader,nounits"],
                    capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.05)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"],
                    "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                 "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 4 + i and r[4 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ------------------------------------------------------------- roofline --
def hbm_peak():
    try:
        peak = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))["hbm_gbs"]
        if peak:
            return float(peak), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        pass
    return 6650.0, "fallback (B200_PROFILING.md)"


def lib_sha():
    """Hash of the CUDA library's sources and build recipe (the build is a
    deterministic function of them)."""
    import glob
    h = hashlib.sha256()
    csrc = os.path.join(REPO, "paper_1608_07411_b200", "csrc")
    for f in sorted(glob.glob(os.path.join(csrc, "*"))) + [
            os.path.join(REPO, "include", "octfuse_b200.h")]:
        h.update(os.path.basename(f).encode())
        with open(f, "rb") as fp:
            h.update(fp.read())
    return h.hexdigest()[:16]


def ncu_traffic(kernel, workload):
    """DRAM bytes (read + write) per launch of ``kernel`` on ``workload``
    from the committed ncu --set full capture (profiles/r*/ncu_traffic.json)
    -- only when it was captured from this exact library source (lib_sha),
    else None: a changed kernel has no measured traffic yet."""
    import glob
    sha = lib_sha()
    for path in sorted(glob.glob(os.path.join(REPO, "profiles", "r*",
                                              "ncu_traffic.json")))[::-1]:
        try:
            rec = json.load(open(path))
        except Exception:
            continue
        for e in rec.get("entries", []):
            if (e.get("kernel") == kernel and e.get("workload") == workload
                    and e.get("lib_sha") == sha):
                return {"bytes": e["dram_bytes_per_launch"],
                        "source": os.path.relpath(path, REPO)}
    return None


def roofline(kernel, nleaves, b_leaf, kernel_ms, workload):
    peak, src = hbm_peak()
    ach = nleaves * b_leaf / (kernel_ms / 1e3) / 1e9
    tr = ncu_traffic(kernel, workload)
    return {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
            "frac": ach / peak,
            "traffic": tr["bytes"] if tr else None,
            "traffic_source": tr["source"] if tr else
            "no ncu capture of this library build",
            "kernel": kernel, "kernel_ms": kernel_ms,
            "bytes_per_leaf": b_leaf, "leaves_per_launch": nleaves,
            "peak_source": src}


# ------------------------------------------------------------ GPU workload --
def build_cfg5(args):
    import torch
    from paper_1608_07411_b200 import scenes
    u0, samples, info = scenes.cfg5_inputs(args.leaves, nviews=args.views,
                                           device="cuda")
    torch.cuda.synchronize()
    return u0, samples, info


def _timed(solver, t0, k, stream=None):
    """Device time (CUDA events on the launch stream) of passes t0..t0+k-1."""
    import torch
    stream = stream or torch.cuda.current_stream()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    solver.run(t0, k)
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


def run_cuda(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_1608_07411_b200 import fusion

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    u0, samples, info = build_cfg5(args)
    p = cfg5_params()
    if world > 1:
        from paper_1608_07411_b200 import shard
        # the plan is built once (rank 0) and each rank receives its part
        h = u0.to_host(scratch=False) if rank == 0 else None
        plan = shard.plan_scattered(h.child if h else None, u0.d_max, world,
                                    rank, used=u0.used)
        del h
        sharded = shard.ShardedSolver(u0, None, p, plan, rank,
                                      precision="fp32", samples=samples)
        solver = sharded.s
        runner = sharded
        nleaves = int(plan.leaves_per_rank.sum())
        my_leaves = int(plan.leaves_per_rank[rank])
    else:
        solver = fusion.Solver(u0, None, p, precision="fp32", samples=samples)
        runner = solver
        nleaves = my_leaves = solver.ctx.info()["leaves"]
    runner.run(0, args.warmup)
    dinfo = solver.ctx.info()
    solver.ctx.profile(True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clocks:
        e0.record(stream)
        runner.run(args.warmup, args.steps)
        e1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    prof = solver.ctx.profile(False)
    ms_t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    ms_step = ms_max / args.steps
    value = nleaves * args.steps / (ms_max / 1e3)
    # algorithmic bytes per leaf-update: snapshot read +
    # u write (fp32) + the N fp32 samples (all valid: no validity bits)
    b_leaf = 4 + 4 + 4 * args.views
    leaf_ms = (prof["leaf_ms"] / prof["leaf_launches"]
               if prof["leaf_launches"] else None)
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (seeded generator paper_1608_07411_b200/scenes.py "
                "cfg5_inputs)",
        "config": {"workload": CONFIG_NAME, "leaves": nleaves,
                   "leaves_per_gpu": my_leaves, "nodes": info["nodes"],
                   "leaves_per_level": info["leaves_per_level"],
                   "samples_per_leaf": args.views, "d_max": 12,
                   "solver": "descent (the reference's update, "
                             "_kernels.pyx:205-253)",
                   "parallelism": (f"{world} Morton-range shards, NCCL halo "
                                   "exchange" if world > 1 else "single GPU"),
                   "l2": "inputs larger than L2 (13.6 GB streamed per pass)",
                   "step": "iterate + propagate + energy (reference fuse loop)"},
        "roofline": (roofline("k_leaf_pass", my_leaves, b_leaf, leaf_ms, "cfg5")
                     if leaf_ms else None),
        "breakdown_ms": {"leaf_update_and_energy": leaf_ms,
                         "rest": ms_step - leaf_ms if leaf_ms else None},
        "gpu_launches": prof["launches"],
        "clocks": clocks.summary(),
        "store": {"mask_format": bool(dinfo["mask_samples"]),
                  "tiles": dinfo["tiles"]},
    }
    solver.close()
    del solver, runner
    torch.cuda.empty_cache()
    if rank != 0:
        return out
    if not args.no_pd:
        out["pd_mode"] = run_pd_mode(u0, samples, p, args, nleaves)
        torch.cuda.empty_cache()
    if not args.no_parity:
        out["parity"] = {"cfg5": parity_cfg5(u0, samples, p)}
        torch.cuda.empty_cache()
    if not args.no_e2e:
        out["e2e"] = run_e2e(u0, samples, p, args, info)
        torch.cuda.empty_cache()
    del u0, samples
    torch.cuda.empty_cache()
    if not args.no_cfg2:
        c2 = run_cfg2(args)
        if "parity" in out and "parity" in c2:
            out["parity"]["cfg2"] = c2.pop("parity")
        out["cfg2"] = c2
        torch.cuda.empty_cache()
    if world == 1 and not args.no_cpu:
        out["cpu_baseline"] = cpu_baseline(args)
    return out


def run_pd_mode(u0, samples, p, args, nleaves):
    """The north_star's TV-L1 primal-dual iteration (solver='pd') on the same
    tree: one step = one primal-dual pass (dual + primal + prox + propagate
    of u, ubar, p) with its energy.  Parity is against its own CPU
    restatement (oracle/pd_oracle.c; the reference has no such solver)."""
    from paper_1608_07411_b200 import fusion
    s = fusion.PDSolver(u0, None, p, precision="fp32", samples=samples)
    s.run(0, args.warmup)
    s.ctx.profile(True)
    ms = _timed(s, args.warmup, args.steps)
    prof = s.ctx.profile(False)
    s.close()
    kms = prof["leaf_ms"] / max(prof["leaf_launches"], 1)
    # u, ubar, px, py, pz read + written (fp32) + the N sorted samples
    b_leaf = 10 * 4 + 4 * args.views
    return {"solver": "pd", "value": nleaves * args.steps / (ms / 1e3),
            "unit": UNIT, "ms_per_step": ms / args.steps,
            "roofline": roofline("k_pd_pass", nleaves, b_leaf, kms, "cfg5"),
            "gpu_launches": prof["launches"],
            "note": "north_star TV-L1 primal-dual; parity vs its CPU "
                    "restatement (tests/test_gpu_pd.py, test_gpu_cfg5.py), "
                    "unpinned vs reference"}


def _max_diff(a, b, used):
    return float((a[:used].double() - b[:used].double()).abs().max().item())


def parity_cfg5(u0, samples, p):
    """fp32 throughput mode vs the fp64 parity mode after the configuration's
    whole schedule (K = 100), full size, every live node; both solvers.  The
    fp64 mode equals the CPU oracle bit for bit (tests/test_gpu_cfg5.py)."""
    from paper_1608_07411_b200 import fusion
    k = p.iterations
    out = {"K": k}
    for name, cls in (("descent", fusion.Solver), ("pd", fusion.PDSolver)):
        res = []
        for prec in ("fp32", "fp64"):
            s = cls(u0, None, p, precision=prec, samples=samples)
            s.run(0, k)
            v = s.cur if cls is fusion.Solver else s.state[0]
            res.append(v[:u0.used].clone())
            s.close()
            del s
        out[f"max_abs_u_fp32_vs_fp64_{name}"] = _max_diff(res[0], res[1],
                                                          u0.used)
    out["tolerance"] = 1e-4
    out["fp64_vs_oracle"] = ("bit-exact (tests/test_gpu_cfg5.py: descent and "
                             "pd, K=100 at 60k leaves)")
    return out


def run_e2e(u0, samples, p, args, info):
    """Same metric through the public API with host inputs: pinned host
    reference-layout u0 pool + per-slot sample arrays -> one fusion.fuse call
    running the configuration's whole schedule (100 iterations) -> the final
    pool back on the host.  Bytes per step = the call's copies / iterations."""
    import torch
    from paper_1608_07411_b200 import fusion, octree

    def pinned(t):
        h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        h.copy_(t)
        return h

    F = samples[0]
    hF = pinned(F)
    hu = (pinned(u0.value[:u0.used]), pinned(u0.child[:u0.used]),
          u0.state.copy())
    h2d = hF.numel() * 4 + sum(a.numel() * a.element_size() for a in hu[:2])
    k = args.e2e_iters
    pk = fusion.FusionParams(**{**p.__dict__, "iterations": k})
    runs = []
    for _ in range(2):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        w0 = time.perf_counter()
        dF = hF.to("cuda", non_blocking=True)
        du = octree.OctreeField.from_host(hu[0], hu[1], hu[2], u0.d_max)
        torch.cuda.synchronize()
        w1 = time.perf_counter()
        res = fusion.fuse(du, None, pk, precision="fp32", samples=(dF, None))
        torch.cuda.synchronize()
        w2 = time.perf_counter()
        host = res.field.to_host(scratch=False)
        e1.record()
        torch.cuda.synchronize()
        w3 = time.perf_counter()
        ms = e0.elapsed_time(e1)
        d2h = host.value.nbytes + host.child.nbytes
        nleaves = int((host.child < 0).sum())
        runs.append({"value": nleaves * k / (ms / 1e3), "unit": UNIT,
                     "h2d_bytes_per_step": int(h2d // k),
                     "d2h_bytes_per_step": int(d2h // k),
                     "ms_total": ms, "steps": k,
                     "phases_ms": {"h2d": (w1 - w0) * 1e3,
                                   "fuse": (w2 - w1) * 1e3,
                                   "d2h": (w3 - w2) * 1e3}})
        del dF, du, res, host
        torch.cuda.empty_cache()
    best = min(runs, key=lambda r: r["ms_total"])
    return dict(best, repeats_ms=[r["ms_total"] for r in runs],
                statistic="faster of 2 end-to-end calls (the first also "
                          "warms the allocator)",
                api=("paper_1608_07411_b200.fusion.fuse(u0, None, params, "
                     "samples=...) on pinned host pools: the configuration's "
                     "whole schedule in one call"))


# ------------------------------------------------------------------ cfg2 --
def build_cfg2(depth, nviews=16, seed=0):
    """cfg2 views and u0 built on the GPU from the seeded dense sample grids."""
    import torch
    from paper_1608_07411_b200 import fusion, octree, scenes
    fs, ws = scenes.make_cfg2_samples(d_max=depth, n_samples=nviews, seed=seed)
    n = 1 << depth
    wf = torch.zeros((n, n, n), dtype=torch.float64, device="cuda")
    wsum = torch.zeros_like(wf)
    views = []
    for f, w in zip(fs, ws):
        fd = torch.from_numpy(f).cuda()
        wd = torch.from_numpy(w).cuda()
        views.append(octree.build_octree(fd, wd, tau=-1.0, dtype=np.float32))
        wf += fd.double() * wd.double()     # reference cli.py:148-149
        wsum += wd.double()
    del fs, ws
    p = cfg2_params()
    u0 = octree.build_octree(fusion.initial_field(wf, wsum, p.gamma), tau=-1.0)
    torch.cuda.synchronize()
    return views, u0, p


def run_cfg2(args):
    """BASELINE config 1 (fixed-structure solver test) as an extra line:
    descent fp32, pd fp32, and the fp32-vs-fp64 parity after the whole
    200-pass schedule."""
    from paper_1608_07411_b200 import fusion
    views, u0, p = build_cfg2(args.cfg2_depth)
    out = {"workload": CFG2_NAME}
    for name, cls, b_leaf, kern in (
            ("descent", fusion.Solver, 4 + 4 + 64 + 2, "k_leaf_pass"),
            ("pd", fusion.PDSolver, 40 + 64 + 2, "k_pd_pass")):
        s = cls(u0, views, p, precision="fp32")
        s.run(0, args.warmup)
        n = s.ctx.info()["leaves"]
        s.ctx.profile(True)
        ms = _timed(s, args.warmup, args.steps)
        prof = s.ctx.profile(False)
        s.close()
        kms = prof["leaf_ms"] / max(prof["leaf_launches"], 1)
        out[name] = {"value": n * args.steps / (ms / 1e3), "unit": UNIT,
                     "ms_per_step": ms / args.steps, "leaves": n,
                     "roofline": roofline(kern, n, b_leaf, kms, "cfg2")}
    if not args.no_parity:
        k = p.iterations
        par = {"K": k}
        for name, cls in (("descent", fusion.Solver), ("pd", fusion.PDSolver)):
            res = []
            for prec in ("fp32", "fp64"):
                s = cls(u0, views, p, precision=prec)
                s.run(0, k)
                res.append((s.cur if cls is fusion.Solver
                            else s.state[0])[:u0.used].clone())
                s.close()
            par[f"max_abs_u_fp32_vs_fp64_{name}"] = _max_diff(res[0], res[1],
                                                              u0.used)
        par["tolerance"] = 1e-4
        par["fp64_vs_oracle"] = ("bit-exact (tests/test_gpu_fullsize.py at "
                                 "depth 8; tests/test_gpu_parity.py K=200 at "
                                 "depth 5)")
        out["parity"] = par
    return out


# ---------------------------------------------------------- CPU reference --
def _ref_kernels():
    """The reference's own compiled kernels (oracle/_ref) if present, else
    the C restatement (oracle/liboctfuse_oracle.so)."""
    import glob
    import importlib.util
    so = glob.glob(os.path.join(REPO, "oracle", "_ref", "_kernels*.so"))
    if so:
        spec = importlib.util.spec_from_file_location("_kernels", so[0])
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        return mod, "reference"
    from oracle import oracle as orc
    return orc, "port"


def _cpu_instance(leaves, nviews):
    """The cfg5 generator at ``leaves`` on the host (torch CPU tree build,
    numpy samples): u pool + one view pool per sample index with the tree's
    structure (the reference reads a view at the leaf's own slot), u0 inner
    nodes by the reference's own propagate -- the pool-level driver of
    SURVEY.md §8(d)."""
    from oracle import oracle as orc
    from paper_1608_07411_b200 import scenes
    kern, _ = _ref_kernels()
    child, d, info = scenes.cfg5_tree(leaves, 12, 0, device="cpu")
    child = child.numpy().astype(np.int32)
    used = child.shape[0]
    rng = np.random.default_rng(1)
    F = rng.uniform(-1.0, 1.0, (nviews, used)).astype(np.float32)
    fsum = np.zeros(used, dtype=np.float64)
    for v in range(nviews):                 # view order (cli.py:148-149)
        fsum += F[v].astype(np.float64)
    state = np.array([used, -1, used], dtype=np.int64)
    ones = np.ones(used, dtype=np.float32)
    views = [orc.Pool(F[v], child, state.copy(), d, weight=ones)
             for v in range(nviews)]
    u0 = orc.Pool(fsum / (nviews + 1e-4), child.copy(), state.copy(), d)
    kern.propagate(u0.value, u0.child)
    return orc.solver_pool(u0, cap=used), views, info["leaves"]


def _cpu_pass(kern, u, views, p, t):
    from oracle import oracle as orc
    vv = [v.value for v in views]
    vw = [v.weight for v in views]
    vc = [v.child for v in views]
    xi = orc.step_scale(t, p)
    kern.iterate_pass(u.value, u.snap, u.child, u.joined, u.state, vv, vw, vc,
                      u.d_max, p.lam, p.eps, p.gamma, xi, p.tau_split,
                      p.tau_join, p.clamp, False, None)
    kern.propagate(u.value, u.child)
    kern.tree_energy(u.value, u.child, vv, vw, vc, u.d_max, p.lam, p.eps,
                     p.gamma)


def cpu_baseline(args):
    kern, kind = _ref_kernels()
    u, views, nleaves = _cpu_instance(args.cpu_leaves, args.views)
    p = cfg5_params()
    _cpu_pass(kern, u, views, p, 0)
    t0 = time.perf_counter()
    for t in range(1, 1 + args.cpu_passes):
        _cpu_pass(kern, u, views, p, t)
    dt = time.perf_counter() - t0
    return {"value": nleaves * args.cpu_passes / dt, "unit": UNIT, "cores": 1,
            "kind": kind,
            "sample": f"cfg5 generator at {nleaves} leaves ({args.views} "
                      f"samples per leaf), {args.cpu_passes} passes of "
                      f"iterate+propagate+energy, 1 thread (the reference is "
                      f"single-threaded; the full 100M-leaf tree exceeds its "
                      f"int32 pool)",
            "cpu": _cpu_model(), "host_cpus": os.cpu_count()}


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


_INST = None


def _replica_worker(args, steps, barrier, q):
    try:
        kern, kind = _ref_kernels()
        u, views, _ = _INST
        p = cfg5_params()
        times = []
        for t in range(steps):
            barrier.wait(timeout=1800)
            t0 = time.perf_counter()
            _cpu_pass(kern, u, views, p, t)
            times.append(time.perf_counter() - t0)
        q.put((kind, times))
    except BaseException as exc:  # never leave the others at the barrier
        barrier.abort()
        q.put(("error", repr(exc)))


def run_reference(args, world):
    """All host cores: one independent replica of the bounded sample per
    core (forked copies of one instance), passes in lock-step; step time =
    slowest replica."""
    import multiprocessing as mp
    global _INST
    nproc = os.cpu_count() or 1
    _INST = _cpu_instance(args.cpu_leaves, args.views)
    nleaves = _INST[2]
    ctx = mp.get_context("fork")
    steps = args.warmup + args.steps
    barrier = ctx.Barrier(nproc)
    q = ctx.Queue()
    procs = [ctx.Process(target=_replica_worker, args=(args, steps, barrier, q))
             for _ in range(nproc)]
    for pr in procs:
        pr.start()
    res = [q.get() for _ in procs]
    for pr in procs:
        pr.join()
    errs = [r[1] for r in res if r[0] == "error"]
    if errs:
        raise RuntimeError(f"reference replica failed: {errs[0]}")
    kind = res[0][0]
    step_t = [max(r[1][i] for r in res) for i in range(args.warmup, steps)]
    total = sum(step_t)
    value = nproc * nleaves * args.steps / total
    sample = (f"cfg5 generator at {nleaves} leaves ({args.views} samples per "
              f"leaf) per replica; {nproc} replicas = one per host core, "
              f"lock-stepped passes of iterate+propagate+energy (the full "
              f"100M-leaf tree exceeds the reference's int32 pool)")
    return {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generator paper_1608_07411_b200/scenes.py "
                "cfg5_tree)",
        "config": {"workload": CONFIG_NAME, "parallelism": f"cpu{nproc}",
                   "leaves_per_replica": nleaves},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": nproc,
                         "kind": kind, "sample": sample, "cpu": _cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args, world)), flush=True)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl")
    out = run_cuda(args, rank, world, local_rank)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
