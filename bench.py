#!/usr/bin/env python
"""Benchmark: octree leaf-updates/s per solver iteration (BASELINE.json metric)
on BASELINE config 1, the fixed-structure solver test:

  full uniform octree at depth 8 (256^3 leaves), N=16 per-leaf fp32 TSDF
  samples = clip(torus signed distance + N(0, 0.01), +-0.04) with 10% marked
  invalid, lambda = 1.0, split/join disabled (tau_split 0, tau_join 1.5).

A step = one full solver pass exactly as the reference's fuse loop runs it
(reference fusion.py:218-236): iterate (descent update of every leaf) +
propagate + energy.  Throughput mode: fp32 iterate (north_star: u within
1e-4); parity of the same code path is covered by tests/.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl cuda|reference]

Prints ONE JSON line (rank 0).  ``--impl reference`` times the reference's own
compiled kernels (oracle/_ref, built from /root/reference/.../_kernels.pyx) on
all host cores (one independent replica per core) on a bounded sample of the
same workload.
"""

from __future__ import annotations

import argparse
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
CONFIG_NAME = ("cfg2 fixed-structure solver test: full octree depth 8 "
               "(256^3 leaves), N=16 fp32 samples, 10% invalid, lambda=1, "
               "split/join off")


def parse():
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("cuda", "reference"), default="cuda")
    ap.add_argument("--depth", type=int, default=8)
    ap.add_argument("--views", type=int, default=16)
    ap.add_argument("--precision", choices=("fp32", "fp64"), default="fp32")
    ap.add_argument("--cpu-depth", type=int, default=6,
                    help="depth of the bounded CPU-baseline sample")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-parity-mode", action="store_true")
    ap.add_argument("--e2e-iters", type=int, default=200,
                    help="iterations of the e2e fuse() call (config: 200)")
    ap.add_argument("--no-pd", action="store_true")
    return ap.parse_args()


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
            self._stop.wait(0.2)

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


# ------------------------------------------------------------ GPU workload --
def build_gpu_workload(depth, nviews, seed=0):
    """Views and u0 built on the GPU from the seeded dense sample grids."""
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


def run_cuda(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_1608_07411_b200 import fusion, octree

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    views, u0, p = build_gpu_workload(args.depth, args.views)
    if world > 1:
        # Morton-range shards of the one cfg2 tree: fixed total work
        from paper_1608_07411_b200 import shard
        h = u0.to_host()
        plan = shard.plan(h.child, h.d_max, world, used=h.used)
        sharded = shard.ShardedSolver(u0, views, p, plan, rank,
                                      precision=args.precision)
        solver = sharded.s
        sharded.run(0, args.warmup)
        nleaves = int(plan.leaves_per_rank.sum())
        my_leaves = int(plan.leaves_per_rank[rank])
    else:
        sharded = None
        solver = fusion.Solver(u0, views, p, precision=args.precision)
        solver.run(0, args.warmup)
    info = solver.ctx.info()
    if sharded is None:
        nleaves = my_leaves = info["leaves"]
    solver.ctx.profile(True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clocks:
        e0.record(stream)
        (sharded or solver).run(args.warmup, args.steps)
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

    # roofline of the dominant kernel (the leaf-update kernel)
    import json as _json
    peaks = {}
    try:
        peaks = _json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak = peaks.get("hbm_gbs")
    peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)"
    if not peak:
        peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
    mask_fmt = bool(info["mask_samples"])
    vsz = 4 if args.precision == "fp32" else 8
    b_leaf = 2 * vsz + 4 * args.views + ((args.views + 7) // 8 if mask_fmt
                                          else 4 * args.views)
    leaf_ms = prof["leaf_ms"] / max(prof["leaf_launches"], 1)
    achieved = my_leaves * b_leaf / (leaf_ms / 1e3) / 1e9
    energy_ms = prof["energy_ms"] / max(prof["energy_launches"], 1)

    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
        "dtype": "f32" if args.precision == "fp32" else "f64",
        "data": "synthetic (seeded generator paper_1608_07411_b200/scenes.py)",
        "config": {"workload": CONFIG_NAME, "leaves": nleaves,
                   "leaves_per_gpu": my_leaves,
                   "samples_per_leaf": args.views, "depth": args.depth,
                   "parallelism": (f"morton-range shards x{world}, NCCL halo "
                                   "exchange" if world > 1 else "single"),
                   "l2": "inputs larger than L2 (>= 1.1 GB streamed per pass)",
                   "step": "iterate + propagate + energy (reference fuse loop)"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": achieved / peak,
                     "traffic": _ncu_traffic(args),
                     "kernel": "k_leaf_pass", "kernel_ms": leaf_ms,
                     "bytes_per_leaf": b_leaf, "peak_source": peak_src},
        "breakdown_ms": {"leaf_update_and_energy": leaf_ms,
                         "separate_energy": energy_ms,
                         "rest": ms_step - leaf_ms - energy_ms},
        "gpu_launches": prof["launches"],
        "clocks": clocks.summary(),
    }
    solver.close()
    if rank == 0 and not args.no_e2e:
        # first after the main timing, with torch's cached blocks released:
        # device allocation on a fragmented heap made single calls noisy
        # (120-700 ms for the same 20 passes); median of three calls, each
        # timed in full, all three listed
        import torch
        torch.cuda.empty_cache()
        runs = [run_e2e(views, u0, p, args) for _ in range(3)]
        runs.sort(key=lambda r: r["ms_total"])
        out["e2e"] = dict(runs[1], repeats_ms=[r["ms_total"] for r in runs],
                          statistic="median of 3 end-to-end calls")
    if rank == 0 and args.precision == "fp32" and not args.no_parity_mode:
        out["parity_mode"] = run_parity_mode(views, u0, p, args, nleaves)
    if rank == 0 and not args.no_pd:
        out["pd_mode"] = run_pd_mode(views, u0, p, args, nleaves, peak)
    if rank == 0 and world == 1 and not args.no_cpu:
        out["cpu_baseline"] = cpu_baseline(args, threads=1)
    return out


def _ncu_traffic(args):
    """dram bytes (read + write) per launch of the leaf kernel from the
    committed ncu --set full capture of this workload (profiles/), or None."""
    import glob
    if (args.depth, args.views, args.precision) != (8, 16, "fp32"):
        return None
    for path in sorted(glob.glob(os.path.join(REPO, "profiles", "r*",
                                              "ncu_traffic.json")))[::-1]:
        try:
            return json.load(open(path))["traffic_bytes_per_launch"]
        except Exception:
            continue
    return None


def run_parity_mode(views, u0, p, args, nleaves):
    """The same workload in the bit-exact fp64 mode (pools identical to the
    reference's kernels), timed the same way."""
    import torch
    from paper_1608_07411_b200 import fusion
    solver = fusion.Solver(u0, views, p, precision="fp64")
    solver.run(0, args.warmup)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    solver.run(args.warmup, args.steps)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    solver.close()
    return {"dtype": "f64", "value": nleaves * args.steps / (ms / 1e3),
            "unit": UNIT, "ms_per_step": ms / args.steps,
            "note": "bit-exact parity mode (tests/test_gpu_parity.py)"}


def run_pd_mode(views, u0, p, args, nleaves, peak):
    """The north_star's TV-L1 primal-dual iteration (solver='pd') on the same
    workload: one step = one primal-dual pass (dual + primal + prox +
    propagate of u, ubar, p) with its energy.  Parity is against its own CPU
    restatement (oracle/pd_oracle.c; the reference has no such solver)."""
    import torch
    from paper_1608_07411_b200 import fusion
    s = fusion.PDSolver(u0, views, p, precision=args.precision)
    s.run(0, args.warmup)
    s.ctx.profile(True)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    s.run(args.warmup, args.steps)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    prof = s.ctx.profile(False)
    s.close()
    kms = prof["leaf_ms"] / max(prof["leaf_launches"], 1)
    vsz = 4 if args.precision == "fp32" else 8
    b_leaf = 10 * vsz + 4 * args.views + (args.views + 7) // 8
    ach = nleaves * b_leaf / (kms / 1e3) / 1e9
    return {"solver": "pd", "value": nleaves * args.steps / (ms / 1e3),
            "unit": UNIT, "ms_per_step": ms / args.steps,
            "roofline": {"bound": "hbm", "achieved": ach, "peak": peak,
                         "unit": "GB/s", "frac": ach / peak,
                         "kernel": "k_pd_pass", "kernel_ms": kms,
                         "bytes_per_leaf": b_leaf},
            "note": "north_star TV-L1 primal-dual; parity vs its CPU "
                    "restatement (tests/test_gpu_pd.py), unpinned vs reference"}


def run_e2e(views, u0, p, args):
    """Same metric through the public API with host inputs: pinned host
    reference-layout pools -> one fuse() call running the configuration's
    whole schedule (BASELINE config 1: 200 iterations; --e2e-iters) -> final
    pool back on the host.  Bytes per step = the call's copies / iterations."""
    import torch
    from paper_1608_07411_b200 import fusion, octree

    def pinned(t):
        h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        h.copy_(t)
        return h

    hv = [(pinned(v.value), pinned(v.weight), pinned(v.child), v.state.copy())
          for v in views]
    hu = (pinned(u0.value), pinned(u0.child), u0.state.copy())
    h2d = sum(a.numel() * a.element_size() + b.numel() * b.element_size()
              + c.numel() * c.element_size() for a, b, c, _ in hv)
    h2d += sum(a.numel() * a.element_size() for a in hu[:2])
    k = args.e2e_iters
    pk = fusion.FusionParams(**{**p.__dict__, "iterations": k})
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    w0 = time.perf_counter()
    dv = [octree.OctreeField.from_host(a, c, st, u0.d_max, weight=b)
          for a, b, c, st in hv]
    du = octree.OctreeField.from_host(hu[0], hu[1], hu[2], u0.d_max)
    torch.cuda.synchronize()
    w1 = time.perf_counter()
    res = fusion.fuse(du, dv, pk, precision=args.precision)
    torch.cuda.synchronize()
    w2 = time.perf_counter()
    host = res.field.to_host(scratch=False)
    e1.record()
    torch.cuda.synchronize()
    w3 = time.perf_counter()
    ms = e0.elapsed_time(e1)
    d2h = host.value.nbytes + host.child.nbytes
    nleaves = (host.child < 0).sum()
    return {"value": float(nleaves) * k / (ms / 1e3), "unit": UNIT,
            "h2d_bytes_per_step": int(h2d // k), "d2h_bytes_per_step": int(d2h // k),
            "ms_total": ms, "steps": k,
            "phases_ms": {"h2d": (w1 - w0) * 1e3, "fuse": (w2 - w1) * 1e3,
                          "d2h": (w3 - w2) * 1e3},
            "api": ("paper_1608_07411_b200.fusion.fuse on host (pinned) pools, "
                    "the configuration's whole schedule in one call")}


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


def _cpu_instance(depth, nviews):
    from oracle import oracle as orc
    from paper_1608_07411_b200 import scenes
    fs, ws = scenes.make_cfg2_samples(d_max=depth, n_samples=nviews)
    views = [orc.build_octree(f, w, tau=-1.0, dtype=np.float32)
             for f, w in zip(fs, ws)]
    wf = sum(w.astype(np.float64) * f.astype(np.float64) for f, w in zip(fs, ws))
    wsum = sum(w.astype(np.float64) for w in ws)
    u0 = orc.build_octree(orc.initial_field(wf, wsum, 1e-4), tau=-1.0)
    return orc.solver_pool(u0), views


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


def cpu_baseline(args, threads=1, passes=4):
    kern, kind = _ref_kernels()
    u, views = _cpu_instance(args.cpu_depth, args.views)
    p = cfg2_params()
    nleaves = 8 ** args.cpu_depth
    _cpu_pass(kern, u, views, p, 0)
    t0 = time.perf_counter()
    for t in range(1, 1 + passes):
        _cpu_pass(kern, u, views, p, t)
    dt = time.perf_counter() - t0
    return {"value": nleaves * passes / dt, "unit": UNIT, "cores": threads,
            "kind": kind,
            "sample": f"cfg2 generator at depth {args.cpu_depth} "
                      f"({nleaves} leaves, {args.views} samples), {passes} "
                      f"passes of iterate+propagate+energy, 1 thread "
                      f"(the reference is single-threaded)",
            "cpu": _cpu_model(), "host_cpus": os.cpu_count()}


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def _replica_worker(args, steps, barrier, q):
    try:
        kern, kind = _ref_kernels()
        u, views = _cpu_instance(args.cpu_depth, args.views)
        p = cfg2_params()
        times = []
        for t in range(steps):
            barrier.wait(timeout=900)
            t0 = time.perf_counter()
            _cpu_pass(kern, u, views, p, t)
            times.append(time.perf_counter() - t0)
        q.put((kind, times))
    except BaseException as exc:  # never leave the others at the barrier
        barrier.abort()
        q.put(("error", repr(exc)))


def run_reference(args, world):
    """All host cores: one independent replica of the bounded sample per
    core, passes in lock-step; step time = slowest replica."""
    import multiprocessing as mp
    nproc = os.cpu_count() or 1
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
    nleaves = 8 ** args.cpu_depth
    value = nproc * nleaves * args.steps / total
    sample = (f"cfg2 generator at depth {args.cpu_depth} ({nleaves} leaves, "
              f"{args.views} samples) per replica; {nproc} replicas = one per "
              f"host core, lock-stepped passes of iterate+propagate+energy")
    return {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generator paper_1608_07411_b200/scenes.py)",
        "config": {"workload": CONFIG_NAME, "parallelism": f"cpu{nproc}"},
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
