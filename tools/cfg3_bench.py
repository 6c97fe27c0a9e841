"""BASELINE config 2 (cfg3, adaptive single object) at full size on one GPU:
64 sphere-traced 640x480 depth maps of the noisy blob, d_max 9 (512^3),
split/join after every pass.  ``--config cfg4`` runs BASELINE config 3 (the
room, 300 frames) at ``--depth`` (default 9; the full depth 11 needs a
sparse build).  Times the input stage (TSDF + view trees + u0)
and K solver passes (iterate + restructure + propagate + energy, host sync
per pass as the reference's loop), reporting leaf-updates/s = pre-pass leaves
/ pass time and the leaf kernel's share.

  python tools/cfg3_bench.py [--passes 20] [--precision fp32] [--views 64]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_1608_07411_b200 import fusion, scenes, volume  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--passes", type=int, default=20)
ap.add_argument("--precision", default="fp32")
ap.add_argument("--views", type=int, default=None)
ap.add_argument("--depth", type=int, default=9)
ap.add_argument("--config", choices=("cfg3", "cfg4"), default="cfg3")
ap.add_argument("--solver", choices=("descent", "pd"), default="descent")
ap.add_argument("--mesh", action="store_true",
                help="also time densify + marching cubes of the result")
ap.add_argument("--save-scene", default=None, help="pickle the rendered scene")
ap.add_argument("--load-scene", default=None, help="reuse a pickled scene")
ap.add_argument("--untimed", action="store_true",
                help="leave the library's phase timers off (their host "
                     "synchronisations cost ~0.05 ms per pass): pass times "
                     "only")
ap.add_argument("--profile-passes", default=None,
                help="a:b -- cudaProfilerStart before pass a, Stop after "
                     "pass b-1 (ncu --profile-from-start off)")
ap.add_argument("--batched", action="store_true",
                help="after the per-pass loop, time the same number of "
                     "further passes in one Solver.run call (the library's "
                     "multi-pass loop, no Python between passes)")
ap.add_argument("--boxed", action="store_true",
                help="box-wise input stage (fusion.prepare_boxed: no dense grid)")
args = ap.parse_args()

t0 = time.time()
if args.load_scene:
    import pickle
    with open(args.load_scene, "rb") as fp:
        sc = pickle.load(fp)
elif args.config == "cfg4":
    sc = scenes.make_cfg4(d_max=args.depth, n_frames=args.views or 300,
                          device="cuda")
else:
    sc = scenes.make_cfg3(d_max=args.depth, n_views=args.views or 64,
                          device="cuda")
if args.save_scene:
    import pickle
    with open(args.save_scene, "wb") as fp:
        pickle.dump(sc, fp)
torch.cuda.synchronize()
t_render = time.time() - t0
p = fusion.FusionParams(**dict(sc.params, iterations=args.passes))
dom = volume.VolumeDomain(sc.origin, sc.voxel_size, sc.resolution)
torch.cuda.synchronize()
t0 = time.time()
if args.boxed:
    views, u0, seen = fusion.prepare_boxed(sc.depths, sc.cameras, dom, p)
else:
    views, u0, seen = fusion.prepare(sc.depths, sc.cameras, dom, p)
torch.cuda.synchronize()
t_prep = time.time() - t0
view_nodes = sum(v.node_count for v in views)
print(json.dumps({"after_prepare": {
    "view_nodes": view_nodes, "u0_nodes": u0.node_count,
    "torch_allocated_gb": torch.cuda.memory_allocated() / 1e9,
    "torch_reserved_gb": torch.cuda.memory_reserved() / 1e9,
    "device_free_gb": torch.cuda.mem_get_info()[0] / 1e9}}), file=sys.stderr,
    flush=True)

if args.solver == "pd":
    s = fusion.PDSolver(u0, views, p, precision=args.precision)
else:
    s = fusion.Solver(u0, views, p, precision=args.precision)
s.ctx.profile(not args.untimed)
passes = []
acc = {}  # per-pass profiles summed (profile(True) reads and resets)
prof_a, prof_b = (map(int, args.profile_passes.split(":"))
                  if args.profile_passes else (-1, -1))
for t in range(args.passes):
    if t == prof_a:
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
    if t == prof_b:
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    st = s.run(t, 1)[0] if args.solver == "pd" else s.step(t)
    e1.record()
    torch.cuda.synchronize()
    pr = s.ctx.profile(not args.untimed)
    for key, val in pr.items():
        if isinstance(val, (int, float)):
            acc[key] = acc.get(key, 0) + val
    passes.append({"ms": e0.elapsed_time(e1), "nodes": st.node_count,
                   "splits": st.splits, "joins": st.joins,
                   "leaf_ms": pr["leaf_ms"], "prepare_ms": pr["prepare_ms"],
                   "gather_ms": pr["gather_ms"],
                   "restructure_ms": pr["restructure_ms"],
                   **({"rebuild_phases_ms": pr["rebuild_phases_ms"]}
                      if os.environ.get("OCTF_PHASES") == "1" else {})})
batched_ms = None
if args.batched and args.solver == "descent":
    s.ctx.profile(False)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    n_before = (7 * s.u.node_count + 1) // 8
    e0.record()
    sts = s.run(args.passes, args.passes)
    e1.record()
    torch.cuda.synchronize()
    batched_ms = e0.elapsed_time(e1) / args.passes
    lv_b = [n_before] + [(7 * q.node_count + 1) // 8 for q in sts[:-1]]
    batched_rate = sum(lv_b) / (e0.elapsed_time(e1) / 1e3)
pr = s.ctx.profile(False)
for key, val in pr.items():
    if isinstance(val, (int, float)):
        acc[key] = acc.get(key, 0) + val
prof = acc
res = s.result()
mesh_info = None
if args.mesh:
    from paper_1608_07411_b200 import mesh, octree
    torch.cuda.synchronize()
    m0 = time.time()
    if args.boxed:   # seen is a tree: the leaf-store readout
        m1 = time.time()
        tm = mesh.marching_cubes_tree(res.field, seen, dom)
    else:
        dense = octree.densify_device(res.field)
        torch.cuda.synchronize()
        m1 = time.time()
        tm = mesh.marching_cubes(dense, seen, dom)
    torch.cuda.synchronize()
    m2 = time.time()
    mesh_info = {"densify_s": m1 - m0, "marching_cubes_s": m2 - m1,
                 "vertices": tm.vertex_count, "faces": tm.face_count}
h = res.field.to_host()
leaves_end = int((h.child[:h.used] < 0).sum())
steady = passes[3:] if len(passes) > 6 else passes
ms = sorted(q["ms"] for q in steady)[len(steady) // 2]
# leaves before each pass ~ nodes*7/8 (complete-children tree: leaves =
# 7*inner + 1 = (7*nodes + 1)/8)
lv = [(7 * q["nodes"] + 1) // 8 for q in passes]
out = {"workload": ("cfg3 adaptive object (BASELINE config 2)"
                    if args.config == "cfg3" else
                    ("cfg4 room (BASELINE config 3) at its configured depth 11"
                     if args.depth >= 11 else
                     "cfg4 room (BASELINE config 3) at reduced depth")),
       "depth": args.depth, "views": len(sc.depths),
       "precision": args.precision,
       "solver": args.solver,
       "render_s": t_render, "prepare_s": t_prep,
       "u0_nodes": u0.node_count, "leaves_end": leaves_end,
       "view_nodes": view_nodes, "boxed": args.boxed,
       "peak_gb": torch.cuda.max_memory_allocated() / 1e9,
       "median_pass_ms": ms,
       **({"batched_ms_per_pass": batched_ms,
           "batched_leaf_updates_per_s": batched_rate}
          if batched_ms is not None else {}),
       "leaf_updates_per_s": lv[-1] / (ms / 1e3),
       "leaf_kernel_ms_per_pass": prof["leaf_ms"] / max(prof["leaf_launches"], 1),
       "profile": prof,
       "mesh": mesh_info, "passes": passes}
print(json.dumps(out))
