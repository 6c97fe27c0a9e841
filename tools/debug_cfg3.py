"""Pass-by-pass GPU vs oracle comparison on the reduced cfg3 scene: reports
the first pass whose pools differ and what the differing nodes are."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from paper_1608_07411_b200 import fusion, scenes, volume  # noqa: E402
from tests.test_gpu_cfg34 import oracle_prepare  # noqa: E402

sc = scenes.make_cfg3(d_max=7, n_views=16, width=320, height=240, focal=262.5,
                      device="cuda")
kw = dict(sc.params, iterations=6)
pg, po = fusion.FusionParams(**kw), orc.Params(**kw)
dom = volume.VolumeDomain(sc.origin, sc.voxel_size, sc.resolution)
views, u0, _ = fusion.prepare(sc.depths, sc.cameras, dom, pg)
oviews, ou0 = oracle_prepare(sc, po)
s = fusion.Solver(u0, views, pg, precision="fp64")
u = orc.solver_pool(ou0, s.u.capacity)
vv = [v.value for v in oviews]
vw = [v.weight for v in oviews]
vc = [v.child for v in oviews]


def levels(child, used):
    lv = np.full(used, -1)
    lv[0] = 0
    order = [0]
    for n in order:
        b = child[n]
        if b >= 0:
            for q in range(8):
                lv[b + q] = lv[n] + 1
                order.append(b + q)
    return lv


dead_prev = None
for t in range(6):
    prev_child = u.child.copy()
    st = s.step(t)
    xi = orc.step_scale(t, po)
    sp, jo, _ = orc.iterate_pass(u.value, u.snap, u.child, u.joined, u.state,
                                 vv, vw, vc, u.d_max, po.lam, po.eps, po.gamma,
                                 xi, po.tau_split, po.tau_join, po.clamp, False,
                                 None)
    orc.propagate(u.value, u.child)
    used = int(u.state[0])
    gv = s.cur[:used].cpu().numpy()
    gc = s.u.child[:used].cpu().numpy()
    lv = levels(u.child, used)
    dead = lv < 0
    print(f"pass {t}: gpu splits/joins {st.splits}/{st.joins} oracle {sp}/{jo}"
          f" used {used} child_eq {np.array_equal(gc, u.child[:used])} "
          f"dead {int(dead.sum())}")
    d = np.nonzero(gv != u.value[:used])[0]
    if len(d):
        live = d[~dead[d]]
        old = d[dead[d] & dead_prev[d]] if dead_prev is not None else d[:0]
        new = d[dead[d] & ~dead_prev[d]] if dead_prev is not None else d
        print(f"  value diffs {len(d)}: live {len(live)} dead-before {len(old)} "
              f"newly-dead {len(new)}")
        for n in live[:6]:
            print(f"   live node {n} L{lv[n]} leaf {u.child[n] < 0} gpu {gv[n]!r} "
                  f"orc {u.value[n]!r}")
        for n in old[:6]:
            print(f"   old-dead node {n} gpu {gv[n]!r} orc {u.value[n]!r}")
        for n in new[:6]:
            print(f"   new-dead node {n} gpu {gv[n]!r} orc {u.value[n]!r}")
        break
    dead_prev = np.concatenate([dead, np.zeros(0, bool)])
