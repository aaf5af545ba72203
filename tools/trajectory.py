"""Hybrid (Alg. 3) or pure domdec trajectory probe: per cycle entry errors,
flow objective, flow time (development aid)."""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2405_09400_b200 import DomDec  # noqa: E402
from synth import make_problem  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--kind", default="gm")
ap.add_argument("--N", type=int, default=256)
ap.add_argument("--s", type=int, default=4)
ap.add_argument("--eps", type=float, default=2.0)
ap.add_argument("--theta", type=float, default=20.0)
ap.add_argument("--cycles", type=int, default=200)
ap.add_argument("--seconds", type=float, default=120)
ap.add_argument("--flow", type=int, default=1, help="flow period in cycles (0 = pure domdec)")
a = ap.parse_args()
p = make_problem(a.kind, a.N, a.s, eps_factor=a.eps, theta_deg=a.theta, seed=0)
dd = DomDec.from_problem(p)
t0 = time.time()
for c in range(a.cycles):
    try:
        sa = dd.sweep("A", stats=True)
        sb = dd.sweep("B", stats=True)
    except Exception as ex:
        print("ERROR", ex, flush=True)
        off, ext, pos, data = dd.export_cells()
        area = ext[:, 0] * ext[:, 1]
        for k in area.argsort()[-5:]:
            print("  big cell", k, off[k], ext[k], data[pos[k]:pos[k]+area[k]].sum(), flush=True)
        break
    fs = None
    tf = 0.0
    if a.flow and (c + 1) % a.flow == 0:
        t1 = time.time()
        fs = dd.flow_update(stats=True)
        tf = time.time() - t1
    cost = float(dd.export_plan_cost().sum()) * p.h * p.h if c % 5 == 0 else float("nan")
    print(f"c{c:4d} t={2 * (c + 1) / p.n:6.3f} e0A={sa['l1x_entry']:.3e} e0B={sb['l1x_entry']:.3e} "
          f"it={(sa['iters_total'] + sb['iters_total']) / (sa['cells'] + sb['cells']):5.1f} "
          f"nc={sa['nonconverged'] + sb['nonconverged']} itmax={max(sa['iters_max'], sb['iters_max'])} cost={cost:.6f} "
          + (f"flow obj={fs['objective']} stat={fs['stationary']} cert={fs['certificate']} moved={fs['changed_cells']} "
             f"rounds={fs['rounds']} {tf:.2f}s" if fs else ""), flush=True)
    if c % 10 == 0 or c == a.cycles - 1:
        off, ext, pos, data = dd.export_cells()
        area = ext[:, 0] * ext[:, 1]
        k = int(area.argmax())
        print(f"   boxes: max ext {ext.max(0)} mean {ext.mean(0)} worst cell {k} off {off[k]} ext {ext[k]} "
              f"mass {data[pos[k]:pos[k]+area[k]].sum():.3e}", flush=True)
    if max(sa["l1x_entry"], sb["l1x_entry"]) <= 1e-4:
        print("converged (R14)", time.time() - t0, flush=True)
        break
    if time.time() - t0 > a.seconds:
        print("time cap", flush=True)
        break
print("marginal_error", dd.marginal_error())
