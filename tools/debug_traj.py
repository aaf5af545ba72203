"""Run a hybrid trajectory until a sweep reports left-unchanged cells, then
report NaN/inf in the state (development aid; run with DD_DEBUG_OVF=1)."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2405_09400_b200 import DomDec, DomDecError  # noqa: E402
from synth import make_problem  # noqa: E402

N, s, theta, cycles = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3]), int(sys.argv[4])
p = make_problem("gm", N, s, eps_factor=2.0, theta_deg=theta, seed=0)
dd = DomDec.from_problem(p)
t0 = time.time()


def report(tag):
    off, ext, pos, data = dd.export_cells()
    area = ext[:, 0].astype(np.int64) * ext[:, 1]
    bad = ~np.isfinite(data)
    print(tag, "nonfinite entries", int(bad.sum()), "max ext", ext.max(0), "mean ext", ext.mean(0), flush=True)
    for part in ("A", "B"):
        try:
            a = dd.export_alpha(part)
            print(tag, "alpha", part, "nonfinite", int((~np.isfinite(a)).sum()), "absmax", np.nanmax(np.abs(a)), flush=True)
        except DomDecError as ex:
            print(tag, "alpha", part, ex)
    big = np.argsort(area)[-6:]
    for k in big:
        d = data[pos[k]:pos[k] + area[k]]
        print(f"   cell {k} off {off[k]} ext {ext[k]} mass {d.sum():.3e} min {d.min():.3e} max {d.max():.3e}", flush=True)


for c in range(cycles):
    ok = True
    for part in ("A", "B"):
        try:
            st = dd.sweep(part, stats=True)
        except DomDecError as ex:
            print(f"cycle {c} sweep {part}: {ex}", flush=True)
            ok = False
            break
    if not ok:
        report("after failure")
        break
    fs = dd.flow_update(stats=True)
    if c % 5 == 0:
        report(f"c{c} e0={st['l1x_entry']:.3e} flow_ms={fs['solver_ms']:.0f}")
print("done", time.time() - t0)
