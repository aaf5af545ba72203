"""Warm-started flow updates (ctx) vs the cold standalone solver on the same
instances along a hybrid trajectory: exact objective equality and timings
(development aid)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2405_09400_b200 import DomDec, mincost_flow  # noqa: E402
from synth import make_problem  # noqa: E402

for N, s, cycles in [tuple(int(v) for v in a.split(",")) for a in sys.argv[1:]]:
    p = make_problem("gm", N, s, eps_factor=2.0, theta_deg=20, seed=0)
    dd = DomDec.from_problem(p)
    for c in range(cycles):
        dd.sweep("A")
        dd.sweep("B")
        _, C, q = dd.edge_costs()
        t = time.time()
        _, obj_cold, st_cold = mincost_flow(p.n, p.n, q, C)
        t_cold = time.time() - t
        fs = dd.flow_update(stats=True)
        print(N, c, "obj equal" if fs["objective"] == obj_cold else f"MISMATCH {fs['objective']} {obj_cold}",
              f"cold {st_cold['solver_ms']:.1f} ms ({st_cold['rounds']} r, {st_cold['label_rounds']} lr)",
              f"warm {fs['solver_ms']:.1f} ms ({fs['rounds']} r, {fs['label_rounds']} lr)", flush=True)
    dd.close()
