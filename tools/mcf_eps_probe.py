"""Exact vs eps-optimal min-cost flow on the bench trajectory instances
(development aid): for cycles 0..C-1 of the 1024^2 T_20 trajectory (exact
warm flows drive the trajectory) the instance (C, q) is also solved cold by
the standalone solver exactly and with DD_MCF_EPSMIN = k (eps = k SC, i.e.
k-optimal in the integer costs): objective gap and solver time."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2405_09400_b200 import DomDec, mincost_flow
from synth import make_problem

N = int(os.environ.get("N", "1024"))
p = make_problem("gm", N, 4, eps_factor=2.0, theta_deg=20, seed=0)
dd = DomDec.from_problem(p)
n = N // 4
for c in range(int(os.environ.get("CYCLES", "4"))):
    dd.sweep("A"); dd.sweep("B")
    _, C, q = dd.edge_costs()
    row = {"cycle": c}
    for k in (0, 1, 16, 256):
        if k: os.environ["DD_MCF_EPSMIN"] = str(k)
        else: os.environ.pop("DD_MCF_EPSMIN", None)
        w, obj, st = mincost_flow(n, n, q, C)
        row[f"k{k}"] = {"obj": int(obj), "ms": round(st["solver_ms"], 1), "rounds": st["rounds"], "label_rounds": st["label_rounds"]}
    os.environ.pop("DD_MCF_EPSMIN", None)
    row["gap_rel"] = {k: (row[k]["obj"] - row["k0"]["obj"]) / abs(row["k0"]["obj"]) if row["k0"]["obj"] else 0 for k in ("k1", "k16", "k256")}
    print(json.dumps(row), flush=True)
    dd.flow_update()
dd.close()
