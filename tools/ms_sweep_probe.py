"""Multiscale time to 1e-4 and single-scale sweep probe (development aid):
the multiscale time to 1e-4 at 1024^2 (T_20 and T_5 pairs) and the
pure-sweep time / Sinkhorn passes per cell along the single-scale bench
trajectory (cycles 5-12), for the current build (DD_H_CLUSTER selects the
huge-class path)."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from paper_2405_09400_b200 import DomDec, multiscale_solve
from synth import make_problem

out = {"h_cluster": os.environ.get("DD_H_CLUSTER", "8"), "levels": os.environ.get("LEVELS", "5"), "max_iter": os.environ.get("MAX_ITER", "2000"), "eps_scale": os.environ.get("EPS_SCALE", "1")}
for th in (20.0, 5.0):
    p = make_problem("gm", 1024, 4, eps_factor=2.0, theta_deg=th, seed=0)
    reps = []
    for rep in range(int(os.environ.get("REPS", "2"))):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dd, st = multiscale_solve(p.mu, p.nu, 4, p.eps, p.E, levels=int(os.environ.get("LEVELS", "5")), conv=1e-4, max_cycles=3000, flow_every=1, max_iter=int(os.environ.get("MAX_ITER", "2000")), eps_scale=float(os.environ.get("EPS_SCALE", "1")), eps_stage_cycles=int(os.environ.get("STAGE_CYCLES", "0")))
        torch.cuda.synchronize()
        sec = time.perf_counter() - t0
        ex, ey = dd.marginal_error()
        dd.close()
        reps.append((round(sec, 3), [round(x, 3) for x in st["seconds"]], [round(x, 3) for x in st["init_seconds"]]))
    out[f"ms_T{th:g}"] = {"seconds": sec, "reps": reps, "cycles": st["cycles"],
                          "layer_s": [round(x, 3) for x in st["seconds"]],
                          "init_s": [round(x, 3) for x in st["init_seconds"]],
                          "flow_s": [round(x, 3) for x in st["flow_seconds"]],
                          "l1x": ex, "l1y": ey, "converged": all(st["converged"])}
p = make_problem("gm", 1024, 4, eps_factor=2.0, theta_deg=20, seed=0)
dd = DomDec.from_problem(p)
ms, it = [], []
for c in range(12):
    for part in "AB":
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); s = dd.sweep(part, stats=True); e1.record(); torch.cuda.synchronize()
        if c >= 5:
            ms.append(e0.elapsed_time(e1)); it.append(s["iters_total"] / s["cells"])
    dd.flow_update()
ex, ey = dd.marginal_error()
out["single_scale_sweep"] = {"ms": float(np.mean(ms)), "iters_per_cell": float(np.mean(it)), "l1x": ex}
dd.close()
print(json.dumps(out), flush=True)
