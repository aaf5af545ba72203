"""Pure-sweep throughput and MUFU fraction on the bench-side configs
(development aid; DD_LIB_PATH selects the build): cfg5 2048^2 s=2, cfg3 256^2
s=4 (eps (2h)^2), and the 1024^2 s=4 bench workload after 8 hybrid cycles."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2405_09400_b200 import DomDec, mufu_peak
from synth import make_problem

peak = 148 * 16 * 1965e6
def sweeps(dd, nwarm=4, nt=6):
    for k in range(nwarm):
        dd.sweep("AB"[k % 2])
    torch.cuda.synchronize()
    dd.reset_counters()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for k in range(nt):
        dd.sweep("AB"[k % 2])
    e1.record()
    torch.cuda.synchronize()
    s = e0.elapsed_time(e1) / 1e3
    cnt = dd.counters()
    return {"sweep_ms": round(1e3 * s / nt, 3), "frac": round(cnt["mufu_ops"] / s / peak, 4),
            "iters": cnt["iters"] / max(1, cnt["cells"]), "cells": cnt["cells"], "iters_total": cnt["iters"]}

out = {"lib": os.environ.get("DD_LIB_PATH", "current")[-24:]}
dd = DomDec.from_problem(make_problem("gm", 2048, 2, eps_factor=2.0, theta_deg=20, seed=0))
out["cfg5"] = sweeps(dd, 2, 4); dd.close()
dd = DomDec.from_problem(make_problem("gm", 256, 4, eps_factor=2.0, theta_deg=5, seed=0))
out["cfg3"] = sweeps(dd); dd.close()
dd = DomDec.from_problem(make_problem("gm", 1024, 4, eps_factor=2.0, theta_deg=20, seed=0))
for c in range(8):
    dd.sweep("A"); dd.sweep("B"); dd.flow_update()
out["cfg4_c8"] = sweeps(dd, 2, 6); dd.close()
print(json.dumps(out), flush=True)
