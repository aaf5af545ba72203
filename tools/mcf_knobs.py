"""Warm min-cost-flow timing along the bench trajectory (1024^2, T_20) for a
few solver knob settings (development aid; the knobs are read per call)."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
from paper_2405_09400_b200 import DomDec
from synth import make_problem

SETTINGS = [{}, {"DD_MCF_GUT": "8"}, {"DD_MCF_GUT": "32"}, {"DD_MCF_R": "32"}, {"DD_MCF_SWEEPS": "64"},
            {"DD_MCF_SWEEPS": "16"}, {"DD_MCF_WDIV": "4096"}]
C = int(os.environ.get("CYCLES", "12"))
p = make_problem("gm", 1024, 4, eps_factor=2.0, theta_deg=20, seed=0)
for st in SETTINGS:
    for k in ("DD_MCF_GUT", "DD_MCF_R", "DD_MCF_SWEEPS", "DD_MCF_WDIV"):
        os.environ.pop(k, None)
    os.environ.update(st)
    dd = DomDec.from_problem(p)
    ms, lr, ph = [], [], []
    for c in range(C):
        dd.sweep("A")
        dd.sweep("B")
        fs = dd.flow_update(stats=True)
        if c >= 4:
            ms.append(fs["solver_ms"]); lr.append(fs["label_rounds"]); ph.append(fs["rounds"])
    dd.close()
    print(json.dumps({"setting": st, "solver_ms_mean": float(np.mean(ms)), "label_rounds": float(np.mean(lr)),
                      "tile_phases": float(np.mean(ph)), "ms": [round(x) for x in ms]}), flush=True)
