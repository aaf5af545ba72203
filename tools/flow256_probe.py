"""Where the flow-update time of the 256^2 single-scale time-to-1e-4 run goes
(development aid): per update the solver's own time, the stationary flag and
the wall time of the flow_update call (with stats, i.e. one synchronisation)."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from paper_2405_09400_b200 import DomDec
from synth import make_problem

p = make_problem("gm", 256, 4, eps_factor=2.0, theta_deg=5.0, seed=0)
dd = DomDec.from_problem(p)
rec = []
for c in range(620):
    dd.sweep("A"); dd.sweep("B")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fs = dd.flow_update(stats=True)
    rec.append((time.perf_counter() - t0, fs["solver_ms"], fs["stationary"], fs["certificate"], fs["label_rounds"]))
dd.close()
a = np.array(rec)
st = a[:, 2] == 1
print(json.dumps({"n": len(rec), "stationary": int(st.sum()),
                  "wall_ms_stationary_mean": 1e3 * float(a[st, 0].mean()), "solver_ms_stationary_mean": float(a[st, 1].mean()),
                  "label_rounds_stationary_mean": float(a[st, 4].mean()),
                  "wall_ms_nonstat": [round(1e3 * x, 2) for x in a[~st, 0]], "solver_ms_nonstat": [round(x, 2) for x in a[~st, 1]],
                  "total_wall_s": float(a[:, 0].sum()), "cert_count": int(a[:, 3].sum())}))
