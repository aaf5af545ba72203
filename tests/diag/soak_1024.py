"""Long-run soak at the bench workload (development aid): 1024^2, s = 4,
T_20, 240 hybrid cycles through domdec_run_cycles (CUDA-graph units), then
the marginal errors, counters and the primal-dual gap must be sane (no pool
exhaustion, no invalid state, errors at the stopping level)."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
from paper_2405_09400_b200 import DomDec
from synth import make_problem

p = make_problem("gm", 1024, 4, eps_factor=2.0, theta_deg=20, seed=0)
dd = DomDec.from_problem(p)
t0 = time.perf_counter()
out = []
for chunk in range(6):
    n, e, moved = dd.run_cycles(40, flow_every=1, conv=0.0)
    ex, ey = dd.marginal_error()
    out.append({"cycles": (chunk + 1) * 40, "entry_error": e, "moved": moved, "l1x": ex, "l1y": ey,
                "t": round(time.perf_counter() - t0, 1)})
    print(json.dumps(out[-1]), flush=True)
print(json.dumps({"counters": dd.counters()}), flush=True)
dd.close()
