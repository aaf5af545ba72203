"""MCF in-kernel timers along the bench trajectory (development aid): 1024^2,
s = 4, GM(0)+T_20, hybrid cycles 0..C-1 with DD_MCF_TIMERS=1 (the solver
prints refine / price-update / tile-phase / barrier-wait ms per solve)."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["DD_MCF_TIMERS"] = "1"
from paper_2405_09400_b200 import DomDec
from synth import make_problem

C = int(os.environ.get("CYCLES", "10"))
p = make_problem("gm", 1024, 4, eps_factor=2.0, theta_deg=20, seed=0)
dd = DomDec.from_problem(p)
for c in range(C):
    dd.sweep("A")
    dd.sweep("B")
    fs = dd.flow_update(stats=True)
    print(json.dumps({"cycle": c, **{k: fs[k] for k in ("solver_ms", "rounds", "label_rounds", "refines", "stationary",
                                                          "changed_cells")}}), flush=True)
dd.close()
