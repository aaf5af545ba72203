"""Device time of the first A and B sweeps of the refined 1024^2 layer (the
wide-hull cells on clusters; development aid, DD_LIB_PATH selects a build)."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch
from paper_2405_09400_b200 import multiscale_solve
from oracle.multiscale import coarsen   # input preparation only (2x2 sums)
from synth import make_problem

p = make_problem("gm", 1024, 4, eps_factor=2.0, theta_deg=20, seed=0)
mu2, nu2 = coarsen(p.mu), coarsen(p.nu)
dd, st = multiscale_solve(mu2, nu2, 4, p.eps * 4, p.E, levels=7, conv=1e-4, max_cycles=3000, flow_every=1)
out = {"lib": os.environ.get("DD_LIB_PATH", "current")[-20:]}
for rep in range(2):
    f = dd.refine(p.mu, p.nu, p.eps, p.E)
    ms = []
    for part in "ABAB":
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); s = f.sweep(part, stats=True); e1.record(); torch.cuda.synchronize()
        ms.append((round(e0.elapsed_time(e1), 2), s["iters_max"], s["l1x_final"]))
    out[f"rep{rep}"] = ms
    f.close()
dd.close()
print(json.dumps(out), flush=True)
