"""cfg5 (2048^2, s = 2) multiscale time-to-1e-4 variance probe (development
aid): REPS solves as in bench.py, per-solve seconds, per-layer construction
(init) seconds and the device memory in use after each solve."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2405_09400_b200 import multiscale_solve
from synth import make_problem

p = make_problem("gm", 2048, 2, eps_factor=2.0, theta_deg=20, seed=0)
out = {"reserve_gb": os.environ.get("DD_POOL_RESERVE_GB", "default"), "solves": []}
for r in range(int(os.environ.get("REPS", "5"))):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dd, st = multiscale_solve(p.mu, p.nu, 2, p.eps, p.E, levels=10, conv=1e-4, max_cycles=3000,
                              flow_every=1, eps_scale=4.0, eps_stage_cycles=1)
    torch.cuda.synchronize()
    sec = time.perf_counter() - t0
    dd.close()
    fr, tot = torch.cuda.mem_get_info()
    out["solves"].append({"s": round(sec, 3), "init": [round(x, 3) for x in st["init_seconds"]],
                          "layer": [round(x, 3) for x in st["seconds"]], "used_gb": round((tot - fr) / 2**30, 1)})
print(json.dumps(out), flush=True)
