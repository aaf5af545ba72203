"""cfg5 (2048^2, s = 2) multiscale solves in one process with per-layer init
times (development aid; DD_MS_TIMERS=1 prints the init checkpoints)."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
from paper_2405_09400_b200 import multiscale_solve
from synth import make_problem

p = make_problem("gm", 2048, 2, eps_factor=2.0, theta_deg=20, seed=0)
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    dd, st = multiscale_solve(p.mu, p.nu, 2, p.eps, p.E, levels=10, conv=1e-4, max_cycles=3000, flow_every=1,
                              eps_scale=4.0, eps_stage_cycles=1)
    torch.cuda.synchronize()
    print(json.dumps({"rep": rep, "s": round(time.perf_counter() - t0, 3), "init": [round(v, 3) for v in st["init_seconds"]],
                      "layer": [round(v, 3) for v in st["seconds"]]}), flush=True)
    dd.close()
