"""Multiscale (f3) time-to-convergence probe (development aid): levels,
conv tolerance and flow period from argv/env; prints the per-layer stats."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: F401  (CUDA context / clocks like the bench)
from paper_2405_09400_b200 import multiscale_solve
from synth import make_problem

N = int(os.environ.get("N", "1024"))
theta = float(os.environ.get("THETA", "20"))
for levels in [int(x) for x in os.environ.get("LEVELS", "5,6").split(",")]:
    for fe in [int(x) for x in os.environ.get("FLOW_EVERY", "1").split(",")]:
        p = make_problem("gm", N, 4, eps_factor=2.0, theta_deg=theta, seed=0)
        t0 = time.perf_counter()
        dd, st = multiscale_solve(p.mu, p.nu, 4, p.eps, p.E, levels=levels, conv=1e-4, max_cycles=3000,
                                  flow_every=fe)
        wall = time.perf_counter() - t0
        ex, ey = dd.marginal_error()
        print(json.dumps({"N": N, "levels": levels, "flow_every": fe, "wall": wall, "l1x": ex, "l1y": ey, **st}),
              flush=True)
        dd.close()
