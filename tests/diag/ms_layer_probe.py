"""Per-sweep timing of the multiscale layers (development aid): builds the
layers by hand through the C-ABI (product init, refine) and prints per sweep
the device time, iterations per cell, max iterations and MUFU work."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import torch
from paper_2405_09400_b200 import DomDec
from oracle.multiscale import layers   # input preparation only (2x2 sums), not the product path
from synth import make_problem

N = int(os.environ.get("N", "1024")); L = int(os.environ.get("LEVELS", "5"))
p = make_problem("gm", N, 4, eps_factor=2.0, theta_deg=float(os.environ.get("THETA_DEG", "20")), seed=0)
lay = layers(p.mu, p.nu, L)
dd = None
for lv, (mu, nu) in enumerate(lay):
    h = 2.0 / mu.shape[0]
    eps = p.eps_prime * h * h
    t0 = time.perf_counter()
    nd = DomDec.product(mu, nu, 4, eps, h, p.E) if dd is None else dd.refine(mu, nu, eps, p.E)
    torch.cuda.synchronize()
    tinit = time.perf_counter() - t0
    if dd is not None:
        dd.close()
    dd = nd
    recs = []
    for cyc in range(3000):
        out = {}
        for part in "AB":
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            st = dd.sweep(part, stats=True)
            e1.record(); torch.cuda.synchronize()
            out[part] = (round(e0.elapsed_time(e1), 2), round(st["iters_total"] / st["cells"], 1), st["iters_max"],
                         round(st["mufu_ops"] / 1e9, 2), st["l1x_entry"])
        fs = dd.flow_update(stats=True)
        recs.append((cyc, out, fs["stationary"], round(fs["solver_ms"], 2)))
        if max(out["A"][4], out["B"][4]) <= 1e-4:
            break
    print(json.dumps({"level": lv, "N": mu.shape[0], "init_s": tinit, "cycles": len(recs),
                      "first": recs[:3], "last": recs[-1]}), flush=True)
dd.close()
