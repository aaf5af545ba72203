"""Debug aid: per-sweep iteration distribution and the slowest cells of the
multiscale layers (hull side, mass, iterations)."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import torch
from paper_2405_09400_b200 import DomDec
from oracle.multiscale import layers
from oracle.partitions import composite_partition
from synth import make_problem

N = int(os.environ.get("N", "1024")); L = int(os.environ.get("LEVELS", "6"))
p = make_problem("gm", N, 4, eps_factor=2.0, theta_deg=20, seed=0)
lay = layers(p.mu, p.nu, L)
dd = None
for lv, (mu, nu) in enumerate(lay):
    h = 2.0 / mu.shape[0]
    eps = p.eps_prime * h * h
    nd = DomDec.product(mu, nu, 4, eps, h, p.E) if dd is None else dd.refine(mu, nu, eps, p.E)
    if dd is not None:
        dd.close()
    dd = nd
    n = mu.shape[0] // 4
    m = mu.reshape(n, 4, n, 4).sum(axis=(1, 3)).ravel()
    for cyc in range(3000):
        es = {}
        for part in "AB":
            e0_, e1_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0_.record()
            st = dd.sweep(part, stats=True)
            e1_.record(); torch.cuda.synchronize()
            es[part] = st["l1x_entry"]
            if lv >= L - 2:
                it, e0, e = dd.cell_stats(part)
                off, ext, pos, data = dd.export_cells()
                comp = composite_partition(n, n, part)
                top = np.argsort(it)[::-1][:5]
                info = []
                for k in top:
                    mem = comp[k]
                    r0 = min(off[i, 0] for i in mem); r1 = max(off[i, 0] + ext[i, 0] for i in mem)
                    c0 = min(off[i, 1] for i in mem); c1 = max(off[i, 1] + ext[i, 1] for i in mem)
                    info.append((int(k), int(it[k]), int(max(r1 - r0, c1 - c0)), float(sum(m[i] for i in mem)), len(mem)))
                print(json.dumps({"lv": lv, "cyc": cyc, "part": part, "ms": round(e0_.elapsed_time(e1_), 2),
                                  "it_mean": float(it.mean()), "it_p99": float(np.percentile(it, 99)),
                                  "n_over_50": int((it > 50).sum()), "top": info}), flush=True)
        dd.flow_update()
        if max(es.values()) <= 1e-4:
            break
