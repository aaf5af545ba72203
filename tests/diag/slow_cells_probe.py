"""Slowest composite cells of the finest multiscale layer (development aid):
solve 4 layers to 512^2 (multiscale_solve), refine to 1024^2, then for the
first cycles print per sweep the cells with the most Sinkhorn passes: their
hull side, X-mass relative to the mean cell, entry error relative to the
cell's budget and the member boxes."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import torch
from paper_2405_09400_b200 import multiscale_solve
from oracle.multiscale import coarsen   # input preparation only (2x2 sums)
from oracle.partitions import composite_partition
from synth import make_problem

th = float(os.environ.get("THETA_DEG", "20"))
p = make_problem("gm", 1024, 4, eps_factor=2.0, theta_deg=th, seed=0)
mu2, nu2 = coarsen(p.mu), coarsen(p.nu)
dd, st = multiscale_solve(mu2, nu2, 4, p.eps * 4, p.E, levels=4, conv=1e-4, max_cycles=3000, flow_every=1)
f = dd.refine(p.mu, p.nu, p.eps, p.E)
dd.close()
s, n = 4, 256
comp = {"A": composite_partition(n, n, "A"), "B": composite_partition(n, n, "B")}
mcell = p.mu.reshape(n, s, n, s).sum(axis=(1, 3)).ravel()
for cyc in range(4):
    for part in "AB":
        boxes = f.boxes()   # state entering the sweep
        stt = f.sweep(part, stats=True)
        it, e0, e = f.cell_stats(part)
        order = np.argsort(-it)[:8]
        avg = p.mu.sum() / len(comp[part])
        rows = []
        for J in order:
            mem = comp[part][J]
            r0 = min(boxes[i][0] for i in mem); c0 = min(boxes[i][1] for i in mem)
            r1 = max(boxes[i][0] + boxes[i][2].shape[0] for i in mem)
            c1 = max(boxes[i][1] + boxes[i][2].shape[1] for i in mem)
            mJ = float(mcell[list(mem)].sum())
            rows.append({"J": int(J), "iters": int(it[J]), "hull": [r1 - r0, c1 - c0], "m_rel": mJ / avg,
                         "e0_rel": float(e0[J] / (1e-4 * mJ)), "e_rel": float(e[J] / (1e-4 * mJ)),
                         "boxes": [list(boxes[i][2].shape) for i in mem],
                         "box_mass": [float(boxes[i][2].sum() / mcell[i]) for i in mem]})
        hull_hist = np.bincount(np.minimum(it, 1000) // 50)
        print(json.dumps({"cycle": cyc, "part": part, "iters_max": stt["iters_max"],
                          "iters_mean": stt["iters_total"] / stt["cells"], "n_over_100": int((it > 100).sum()),
                          "iters_hist_50": hull_hist.tolist(), "top": rows}), flush=True)
    f.flow_update()
f.close()
