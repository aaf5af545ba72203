"""Debug aid: find composite cells with non-finite sweep-entry errors in the
multiscale layers (per-cell stats through the C-ABI)."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
from paper_2405_09400_b200 import DomDec
from oracle.multiscale import layers
from synth import make_problem

N = int(os.environ.get("N", "256")); L = int(os.environ.get("LEVELS", "4"))
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
    for cyc in range(3000):
        sts = {}
        for part in "AB":
            st = dd.sweep(part, stats=True)
            it, e0, e = dd.cell_stats(part)
            bad = np.flatnonzero(~np.isfinite(e0) | ~np.isfinite(e))
            if len(bad):
                off, ext, pos, data = dd.export_cells()
                print(json.dumps({"level": lv, "cycle": cyc, "part": part, "nbad": int(len(bad)),
                                  "cells": bad[:10].tolist(), "iters": it[bad[:10]].tolist(),
                                  "e0": [float(x) for x in e0[bad[:10]]], "e": [float(x) for x in e[bad[:10]]],
                                  "maxext": int(ext.max()), "data_finite": bool(np.isfinite(data).all())}), flush=True)
                a = dd.export_alpha(part)
                print("alpha finite", bool(np.isfinite(a).all()), flush=True)
                sys.exit(0)
            sts[part] = st["l1x_entry"]
        dd.flow_update()
        if max(sts.values()) <= 1e-4:
            break
    print("level", lv, "cycles", cyc + 1, "ok", flush=True)
