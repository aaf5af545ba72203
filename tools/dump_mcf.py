"""Dump real flow-update min-cost-flow instances (C, q) from GPU runs for
offline solver tuning (development aid)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2405_09400_b200 import DomDec  # noqa: E402
from synth import make_problem  # noqa: E402

for N, s, cycles in ((256, 4, 2), (1024, 4, 1)):
    p = make_problem("gm", N, s, eps_factor=2.0, theta_deg=20, seed=0)
    dd = DomDec.from_problem(p)
    for c in range(cycles):
        dd.sweep("A")
        st = dd.sweep("B", stats=True)
        cbar, C, q = dd.edge_costs()
        np.savez_compressed(os.path.join(ROOT, "gpurun_out", f"mcf_N{N}_c{c}.npz"), C=C, q=q, n=p.n)
        print(N, c, st, flush=True)
        if c + 1 < cycles:
            print(dd.flow_update(stats=True), flush=True)
