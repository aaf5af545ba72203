"""Dump consecutive flow-update min-cost-flow instances (C, q) and the GPU
solver's optimal flows w along a hybrid trajectory (development aid for
solver work; the flow update is run step by step through the C-ABI hooks
flow_edge_costs -> dd_mincost_flow -> flow_apply)."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2405_09400_b200 import DomDec, mincost_flow  # noqa: E402
from synth import make_problem  # noqa: E402

out = os.path.join(ROOT, "gpurun_out", "data")
os.makedirs(out, exist_ok=True)
for N, s, cycles in [tuple(int(v) for v in a.split(",")) for a in sys.argv[1:]]:
    p = make_problem("gm", N, s, eps_factor=2.0, theta_deg=20, seed=0)
    dd = DomDec.from_problem(p)
    for c in range(cycles):
        dd.sweep("A")
        st = dd.sweep("B", stats=True)
        cbar, C, q = dd.edge_costs()
        t = time.time()
        w, obj, fst = mincost_flow(p.n, p.n, q, C)
        dt = time.time() - t
        np.savez_compressed(os.path.join(out, f"seq_N{N}_s{s}_c{c:02d}.npz"), C=C, q=q, w=w, n=p.n, obj=obj)
        if obj < 0:
            dd.apply_flow(w)
        print(N, c, f"solve {dt:.3f}s obj {obj}", fst, "entry", st.get("l1x_entry"), flush=True)
    dd.close()
