"""Small end-to-end run of every kernel family through the C-ABI, for
compute-sanitizer (tests/test_sanitizer.py): sweeps of every size class,
flow updates (edge costs, min-cost flow, apply), diagnostics, the primal-dual
gap, halo pack/unpack, multiscale refinement and the global Sinkhorn."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402,F401
import torch  # noqa: E402

from paper_2405_09400_b200 import DomDec, mincost_flow, multiscale_solve, sinkhorn_global  # noqa: E402
from synth import make_problem, random_mcf_instance  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
N, s = {"cfg1": (16, 2), "cfg2": (64, 2)}[which]
p = make_problem("gm", N, s, eps_factor=2.0, theta_deg=20, seed=0)
for cap in (0, 6):   # automatic classes, then every larger hull through the global-scratch class
    dd = DomDec.from_problem(p, track_primal=True, comp_cap=cap)
    for _ in range(2):
        dd.sweep("A", stats=True)
        dd.sweep("B", stats=True)
        dd.flow_update(stats=True)
    dd.marginal_error()
    dd.primal_dual_gap()
    cap = dd.halo_capacity()
    buf = torch.zeros(cap, dtype=torch.uint8, device="cuda")
    dd.halo_pack(1, buf.data_ptr(), cap)      # row 1 out and back in (device-side metadata)
    dd.halo_unpack(1, buf.data_ptr(), cap)
    dd.sweep("A", stats=True)
    dd.marginal_error()
    dd.close()
q, C = random_mcf_instance(8, 8, seed=3)
mincost_flow(8, 8, q, C)
ms, st = multiscale_solve(p.mu, p.nu, s, p.eps, p.E, levels=2, conv=1e-3, max_cycles=20)
ms.close()
sinkhorn_global(p.mu, p.nu, p.eps_prime, err=1e-3, max_iter=50, check_every=5)
print("sanitize run ok", which)
