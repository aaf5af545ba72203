"""Time the global separable Sinkhorn (dd_sinkhorn_global) at 256^2 and 1024^2 (dev aid)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_09400_b200 import sinkhorn_global
from synth import make_problem
runs = ((256, 4, 20000, 1e-4), (1024, 4, 20, 0.0))
if os.environ.get("SG_NCU"):
    runs = ((1024, 4, 3, 0.0),)
for N, s, K, err in runs:
    p = make_problem("gm", N, s, theta_deg=5.0, seed=0)
    a, b, it, e, ms = sinkhorn_global(p.mu, p.nu, p.eps_prime, err=err, max_iter=K, check_every=10)
    print(f"N={N} iters={it} l1_x={e:.3e} ms={ms:.1f} ms/iter={ms/it:.3f}", flush=True)
