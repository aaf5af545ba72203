"""Driver for an ncu capture of the huge class on clusters (development aid):
multiscale to 512^2, refine to 1024^2 (T_20 pair), then the first A and B
sweeps of the fine layer, where wide-hull cells run on 8-CTA clusters."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_2405_09400_b200 import multiscale_solve
from oracle.multiscale import coarsen   # input preparation only (2x2 sums)
from synth import make_problem

p = make_problem("gm", 1024, 4, eps_factor=2.0, theta_deg=20, seed=0)
mu2, nu2 = coarsen(p.mu), coarsen(p.nu)
os.environ["DD_H_CLUSTER"] = "0"   # coarse layers without clusters: the fine sweeps launch the only cluster kernels
dd, st = multiscale_solve(mu2, nu2, 4, p.eps * 4, p.E, levels=7, conv=1e-4, max_cycles=3000, flow_every=1)
os.environ.pop("DD_H_CLUSTER")
f = dd.refine(p.mu, p.nu, p.eps, p.E)
dd.close()
print(f.sweep("A", stats=True))
print(f.sweep("B", stats=True))
f.close()
