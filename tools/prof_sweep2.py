"""Driver for ncu captures of the sweep kernels in the bench trajectory
(1024^2, s = 4, eps = (2h)^2, GM(0) + T_20): CYCLES hybrid cycles, then one A
and one B sweep with stats (development aid)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2405_09400_b200 import DomDec  # noqa: E402
from synth import make_problem  # noqa: E402

p = make_problem("gm", 1024, 4, eps_factor=2.0, theta_deg=20, seed=0)
dd = DomDec.from_problem(p)
for c in range(int(os.environ.get("CYCLES", "10"))):
    dd.sweep("A")
    dd.sweep("B")
    dd.flow_update()
print(dd.sweep("A", stats=True))
print(dd.sweep("B", stats=True))
dd.close()
