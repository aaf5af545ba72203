"""Config 5 probe (2048^2, s = 2: 1,048,576 basic cells): init, A and B sweeps
and one flow update on one GPU, with timings (development aid)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2405_09400_b200 import DomDec  # noqa: E402
from synth import make_problem  # noqa: E402

t = time.time()
p = make_problem("gm", 2048, 2, eps_factor=2.0, theta_deg=20, seed=0)
print("generate", f"{time.time() - t:.1f}s", flush=True)
t = time.time()
dd = DomDec.from_problem(p)
torch.cuda.synchronize()
print("init", f"{time.time() - t:.1f}s", flush=True)
for c in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    for part in ("A", "B"):
        t = time.time()
        st = dd.sweep(part, stats=True)
        print(c, part, f"{(time.time() - t) * 1e3:.1f} ms", {k: st[k] for k in ("cells", "iters_total", "iters_max",
                                                                           "nonconverged", "l1x_entry")}, flush=True)
    t = time.time()
    fs = dd.flow_update(stats=True)
    print(c, "flow", f"{time.time() - t:.2f} s", fs, flush=True)
print("marginal_error", dd.marginal_error(), flush=True)
