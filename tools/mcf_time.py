"""Time the GPU min-cost-flow solver on dumped flow-update instances (dev aid).
A tiny warm-up solve first, so module loading is not timed."""
import glob, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
from paper_2405_09400_b200 import mincost_flow
from synth import random_mcf_instance
q, C = random_mcf_instance(8, 8, 0)
mincost_flow(8, 8, q, C)
for f in sorted(glob.glob(os.path.join(ROOT, "tools", "data", os.environ.get("MCF_GLOB", "mcf_N*_c*.npz")))):
    d = np.load(f)
    n = int(d["n"])
    t = time.time()
    w, obj, st = mincost_flow(n, n, d["q"], d["C"])
    print(os.path.basename(f), f"{time.time()-t:.3f}s", obj, st, flush=True)
