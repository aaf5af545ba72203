import os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np
from paper_2405_09400_b200 import mincost_flow, DomDecError
from synth import random_mcf_instance
which = sys.argv[1]
for k in range(int(sys.argv[2])):
    if which == "tiny":
        q, C = random_mcf_instance(8, 8, 0); n = 8
    else:
        d = np.load(f"tools/data/{which}.npz"); n = int(d["n"]); q, C = d["q"], d["C"]
    t = time.time()
    try:
        w, obj, st = mincost_flow(n, n, q, C)
        print(which, k, f"{time.time()-t:.3f}s", obj, st["rounds"], st["label_rounds"], flush=True)
    except DomDecError as e:
        print(which, k, "FAILED", e, f"{time.time()-t:.3f}s", flush=True)
