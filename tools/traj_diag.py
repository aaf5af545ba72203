"""Bench-trajectory diagnostics (development aid): the bench workload (1024^2,
s = 4, eps = (2h)^2, GM(0) + T_20) for C hybrid cycles; per sweep the device
time (CUDA events), iterations, and at selected cycles the distribution of
composite hull sides of both partitions (from the exported boxes).  Prints one
JSON line per cycle."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2405_09400_b200 import DomDec  # noqa: E402
from synth import make_problem  # noqa: E402

C = int(os.environ.get("CYCLES", "25"))
N = int(os.environ.get("N", "1024"))
THETA = float(os.environ.get("THETA", "20"))
p = make_problem("gm", N, 4, eps_factor=2.0, theta_deg=THETA, seed=0)
n = N // 4


def hulls(off, ext, part):
    r0, c0 = off[:, 0].reshape(n, n), off[:, 1].reshape(n, n)
    r1, c1 = r0 + ext[:, 0].reshape(n, n), c0 + ext[:, 1].reshape(n, n)
    sides = []
    if part == "A":
        groups = [(slice(2 * a, 2 * a + 2), slice(2 * b, 2 * b + 2)) for a in range(n // 2) for b in range(n // 2)]
    else:
        groups = [(slice(max(0, 2 * a - 1), min(n, 2 * a + 1)), slice(max(0, 2 * b - 1), min(n, 2 * b + 1)))
                  for a in range(n // 2 + 1) for b in range(n // 2 + 1)]
    for gr, gc in groups:
        h1 = r1[gr, gc].max() - r0[gr, gc].min()
        h2 = c1[gr, gc].max() - c0[gr, gc].min()
        sides.append(max(h1, h2))
    s = np.array(sides)
    return {"p50": float(np.median(s)), "p90": float(np.percentile(s, 90)), "p99": float(np.percentile(s, 99)),
            "max": int(s.max()), "gt32": int((s > 32).sum()), "gt48": int((s > 48).sum()),
            "gt64": int((s > 64).sum()), "gt96": int((s > 96).sum()), "n": len(s)}


st = torch.cuda.Stream()
with torch.cuda.stream(st):
    dd = DomDec.from_problem(p, stream=st.cuda_stream)
    for c in range(C):
        rec = {"cycle": c}
        for part in ("A", "B"):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            s = dd.sweep(part, stats=True)
            e1.record(st)
            torch.cuda.synchronize()
            rec[part] = {"ms": e0.elapsed_time(e1), "iters": s["iters_total"] / max(1, s["cells"]),
                         "mufu": s["mufu_ops"], "e0": s["l1x_entry"]}
        fs = dd.flow_update(stats=True)
        rec["flow"] = {"ms": fs["solver_ms"], "stationary": fs["stationary"], "changed": fs["changed_cells"]}
        if c in (0, 2, 5, 10, 15, 20, 24) or c == C - 1:
            off, ext, pos, data = dd.export_cells()
            rec["hullA"] = hulls(off, ext, "A")
            rec["hullB"] = hulls(off, ext, "B")
        print(json.dumps(rec), flush=True)
    dd.close()
