"""Quick GPU probe: per-sweep device time, MUFU count and flow-update cost on
a config (development aid; bench.py is the contract)."""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2405_09400_b200 import DomDec  # noqa: E402
from synth import make_problem  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=int, default=1024)
    ap.add_argument("--s", type=int, default=4)
    ap.add_argument("--eps", type=float, default=2.0)
    ap.add_argument("--theta", type=float, default=20.0)
    ap.add_argument("--cycles", type=int, default=6)
    ap.add_argument("--flow", type=int, default=1)
    a = ap.parse_args()
    t0 = time.time()
    p = make_problem("gm", a.N, a.s, eps_factor=a.eps, theta_deg=a.theta, seed=0)
    print(f"gen {time.time()-t0:.2f}s", flush=True)
    stream = torch.cuda.current_stream()
    t0 = time.time()
    dd = DomDec.from_problem(p, stream=stream.cuda_stream)
    torch.cuda.synchronize()
    print(f"init {time.time()-t0:.2f}s", flush=True)
    for c in range(a.cycles):
        for part in "AB":
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            dd.sweep(part)
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            print(f"cycle {c} {part}: {ms:.3f} ms", flush=True)
        if c == 0:
            try:
                print("stats B", dd.sweep("B", stats=True), flush=True)
            except Exception as ex:
                print("stats B error", ex, flush=True)
        st = None
        if a.flow:
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fs = dd.flow_update(stats=True)
            e1.record(stream)
            torch.cuda.synchronize()
            print(f"cycle {c} F: {e0.elapsed_time(e1):.3f} ms {fs}", flush=True)
    s = dd.sweep("A", stats=True)
    torch.cuda.synchronize()
    print("stats", s)
    print("marginal_error", dd.marginal_error())


if __name__ == "__main__":
    main()
