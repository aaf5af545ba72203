"""Sweep-only timing probe: per-sweep device time and MUFU rate (dev aid)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2405_09400_b200 import DomDec
from synth import make_problem
N = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
s = int(sys.argv[2]) if len(sys.argv) > 2 else 4
cyc = int(sys.argv[3]) if len(sys.argv) > 3 else 8
p = make_problem("gm", N, s, eps_factor=2.0, theta_deg=20, seed=0)
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    dd = DomDec.from_problem(p, stream=st.cuda_stream)
    for c in range(cyc):
        for part in "AB":
            dd.reset_counters()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(st); dd.sweep(part); e1.record(st); torch.cuda.synchronize()
            ms = e0.elapsed_time(e1); cnt = dd.counters()
            print(f"{os.environ.get('DOMDEC_LIB','default')[-20:]} c{c}{part} {ms:.3f} ms  it/cell {cnt['iters']/cnt['cells']:.2f}  MUFU {cnt['mufu_ops']/ms/1e9:.3f} TOP/s", flush=True)
