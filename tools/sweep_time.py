"""Device time per sweep (CUDA events) at the bench grid, pure domdec
sequence: 6 warm-up sweeps then 10 timed (development A/B aid; pick the
library with DD_LIB_PATH)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2405_09400_b200 import DomDec  # noqa: E402
from synth import make_problem  # noqa: E402

p = make_problem("gm", 1024, 4, eps_factor=2.0, theta_deg=20, seed=0)
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    dd = DomDec.from_problem(p, stream=st.cuda_stream)
    for k in range(6):
        dd.sweep("AB"[k % 2])
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
    it = 0
    for k in range(10):
        ev[k][0].record(st)
        s = dd.sweep("AB"[k % 2], stats=True)
        ev[k][1].record(st)
        it += s["iters_total"]
    torch.cuda.synchronize()
    ms = [a.elapsed_time(b) for a, b in ev]
    print(os.path.basename(os.environ.get("DD_LIB_PATH", "default")), f"mean {sum(ms)/len(ms):.3f} ms/sweep",
          f"min {min(ms):.3f}", "iters", it, flush=True)
