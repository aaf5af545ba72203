"""Per-sweep GPU vs oracle statistics along the hybrid schedule on config 1
in tolerance mode (development aid)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle as O  # noqa: E402
from parity import CONFIGS, gpu_ctx, gpu_transport_cost, oracle_state  # noqa: E402

err = float(sys.argv[1]) if len(sys.argv) > 1 else 1e-6
p = CONFIGS["cfg1_gm"]()
st = oracle_state(p)
q = p.supplies()
dd = gpu_ctx(p, err=err)
for c in range(12):
    for part in ("A", "B"):
        o = O.domdec_sweep(st, part, err=err)
        g = dd.sweep(part, stats=True)
        print(c, part, "iters", g["iters_total"], sum(o["iters"]), "e0", g["l1x_entry"], o["e0_sum"], "e", g["l1x_final"],
              o["e_sum"], flush=True)
    O.flow_update(st, q)
    dd.flow_update()
    print("  cost", gpu_transport_cost(dd, p.h), O.transport_cost(st), flush=True)
